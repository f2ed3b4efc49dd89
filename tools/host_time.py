"""Diagnosis only: host-side wall time of each call of the bench step (device
inputs), without extra synchronisation, to find host work the GPU waits for.
LOBE_TRACE_HOST=1 adds the library's load-phase marks (stderr)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01767_b200 import lobe
from paper_2510_01767_b200.engine import Engine
from synth import make_scene

sc = make_scene(sys.argv[1] if len(sys.argv) > 1 else "matrixcity")
class DG: pass
dg = DG()
for k in ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity"):
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
cams = lobe.make_cameras(sc)
m, n = sc.cfg.m, sc.cfg.n
W64 = (sc.G + 63) // 64
crop = torch.empty(m * n * W64, dtype=torch.int64, device="cuda")
elig = torch.empty_like(crop)
stream = torch.cuda.current_stream()
for it in range(8):
    T = [time.perf_counter()]
    eng = Engine.from_scene(dg, cams, stream=stream); T.append(time.perf_counter())
    eng.crop_masks_into(m, n, crop, elig); T.append(time.perf_counter())
    eng.block_loads(m, n); T.append(time.perf_counter())
    eng.assign_cameras(m, n); T.append(time.perf_counter())
    eng.stats(); T.append(time.perf_counter())
    eng.close(); T.append(time.perf_counter())
    names = ("load", "crop", "loads", "assign", "stats", "close")
    print(" ".join(f"{a} {1e3 * (T[i + 1] - T[i]):.3f}" for i, a in enumerate(names)), f"total {1e3 * (T[-1] - T[0]):.3f} ms")
