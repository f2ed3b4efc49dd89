"""Diagnosis only: host timeline of lobe_load_scene (LOBE_TRACE_HOST=1) for two
bench steps after warm-up, with the Python-side call boundaries."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01767_b200 import lobe
from paper_2510_01767_b200.engine import Engine
from synth import make_scene

sc = make_scene(sys.argv[1] if len(sys.argv) > 1 else "matrixcity")
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")
class DG: pass
dg = DG()
for k in names:
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
cams = lobe.make_cameras(sc)
m, n = sc.cfg.m, sc.cfg.n
W64 = (sc.G + 63) // 64
crop = torch.empty(m * n * W64, dtype=torch.int64, device="cuda")
elig = torch.empty_like(crop)
stream = torch.cuda.current_stream()
T0 = time.perf_counter()
def mark(w):
    print(f"[py] {w:30s} {1e6 * (time.perf_counter() - T0):10.1f} us", file=sys.stderr, flush=True)
def step(trace):
    if trace: mark("step start")
    eng = Engine.from_scene(dg, cams, stream=stream)
    if trace: mark("load returned")
    eng.crop_masks_into(m, n, crop, elig)
    if trace: mark("crop returned")
    eng.block_loads(m, n)
    if trace: mark("block_loads returned")
    eng.assign_cameras(m, n)
    if trace: mark("assign returned")
    eng.close()
    if trace: mark("close returned")
for _ in range(3):
    step(False)
torch.cuda.synchronize()
os.environ["LOBE_TRACE_HOST"] = "1"
for _ in range(2):
    step(True)
torch.cuda.synchronize()
