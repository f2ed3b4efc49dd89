"""Diagnosis only: host-side (Python + C ABI call) time of the bench step with
device-resident inputs, per phase, and a cProfile of 20 steps."""
import sys, os, time, cProfile, pstats
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
B = m * n; W64 = (sc.G + 63) // 64
crop = torch.empty(B * W64, dtype=torch.int64, device="cuda")
elig = torch.empty(B * W64, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream()
T = {}
def step():
    t0 = time.perf_counter()
    eng = Engine.from_scene(dg, cams, stream=stream)
    t1 = time.perf_counter()
    eng.crop_masks_into(m, n, crop, elig)
    t2 = time.perf_counter()
    eng.block_loads(m, n)
    t3 = time.perf_counter()
    eng.assign_cameras(m, n)
    t4 = time.perf_counter()
    st = eng.local.stats()
    eng.close()
    t5 = time.perf_counter()
    for k, v in (("load", t1 - t0), ("crop", t2 - t1), ("loads", t3 - t2), ("assign", t4 - t3), ("stats+close", t5 - t4)):
        T.setdefault(k, []).append(v * 1e3)
for _ in range(3):
    step()
torch.cuda.synchronize()
T.clear()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step()
pr.disable()
torch.cuda.synchronize()
print({k: round(sorted(v)[len(v) // 2], 3) for k, v in T.items()})
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
