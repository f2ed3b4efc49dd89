"""Diagnosis only: end-to-end steps from pinned host buffers, one or two host
threads (own stream each), per-step wall times."""
import sys, os, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01767_b200 import lobe
from paper_2510_01767_b200.engine import Engine
from synth import make_scene

sc = make_scene(sys.argv[1] if len(sys.argv) > 1 else "matrixcity")
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")
class HG: pass
hg = HG()
for k in names:
    t = torch.empty(sc.G, dtype=torch.float32, pin_memory=True); t.numpy()[:] = getattr(sc, k); setattr(hg, k, t)
cams = lobe.make_cameras(sc)
m, n = sc.cfg.m, sc.cfg.n
B = m * n; W64 = (sc.G + 63) // 64
NT = 4
outs = [(torch.empty(B * W64, dtype=torch.int64, pin_memory=True), torch.empty(B * W64, dtype=torch.int64, pin_memory=True)) for _ in range(NT)]
strms = [torch.cuda.Stream() for _ in range(NT)]

def step(i, log):
    t0 = time.perf_counter()
    eng = Engine.from_scene(hg, cams, stream=strms[i])
    t1 = time.perf_counter()
    eng.crop_masks_into(m, n, outs[i][0], outs[i][1])
    t2 = time.perf_counter()
    eng.block_loads(m, n)
    t3 = time.perf_counter()
    eng.assign_cameras(m, n)
    t4 = time.perf_counter()
    eng.close()
    t5 = time.perf_counter()
    log.append((i, round((t1-t0)*1e3, 2), round((t2-t1)*1e3, 2), round((t3-t2)*1e3, 2), round((t4-t3)*1e3, 2), round((t5-t4)*1e3, 2)))

def run(nthreads, steps_each, log):
    th = [threading.Thread(target=lambda i=i: [step(i, log) for _ in range(steps_each)]) for i in range(nthreads)]
    [t.start() for t in th]; [t.join() for t in th]

run(NT, 2, [])   # grow the pool for NT scenes in flight
torch.cuda.synchronize()
for nthreads in (1, 2, 3, 4, 2, 3):
    log = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(nthreads, 12 // nthreads, log)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 12
    print(f"threads={nthreads}: {dt*1e3:.2f} ms/step; load ms per step: {[l[1] for l in log]}", flush=True)
