"""Diagnosis only (numbers under a profiler are never bench values): one engine
step under torch.profiler (CUPTI), then the gaps on the library stream and the
host-side time between kernel launches, to find synchronisation bubbles.
--host: inputs and crop outputs in pinned host memory (the bench's e2e step).
--aniso: the anisotropic predicate. --two: two back-to-back steps."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01767_b200 import lobe
from paper_2510_01767_b200.engine import Engine
from synth import make_scene

args = [a for a in sys.argv[1:] if not a.startswith("--")]
HOST = "--host" in sys.argv
PRED = 1 if "--aniso" in sys.argv else 0
cfg = args[0] if args else "matrixcity"
sc = make_scene(cfg)
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")
class DG: pass
dg = DG()
for k in names:
    if HOST:
        t = torch.empty(sc.G, dtype=torch.float32, pin_memory=True)
        t.numpy()[:] = getattr(sc, k)
        setattr(dg, k, t)
    else:
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
cams = lobe.make_cameras(sc)
m, n = sc.cfg.m, sc.cfg.n
B = m * n
W64 = (sc.G + 63) // 64
crop = torch.empty(B * W64, dtype=torch.int64, device="cuda") if not HOST else torch.empty(B * W64, dtype=torch.int64, pin_memory=True)
elig = torch.empty_like(crop) if not HOST else torch.empty(B * W64, dtype=torch.int64, pin_memory=True)
stream = torch.cuda.current_stream()

def step():
    eng = Engine.from_scene(dg, cams, stream=stream, predicate=PRED)
    eng.crop_masks_into(m, n, crop, elig)
    eng.block_loads(m, n)
    eng.assign_cameras(m, n)
    eng.close()

import time
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    print("step wall ms %.2f" % (1e3 * (time.perf_counter() - t0)))
from torch.profiler import profile, ProfilerActivity
TWO = "--two" in sys.argv   # two back-to-back steps: the host gap between them
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    if TWO:
        step()
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
tf = "gpurun_out/trace_step%s%s.json" % ("_host" if HOST else "", "_aniso" if PRED else "")
prof.export_chrome_trace(tf)
ev = json.load(open(tf))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0 = k[0]["ts"]
prev_end = t0
print(f"{'start':>9} {'dur':>8} {'gap':>8}  name")
for e in k:
    gap = e["ts"] - prev_end
    print(f"{e['ts']-t0:9.1f} {e['dur']:8.1f} {gap:8.1f}  s{e.get('args', {}).get('stream', '?')} {e['name'][:66]}")
    prev_end = max(prev_end, e["ts"] + e["dur"])
print("span", prev_end - t0, "busy", sum(e["dur"] for e in k))
rt = sorted([e for e in ev if e.get("cat") == "cuda_runtime" and e.get("dur", 0) > 50], key=lambda e: -e["dur"])
# host-side API calls (python_function / user annotations are not recorded; cuda_runtime calls show the host's pace)
rc = sorted([e for e in ev if e.get("cat") == "cuda_runtime"], key=lambda e: e["ts"])
if TWO and rc:
    print("runtime calls between the two steps' GPU work (ts, dur, name):")
    for e in rc:
        if 0 <= e["ts"] - t0 and e["name"] in ("cudaStreamSynchronize", "cudaEventSynchronize", "cudaFreeAsync",
                                                 "cudaMallocAsync", "cudaHostAlloc", "cudaFreeHost", "cudaFree",
                                                 "cudaMalloc", "cudaStreamCreateWithFlags", "cudaEventCreate"):
            print(f"{e['ts']-t0:9.1f} {e['dur']:8.1f}  {e['name']}")
print("slow runtime calls:")
for e in rt[:25]:
    print(f"{e['ts']-t0:9.1f} {e['dur']:8.1f}  {e['name']}")
