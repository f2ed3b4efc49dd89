"""Diagnosis only (profiler numbers are never bench values): the depth-render
camera selection under torch.profiler -- device time per kernel name, total
busy time and span, and the slowest host runtime calls."""
import sys, os, json, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01767_b200 import lobe
from synth import make_scene

sc = make_scene(sys.argv[1] if len(sys.argv) > 1 else "matrixcity")
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")
class DG: pass
dg = DG()
for k in names:
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
S = lobe.Scene(dg, lobe.make_cameras(sc))
S.render_select(dg)  # warm
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    S.render_select(dg)
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/trace_render.json")
ev = json.load(open("gpurun_out/trace_render.json"))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
agg = collections.defaultdict(lambda: [0, 0.0])
for e in k:
    nm = e["name"].split("(")[0][:60]
    agg[nm][0] += 1
    agg[nm][1] += e["dur"]
span = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
busy = sum(e["dur"] for e in k)
print(f"span {span/1e3:.1f} ms, busy {busy/1e3:.1f} ms")
for nm, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{d/1e3:9.2f} ms  x{c:5d}  {nm}")
rt = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    if e.get("cat") == "cuda_runtime":
        rt[e["name"]][0] += 1
        rt[e["name"]][1] += e.get("dur", 0)
print("host runtime calls:")
for nm, (c, d) in sorted(rt.items(), key=lambda x: -x[1][1])[:10]:
    print(f"{d/1e3:9.2f} ms  x{c:5d}  {nm}")
S.close()
