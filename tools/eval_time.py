"""Time one evaluation (a5-a8 at the uniform cuts) and the isolated a4 on a
config (diagnosis): medians of the library's CUDA-event stage times."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOBE_A4_STREAM"] = "0"
import torch  # noqa: F401
from paper_2510_01767_b200 import lobe
from synth import make_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "matrixcity"
sc = make_scene(cfg)
m, n = sc.cfg.m, sc.cfg.n
ev, vis, dep = [], [], []
for _ in range(3):
    with lobe.Scene(sc, sc, device=0) as S:
        for _ in range(5):
            S.block_loads(m, n)
            st = S.stats()
            ev.append(st.t_hist_ms + st.t_loads_ms)
        S.assign_cameras(m, n)
        st = S.stats()
        vis.append(st.t_vis_ms)
        dep.append(st.t_depth_ms)
print(f"{cfg}: evaluation {statistics.median(ev):.4f} ms  vis {statistics.median(vis):.4f} ms  "
      f"a4 {statistics.median(dep):.4f} ms")
