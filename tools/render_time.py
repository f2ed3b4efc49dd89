"""Wall time of the depth-render camera selection on a config, called
repeatedly on one scene (diagnosis; LOBE_TRACE_ALLOC=1 prints slow pool
allocations)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01767_b200 import lobe
from synth import make_scene

sc = make_scene(sys.argv[1] if len(sys.argv) > 1 else "matrixcity")
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")


class DG:
    pass


dg = DG()
for k in names:
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
S = lobe.Scene(dg, lobe.make_cameras(sc))
for r in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.render_select(dg)
    torch.cuda.synchronize()
    st = S.stats()
    print(f"render_select {r}: {time.perf_counter() - t0:.3f} s  k_render {st.t_render_kernel_ms:.1f} ms", flush=True)
S.close()
