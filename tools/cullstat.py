import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2510_01767_b200 import lobe
from synth import make_scene
for cfg in sys.argv[1:]:
    sc = make_scene(cfg)
    class DG: pass
    dg = DG()
    for k in ("x","y","z","sx","sy","sz","qw","qx","qy","qz","opacity"):
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
    S = lobe.Scene(dg, lobe.make_cameras(sc))
    st = S.stats()
    n_tiles = (st.n_gaussians + 16383)//16384*16
    tot = n_tiles * st.n_local_cameras
    print(cfg, "logical", st.tests_executed, "dense", st.dense_tests, "kept frac %.4f" % (st.dense_tests/1024/tot),
          "nonempty frac %.4f" % (st.tile_pairs/tot), "t_vis %.2f t_cull %.2f" % (st.t_vis_ms, st.t_cull_ms))
    S.close()
