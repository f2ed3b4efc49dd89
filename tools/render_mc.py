"""Timing of the depth-render camera selection (NEXT-1) on a named config."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2510_01767_b200 import lobe
from synth import make_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "matrixcity"
sc = make_scene(cfg)
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")
class DG: pass
dg = DG()
for k in names:
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
S = lobe.Scene(dg, lobe.make_cameras(sc))
m, n = sc.cfg.m, sc.cfg.n
a0 = S.assign_cameras(m, n)
torch.cuda.synchronize()
t0 = time.perf_counter()
S.render_select(dg)
torch.cuda.synchronize()
t1 = time.perf_counter()
off, gu, gv = S.camera_clouds()
a1 = S.assign_cameras(m, n)
L0 = None
res = {"config": cfg, "render_select_s": t1 - t0, "cloud_points": int(off[-1]),
       "mean_points_per_camera": float(off[-1]) / sc.N,
       "cameras_with_changed_member_set": int((a0["member"] != a1["member"]).sum()),
       "mean_memberships_gaussian_cloud": float(np.mean([bin(int(v)).count("1") for v in a0["member"]])),
       "mean_memberships_render_cloud": float(np.mean([bin(int(v)).count("1") for v in a1["member"]]))}
t2 = time.perf_counter()
r = S.balance_partition(m, n, L=100, seed=0)
res["bo_render_mode_s"] = time.perf_counter() - t2
res["objective_uniform"] = int(r["history"][0])
res["objective_best"] = int(r["history"].min())
print(json.dumps(res))
S.close()
