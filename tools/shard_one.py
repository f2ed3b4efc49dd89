"""Load rank r of W (cameras [rN/W, (r+1)N/W), the full scene's frame) alone on
one GPU and run a few evaluations -- the per-rank kernel mix for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOBE_A4_STREAM"] = "0"
import torch
from paper_2510_01767_b200 import lobe
from synth import make_scene

cfg, r, W = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
sc = make_scene(cfg)
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")


class DG:
    pass


dg = DG()
for k in names:
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
with lobe.Scene(dg, lobe.make_cameras(sc)) as S0:
    frame = dict(S0.frame)
sub = sc.subset_cameras(list(range(r * sc.N // W, (r + 1) * sc.N // W)))
S = lobe.Scene(dg, lobe.make_cameras(sub), frame=frame)
for _ in range(3):
    S.block_loads(sc.cfg.m, sc.cfg.n)
torch.cuda.synchronize()
S.close()
