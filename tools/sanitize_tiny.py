"""compute-sanitizer target: the whole hot path once on the tiny config through
the C ABI (isotropic and anisotropic load, assignment, block loads, crop, a short
BO loop, the depth-render selection, the block pipeline calls, a collective
NCCL-comm scene at world 1). Run as
  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_tiny.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_01767_b200 import lobe
from synth import make_scene

sc = make_scene("tiny")
m, n = sc.cfg.m, sc.cfg.n
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")


class DG:
    pass


dg = DG()
for k in names:
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
for pred in (0, 1):
    with lobe.Scene(sc, sc, predicate=pred) as S:
        a = S.assign_cameras(m, n)
        L = S.block_loads(m, n)
        c, e = S.crop_masks(m, n)
        r = S.balance_partition(m, n, L=4, seed=1)
        S.export_rows(0, 3)
        sub = S.block_subscene(m, n, 0, dg)
        S.prune_outside(m, n, 0, sub)
        if pred == 0:
            S.render_select(dg)
            S.assign_cameras(m, n)
            S.block_loads(m, n)
        print("pred", pred, "objective", L["objective"], "bo", int(r["history"].min()))
nid = lobe.nccl_unique_id()
with lobe.Scene(sc, sc, nccl_id=nid) as S:
    S.assign_cameras(m, n)
    S.block_loads(m, n)
    S.crop_masks(m, n)
lobe.release_comms()
torch.cuda.synchronize()
print("sanitize target ok")
