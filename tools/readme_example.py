"""The README usage example (runs on a GPU box: python tools/readme_example.py)."""
import torch, sys
sys.path.insert(0, ".")
from paper_2510_01767_b200 import lobe
from synth import make_scene

sc = make_scene("rubble")
class G: pass
g = G()
for k in ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity"):
    setattr(g, k, torch.from_numpy(getattr(sc, k)).cuda())
with lobe.Scene(g, lobe.make_cameras(sc)) as S:
    loads = S.block_loads(3, 3)
    cams = S.assign_cameras(3, 3)
    crop, eligible = S.crop_masks(3, 3)
    best = S.balance_partition(3, 3, L=100)
print("objective", loads["objective"], "best", int(best["history"].min()), "K>0", int((cams["K"] > 0).sum()), crop.shape)
