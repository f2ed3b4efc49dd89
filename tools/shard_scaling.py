"""Per-rank work of the camera-sharded engine, measured on one GPU (SURVEY
§8(e)): for W ranks, rank r owns cameras [rN/W, (r+1)N/W) and all
G Gaussians. Each rank's scene is loaded alone (world 1, the full scene's
frame passed explicitly so every rank sees the same grid coordinates) and its
stage times are taken with nothing else on the device: the visibility pass
(a3), one evaluation (a5-a8) and the load / step pieces. The exchange (a11)
is not run here (one GPU): its bytes per rank are reported for the model.

python tools/shard_scaling.py [config] [W ...]   -> one JSON line per W"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOBE_A4_STREAM"] = "0"  # a4 alone, after the evaluations
import torch
from paper_2510_01767_b200 import lobe
from synth import make_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "matrixcity"
Ws = [int(w) for w in sys.argv[2:]] or [1, 2, 4, 8]
sc = make_scene(cfg)
m, n = sc.cfg.m, sc.cfg.n
B = m * n
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")


class DG:
    pass


dg = DG()
for k in names:
    setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
with lobe.Scene(dg, lobe.make_cameras(sc)) as S0:
    frame = dict(S0.frame)


def rank_times(c0, c1, reps=3):
    sub = sc.subset_cameras(list(range(c0, c1)))
    cams = lobe.make_cameras(sub)
    vis, ev, dep, load = [], [], [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S = lobe.Scene(dg, cams, frame=frame)
        for _ in range(3):
            S.block_loads(m, n)
            st = S.stats()
            ev.append(st.t_hist_ms + st.t_loads_ms)
        S.assign_cameras(m, n)
        st = S.stats()
        vis.append(st.t_vis_ms)
        dep.append(st.t_depth_ms)
        load.append(st.t_prep_ms)
        S.close()
    med = statistics.median
    return dict(cams=c1 - c0, t_vis_ms=med(vis), t_eval_ms=med(ev), t_depth_ms=med(dep), t_prep_ms=med(load))


for W in Ws:
    ranks = [rank_times(r * sc.N // W, (r + 1) * sc.N // W) for r in range(W)]
    worst = {k: max(rk[k] for rk in ranks) for k in ("t_vis_ms", "t_eval_ms", "t_depth_ms", "t_prep_ms")}
    words = (sc.G + 1023) // 1024 * 32
    own_blocks = max(((j + 1) * B // W) - (j * B // W) for j in range(W))
    line = {"config": cfg, "W": W, "ranks": ranks, "max_over_ranks": worst,
            "engine_eval_compute_ms": worst["t_vis_ms"] + worst["t_eval_ms"],
            "exchange_bytes_per_rank": {"partial_masks_all_to_all": (W - 1) * own_blocks * words * 4 if W > 1 else 0,
                                        "combine_reads": W * own_blocks * words * 4 if W > 1 else 0}}
    print(json.dumps(line), flush=True)
