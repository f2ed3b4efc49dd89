"""Per-rank work of the Gaussian-sharded alternative (SURVEY §8(e):
"shard Gaussians and replicate cameras"), measured on one GPU. The Gaussians
are ordered by a 3D Morton code of their positions (host, numpy: any
spatially coherent order serves for timing) and rank r owns the contiguous
range [rG/W, (r+1)G/W) with all N cameras. Each rank's scene is loaded alone
(world 1, the full scene's frame passed explicitly) and its stage times are
taken with nothing else on the device. In this scheme a rank's masks are its
own Gaussians' (no OR-combine); the exchange is an all-reduce of the per-camera
histograms (N x B u32 twice) and of the B counts, modelled, not run here.

python tools/shard_scaling_gauss.py [config] [W ...]   -> one JSON line per W"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOBE_A4_STREAM"] = "0"
import numpy as np
import torch
from paper_2510_01767_b200 import lobe
from synth import make_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "matrixcity"
Ws = [int(w) for w in sys.argv[2:]] or [1, 2, 4, 8]
sc = make_scene(cfg)
m, n = sc.cfg.m, sc.cfg.n
names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")
cams = lobe.make_cameras(sc)


def device_arrays(s):
    class DG:
        pass
    dg = DG()
    for k in names:
        setattr(dg, k, torch.from_numpy(np.ascontiguousarray(getattr(s, k))).cuda())
    return dg


with lobe.Scene(device_arrays(sc), cams) as S0:
    frame = dict(S0.frame)


def morton_order(s):
    pts = np.stack([s.x, s.y, s.z], 1).astype(np.float64)
    lo, hi = np.percentile(pts, 1, axis=0), np.percentile(pts, 99, axis=0)
    q = np.clip(((pts - lo) / np.maximum(hi - lo, 1e-12) * 1023).astype(np.int64), 0, 1023)
    code = np.zeros(len(pts), np.int64)
    for b in range(10):
        for a in range(3):
            code |= ((q[:, a] >> b) & 1) << (3 * b + a)
    return np.argsort(code, kind="stable")


order = morton_order(sc)
sorted_sc = sc.permute_gaussians(order)


def rank_times(g0, g1, reps=3):
    sub = sorted_sc.permute_gaussians(np.arange(g0, g1))
    dg = device_arrays(sub)
    vis, ev, dep = [], [], []
    for _ in range(reps):
        S = lobe.Scene(dg, cams, frame=frame)
        for _ in range(3):
            S.block_loads(m, n)
            st = S.stats()
            ev.append(st.t_hist_ms + st.t_loads_ms)
        S.assign_cameras(m, n)
        st = S.stats()
        vis.append(st.t_vis_ms)
        dep.append(st.t_depth_ms)
        S.close()
    med = statistics.median
    return dict(gaussians=g1 - g0, t_vis_ms=med(vis), t_eval_ms=med(ev), t_depth_ms=med(dep))


for W in Ws:
    ranks = [rank_times(r * sc.G // W, (r + 1) * sc.G // W) for r in range(W)]
    worst = {k: max(rk[k] for rk in ranks) for k in ("t_vis_ms", "t_eval_ms", "t_depth_ms")}
    B = m * n
    line = {"config": cfg, "W": W, "sharding": "gaussians (Morton ranges), cameras replicated", "ranks": ranks,
            "max_over_ranks": worst, "engine_eval_compute_ms": worst["t_vis_ms"] + worst["t_eval_ms"],
            "exchange_bytes_per_rank": {"histogram_allreduce": 2 * sc.N * B * 4 if W > 1 else 0,
                                        "counts_allreduce": 3 * B * 8 if W > 1 else 0}}
    print(json.dumps(line), flush=True)
