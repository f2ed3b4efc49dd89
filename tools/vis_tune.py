"""Time every visibility-kernel variant on one scene (default MatrixCity-shaped)
and check each leaves byte-identical outputs. Usage: python tools/vis_tune.py [config] [reps]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2510_01767_b200 import lobe
    from synth import make_scene
    cfg = sys.argv[1] if len(sys.argv) > 1 else "matrixcity"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    variants = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
    sc = make_scene(cfg)
    G, N = sc.G, sc.N

    class DG:
        pass

    dg = DG()
    for k in ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity"):
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
    S = lobe.Scene(dg, lobe.make_cameras(sc))
    m, n = sc.cfg.m, sc.cfg.n
    sel = [0, N // 3, N - 1]
    ref_rows = np.concatenate([S.export_rows(c, 1) for c in sel])
    ref = S.assign_cameras(m, n)
    out = []
    nv = 6
    for v in (variants or range(nv)):
        try:
            ms, grid = S.dev_vis_bench(v, reps)
        except lobe.LobeError as e:
            out.append({"variant": v, "error": str(e)})
            continue
        # outputs after this variant ran (rows, partials) must be identical
        S._keep.append(None)
        rows = np.concatenate([S.export_rows(c, 1) for c in sel])
        S2 = S  # per-camera stats come from partials written by the variant: re-reduce via a fresh grid eval
        a = S2.assign_cameras(m, n, tau=0.15000000000000002)   # different key -> re-evaluates
        same = bool((rows == ref_rows).all()) and all((a[k] == ref[k]).all() for k in ("K", "n", "n0", "member"))
        tests = G * N
        out.append({"variant": v, "ms": ms, "grid": grid, "tests_per_s": tests / (ms * 1e-3),
                    "frac_fp32": 22 * tests / (ms * 1e-3) / 74.45e12, "identical": same})
        print(json.dumps(out[-1]), flush=True)
    S.close()


if __name__ == "__main__":
    main()
