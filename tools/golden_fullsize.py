"""Write tests/golden/<config>_oracle.json: the ORACLE's outputs for a full-size
BASELINE config, as SHA-256 digests (rows, per-camera integer arrays, crop and
eligible masks per block), block records in full and D_c values.

Calls only oracle/ and synth/ (test infrastructure; "a stored value
is ... written by a committed script that calls only oracle/"). The GPU test
tests/test_gpu_fullsize.py regenerates the same seeded scene (checking the
array hashes stored here), runs the CUDA path through the C ABI and compares.

python tools/golden_fullsize.py matrixcity      (~7 min on 8 cores, ~8 GB RAM)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import make_scene, array_hashes  # noqa: E402

# the second grid of every golden file: fixed non-uniform cuts (fp32), tau 0.3
RAND_CUTS = {"v": [0.23, 0.41, 0.5, 0.66, 0.8], "h": [0.12, 0.35, 0.47, 0.71, 0.9]}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def grid_list(m, n):
    g2 = oracle.default_grid(m, n, v=np.asarray(RAND_CUTS["v"][:m - 1], np.float32),
                             h=np.asarray(RAND_CUTS["h"][:n - 1], np.float32), tau=0.3)
    return [("uniform", oracle.default_grid(m, n)), ("cuts_tau0.3", g2)]


def loads_json(bl):
    out = {k: [int(x) for x in bl[k]] for k in ("n_cams", "g_blk", "g_vis", "incidences")}
    out["area"] = [float(x).hex() for x in bl["area"]]
    out["g_avgvis"] = [float(x).hex() for x in bl["g_avgvis"]]
    out["lohi"] = [[float(np.float32(y)).hex() for y in row] for row in np.asarray(bl["lohi"]).reshape(len(bl["n_cams"]), -1)]
    out["objective"] = int(bl["objective"])
    return out


def main(name):
    t0 = time.time()
    sc = make_scene(name)
    m, n = sc.cfg.m, sc.cfg.n
    print(f"{name}: G={sc.G} N={sc.N} grid {m}x{n}", flush=True)
    o = oracle.run(sc, masks=True)
    print(f"oracle pass {time.time() - t0:.0f} s", flush=True)
    vis = o["vis"]
    gold = {
        "_about": f"Oracle outputs for the full-size {name}-shaped config, written by tools/golden_fullsize.py "
                  "(calls only oracle/ and synth/). Digests are SHA-256 of the C-contiguous little-endian "
                  "arrays: rows = N x ceil(G/32) u32 in caller order (bit i%32 of word i/32); K u32; zmin, zmax "
                  "f32; n, n0 N x B u32; member u64; home i32; crop / eligible = per block ceil(G/64) u64. "
                  "D_c as float.hex (compared within 1e-6 relative). Floats of the records as float.hex.",
        "config": name, "G": sc.G, "N": sc.N, "m": m, "n": n,
        "scene_hashes": array_hashes(sc),
        "frame": {"center": [float(x).hex() for x in o["frame"][0]], "radius": float(o["frame"][1]).hex()},
        "rows_sha256": sha(vis["rows"]),
        "K_sha256": sha(np.asarray(vis["K"], np.uint32)),
        "K_sum": int(np.asarray(vis["K"], np.int64).sum()),
        "zmin_sha256": sha(np.asarray(vis["zmin"], np.float32)),
        "zmax_sha256": sha(np.asarray(vis["zmax"], np.float32)),
        "D": [float(x).hex() for x in vis["D"]],
        "grids": {},
    }
    for gname, g in grid_list(m, n):
        if gname == "uniform":
            asg, bl, cr, el = o["asg"], o["loads"], o["crop"], o["eligible"]
        else:
            asg = oracle.assign(sc, o["pre"], vis, g)
            bl = oracle.block_loads(sc, o["pre"], vis, asg, g, masks=True)
            cr, el = oracle.crop(sc, o["pre"], g, bl["M"])
        gold["grids"][gname] = {
            "v": [float(x).hex() for x in g["v"]], "h": [float(x).hex() for x in g["h"]], "tau": float(g["tau"]),
            "n_sha256": sha(np.asarray(asg["n"], np.uint32)), "n0_sha256": sha(np.asarray(asg["n0"], np.uint32)),
            "member_sha256": sha(np.asarray(asg["member"], np.uint64)),
            "home_sha256": sha(np.asarray(asg["home"], np.int32)),
            "loads": loads_json(bl),
            "crop_sha256": [sha(np.asarray(cr[b], np.uint64)) for b in range(m * n)],
            "eligible_sha256": [sha(np.asarray(el[b], np.uint64)) for b in range(m * n)],
        }
        print(f"grid {gname}: objective {bl['objective']}  {time.time() - t0:.0f} s", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"{name}_oracle.json")
    with open(out, "w") as f:
        json.dump(gold, f, indent=1)
    print("wrote", out, f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "matrixcity")
