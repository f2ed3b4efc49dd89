"""Full-size oracle parity of every output (§4.3: G_vis
is the objective), at the BASELINE configs' full sizes and in the launch
configuration bench.py times.

- Rubble-, Building- and Residence-shaped (and Rubble in the anisotropic
  mode): the oracle runs live on the host cores (tens of seconds each) and
  every output is compared element by element:
  rows of all cameras, K, D_c (1e-6 relative), z_min, z_max, n, n0, member, home,
  all block records, crop and eligible masks, on the uniform cuts and a second
  grid with non-uniform cuts and tau = 0.3.
- MatrixCity-shaped (10M x 5620; the oracle needs ~7 min on 8 cores): against
  tests/golden/matrixcity_oracle.json, written by tools/golden_fullsize.py,
  which calls only oracle/ -- SHA-256 digests of the rows (7 GB, hashed in camera
  chunks), per-camera arrays and every block's crop / eligible mask, the block
  records in full and D_c within 1e-6.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from synth import make_scene, array_hashes
from tests.test_gpu_parity import _lobe, full_parity, check_i16, D_RTOL

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RAND_CUTS = {"v": [0.23, 0.41, 0.5, 0.66, 0.8], "h": [0.12, 0.35, 0.47, 0.71, 0.9]}  # tools/golden_fullsize.py


def _grids(m, n):
    return [oracle.default_grid(m, n),
            oracle.default_grid(m, n, v=np.asarray(RAND_CUTS["v"][:m - 1], np.float32),
                                h=np.asarray(RAND_CUTS["h"][:n - 1], np.float32), tau=0.3)]


@pytest.mark.parametrize("name", ["rubble", "building", "residence"])
def test_fullsize_live_oracle(name):
    sc = make_scene(name)
    full_parity(sc, _grids(sc.cfg.m, sc.cfg.n))


def test_fullsize_bo_trajectory_rubble():
    """a10 at full Rubble size: every evaluation of lobe_balance_partition (L = 8:
    the uniform cuts, Sobol points, then GP + EI proposals) equals the oracle's
    objective at the recorded cuts, so an oracle-backed BO follows the same
    trajectory."""
    lobe = _lobe()
    sc = make_scene("rubble")
    m, n = sc.cfg.m, sc.cfg.n
    o = oracle.run(sc, masks=False)
    with lobe.Scene(sc, sc) as S:
        r = S.balance_partition(m, n, L=8, seed=2)
    for row, val in zip(r["cut_history"], r["history"]):
        g = oracle.default_grid(m, n, v=row[:m - 1], h=row[m - 1:])
        assert oracle.evaluate_cuts(sc, o["pre"], o["vis"], g) == val
    assert r["best"]["objective"] == r["history"].min() <= r["history"][0]


def test_fullsize_live_oracle_aniso_rubble():
    """The anisotropic (EWA) predicate mode at the full Rubble-shaped size: every
    output against the oracle's O6a, element by element (~30 s of oracle on
    16 cores)."""
    sc = make_scene("rubble")
    full_parity(sc, _grids(sc.cfg.m, sc.cfg.n), predicate=1)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _fx(h):
    return float.fromhex(h)


@pytest.mark.parametrize("name", ["matrixcity"])
def test_fullsize_golden(name):
    path = os.path.join(GOLDEN, f"{name}_oracle.json")
    gold = json.load(open(path))
    lobe = _lobe()
    sc = make_scene(name)
    assert array_hashes(sc) == gold["scene_hashes"], "generated scene differs from the golden file's"
    m, n = sc.cfg.m, sc.cfg.n
    with lobe.Scene(sc, sc) as S:
        assert [float(x) for x in S.frame["center"]] == [_fx(x) for x in gold["frame"]["center"]]
        assert float(S.frame["radius"]) == _fx(gold["frame"]["radius"])
        h = hashlib.sha256()
        step = 256
        for c0 in range(0, sc.N, step):
            h.update(S.export_rows(c0, min(step, sc.N - c0)).tobytes())
        assert h.hexdigest() == gold["rows_sha256"]
        for gname, g in zip(("uniform", "cuts_tau0.3"), _grids(m, n)):
            gg = gold["grids"][gname]
            assert [float(x).hex() for x in g["v"]] == gg["v"] and [float(x).hex() for x in g["h"]] == gg["h"]
            kw = dict(v=g["v"], h=g["h"], delta_v=float(g["dv"]), delta_h=float(g["dh"]), tau=float(g["tau"]))
            a = S.assign_cameras(m, n, **kw)
            if gname == "uniform":
                assert _sha(a["K"]) == gold["K_sha256"]
                assert _sha(a["zmin"]) == gold["zmin_sha256"] and _sha(a["zmax"]) == gold["zmax_sha256"]
                D = np.array([_fx(x) for x in gold["D"]])
                np.testing.assert_allclose(a["D"], D, rtol=D_RTOL, atol=0)
                assert ((a["D"] == 0) == (D == 0)).all()
                check_i16(S.stats(), sc.G, sc.N, gold["K_sum"])
            for k in ("n", "n0", "member", "home"):
                assert _sha(a[k]) == gg[f"{k}_sha256"], (gname, k)
            L = S.block_loads(m, n, **kw)
            gl = gg["loads"]
            for k in ("n_cams", "g_blk", "g_vis", "incidences"):
                assert [int(x) for x in L[k]] == gl[k], (gname, k)
            assert [float(x).hex() for x in L["area"]] == gl["area"]
            assert [float(x).hex() for x in L["g_avgvis"]] == gl["g_avgvis"]
            assert [[float(y).hex() for y in r] for r in L["lohi"]] == gl["lohi"]
            assert L["objective"] == gl["objective"]
            c, e = S.crop_masks(m, n, **kw)
            assert [_sha(c[b]) for b in range(m * n)] == gg["crop_sha256"], gname
            assert [_sha(e[b]) for b in range(m * n)] == gg["eligible_sha256"], gname
