"""BO driver (host C++ in liblobe.so, no GPU needed) with the oracle objective.

Pins: SPEC.md:486-495 / SURVEY.md §8c I15 and P3 -- L=1 returns the uniform
cuts, the incumbent never gets worse than uniform, every evaluated cut lies in
the halfway bounds and is strictly increasing, and on 1x2 grids
BO with L >= 30 lands within 5 % of an exhaustive 101-point scan.
"""
import numpy as np
import pytest

import oracle
from paper_2510_01767_b200 import lobe
from synth import make_scene, make_config


@pytest.fixture(scope="module")
def skewed():
    sc = make_scene(make_config("rubble", G=30_000, N=60, m=1, n=2, seed=0xB0, skew=2.0, clusters=6))
    out = oracle.run(sc, grid=oracle.default_grid(1, 2))
    return sc, out


def _objective(sc, out, m, n):
    def f(v, h):
        g = oracle.default_grid(m, n, v=v, h=h)
        return oracle.evaluate_cuts(sc, out["pre"], out["vis"], g)
    return f


def test_L1_returns_uniform(skewed):
    sc, out = skewed
    r = lobe.bo_run(1, 2, _objective(sc, out, 1, 2), L=1)
    assert list(r["h"]) == [np.float32(0.5)]
    assert r["history"][0] == oracle.evaluate_cuts(sc, out["pre"], out["vis"], oracle.default_grid(1, 2))


def test_incumbent_bounds_and_monotone(skewed):
    sc, out = skewed
    m, n = 3, 3
    f = _objective(sc, out, m, n)
    r = lobe.bo_run(m, n, f, L=25, seed=3)
    hist = r["history"].astype(np.int64)
    best = np.minimum.accumulate(hist)
    assert (np.diff(best) <= 0).all()
    assert best[-1] <= hist[0]                              # never worse than uniform
    ch = r["cut_history"]
    for row in ch:
        v, h = row[:m - 1], row[m - 1:]
        for cuts, k in ((v, m), (h, n)):
            assert (np.diff(cuts) > 0).all()
            for i, c in enumerate(cuts, start=1):           # halfway bounds
                assert (2 * i - 1) / (2 * k) <= c <= (2 * i + 1) / (2 * k)
    # returned cuts are the incumbent and re-evaluate to the best value
    assert f(r["v"], r["h"]) == best[-1]
    # determinism
    r2 = lobe.bo_run(m, n, f, L=25, seed=3)
    assert (r2["history"] == r["history"]).all() and (r2["cut_history"] == r["cut_history"]).all()


def test_P3_one_cut_within_5pct_of_scan(skewed):
    sc, out = skewed
    f = _objective(sc, out, 1, 2)
    lo, hi = 0.25 + 1e-6, 0.75 - 1e-6
    scan = min(f(np.zeros(0, np.float32), np.array([np.float32(lo + k * (hi - lo) / 100)], np.float32))
               for k in range(101))
    uniform = f(np.zeros(0, np.float32), np.array([0.5], np.float32))
    fails = 0
    for seed in range(10):
        r = lobe.bo_run(1, 2, f, L=30, seed=seed)
        if int(r["history"].min()) > 1.05 * scan:
            fails += 1
    assert fails == 0, (scan, uniform)
