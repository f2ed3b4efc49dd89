"""Pins of the block-pipeline oracle (SPEC.md:529-571 with
its examples; acceptance criteria #8 and #9 of SPEC.md; ledger L25)."""
import numpy as np
import pytest

import oracle
from tests.helpers import mini_scene

F = np.float32


def _setup(sc, m=2, n=2):
    oracle.validate(sc)
    fr = oracle.frame(sc)
    pre = oracle.prep(sc, fr)
    grid = oracle.default_grid(m, n)
    vis = oracle.visibility(sc, pre)
    asg = oracle.assign(sc, pre, vis, grid)
    bl = oracle.block_loads(sc, pre, vis, asg, grid)
    crop, elig = oracle.crop(sc, pre, grid, bl["M"])
    return fr, pre, grid, vis, asg, bl, crop, elig


def test_subscene_bits_3_7():
    """a crop mask {3, 7} gives a sub-scene of 2 with origin_index {3, 7}."""
    sc = mini_scene([dict(mu=(0.1 * i, 0.0, 5.0)) for i in range(10)],
                    [dict(fx=100.0, fy=100.0, cx=50.0, cy=50.0, width=100, height=100, R=np.eye(3),
                          t=np.zeros(3), z_near=0.1, z_far=100.0)])
    crop = np.zeros(1, np.uint64)
    crop[0] = (1 << 3) | (1 << 7)
    elig = np.zeros(1, np.uint64)
    elig[0] = 1 << 7
    sub = oracle.subscene(sc, crop, elig)
    assert list(sub["origin"]) == [3, 7] and list(sub["in_block"]) == [0, 1]
    assert sub["x"][1] == sc.x[7]


def _sub_manual(n, in_block, s=0.01):
    sub = {k: np.zeros(n, np.float32) for k in oracle.SUB_FIELDS}
    sub["x"] = np.linspace(-0.5, 0.5, n).astype(np.float32)
    sub["z"][:] = 0.0
    for k in ("sx", "sy", "sz"):
        sub[k][:] = s
    sub["qw"][:] = 1.0
    sub["opacity"][:] = 0.5
    sub["origin"] = np.arange(n, dtype=np.int64)
    sub["in_block"] = np.asarray(in_block, np.uint8)
    return sub


def _frame_for(sc):
    fr = oracle.frame(sc)
    pre = oracle.prep(sc, fr)
    return fr, pre["minmax"]


@pytest.fixture(scope="module")
def small():
    from synth.scenes import make_config, make_scene
    sc = make_scene(make_config("tiny", G=2000, N=24, seed=0x2510AB))
    return sc, _setup(sc, 3, 3)


def test_densify_below_threshold_unchanged(small):
    """all grad < tau -> sub-scene unchanged, field for field."""
    sc, (fr, pre, grid, vis, asg, bl, crop, elig) = small
    sub = oracle.subscene(sc, crop[4], elig[4])
    n = len(sub["x"])
    out = oracle.densify_step(sub, np.full(n, 0.1, np.float32), np.zeros((n, 6), np.float32), 1.0, 0.01,
                              fr, pre["minmax"], grid, 4)
    for k in sub:
        assert np.array_equal(out[k], sub[k]), k


def test_densify_split_one_large(small):
    """one eligible large Gaussian above threshold -> count + 1, child
    scales = parent / 1.6, children origin -1; with q = identity the children
    sit at mu + s * n exactly."""
    sc, (fr, pre, grid, vis, asg, bl, crop, elig) = small
    sub = oracle.subscene(sc, crop[4], elig[4])
    j = int(np.flatnonzero(sub["in_block"])[0])
    sub["qw"][j], sub["qx"][j], sub["qy"][j], sub["qz"][j] = 1.0, 0.0, 0.0, 0.0
    n = len(sub["x"])
    grad = np.zeros(n, np.float32)
    grad[j] = 5.0
    nrm = np.zeros((n, 6), np.float32)
    nrm[j] = [0.5, -1.0, 2.0, -0.25, 0.75, 1.5]
    out = oracle.densify_step(sub, grad, nrm, 1.0, 0.0, fr, pre["minmax"], grid, 4)  # scale_split 0: split
    assert len(out["x"]) == n + 1
    for k in range(2):
        c = j + k
        assert out["origin"][c] == -1
        assert out["sx"][c] == F(sub["sx"][j] / F(1.6)) and out["sz"][c] == F(sub["sz"][j] / F(1.6))
        assert out["x"][c] == F(sub["x"][j] + sub["sx"][j] * nrm[j, 3 * k])
        assert out["z"][c] == F(sub["z"][j] + sub["sz"][j] * nrm[j, 3 * k + 2])
    # the rest is untouched and in order
    assert np.array_equal(out["origin"][:j], sub["origin"][:j])
    assert np.array_equal(out["origin"][j + 2:], sub["origin"][j + 1:])


def test_densify_split_rotated():
    """Split offsets follow R(q): a 90 degree turn about z maps (sx nx, sy ny, sz nz)
    to (-sy ny, sx nx, sz nz) (closed form, fp32 rounding of R only)."""
    sub = _sub_manual(1, [1], s=0.02)
    sub["sx"][0], sub["sy"][0], sub["sz"][0] = 0.02, 0.05, 0.01
    c = np.cos(np.pi / 4)
    sub["qw"][0], sub["qz"][0] = c, c
    cam = dict(fx=100.0, fy=100.0, cx=50.0, cy=50.0, width=100, height=100, R=np.eye(3), t=np.zeros(3),
               z_near=0.1, z_far=100.0)
    sc = mini_scene([dict(mu=(-1, -1, 0)), dict(mu=(1, 1, 0.5))],
                    [dict(cam, t=np.array([0.0, 0.0, 5.0])), dict(cam, t=np.array([0.3, 0.1, 5.0]))])
    fr, mm = _frame_for(sc)
    grid = oracle.default_grid(1, 1)
    nrm = np.array([[1.0, 2.0, -1.0, 0.0, 0.0, 0.0]], np.float32)
    out = oracle.densify_step(sub, np.ones(1, np.float32), nrm, 0.5, 0.0, fr, mm, grid, 0)
    d = np.array([out["x"][0] - sub["x"][0], out["y"][0] - sub["y"][0], out["z"][0] - sub["z"][0]])
    want = np.array([-0.05 * 2.0, 0.02 * 1.0, 0.01 * -1.0])
    assert np.allclose(d, want, atol=1e-7)


def test_densify_clone_and_outside(small):
    """Clone (max s < scale_split): both copies jittered by 0.1 s n, the first
    keeps its origin; an out-of-block Gaussian with a huge gradient is untouched."""
    sc, (fr, pre, grid, vis, asg, bl, crop, elig) = small
    sub = oracle.subscene(sc, crop[4], elig[4])
    j = int(np.flatnonzero(sub["in_block"])[0])
    o = int(np.flatnonzero(sub["in_block"] == 0)[0])
    n = len(sub["x"])
    grad = np.zeros(n, np.float32)
    grad[j] = 2.0
    grad[o] = 1e30
    nrm = np.zeros((n, 6), np.float32)
    nrm[j] = [1.0, -2.0, 0.5, 3.0, 0.0, -1.0]
    out = oracle.densify_step(sub, grad, nrm, 1.0, 10.0, fr, pre["minmax"], grid, 4)
    assert len(out["x"]) == n + 1
    jj = j  # clone pair at j, j + 1 (o is before or after; indices shift by one after j)
    assert out["origin"][jj] == sub["origin"][j] and out["origin"][jj + 1] == -1
    for k in range(2):
        assert out["x"][jj + k] == F(sub["x"][j] + F(F(0.1) * sub["sx"][j]) * nrm[j, 3 * k])
        assert out["sx"][jj + k] == sub["sx"][j]
    oo = o if o < j else o + 1
    for key in oracle.SUB_FIELDS:
        assert out[key][oo] == sub[key][o], key


def test_prune_identity_equals_eligible(small):
    """pruning the unchanged sub-scene keeps exactly its in-block
    Gaussians (the eligible mask from the crop step, computed from gu, gv)."""
    sc, (fr, pre, grid, vis, asg, bl, crop, elig) = small
    for b in (0, 4, 8):
        sub = oracle.subscene(sc, crop[b], elig[b])
        pr = oracle.prune_outside(sub, fr, pre["minmax"], grid, b)
        assert np.array_equal(pr["origin"], sub["origin"][sub["in_block"] == 1])


def test_merge_identity_acceptance_9(small):
    """Acceptance #9: the identity pipeline (no densification) merged over a 3x3
    grid recovers, via origin_index, exactly the Gaussians visible from at least
    one assigned camera of their containing block, with no duplicates; set
    computed independently from the rows, the members and the cells."""
    sc, (fr, pre, grid, vis, asg, bl, crop, elig) = small
    subs = []
    for b in range(9):
        sub = oracle.subscene(sc, crop[b], elig[b])
        subs.append(oracle.prune_outside(sub, fr, pre["minmax"], grid, b))
    merged, ok = oracle.merge_blocks(subs)
    assert ok
    G = sc.G
    rows = np.unpackbits(vis["rows"].view(np.uint8), bitorder="little").reshape(sc.N, -1)[:, :G].astype(bool)
    U = np.searchsorted(np.asarray(grid["v"], np.float64), pre["gu"], side="right")
    V = np.searchsorted(np.asarray(grid["h"], np.float64), pre["gv"], side="right")
    cell = U * 3 + V
    want = set()
    for i in range(G):
        b = int(cell[i])
        for c in range(sc.N):
            if (int(asg["member"][c]) >> b) & 1 and rows[c, i]:
                want.add(i)
                break
    assert set(merged["origin"].tolist()) == want and len(merged["origin"]) == len(want)


def test_merge_duplicate_is_integrity_error():
    """an origin index present in two blocks (delta not zeroed before
    pruning) is a merge-integrity error."""
    a = _sub_manual(3, [1, 1, 1])
    b = _sub_manual(2, [1, 1])
    b["origin"][:] = [5, 1]
    _, ok = oracle.merge_blocks([a, b])
    assert not ok
    b["origin"][:] = [5, -1]
    c = _sub_manual(1, [1])
    c["origin"][:] = [-1]
    _, ok = oracle.merge_blocks([a, b, c])
    assert ok


def test_acceptance_8_selective_densification(small):
    """Acceptance #8: 5 densify steps with adversarial gradients (huge outside
    the block): no created Gaussian has an out-of-block parent, and every
    ineligible Gaussian is unchanged field for field."""
    sc, (fr, pre, grid, vis, asg, bl, crop, elig) = small
    rng = np.random.default_rng(5)
    sub = oracle.subscene(sc, crop[4], elig[4])
    for step in range(5):
        n = len(sub["x"])
        grad = np.where(sub["in_block"] == 1, rng.uniform(0, 2, n), 1e30).astype(np.float32)
        nrm = rng.normal(size=(n, 6)).astype(np.float32)
        out = oracle.densify_step(sub, grad, nrm, 1.0, 0.004, fr, pre["minmax"], grid, 4)
        # walk input / output in order: selected Gaussians become two entries
        k = 0
        for i in range(n):
            sel = sub["in_block"][i] == 1 and grad[i] >= 1.0
            if not sel:
                for key in oracle.SUB_FIELDS + ("origin", "in_block"):
                    assert out[key][k] == sub[key][i]
                k += 1
            else:
                assert sub["in_block"][i] == 1  # parent in the block
                k += 2
        assert k == len(out["x"])
        sub = out
