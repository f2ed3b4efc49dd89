"""Oracle pins against things other than itself: float64 brute force of SPEC's
formula (B1), set-level enumeration (B2), invariants I1-I14 and special
cases P1-P6 of SURVEY.md §8(c).
"""
import numpy as np
import pytest

import oracle
from oracle.brute import predicate_f64
from synth import make_scene, make_config
from tests.helpers import bits_of_row, bits_of_mask64


@pytest.fixture(scope="module")
def tiny_run(tiny_scene):
    return oracle.run(tiny_scene)


@pytest.fixture(scope="module")
def small_scene():
    return make_scene(make_config("rubble", G=20_000, N=48, seed=0x1234))


@pytest.fixture(scope="module")
def small_run(small_scene):
    return oracle.run(small_scene)


def _unpack_rows(rows, G):
    bits = np.unpackbits(rows.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :G].astype(bool)


# ------------------------------------------------------------------ B1
@pytest.mark.parametrize("which", ["tiny", "small"])
def test_B1_fp64_spec_formula(which, tiny_scene, tiny_run, small_scene, small_run):
    """The pinned fp32 predicate agrees with SPEC.md:243/:299 evaluated in
    float64 on every pair whose float64 margin exceeds 1e-5."""
    sc, out = (tiny_scene, tiny_run) if which == "tiny" else (small_scene, small_run)
    vis64, margin = predicate_f64(sc)
    vis32 = _unpack_rows(out["vis"]["rows"], sc.G)
    outside = margin > 1e-5
    bad = (vis64 != vis32) & outside
    assert bad.sum() == 0, f"{bad.sum()} disagreements outside the boundary band"
    inband = (vis64 != vis32) & ~outside
    assert inband.sum() <= 10  # reported: expected ~0 on generic data
    assert vis32.sum() > 0.05 * vis32.size if which == "tiny" else vis32.sum() > 0


# ------------------------------------------------------------------ B2
@pytest.mark.parametrize("G,N,seed", [(12, 3, 1), (200, 6, 2), (1000, 16, 3)])
def test_B2_set_enumeration(G, N, seed):
    """Assignments, G_vis and crops from plain Python sets:
    V_c from the float64 brute force (B1), ratio test with exact rationals
    n * 20 >= 3 * K (tau = 3/20), regions from the paper's
    interval definition evaluated on the oracle's grid coords."""
    sc = make_scene(make_config("tiny", G=G, N=N, seed=seed))
    out = oracle.run(sc)
    pre, grid = out["pre"], out["grid"]
    vis64, margin = predicate_f64(sc)
    V = [set(np.nonzero(vis64[c])[0].tolist()) for c in range(N)]
    for c in range(N):
        if (margin[c] > 1e-5).all():
            assert V[c] == bits_of_row(out["vis"]["rows"][c], G)
    V = [bits_of_row(out["vis"]["rows"][c], G) for c in range(N)]
    m, n = grid["m"], grid["n"]
    gu, gv = pre["gu"].astype(float), pre["gv"].astype(float)

    def bounds(cuts, cnt, delta):
        edges = [0.0] + [float(c) for c in cuts] + [1.0]
        res = []
        for p in range(cnt):
            lo, hi = edges[p], edges[p + 1]
            elo = float(np.float32(max(0.0, float(np.float32(np.float32(lo) - np.float32(delta))))))
            ehi = float(np.float32(min(1.0, float(np.float32(np.float32(hi) + np.float32(delta))))))
            res.append(((lo, hi), (elo, ehi)))
        return res

    def inside(x, lo, hi):
        return x >= lo and (x < hi or (hi == 1.0 and x <= 1.0))

    U = bounds(grid["v"], m, grid["dv"])
    Vb = bounds(grid["h"], n, grid["dh"])
    members = []
    for c in range(N):
        K = len(V[c])
        mem = set()
        for p in range(m):
            for q in range(n):
                cnt = sum(1 for i in V[c] if inside(gu[i], *U[p][1]) and inside(gv[i], *Vb[q][1]))
                if K > 0 and cnt * 20 >= 3 * K:
                    mem.add(p * n + q)
        members.append(mem)
        assert mem == {b for b in range(m * n) if (int(out["asg"]["member"][c]) >> b) & 1}
    for b in range(m * n):
        cams = [c for c in range(N) if b in members[c]]
        union = set().union(*[V[c] for c in cams]) if cams else set()
        assert out["loads"]["g_vis"][b] == len(union)
        assert out["loads"]["n_cams"][b] == len(cams)
        assert bits_of_mask64(out["crop"][b], G) == union
        p, q = divmod(b, n)
        cell = {i for i in range(G) if inside(gu[i], *U[p][0]) and inside(gv[i], *Vb[q][0])}
        assert bits_of_mask64(out["eligible"][b], G) == union & cell
        assert out["loads"]["g_blk"][b] == len(cell)
    assert out["loads"]["objective"] == max(out["loads"]["g_vis"])


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("which", ["tiny", "small"])
def test_invariants_I1_to_I10(which, tiny_scene, tiny_run, small_scene, small_run):
    sc, out = (tiny_scene, tiny_run) if which == "tiny" else (small_scene, small_run)
    G, N = sc.G, sc.N
    vis, asg, L = out["vis"], out["asg"], out["loads"]
    B = out["grid"]["m"] * out["grid"]["n"]
    rows = _unpack_rows(vis["rows"], G)
    crops = [np.unpackbits(out["crop"][b].view(np.uint8), bitorder="little")[:G].astype(bool) for b in range(B)]
    member = asg["member"].astype(np.uint64)
    for b in range(B):
        cams = [c for c in range(N) if (int(member[c]) >> b) & 1]
        for c in cams:                                            # I1 crop superset
            assert not (rows[c] & ~crops[b]).any()
        Ks = [int(vis["K"][c]) for c in cams]                     # I9 bounds
        if cams:
            assert max(Ks) <= L["g_vis"][b] <= min(G, sum(Ks))
            assert L["g_avgvis"][b] * L["n_cams"][b] == pytest.approx(L["g_vis"][b], rel=1e-15)   # I10
        else:
            assert L["g_vis"][b] == 0 and L["g_avgvis"][b] == 0
    assert int(L["incidences"].sum()) == int(vis["K"].astype(np.int64).sum())    # I2
    assert ((asg["home"] >= 0) & (asg["home"] < B)).all()                          # I3
    assert int(L["g_blk"].astype(np.int64).sum()) == G                            # I4
    assert (asg["n0"].sum(axis=1) == vis["K"]).all()                               # I5
    assert (asg["n"] >= asg["n0"]).all()                                           # I6
    assert (vis["K"] == rows.sum(axis=1)).all()
    # depth statistic sanity (D_c parity is otherwise unpinned, ledger L4)
    k = vis["K"] > 0
    assert (vis["D"][k] >= vis["zmin"][k] - 1e-6).all() and (vis["D"][k] <= vis["zmax"][k] + 1e-6).all()
    assert (vis["D"][~k] == 0).all()
    # home cell holds the most points (argmax definition)
    assert (asg["n0"][np.arange(N), asg["home"]] == asg["n0"].max(axis=1))[k].all()


def test_I7_tau_monotone_and_P2(small_scene, small_run):
    sc, out = small_scene, small_run
    prev = None
    for tau in (0.0, 0.05, 0.15, 0.3, 0.6, 1.0):
        grid = dict(out["grid"], tau=tau)
        asg = oracle.assign(sc, out["pre"], out["vis"], grid)
        mem = asg["member"].astype(np.uint64)
        if prev is not None:
            assert ((mem & ~prev) == 0).all()         # C^(b)(tau2) subset of C^(b)(tau1)
        if tau == 0.0:                                # P2: every K>0 camera in every block
            B = grid["m"] * grid["n"]
            full = np.uint64((1 << B) - 1)
            assert (mem[out["vis"]["K"] > 0] == full).all()
        prev = mem


def test_I8_union_monotone(small_scene, small_run):
    out = small_run
    rows = _unpack_rows(out["vis"]["rows"], small_scene.G)
    acc = np.zeros(small_scene.G, bool)
    last = 0
    for c in range(small_scene.N):
        acc |= rows[c]
        assert acc.sum() >= last
        last = acc.sum()


def test_P1_one_block_is_union(small_scene, small_run):
    sc, out = small_scene, small_run
    grid = oracle.default_grid(1, 1)
    asg = oracle.assign(sc, out["pre"], out["vis"], grid)
    bl = oracle.block_loads(sc, out["pre"], out["vis"], asg, grid)
    rows = _unpack_rows(out["vis"]["rows"], sc.G)
    assert bl["g_vis"][0] == rows.any(axis=0).sum()
    assert bl["n_cams"][0] == (out["vis"]["K"] > 0).sum()


def test_P4_delta_zero_cells(small_scene, small_run):
    sc, out = small_scene, small_run
    grid = dict(out["grid"], dv=np.float32(0), dh=np.float32(0))
    asg = oracle.assign(sc, out["pre"], out["vis"], grid)
    assert (asg["n"] == asg["n0"]).all()


def test_P6_duplicate_camera_and_I14_camera_order(small_scene, small_run):
    sc = small_scene
    idx = np.r_[np.arange(sc.N)[::-1], 5]            # reversed order + a duplicate of camera 5
    sc2 = sc.subset_cameras(idx)
    fr = small_run["frame"]
    out2 = oracle.run(sc2, frame_args=dict(center=fr[0], radius=fr[1], axis_u=fr[2], axis_v=fr[3]))
    r1 = small_run["vis"]["rows"]
    r2 = out2["vis"]["rows"]
    assert (r2[:-1] == r1[::-1]).all()
    assert (r2[-1] == r1[5]).all()                     # P6
    assert (out2["asg"]["member"][:-1] == small_run["asg"]["member"][::-1]).all()


def test_I13_permutation_invariance(small_scene, small_run):
    sc = small_scene
    perm = np.random.default_rng(7).permutation(sc.G)
    sc2 = sc.permute_gaussians(perm)
    out2 = oracle.run(sc2)
    for key in ("g_vis", "g_blk", "n_cams", "incidences"):
        assert (out2["loads"][key] == small_run["loads"][key]).all(), key
    assert (out2["vis"]["K"] == small_run["vis"]["K"]).all()
    assert (out2["asg"]["member"] == small_run["asg"]["member"]).all()
    assert (out2["vis"]["zmin"] == small_run["vis"]["zmin"]).all()
    assert out2["vis"]["D"] == pytest.approx(small_run["vis"]["D"], rel=1e-12)
    rows1 = _unpack_rows(small_run["vis"]["rows"], sc.G)
    rows2 = _unpack_rows(out2["vis"]["rows"], sc.G)
    assert (rows2 == rows1[:, perm]).all()
    B = small_run["grid"]["m"] * small_run["grid"]["n"]
    for b in range(B):
        c1 = np.unpackbits(small_run["crop"][b].view(np.uint8), bitorder="little")[:sc.G]
        c2 = np.unpackbits(out2["crop"][b].view(np.uint8), bitorder="little")[:sc.G]
        assert (c2 == c1[perm]).all()


def test_I11_determinism(small_scene, small_run):
    out2 = oracle.run(small_scene)
    assert (out2["vis"]["rows"] == small_run["vis"]["rows"]).all()
    assert (out2["vis"]["S"] == small_run["vis"]["S"]).all()
    assert (out2["crop"] == small_run["crop"]).all()


def test_tiny_every_camera_sees_something(tiny_run):
    """the generator's cameras all see >= 1 Gaussian (tiny config)."""
    assert (tiny_run["vis"]["K"] > 0).all()


def test_modes_home_and_union(small_scene, small_run):
    sc, out = small_scene, small_run
    B = out["grid"]["m"] * out["grid"]["n"]
    lh = oracle.block_loads(sc, out["pre"], out["vis"], out["asg"], out["grid"], mode=oracle.MODE_HOME)
    lu = oracle.block_loads(sc, out["pre"], out["vis"], out["asg"], out["grid"], mode=oracle.MODE_UNION)
    assert int(lh["n_cams"].sum()) == sc.N                      # every camera has exactly one home (I3)
    assert (lu["g_vis"] >= np.maximum(lh["g_vis"], out["loads"]["g_vis"])).all()
    assert (lu["n_cams"] >= lh["n_cams"]).all()


# ------------------------------------------------------------------ D_c, z_min, z_max
@pytest.mark.parametrize("which", ["tiny", "small"])
def test_depth_statistic_float64_route(which, tiny_scene, tiny_run, small_scene, small_run):
    """Ledger L4: D_c is the opacity-weighted mean camera depth over V_c and
    z_min / z_max its extremes. Recomputed by another route -- the camera-frame
    depth (R x + t)_z of each visible Gaussian in float64 from the caller's
    extrinsics (not the oracle's fp32 setup rows), weighted by the caller's
    opacities -- it must match the oracle within the fp32 rounding of w (1e-5).
    A wrong row, sign, translation or weight fails this."""
    sc, out = (tiny_scene, tiny_run) if which == "tiny" else (small_scene, small_run)
    vis = _unpack_rows(out["vis"]["rows"], sc.G)
    P = np.stack([sc.x, sc.y, sc.z], 1).astype(np.float64)
    o = sc.opacity.astype(np.float64)
    checked = 0
    for c in range(sc.N):
        idx = np.flatnonzero(vis[c])
        if len(idx) == 0:
            assert out["vis"]["D"][c] == 0.0
            continue
        depth = P[idx] @ sc.R[c].astype(np.float64)[2] + float(sc.t[c][2])
        D = float((o[idx] * depth).sum() / o[idx].sum())
        assert out["vis"]["D"][c] == pytest.approx(D, rel=1e-5), c
        assert out["vis"]["zmin"][c] == pytest.approx(depth.min(), rel=1e-5), c
        assert out["vis"]["zmax"][c] == pytest.approx(depth.max(), rel=1e-5), c
        checked += 1
    assert checked > 0
