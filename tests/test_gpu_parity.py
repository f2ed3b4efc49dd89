"""GPU <-> oracle parity through the C ABI (csrc/liblobe.so).

Bar (BASELINE.json north_star): counts, assignments, rows and masks bit-exact;
depth statistics within 1e-6 relative.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import make_scene, make_config
from tests.helpers import mini_scene, nadir_camera

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")))
D_RTOL = 1e-6


def _lobe():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_01767_b200 import lobe
    return lobe


def _grid_kw(g):
    return dict(v=g["v"], h=g["h"], delta_v=float(g["dv"]), delta_h=float(g["dh"]), tau=float(g["tau"]))


def _cmp_percam(a, o_vis, o_asg, sel=None):
    sl = slice(None) if sel is None else sel
    assert (a["K"][sl] == o_vis["K"]).all()
    assert (a["zmin"][sl] == o_vis["zmin"]).all() and (a["zmax"][sl] == o_vis["zmax"]).all()
    np.testing.assert_allclose(a["D"][sl], o_vis["D"], rtol=D_RTOL, atol=0)
    assert ((a["D"][sl] == 0) == (o_vis["K"] == 0)).all()
    assert (a["n"][sl] == o_asg["n"]).all()
    assert (a["n0"][sl] == o_asg["n0"]).all()
    assert (a["member"][sl] == o_asg["member"]).all()
    assert (a["home"][sl] == o_asg["home"]).all()


def _cmp_loads(L, o):
    for k in ("n_cams", "g_blk", "g_vis", "incidences"):
        assert (L[k] == o[k]).all(), k
    assert (L["area"] == o["area"]).all()
    assert (L["g_avgvis"] == o["g_avgvis"]).all()
    assert (L["lohi"] == o["lohi"]).all()
    assert L["objective"] == o["objective"]


def check_i16(st, G, n_local, K_sum):
    """I16, measured inside the kernels: every one of the G x N_local
    logical tests of the visibility pass was decided exactly once -- by k_cull's
    chunk / tile bound, by k_vis_tiles' slice bound (rejected / accepted) or by
    the exact test -- and the visible bits the kernel wrote add up to sum_c K_c
    (K comes from the separate depth-statistic kernel)."""
    d = [int(x) for x in st.decided_tests]
    assert sum(d) == G * n_local, (d, G, n_local)
    assert int(st.visible_bits[0]) + int(st.visible_bits[1]) == int(K_sum)
    assert d[3] <= st.dense_tests and d[2] <= st.accepted_tests  # padding only adds to the executed counts


def full_parity(sc, grids, mode=0, predicate=0):
    lobe = _lobe()
    with lobe.Scene(sc, sc, assign_mode=mode, predicate=predicate) as S:
        o0 = oracle.run(sc, grid=grids[0], mode=mode, predicate=predicate)
        c0, rho, au, av = o0["frame"]
        assert (S.frame["center"] == c0).all() and S.frame["radius"] == rho
        rows = S.export_rows()
        assert (rows == o0["vis"]["rows"]).all()
        st = S.stats()
        check_i16(st, sc.G, sc.N, np.asarray(o0["vis"]["K"], np.int64).sum())
        assert st.tests_executed == sc.G * sc.N
        for g in grids:
            o = o0 if g is grids[0] else None
            if o is None:
                asg = oracle.assign(sc, o0["pre"], o0["vis"], g)
                bl = oracle.block_loads(sc, o0["pre"], o0["vis"], asg, g, mode=mode)
                cr, el = oracle.crop(sc, o0["pre"], g, bl["M"])
            else:
                asg, bl, cr, el = o["asg"], o["loads"], o["crop"], o["eligible"]
            a = S.assign_cameras(g["m"], g["n"], **_grid_kw(g))
            _cmp_percam(a, o0["vis"], asg)
            L = S.block_loads(g["m"], g["n"], **_grid_kw(g))
            _cmp_loads(L, bl)
            c, e = S.crop_masks(g["m"], g["n"], **_grid_kw(g))
            assert (c == cr).all() and (e == el).all()
    return st


def _rand_grid(m, n, seed, **kw):
    rng = np.random.default_rng(seed)
    v = np.sort(rng.uniform(0.05, 0.95, m - 1)).astype(np.float32)
    h = np.sort(rng.uniform(0.05, 0.95, n - 1)).astype(np.float32)
    return oracle.default_grid(m, n, v=v, h=h, **kw)


def test_tiny_full(tiny_scene):
    full_parity(tiny_scene, [oracle.default_grid(2, 2), oracle.default_grid(1, 1), _rand_grid(3, 3, 1),
                             oracle.default_grid(2, 2, tau=0.0), oracle.default_grid(2, 2, delta_v=0, delta_h=0)])


@pytest.mark.parametrize("mode", [1, 2])
def test_tiny_modes(tiny_scene, mode):
    full_parity(tiny_scene, [oracle.default_grid(2, 2), _rand_grid(4, 3, 2)], mode=mode)


def test_ragged_multi_tile():
    """G not a multiple of the tile / chunk / word sizes, N not a multiple of the camera group."""
    sc = make_scene(make_config("residence", G=37_123, N=53, seed=0x5151))
    full_parity(sc, [oracle.default_grid(4, 4), _rand_grid(6, 6, 3), _rand_grid(8, 8, 4, tau=0.05),
                     oracle.default_grid(1, 7), oracle.default_grid(2, 2, tau=1.0)])


@pytest.mark.parametrize("groups", ["1", "2"])
def test_block_masks_group_overflow(groups, monkeypatch):
    """k_block_masks groups a tile's cameras by assignment set in a 64-slot hash
    table; with the table cut to 1 or 2 slots (LOBE_MASK_GROUPS, read at every
    launch) most cameras take the direct path. Loads and crop masks must not
    change."""
    monkeypatch.setenv("LOBE_MASK_GROUPS", groups)
    sc = make_scene(make_config("residence", G=37_123, N=53, seed=0x5151))
    full_parity(sc, [_rand_grid(8, 8, 4, tau=0.05), oracle.default_grid(4, 4)])


def test_call_orders(tiny_scene):
    """The evaluation's block counts reach the host asynchronously and the
    per-camera copies run on a side stream: crop first (device outputs), then
    loads and assignment, with a second grid evaluated in between, must give
    the oracle's results for both grids."""
    import torch
    lobe = _lobe()
    sc = tiny_scene
    g1, g2 = oracle.default_grid(2, 2), _rand_grid(3, 2, 7)
    o = oracle.run(sc, grid=g1)
    asg2 = oracle.assign(sc, o["pre"], o["vis"], g2)
    bl2 = oracle.block_loads(sc, o["pre"], o["vis"], asg2, g2)
    with lobe.Scene(sc, sc) as S:
        W64 = (sc.G + 63) // 64
        cd = torch.empty(4 * W64, dtype=torch.int64, device="cuda")
        ed = torch.empty(4 * W64, dtype=torch.int64, device="cuda")
        S.crop_masks_into(2, 2, cd, ed)
        L2 = S.block_loads(3, 2, **_grid_kw(g2))           # another grid in between
        L1 = S.block_loads(2, 2)
        a1 = S.assign_cameras(2, 2)
        torch.cuda.synchronize()
        crop = cd.cpu().numpy().view(np.uint64).reshape(4, W64)
        elig = ed.cpu().numpy().view(np.uint64).reshape(4, W64)
        a2 = S.assign_cameras(3, 2, **_grid_kw(g2))
    _cmp_loads(L1, o["loads"])
    _cmp_loads(L2, bl2)
    _cmp_percam(a1, o["vis"], o["asg"])
    _cmp_percam(a2, o["vis"], asg2)
    assert (crop == o["crop"]).all() and (elig == o["eligible"]).all()


def test_zone_bins_dense_and_aligned_cuts():
    """The zone lookup bins (1/1024 wide): three cuts inside one bin (binary-search
    fallback), cuts exactly on bin edges (0.25, 0.5, 0.75) and a point-dense
    scene, with and without enlargement: counts, assignment, loads and masks
    stay bit-exact."""
    sc = make_scene(make_config("residence", G=37_123, N=53, seed=0x5151))
    v = np.array([0.3, 0.3001, 0.3002], np.float32)
    h = np.array([0.25, 0.5, 0.75], np.float32)
    full_parity(sc, [oracle.default_grid(4, 4, v=v, h=h), oracle.default_grid(4, 4, v=v, h=h, delta_v=0.0,
                                                                               delta_h=0.0),
                     oracle.default_grid(4, 4, v=h, h=v, delta_v=0.0001, delta_h=0.25)])


def test_mid_size():
    sc = make_scene(make_config("matrixcity", G=150_000, N=120, seed=0x77))
    full_parity(sc, [oracle.default_grid(6, 6), _rand_grid(5, 4, 9)])


@pytest.mark.parametrize("case", GOLD["visibility"], ids=[c["id"] for c in GOLD["visibility"]])
def test_hand_visibility_gpu(case):
    lobe = _lobe()
    anchors = [dict(mu=[-50, -50, -50], s=0.01, o=0.0), dict(mu=[50, 50, 50], s=0.01, o=0.0)]
    sc = mini_scene([dict(mu=case["mu"], s=case["s"], o=case["o"])] + anchors, [GOLD["camera_C0"]])
    fr = dict(center=[0, 0, 0], radius=1.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    with lobe.Scene(sc, sc, frame=fr) as S:
        rows = S.export_rows()
        assert bool(rows[0, 0] & 1) == case["visible"], case["id"]


def test_hand_depth_H7_gpu():
    lobe = _lobe()
    d = GOLD["depth_stat"]
    g = [dict(mu=x["mu"], s=x["s"], o=x["o"]) for x in d["gaussians"]]
    g += [dict(mu=[-50, -50, -50], s=0.01, o=0.0), dict(mu=[50, 50, 50], s=0.01, o=0.0)]
    sc = mini_scene(g, [GOLD["camera_C0"]])
    with lobe.Scene(sc, sc, frame=dict(center=[0, 0, 0], radius=1.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])) as S:
        a = S.assign_cameras(1, 1)
        assert a["K"][0] == d["K"] and a["D"][0] == pytest.approx(d["D"], rel=1e-15)
        assert a["zmin"][0] == d["z_min"] and a["zmax"][0] == d["z_max"]


@pytest.mark.parametrize("case", GOLD["frame_auto"]["cases"], ids=[c["id"] for c in GOLD["frame_auto"]["cases"]])
def test_hand_frame_auto_gpu(case):
    """O2 automatic frame resolved by lobe_load_scene equals the hand-worked
    centre and radius (tests/golden/hand_cases.json frame_auto)."""
    from tests.test_oracle_hand import frame_cameras, FRAME_GAUSSIANS
    lobe = _lobe()
    extra = "extra_identity_camera_t" in case
    sc = mini_scene(FRAME_GAUSSIANS, frame_cameras(case, extra=extra))
    with lobe.Scene(sc, sc) as S:
        assert list(S.frame["center"]) == [np.float32(v) for v in case["center"]], case["why"]
        assert S.frame["radius"] == np.float32(case["radius"]), case["why"]
        assert list(S.frame["axis_u"]) == [1, 0, 0] and list(S.frame["axis_v"]) == [0, 1, 0]
    if extra:
        sc0 = mini_scene(FRAME_GAUSSIANS, frame_cameras(case))
        with pytest.raises(lobe.LobeError) as e:
            lobe.Scene(sc0, sc0)
        assert e.value.code == 5  # LOBE_E_DEGENERATE_SCENE


def test_hand_assignment_H9_gpu():
    lobe = _lobe()
    a = GOLD["assignment"]
    rng = np.random.default_rng(0)
    g = [dict(mu=x["mu"], s=x["s"], o=x["o"]) for x in a["anchors"]]
    for cl in (a["cluster_low"], a["cluster_high"]):
        for _ in range(cl["count"]):
            g.append(dict(mu=np.asarray(cl["center"], float) + np.r_[rng.uniform(-0.05, 0.05, 2), 0.0], s=0.001,
                          o=0.9))
    sc = mini_scene(g, [nadir_camera(*a["camera"]["nadir_at"], f=a["camera"]["f"])], m=2, n=2)
    with lobe.Scene(sc, sc, frame=dict(center=[0, 0, 0], radius=10.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])) as S:
        r = S.assign_cameras(2, 2, delta_v=0.05, delta_h=0.05, tau=0.15)
        e = a["expect"]
        assert r["K"][0] == e["K"] and list(r["n"][0]) == e["n"] and list(r["n0"][0]) == e["n0"]
        assert [b for b in range(4) if (int(r["member"][0]) >> b) & 1] == e["member_tau_0.15"]
        assert r["home"][0] == e["home"]
        r = S.assign_cameras(2, 2, delta_v=0.05, delta_h=0.05, tau=0.5)
        assert [b for b in range(4) if (int(r["member"][0]) >> b) & 1] == e["member_tau_0.5"]


def test_determinism_and_permutation(tiny_scene):
    lobe = _lobe()
    sc = tiny_scene
    with lobe.Scene(sc, sc) as A, lobe.Scene(sc, sc) as B:
        assert (A.export_rows() == B.export_rows()).all()
        a, b = A.assign_cameras(2, 2), B.assign_cameras(2, 2)
        for k in a:
            assert (a[k] == b[k]).all(), k                      # I11: identical bytes (D included)
    perm = np.random.default_rng(3).permutation(sc.G)
    sc2 = sc.permute_gaussians(perm)
    with lobe.Scene(sc, sc) as A, lobe.Scene(sc2, sc2) as B:
        la, lb = A.block_loads(2, 2), B.block_loads(2, 2)
        for k in ("g_vis", "g_blk", "n_cams", "incidences"):
            assert (la[k] == lb[k]).all()                       # I13
        ra, rb = A.export_rows(), B.export_rows()
        ua = np.unpackbits(ra.view(np.uint8), axis=1, bitorder="little")[:, :sc.G]
        ub = np.unpackbits(rb.view(np.uint8), axis=1, bitorder="little")[:, :sc.G]
        assert (ub == ua[:, perm]).all()


def test_camera_order_invariance_and_duplicates_gpu():
    """I14: permuting the cameras permutes every per-camera output and leaves the
    block loads and masks unchanged; P6: a duplicated camera gets identical rows
    and per-camera outputs."""
    lobe = _lobe()
    sc = make_scene(make_config("residence", G=37_123, N=53, seed=0x5151))
    perm = np.random.default_rng(5).permutation(sc.N)
    sp = sc.subset_cameras(perm)
    with lobe.Scene(sc, sc) as A, lobe.Scene(sp, sp) as Bs:
        for m, n in ((4, 4), (3, 2)):
            la, lb = A.block_loads(m, n), Bs.block_loads(m, n)
            for k in ("n_cams", "g_vis", "g_blk", "incidences", "g_avgvis", "area", "lohi"):
                assert (la[k] == lb[k]).all(), k
            ca, ea = A.crop_masks(m, n)
            cb, eb = Bs.crop_masks(m, n)
            assert (ca == cb).all() and (ea == eb).all()
            aa, ab = A.assign_cameras(m, n), Bs.assign_cameras(m, n)
            for k in aa:
                assert (aa[k][perm] == ab[k]).all(), k
        assert (A.export_rows()[perm] == Bs.export_rows()).all()
    dup = sc.subset_cameras(np.r_[np.arange(sc.N), [7, 7]])
    with lobe.Scene(dup, dup) as D:
        rows = D.export_rows()
        assert (rows[7] == rows[sc.N]).all() and (rows[7] == rows[sc.N + 1]).all()
        a = D.assign_cameras(4, 4)
        for k in a:
            assert (a[k][7] == a[k][sc.N]).all(), k


def test_world_shards_match_world1():
    """Camera sharding on one GPU, ranks run one after another:
    per-camera outputs concatenate, OR-combined partial masks equal world=1."""
    import torch
    lobe = _lobe()
    sc = make_scene(make_config("rubble", G=60_000, N=41, seed=0x99))
    m, n = 3, 3
    with lobe.Scene(sc, sc) as S1:
        ref = S1.assign_cameras(m, n)
        L1 = S1.block_loads(m, n)
        c1, e1 = S1.crop_masks(m, n)
        words = S1.mask_words()
    for W in (2, 3):
        parts, outs, ncs, incs = [], [], [], []
        scenes = [lobe.Scene(sc, sc, rank=r, world=W) for r in range(W)]
        try:
            for S in scenes:
                outs.append(S.assign_cameras(m, n))
                d = torch.zeros(m * n * words, dtype=torch.int32, device="cuda")
                nc, inc = S.block_partial(m, n, d)
                parts.append(d)
                ncs.append(nc)
                incs.append(inc)
            for k in ref:
                assert (np.concatenate([o[k] for o in outs]) == ref[k]).all(), k
            gathered = torch.cat(parts)
            comb = torch.empty_like(parts[0])
            gv = scenes[0].masks_combine(m * n, gathered, W, comb)
            rec = scenes[0].block_records(m, n, np.sum(ncs, axis=0), np.sum(incs, axis=0), gv)
            for k in ("n_cams", "g_vis", "g_blk", "incidences", "g_avgvis", "area"):
                assert (rec[k] == L1[k]).all(), k
            c, e = scenes[W - 1].crop_from_masks(m, n, comb)
            assert (c == c1).all() and (e == e1).all()
        finally:
            for S in scenes:
                S.close()


def test_bo_trajectory_parity_and_I16():
    """Every evaluation of lobe_balance_partition equals the oracle objective at
    the recorded cuts (so the oracle-backed run follows the same trajectory), and
    the visibility kernels ran exactly once: tests_executed, the sum of the
    kernels' own decision counters, = G N (I16)."""
    lobe = _lobe()
    sc = make_scene(make_config("building", G=40_000, N=48, seed=0x42))
    m, n = sc.cfg.m, sc.cfg.n
    o = oracle.run(sc, grid=oracle.default_grid(m, n), masks=False)
    with lobe.Scene(sc, sc) as S:
        r = S.balance_partition(m, n, L=16, seed=5)
        for row, val in zip(r["cut_history"], r["history"]):
            g = oracle.default_grid(m, n, v=row[:m - 1], h=row[m - 1:])
            assert oracle.evaluate_cuts(sc, o["pre"], o["vis"], g) == val
        assert r["best"]["objective"] == r["history"].min() <= r["history"][0]
        st = S.stats()
        assert st.tests_executed == sc.G * sc.N and st.vis_launches == 1
        check_i16(st, sc.G, sc.N, np.asarray(o["vis"]["K"], np.int64).sum())


@pytest.mark.parametrize("name", ["rubble", "building", "residence", "matrixcity"])
def test_full_size_sampled(name):
    """BASELINE configs at full size, in the launch configuration bench.py times:
    rows / per-camera outputs bit-exact on sampled cameras (the oracle computes
    them one by one), block-level invariants at full size."""
    lobe = _lobe()
    sc = make_scene(name)
    m, n = sc.cfg.m, sc.cfg.n
    rng = np.random.default_rng(11)
    sel = np.sort(rng.choice(sc.N, 6, replace=False))
    with lobe.Scene(sc, sc) as S:
        fr = oracle.frame(sc)
        assert (S.frame["center"] == fr[0]).all() and S.frame["radius"] == fr[1]
        pre = oracle.prep(sc, fr)
        pre["cam_gu_sel"], pre["cam_gv_sel"] = pre["cam_gu"][sel], pre["cam_gv"][sel]
        vis = oracle.visibility(sc, pre, cams=sel)
        rows = np.concatenate([S.export_rows(int(c), 1) for c in sel])
        assert (rows == vis["rows"]).all()
        g = oracle.default_grid(m, n)
        asg = oracle.assign(sc, pre, vis, g)
        a = S.assign_cameras(m, n)
        _cmp_percam(a, vis, asg, sel=sel)
        check_i16(S.stats(), sc.G, sc.N, a["K"].astype(np.int64).sum())
        L = S.block_loads(m, n)
        assert int(L["incidences"].sum()) == int(a["K"].astype(np.int64).sum())      # I2
        assert int(L["g_blk"].astype(np.int64).sum()) == sc.G                         # I4
        assert (a["n0"].sum(axis=1) == a["K"]).all() and (a["n"] >= a["n0"]).all()  # I5, I6
        for b in range(m * n):
            cams = np.nonzero((a["member"] >> np.uint64(b)) & np.uint64(1))[0]
            if len(cams):
                assert a["K"][cams].max() <= L["g_vis"][b] <= min(sc.G, int(a["K"][cams].astype(np.int64).sum()))
        # crop superset (I1) for the sampled cameras
        c, _ = S.crop_masks(m, n, eligible=False)
        for j, cam in enumerate(sel):
            rb = np.unpackbits(rows[j].view(np.uint8), bitorder="little")[:sc.G].astype(bool)
            for b in range(m * n):
                if (int(a["member"][cam]) >> b) & 1:
                    cb = np.unpackbits(c[b].view(np.uint8), bitorder="little")[:sc.G].astype(bool)
                    assert not (rb & ~cb).any()


def test_invalid_camera_gpu():
    """Cameras are validated while the device runs the first kernels of the
    load; an invalid one still fails the load with INVALID_INPUT (no partial
    scene) -- non-orthonormal R, z_near >= z_far, a NaN translation."""
    lobe = _lobe()
    sc = make_scene("tiny")
    for field, value in (("R", 1.5), ("z_near", 9.0), ("t", np.nan)):
        bad = make_scene("tiny")
        arr = getattr(bad, field)
        if arr.ndim > 1:
            arr[7].flat[0] = value
        else:
            arr[7] = value
        with pytest.raises(lobe.LobeError) as e:
            lobe.Scene(sc, bad)
        assert e.value.status == "INVALID_INPUT", field
    with lobe.Scene(sc, sc) as S:  # the valid scene still loads afterwards
        assert S.assign_cameras(2, 2)["K"].sum() > 0


@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("predicate", [0, 1])
def test_invalid_gaussians_gpu(on_device, predicate):
    """Every Gaussian field is validated (O1) whichever path the
    inputs take -- host inputs in the isotropic mode validate the quaternions
    on a side stream after the other fields -- and the message names the first
    invalid Gaussian, as the oracle does."""
    import torch
    lobe = _lobe()
    cases = [(("qw", 700, 0.5),), (("sx", 900, -1.0), ("qx", 700, 3.0)), (("qy", 900, np.nan), ("opacity", 700, 1.5)),
             (("x", 10, np.inf),), (("qz", 9999, 0.9),)]
    for changes in cases:
        bad = make_scene("tiny")
        for field, idx, val in changes:
            getattr(bad, field)[idx] = val
        with pytest.raises(oracle.OracleError) as eo:
            oracle.validate(bad)
        first = min(idx for _, idx, _ in changes)
        assert f"index {first}" in str(eo.value)
        g = bad
        if on_device:
            class DG:
                pass
            g = DG()
            for k in ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity"):
                setattr(g, k, torch.from_numpy(getattr(bad, k)).cuda())
        # a host-input load in the isotropic mode may return before its deferred
        # quaternion check has decided: the verdict is then the next call's
        # status, and every later call on the scene repeats it (include/lobe.h)
        deferred = (not on_device) and predicate == 0 and all(f in ("qw", "qx", "qy", "qz") for f, _, _ in changes)
        with pytest.raises(lobe.LobeError) as e:
            S = lobe.Scene(g, bad, predicate=predicate)
            try:
                assert deferred, "load accepted invalid non-quaternion inputs"
                S.assign_cameras(2, 2)
            finally:
                with pytest.raises(lobe.LobeError) as e2:  # the scene stays unusable
                    S.block_loads(2, 2)
                assert e2.value.status == "INVALID_INPUT" and f"gaussian {first} " in str(e2.value)
                S.close()
        assert e.value.status == "INVALID_INPUT" and f"gaussian {first} " in str(e.value), (changes, str(e.value))
    sc = make_scene("tiny")
    with lobe.Scene(sc, sc, predicate=predicate) as S:  # valid inputs still load
        assert S.assign_cameras(2, 2)["K"].sum() > 0


def test_errors_gpu():
    lobe = _lobe()
    g = [dict(mu=[0, 0, 5], s=0.1, o=1.0), dict(mu=[1, 1, 5], s=0.1, o=1.0)]
    sc = mini_scene(g, [GOLD["camera_C0"]])
    sc.x[0] = np.nan
    fr = dict(center=[0, 0, 0], radius=1.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    with pytest.raises(lobe.LobeError) as e:
        lobe.Scene(sc, sc, frame=fr)
    assert e.value.status == "INVALID_INPUT"
    with pytest.raises(lobe.LobeError) as e:      # one camera: automatic radius is 0
        lobe.Scene(mini_scene(g, [GOLD["camera_C0"]]), mini_scene(g, [GOLD["camera_C0"]]))
    assert e.value.status == "DEGENERATE_SCENE"
    sc = mini_scene([dict(mu=[1, 1, 1], s=0.1, o=1.0)] * 3, [GOLD["camera_C0"]])
    with pytest.raises(lobe.LobeError) as e:
        lobe.Scene(sc, sc, frame=dict(center=[0, 0, 0], radius=1.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0]))
    assert e.value.status == "DEGENERATE_SCENE"
    sc = make_scene(make_config("tiny", G=500, N=4))
    with lobe.Scene(sc, sc) as S:
        with pytest.raises(lobe.LobeError) as e:
            S.block_loads(3, 1, v=np.array([0.6, 0.4], np.float32))
        assert e.value.status == "INVALID_CUTS"
        with pytest.raises(lobe.LobeError) as e:
            S.block_loads(9, 9)
        assert e.value.status == "INVALID_CONFIG"
        S.block_loads(2, 2)   # handle still valid after failures


def _fuzz_scene(seed, G=6000, N=24):
    """Adversarial geometry for the tile culling: Gaussians in a box that the
    cameras sit inside (camera planes cut through tiles, points behind and
    beside every camera), heavy-tailed scales (huge footprints), some gated,
    random intrinsics and depth ranges."""
    from synth.scenes import Scene, SceneConfig
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.asarray(a, dtype=np.float32)
    mu = rng.uniform(-1, 1, size=(G, 3))
    mu[: G // 4] *= rng.uniform(0.0, 0.02, size=(G // 4, 1))      # a dense blob at the origin
    s = np.exp(rng.normal(np.log(0.01), 1.5, size=(G, 3)))
    q = rng.normal(size=(G, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.uniform(0, 1, G)
    op[rng.uniform(size=G) < 0.1] = 0.001                            # gated
    cams = []
    for c in range(N):
        p = rng.uniform(-0.8, 0.8, 3)
        f = rng.normal(size=3)
        f /= np.linalg.norm(f)
        up = np.array([0.0, 0.0, 1.0]) if abs(f[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
        xa = np.cross(f, up)
        xa /= np.linalg.norm(xa)
        ya = np.cross(f, xa)
        R = np.stack([xa, ya, f])
        W, H = int(rng.integers(32, 400)), int(rng.integers(32, 400))
        fx = float(rng.uniform(0.3, 2.0) * W)
        fy = float(fx * rng.uniform(0.8, 1.25))
        zn = float(10 ** rng.uniform(-3, -1))
        cams.append(dict(R=R, t=-R @ p, W=W, H=H, fx=fx, fy=fy, cx=W * rng.uniform(0.3, 0.7),
                         cy=H * rng.uniform(0.3, 0.7), zn=zn, zf=float(zn * 10 ** rng.uniform(1, 4))))
    cfg = SceneConfig("fuzz", G, N, 3, 2, 100, 100, 60.0, (-1, 1, -1, 1), 1.0, 1, 0.0, seed)
    return Scene(cfg, f32(mu[:, 0]), f32(mu[:, 1]), f32(mu[:, 2]), f32(s[:, 0]), f32(s[:, 1]), f32(s[:, 2]),
                 f32(q[:, 0]), f32(q[:, 1]), f32(q[:, 2]), f32(q[:, 3]), f32(op),
                 cam_id=np.arange(N, dtype=np.int32), fx=f32([c["fx"] for c in cams]), fy=f32([c["fy"] for c in cams]),
                 cx=f32([c["cx"] for c in cams]), cy=f32([c["cy"] for c in cams]),
                 width=np.array([c["W"] for c in cams], np.int32), height=np.array([c["H"] for c in cams], np.int32),
                 R=f32([c["R"] for c in cams]), t=f32([c["t"] for c in cams]),
                 z_near=f32([c["zn"] for c in cams]), z_far=f32([c["zf"] for c in cams]))


@pytest.mark.parametrize("seed,G", [(1, 6000), (2, 6000), (3, 50_000), (4, 50_000)])
def test_fuzz_culling_exact(seed, G):
    """Tile culling never drops a visible Gaussian (and the whole path stays
    bit-exact) under adversarial camera placement and footprints."""
    sc = _fuzz_scene(seed, G=G)
    full_parity(sc, [oracle.default_grid(3, 2), _rand_grid(4, 4, seed)])


def _edge_scene(seed, N=16, clusters=12, per=300):
    """Tight clusters (radius 1e-4 of the depth) placed just inside and just
    outside every frustum boundary of every camera -- the four image edges
    dilated by the footprint, the near and the far plane -- so that 256-Gaussian
    slice boxes land on both sides of each condition. Exercises the slice
    accept / reject bounds of k_vis_tiles against the exact test."""
    from synth.scenes import Scene, SceneConfig
    rng = np.random.default_rng(1000 + seed)
    f32 = lambda a: np.asarray(a, dtype=np.float32)
    cams = []
    for c in range(N):
        p = rng.uniform(-0.5, 0.5, 3)
        f = rng.normal(size=3)
        f /= np.linalg.norm(f)
        up = np.array([0.0, 0.0, 1.0]) if abs(f[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
        xa = np.cross(f, up)
        xa /= np.linalg.norm(xa)
        ya = np.cross(f, xa)
        R = np.stack([xa, ya, f])
        W, H = int(rng.integers(64, 400)), int(rng.integers(64, 400))
        fx = float(rng.uniform(0.5, 2.0) * W)
        fy = float(fx * rng.uniform(0.8, 1.25))
        zn = float(10 ** rng.uniform(-2, -1))
        cams.append(dict(R=R, p=p, t=-R @ p, W=W, H=H, fx=fx, fy=fy, cx=W * rng.uniform(0.3, 0.7),
                         cy=H * rng.uniform(0.3, 0.7), zn=zn, zf=float(zn * 10 ** rng.uniform(1, 2))))
    pts, scl = [], []
    for cam in cams:
        for k in range(clusters):
            side = k % 6  # 0..3 image edges, 4 near plane, 5 far plane
            z = rng.uniform(1.5 * cam["zn"], 0.7 * cam["zf"])
            px, py = rng.uniform(0, cam["W"]), rng.uniform(0, cam["H"])
            off = (1 if rng.uniform() < 0.5 else -1) * 10 ** rng.uniform(-3, 1)  # pixels / depth units
            if side == 0:
                px = 0.0 + off
            elif side == 1:
                px = cam["W"] + off
            elif side == 2:
                py = 0.0 + off
            elif side == 3:
                py = cam["H"] + off
            elif side == 4:
                z = cam["zn"] * (1 + off * 1e-2)
            else:
                z = cam["zf"] * (1 + off * 1e-2)
            xc = np.array([(px - cam["cx"]) / cam["fx"] * z, (py - cam["cy"]) / cam["fy"] * z, z])
            centre = cam["R"].T @ xc + cam["p"]
            pts.append(centre + rng.normal(scale=1e-4 * z, size=(per, 3)))
            scl.append(np.full((per, 3), 10 ** rng.uniform(-7, -4)))
    mu = np.concatenate(pts)
    s = np.concatenate(scl) * np.exp(rng.normal(0, 0.3, size=(len(mu), 3)))
    G = len(mu)
    q = rng.normal(size=(G, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.uniform(0.01, 1, G)
    op[rng.uniform(size=G) < 0.05] = 0.001
    cfg = SceneConfig("edge", G, N, 2, 2, 100, 100, 60.0, (-1, 1, -1, 1), 1.0, 1, 0.0, seed)
    return Scene(cfg, f32(mu[:, 0]), f32(mu[:, 1]), f32(mu[:, 2]), f32(s[:, 0]), f32(s[:, 1]), f32(s[:, 2]),
                 f32(q[:, 0]), f32(q[:, 1]), f32(q[:, 2]), f32(q[:, 3]), f32(op),
                 cam_id=np.arange(N, dtype=np.int32), fx=f32([c["fx"] for c in cams]), fy=f32([c["fy"] for c in cams]),
                 cx=f32([c["cx"] for c in cams]), cy=f32([c["cy"] for c in cams]),
                 width=np.array([c["W"] for c in cams], np.int32), height=np.array([c["H"] for c in cams], np.int32),
                 R=f32([c["R"] for c in cams]), t=f32([c["t"] for c in cams]),
                 z_near=f32([c["zn"] for c in cams]), z_far=f32([c["zf"] for c in cams]))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_edge_clusters_exact(seed):
    """Slice bounds (accept / reject) never change a test outcome: clusters
    straddling every frustum boundary, compared in full with the oracle; the
    scene must actually exercise accepted, rejected and exact slices."""
    sc = _edge_scene(seed)
    st = full_parity(sc, [oracle.default_grid(2, 2)])
    assert st.accepted_tests > 0 and st.dense_tests > 0 and st.kept_tests > st.dense_tests + st.accepted_tests


# ---------------------------------------------------------------- anisotropic predicate (NEXT-2, ledger L24)
def test_aniso_tiny_full(tiny_scene):
    """The projected-covariance footprint path: rows, counts, depth statistics,
    assignments, loads and masks equal the oracle's O6a (bit-exact; D_c 1e-6)."""
    full_parity(tiny_scene, [oracle.default_grid(2, 2), _rand_grid(3, 3, 5)], predicate=1)


def test_aniso_ieee_path():
    """A camera with z_far beyond 2^126 disables the branch-free reciprocal /
    square roots for the scene (host check): the IEEE kernel variant must give
    the same O6a results."""
    sc = make_scene("tiny")
    sc.z_far[3] = np.float32(1e38)
    full_parity(sc, [oracle.default_grid(2, 2)], predicate=1)


def test_aniso_ragged():
    from synth.scenes import make_config, make_scene
    sc = make_scene(make_config("residence", G=37_123, N=53, seed=0x2510AA01))
    full_parity(sc, [oracle.default_grid(2, 2), _rand_grid(8, 8, 3)], predicate=1)


@pytest.mark.parametrize("seed,G", [(1, 6000), (3, 50_000)])
def test_aniso_fuzz_culling_exact(seed, G):
    """Box bounds of the anisotropic mode (fp64, radius envelope from trace(Sigma)
    and ||J||_F) never change a decision: cameras inside the cloud, heavy-tailed
    scales and random rotations."""
    full_parity(_fuzz_scene(seed, G=G), [oracle.default_grid(3, 2)], predicate=1)


@pytest.mark.parametrize("seed", [1, 2])
def test_aniso_edge_clusters_exact(seed):
    st = full_parity(_edge_scene(seed), [oracle.default_grid(2, 2)], predicate=1)
    assert st.dense_tests > 0


def test_aniso_overflowing_covariance_not_accepted():
    """scales up to 1e18 are valid (L22); a tight cluster of such
    Gaussians projecting inside the image has A = C = inf in the pinned fp32
    covariance, d = A - C = NaN and the oracle calls it invisible. The slice
    bound must then leave the slice to the exact test instead of accepting it."""
    rng = np.random.default_rng(7)
    g = [dict(mu=[float(x), float(y), 1.0 + float(z)], s=1e18, o=0.9)
         for x, y, z in rng.normal(scale=0.002, size=(300, 3))]
    g += [dict(mu=[float(x), float(y), float(z)], s=0.001, o=0.8)
          for x, y, z in zip(rng.uniform(-0.5, 0.5, 200), rng.uniform(-0.5, 0.5, 200), rng.uniform(0.5, 3, 200))]
    cam1 = dict(GOLD["camera_C0"])
    cam2 = dict(GOLD["camera_C0"], t=[-0.3, 0.1, 0.0])
    sc = mini_scene(g, [cam1, cam2])
    o = oracle.run(sc, predicate=1)
    huge = np.unpackbits(o["vis"]["rows"].view(np.uint8), axis=1, bitorder="little")[:, :300]
    assert not huge.any()  # NaN footprint: never visible in O6a
    assert o["vis"]["K"].min() > 0
    full_parity(sc, [oracle.default_grid(1, 1), oracle.default_grid(2, 2)], predicate=1)


@pytest.mark.parametrize("name", ["rubble", "matrixcity"])
def test_full_size_sampled_aniso(name):
    """The anisotropic mode at full Rubble and MatrixCity size: rows and
    per-camera outputs of sampled cameras equal the oracle's O6a."""
    lobe = _lobe()
    sc = make_scene(name)
    m, n = sc.cfg.m, sc.cfg.n
    rng = np.random.default_rng(23)
    sel = np.sort(rng.choice(sc.N, 4, replace=False))
    with lobe.Scene(sc, sc, predicate=1) as S:
        fr = oracle.frame(sc)
        pre = oracle.prep(sc, fr)
        pre["cam_gu_sel"], pre["cam_gv_sel"] = pre["cam_gu"][sel], pre["cam_gv"][sel]
        vis = oracle.visibility_aniso(sc, pre, cams=sel)
        rows = np.concatenate([S.export_rows(int(c), 1) for c in sel])
        assert (rows == vis["rows"]).all()
        g = oracle.default_grid(m, n)
        asg = oracle.assign(sc, pre, vis, g)
        _cmp_percam(S.assign_cameras(m, n), vis, asg, sel=sel)


def test_dev_vis_bench_variants_identical(tiny_scene):
    """lobe_dev_vis_bench: every visibility kernel variant (the tile-major
    production kernel, the culled and dense camera-inner kernels and their
    other shapes) rewrites the rows with the same bits as the oracle."""
    lobe = _lobe()
    o = oracle.run(tiny_scene)
    with lobe.Scene(tiny_scene, tiny_scene) as S:
        for variant in range(6):
            ms, grid = S.dev_vis_bench(variant, reps=1)
            assert ms > 0 and grid > 0
            assert (S.export_rows() == o["vis"]["rows"]).all(), variant
        with pytest.raises(lobe.LobeError):
            S.dev_vis_bench(99, reps=1)


def test_dev_vis_bench_aniso(tiny_scene):
    """Anisotropic scenes: the production kernel re-run by lobe_dev_vis_bench
    keeps the O6a rows; the camera-inner variants are isotropic only."""
    lobe = _lobe()
    o = oracle.run(tiny_scene, predicate=oracle.PRED_ANISO)
    with lobe.Scene(tiny_scene, tiny_scene, predicate=1) as S:
        S.dev_vis_bench(0, reps=2)
        assert (S.export_rows() == o["vis"]["rows"]).all()
        with pytest.raises(lobe.LobeError) as e:
            S.dev_vis_bench(1, reps=1)
        assert e.value.status == "INVALID_CONFIG"
