"""Oracle pins: hand-worked cases (tests/golden/hand_cases.json) and SPEC examples.

Every expected value here comes from the golden fixture (derived by hand from
the cited definitions) -- never from the oracle itself.
"""
import json
import os

import numpy as np
import pytest

import oracle
from tests.helpers import mini_scene, nadir_camera, bits_of_row, bits_of_mask64

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")))
C0 = GOLD["camera_C0"]


def _run_single(gaussians, cams=(C0,), frame=None):
    sc = mini_scene(gaussians, list(cams))
    oracle.validate(sc)
    fa = frame or dict(center=[0, 0, 0], radius=1.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    fr = oracle.frame(sc, **fa)
    # add two far anchors so the grid normalisation is never degenerate
    pre = oracle.prep(sc, fr)
    vis = oracle.visibility(sc, pre, threads=1)
    return sc, pre, vis


@pytest.mark.parametrize("case", GOLD["visibility"], ids=[c["id"] for c in GOLD["visibility"]])
def test_visibility_hand_case(case):
    anchors = [dict(mu=[-50, -50, -50], s=0.01, o=0.0), dict(mu=[50, 50, 50], s=0.01, o=0.0)]
    g = [dict(mu=case["mu"], s=case["s"], o=case["o"])] + anchors
    sc, pre, vis = _run_single(g)
    got = bool(vis["rows"][0, 0] & 1)
    assert got == case["visible"], f'{case["id"]}: {case["why"]} ({case["cite"]})'
    assert vis["K"][0] == (1 if case["visible"] else 0)


def test_depth_statistic_H7():
    d = GOLD["depth_stat"]
    g = [dict(mu=x["mu"], s=x["s"], o=x["o"]) for x in d["gaussians"]]
    g += [dict(mu=[-50, -50, -50], s=0.01, o=0.0), dict(mu=[50, 50, 50], s=0.01, o=0.0)]
    sc, pre, vis = _run_single(g)
    assert vis["K"][0] == d["K"]
    assert vis["D"][0] == pytest.approx(d["D"], rel=1e-15)
    assert vis["zmin"][0] == np.float32(d["z_min"]) and vis["zmax"][0] == np.float32(d["z_max"])


def _assign_scene(n_low, n_high):
    a = GOLD["assignment"]
    rng = np.random.default_rng(0)
    g = [dict(mu=x["mu"], s=x["s"], o=x["o"]) for x in a["anchors"]]
    for cl, cnt in ((a["cluster_low"], n_low), (a["cluster_high"], n_high)):
        for _ in range(cnt):
            mu = np.asarray(cl["center"], float) + np.r_[rng.uniform(-0.05, 0.05, 2), 0.0]
            g.append(dict(mu=mu, s=0.001, o=0.9))
    cam = nadir_camera(*a["camera"]["nadir_at"], f=a["camera"]["f"])
    sc = mini_scene(g, [cam], m=2, n=2)
    fr = oracle.frame(sc, center=a["frame"]["center"], radius=a["frame"]["radius"], axis_u=[1, 0, 0],
                      axis_v=[0, 1, 0])
    pre = oracle.prep(sc, fr)
    vis = oracle.visibility(sc, pre, threads=1)
    return sc, pre, vis


def test_assignment_H9():
    a = GOLD["assignment"]
    sc, pre, vis = _assign_scene(a["cluster_low"]["count"], a["cluster_high"]["count"])
    e = a["expect"]
    assert vis["K"][0] == e["K"]
    grid = oracle.default_grid(2, 2, delta_v=a["grid"]["delta"], delta_h=a["grid"]["delta"], tau=0.15)
    asg = oracle.assign(sc, pre, vis, grid, threads=1)
    assert list(asg["n"][0]) == e["n"] and list(asg["n0"][0]) == e["n0"]
    assert [b for b in range(4) if (int(asg["member"][0]) >> b) & 1] == e["member_tau_0.15"]
    assert asg["home"][0] == e["home"]
    asg5 = oracle.assign(sc, pre, vis, dict(grid, tau=0.5), threads=1)
    assert [b for b in range(4) if (int(asg5["member"][0]) >> b) & 1] == e["member_tau_0.5"]


def test_assignment_home_tie_H9():
    t = GOLD["assignment"]["tie"]
    sc, pre, vis = _assign_scene(t["cluster_low_count"], t["cluster_high_count"])
    grid = oracle.default_grid(2, 2, delta_v=0.05, delta_h=0.05)
    asg = oracle.assign(sc, pre, vis, grid, threads=1)
    assert asg["home"][0] == t["home"]


@pytest.mark.parametrize("case", GOLD["tau_rule"]["cases"], ids=lambda c: f'n{c["n"]}')
def test_tau_rule_H9b(case):
    """K=20 visible: n in block 0's region, the rest far away in block 3."""
    K = GOLD["tau_rule"]["K"]
    n_low = case["n"]
    sc, pre, vis = _assign_scene(n_low, K - n_low)
    grid = oracle.default_grid(2, 2, delta_v=0.05, delta_h=0.05, tau=0.15)
    asg = oracle.assign(sc, pre, vis, grid, threads=1)
    assert vis["K"][0] == K and asg["n"][0][0] == n_low
    assert bool(int(asg["member"][0]) & 1) == case["member"]


def test_cell_boundary_H10():
    """A Gaussian whose grid coordinate is exactly 0.5 (anchors at x=-1, +1;
    the point at x=0 maps to (0/10 + 0.1)/0.2 = 0.5 exactly)."""
    h = GOLD["cell_boundary"]
    g = [dict(mu=[-1, -1, 0], s=0.01, o=0.0), dict(mu=[1, 1, 0], s=0.01, o=0.0), dict(mu=[0, -0.9, 0], s=0.001, o=1)]
    cam = nadir_camera(0, 0, 3)
    sc = mini_scene(g, [cam], m=2, n=2)
    fr = oracle.frame(sc, center=[0, 0, 0], radius=10.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    pre = oracle.prep(sc, fr)
    assert pre["gu"][2] == np.float32(h["gu"])
    vis = oracle.visibility(sc, pre, threads=1)
    assert vis["K"][0] == 1
    grid = oracle.default_grid(2, 2, delta_v=h["delta"], delta_h=h["delta"])
    asg = oracle.assign(sc, pre, vis, grid, threads=1)
    # gv is near 0.05 -> q = 0; cell p must be the higher one (1); enlarged p in {0,1}
    assert asg["n0"][0][1 * 2 + 0] == 1
    assert [p for p in range(2) if asg["n"][0][p * 2 + 0] == 1] == h["enlarged"]


def test_contraction_H11():
    c = GOLD["contraction"]
    pts = c["norm4"]["points"]
    g = [dict(mu=p, s=0.01, o=1.0) for p in pts] + [dict(mu=[0, 0.3, 0], s=0.01, o=1.0)]
    sc = mini_scene(g, [C0])
    fr = oracle.frame(sc, **c["norm4"]["frame"], axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    pre = oracle.prep(sc, fr)
    assert pre["minmax"][1] == np.float32(c["norm4"]["max_u_before_norm"])
    pts = c["collinear"]["points"]
    g = [dict(mu=p, s=0.01, o=1.0) for p in pts] + [dict(mu=[0, 1, 0], s=0.01, o=1.0)]
    sc = mini_scene(g, [C0])
    fr = oracle.frame(sc, **c["collinear"]["frame"], axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    pre = oracle.prep(sc, fr)
    assert list(pre["gu"][:3]) == [np.float32(v) for v in c["collinear"]["gu"]]


def test_empty_camera_H12():
    g = [dict(mu=[-1, -1, 0], s=0.01, o=1.0), dict(mu=[1, 1, 0], s=0.01, o=1.0), dict(mu=[0.5, 0.5, 0], s=0.01, o=1)]
    up = dict(nadir_camera(0.5, 0.5, 3))
    up["R"] = np.eye(3)                       # looks along +z: away from every Gaussian
    up["t"] = -np.array([0.5, 0.5, 3.0])
    sc = mini_scene(g, [up], m=2, n=2)
    fr = oracle.frame(sc, center=[0, 0, 0], radius=10.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    pre = oracle.prep(sc, fr)
    vis = oracle.visibility(sc, pre, threads=1)
    assert vis["K"][0] == 0 and vis["D"][0] == 0.0
    assert np.isinf(vis["zmin"][0]) and vis["zmin"][0] > 0 and np.isinf(vis["zmax"][0]) and vis["zmax"][0] < 0
    grid = oracle.default_grid(2, 2)
    asg = oracle.assign(sc, pre, vis, grid, threads=1)
    assert asg["member"][0] == 0
    # camera centre (0.5,0.5,3) -> contracted ground coords (0.05, 0.05) -> gu = (0.05+0.1)/0.2 = 0.75 -> cell (1,1)
    assert asg["home"][0] == 3


def test_spec_block_region_and_area():
    e = GOLD["spec_examples"]["block_region"]
    sc, pre, vis = _assign_scene(4, 6)
    for delta, key in ((0.0, "delta0"), (0.05, "delta005")):
        grid = oracle.default_grid(2, 2, delta_v=delta, delta_h=delta)
        asg = oracle.assign(sc, pre, vis, grid, threads=1)
        bl = oracle.block_loads(sc, pre, vis, asg, grid)
        assert [list(map(float, bl["lohi"][0]))] == [[np.float32(v) for v in e[key][0]]]
        assert list(bl["area"]) == [e["area"]] * 4


def test_spec_init_cuts():
    e = GOLD["spec_examples"]["init_cuts"]
    assert list(oracle.default_grid(4, 1)["v"]) == e["m4"]
    assert list(oracle.default_grid(2, 1)["v"]) == e["m2"]
    assert list(oracle.default_grid(1, 1)["v"]) == e["m1"]


def test_spec_crop_single_camera_rows():
    """single camera seeing {3, 7} -> sub-scene {3, 7}."""
    g = [dict(mu=[0, 0, -5], s=0.01, o=1.0) for _ in range(10)]
    for i in (3, 7):
        g[i] = dict(mu=[0.1 * i - 0.5, 0, 5], s=0.01, o=1.0)
    g[0] = dict(mu=[-3, -3, -5], s=0.01, o=1.0)
    g[9] = dict(mu=[3, 3, -5], s=0.01, o=1.0)
    sc = mini_scene(g, [C0], m=1, n=1)
    fr = oracle.frame(sc, center=[0, 0, 0], radius=100.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    pre = oracle.prep(sc, fr)
    vis = oracle.visibility(sc, pre, threads=1)
    assert bits_of_row(vis["rows"][0], sc.G) == {3, 7}
    grid = oracle.default_grid(1, 1)
    asg = oracle.assign(sc, pre, vis, grid, threads=1)
    bl = oracle.block_loads(sc, pre, vis, asg, grid)
    crop, elig = oracle.crop(sc, pre, grid, bl["M"])
    assert bits_of_mask64(crop[0], sc.G) == {3, 7}
    assert bits_of_mask64(elig[0], sc.G) == {3, 7}      # 1x1 grid: every Gaussian is in the block


def test_spec_selective_mask_6_in_4_out():
    """mixed fixture 6-in / 4-out -> exactly 6 eligible."""
    g = [dict(mu=[-1, -1, 0], s=0.001, o=0.0), dict(mu=[1, 1, 0], s=0.001, o=0.0)]
    xs = [-0.8, -0.7, -0.6, -0.75, -0.65, -0.55, 0.6, 0.7, 0.8, 0.75]   # 6 with gu < 0.5, 4 above
    for x in xs:
        g.append(dict(mu=[x, -0.8, 0], s=0.001, o=1.0))
    cam = nadir_camera(0, 0, 3, f=20.0)
    sc = mini_scene(g, [cam], m=2, n=1)
    fr = oracle.frame(sc, center=[0, 0, 0], radius=10.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    pre = oracle.prep(sc, fr)
    vis = oracle.visibility(sc, pre, threads=1)
    assert vis["K"][0] == 10
    grid = oracle.default_grid(2, 1, tau=0.0)        # tau = 0: the camera joins both blocks
    asg = oracle.assign(sc, pre, vis, grid, threads=1)
    assert int(asg["member"][0]) == 0b11
    bl = oracle.block_loads(sc, pre, vis, asg, grid)
    crop, elig = oracle.crop(sc, pre, grid, bl["M"])
    assert len(bits_of_mask64(crop[0], sc.G)) == 10
    assert len(bits_of_mask64(elig[0], sc.G)) == 6
    assert len(bits_of_mask64(elig[1], sc.G)) == 4


def test_visibility_ratio_10_points_4_inside():
    """10-point fixture with 4 points in the region -> ratio 0.4;
    tau = 0.4 admits the camera, tau = 0.41 does not."""
    sc, pre, vis = _assign_scene(4, 6)
    for tau, want in ((0.4, True), (0.41, False)):
        grid = oracle.default_grid(2, 2, delta_v=0.05, delta_h=0.05, tau=tau)
        asg = oracle.assign(sc, pre, vis, grid, threads=1)
        assert bool(int(asg["member"][0]) & 1) == want


def test_errors():
    g = [dict(mu=[0, 0, 5], s=0.1, o=1.0), dict(mu=[1, 1, 5], s=0.1, o=1.0)]
    sc = mini_scene(g, [C0])
    sc.x[0] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.validate(sc)
    assert e.value.status == "INVALID_INPUT"
    sc = mini_scene(g, [C0])
    sc.sx[1] = 0.0
    with pytest.raises(oracle.OracleError):
        oracle.validate(sc)
    sc = mini_scene(g, [dict(C0, z_near=5.0, z_far=1.0)])
    with pytest.raises(oracle.OracleError):
        oracle.validate(sc)
    # all points identical -> degenerate
    sc = mini_scene([dict(mu=[1, 1, 1], s=0.1, o=1.0)] * 3, [C0])
    fr = oracle.frame(sc, center=[0, 0, 0], radius=1.0, axis_u=[1, 0, 0], axis_v=[0, 1, 0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.prep(sc, fr)
    assert e.value.status == "DEGENERATE_SCENE"
    # non-monotone cuts
    sc, pre, vis = _assign_scene(4, 6)
    grid = oracle.default_grid(3, 1, v=[0.6, 0.4])
    with pytest.raises(oracle.OracleError) as e:
        oracle.assign(sc, pre, vis, grid)
    assert e.value.status == "INVALID_CUTS"


# ------------------------------------------------------------------ O2 frame
FRAME = GOLD["frame_auto"]


def frame_cameras(case, extra=False):
    """Cameras of a frame case: identity R with t = -o (so o = -R^T t = the listed
    centre), or the case's rotated pose; F3 optionally adds its identity camera."""
    cams = []
    for o in case["centers"]:
        c = dict(fx=100.0, fy=100.0, cx=50.0, cy=50.0, width=100, height=100, z_near=0.1, z_far=100.0)
        if "rotated" in case:
            c["R"] = np.asarray(case["rotated"]["R"], float)
            c["t"] = np.asarray(case["rotated"]["t"], float)
        else:
            c["R"] = np.eye(3)
            c["t"] = -np.asarray(o, float)
        cams.append(c)
    if extra:
        cams.append(dict(fx=100.0, fy=100.0, cx=50.0, cy=50.0, width=100, height=100, z_near=0.1, z_far=100.0,
                         R=np.eye(3), t=np.asarray(case["extra_identity_camera_t"], float)))
    return cams


FRAME_GAUSSIANS = [dict(mu=[-1, -1, 0], s=0.01, o=0.5), dict(mu=[1, 1, 0.5], s=0.01, o=0.5)]


@pytest.mark.parametrize("case", FRAME["cases"], ids=[c["id"] for c in FRAME["cases"]])
def test_frame_auto_hand_case(case):
    extra = "extra_identity_camera_t" in case
    sc = mini_scene(FRAME_GAUSSIANS, frame_cameras(case, extra=extra))
    c0, rho, au, av = oracle.frame(sc)
    assert list(c0) == [np.float32(v) for v in case["center"]], (case["id"], case["why"])
    assert rho == np.float32(case["radius"]), (case["id"], case["why"])
    assert list(au) == [1, 0, 0] and list(av) == [0, 1, 0]
    if extra:  # without the extra camera every distance is 0: DEGENERATE_SCENE
        assert case["radius_without_extra"] == 0
        with pytest.raises(oracle.OracleError) as e:
            oracle.frame(mini_scene(FRAME_GAUSSIANS, frame_cameras(case)))
        assert e.value.status == "DEGENERATE_SCENE"


def test_frame_auto_overrides():
    """Caller values override each default independently (O2 'Caller-supplied
    values override the defaults'): a given centre changes the radius's
    reference point (F1 about (0,0,0): distances 3,sqrt(41),sqrt(80),sqrt(13),0,
    sqrt(221) -> 6th = sqrt(221))."""
    case = FRAME["cases"][0]
    sc = mini_scene(FRAME_GAUSSIANS, frame_cameras(case))
    c0, rho, _, _ = oracle.frame(sc, center=[0, 0, 0])
    assert list(c0) == [0, 0, 0] and rho == np.float32(np.sqrt(221.0))
    c0, rho, _, _ = oracle.frame(sc, radius=7.5)
    assert list(c0) == [2, 0, 0] and rho == np.float32(7.5)
