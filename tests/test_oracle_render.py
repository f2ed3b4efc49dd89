"""Pins of the depth-render camera selection oracle (
PAPER.md:175-179; SPEC.md:335-360 examples and acceptance #6; ledger L26)."""
import ctypes

import numpy as np
import pytest

import oracle
from tests.helpers import mini_scene

F = np.float32


def _exp(x):
    L = oracle.lib()
    L.exp_l26.restype = ctypes.c_float
    L.exp_l26.argtypes = [ctypes.c_float]
    return L.exp_l26(F(x))


def test_exp_accuracy():
    """exp_l26 on [-4.5, 0]: within 3e-7 relative of float64 exp; exp(0) = 1 exactly."""
    assert _exp(0.0) == 1.0
    xs = np.linspace(-4.5, 0.0, 2001).astype(np.float32)
    got = np.array([_exp(x) for x in xs], np.float64)
    want = np.exp(xs.astype(np.float64))
    assert np.max(np.abs(got - want) / want) < 3e-7


def _cam(ds=4, f=100.0, c=10.5, size=21):
    # full-resolution intrinsics so that the 1/ds image has focal f and principal point c
    return dict(fx=f * ds, fy=f * ds, cx=c * ds, cy=c * ds, width=size * ds, height=size * ds,
                R=np.eye(3), t=np.zeros(3), z_near=0.1, z_far=100.0)


def _render(gs, cam=None, ds=4, stride=2, eps_w=0.1):
    cam = cam or _cam(ds)
    sc = mini_scene(gs + [dict(mu=(50.0, 50.0, -50.0), o=0.001), dict(mu=(-40.0, 60.0, -30.0), o=0.001)],
                    [cam, dict(cam, t=np.array([1.0, 0.0, 0.0]))])
    fr = oracle.frame(sc)
    pre = oracle.prep(sc, fr)
    vis = np.arange(len(gs))
    D, W, pu, pv = oracle.render_camera(sc, pre, fr, 0, vis, ds, stride, eps_w)
    return D, W, pu, pv, sc, fr, pre


def test_single_opaque_gaussian():
    """opacity 1, centred on a pixel at depth 5 -> D = 5, weight = 1 there."""
    D, W, *_ = _render([dict(mu=(0.0, 0.0, 5.0), s=0.01, o=1.0)])
    assert abs(D[10, 10] - 5.0) < 1e-4 and abs(W[10, 10] - 1.0) < 1e-4


def test_two_layer_composite():
    """S:342 / acceptance #6: alpha 0.5 at depths 2 then 4 -> D = 2.0, weight 0.75."""
    D, W, *_ = _render([dict(mu=(0.0, 0.0, 4.0), s=0.01, o=0.5), dict(mu=(0.0, 0.0, 2.0), s=0.01, o=0.5)])
    assert abs(D[10, 10] - 2.0) < 1e-4 and abs(W[10, 10] - 0.75) < 1e-4


def test_empty_scene():
    """nothing visible -> all-zero depth and weight, empty cloud."""
    D, W, pu, pv, *_ = _render([])
    assert not D.any() and not W.any() and len(pu) == 0


def test_footprint_gaussian_value():
    """alpha at an offset pixel = o exp(-d^T Sigma'^-1 d / 2) with the EWA Sigma'
    of an axis-aligned on-axis Gaussian, diag(f^2 sx^2/z^2 + 0.3, f^2 sy^2/z^2 + 0.3)
    (closed form in float64, 1e-5 relative)."""
    z, sx, sy, o = 5.0, 0.03, 0.015, 0.8
    D, W, *_ = _render([dict(mu=(0.0, 0.0, z), s=(sx, sy, 0.01), o=o)])
    f = 100.0
    A = f * f * sx * sx / (z * z) + 0.3
    C = f * f * sy * sy / (z * z) + 0.3
    for (py, px) in [(10, 10), (10, 11), (11, 10), (12, 11), (9, 8)]:
        dx, dy = px + 0.5 - 10.5, py + 0.5 - 10.5
        p = -0.5 * (dx * dx / A + dy * dy / C)
        want = o * np.exp(p) if p >= -4.5 else 0.0
        assert abs(W[py, px] - want) <= 1e-5 * max(want, 1e-12), (py, px, W[py, px], want)


def test_weights_bounded_random():
    """Acceptance #6 property: per pixel sum w <= 1 and D <= max d * sum w on a random scene."""
    rng = np.random.default_rng(3)
    gs = [dict(mu=(rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(3, 8)), s=rng.uniform(0.01, 0.2, 3),
               o=rng.uniform(0.05, 1.0), q=tuple(v / np.linalg.norm(v) for v in [rng.normal(size=4)])[0])
          for _ in range(60)]
    D, W, *_ = _render(gs)
    zs = [g["mu"][2] for g in gs]
    assert (W <= 1.0 + 1e-6).all() and (W >= 0).all()
    assert (D <= max(zs) * W + 1e-4).all()


def test_backproject_optical_axis():
    """the pixel at the principal point with D = d back-projects to the
    world point on the optical axis at depth d (here (0, 0, 5)), whose grid
    coordinates follow the frame's contraction and min/max normalisation
    (recomputed in float64)."""
    D, W, pu, pv, sc, fr, pre = _render([dict(mu=(0.0, 0.0, 5.0), s=0.01, o=1.0)], stride=1)
    # the only pixel with weight >= 0.1 is the centre one (the footprint is tiny)
    assert len(pu) >= 1
    idx = [i for i, (py, px) in enumerate([(py, px) for py in range(21) for px in range(21) if W[py, px] >= 0.1])
           if (py, px) == (10, 10)][0]
    c0, rho, au, av = (np.asarray(a, np.float64) for a in fr)
    h = (np.array([0.0, 0.0, 5.0]) - c0) / rho
    r = np.linalg.norm(h)
    if r > 1:
        h = (2 - 1 / r) * h / r
    ru, rv = h @ au, h @ av
    mm = pre["minmax"].astype(np.float64)
    gu = np.clip((ru - mm[0]) / (mm[1] - mm[0]), 0, 1)
    gv = np.clip((rv - mm[2]) / (mm[3] - mm[2]), 0, 1)
    assert abs(pu[idx] - gu) < 1e-5 and abs(pv[idx] - gv) < 1e-5


def test_weight_floor():
    """every weight below eps_w -> K = 0."""
    *_, pu, pv, sc, fr, pre = _render([dict(mu=(0.0, 0.0, 5.0), s=0.05, o=0.05)])
    assert len(pu) == 0


def test_visibility_ratio_hand_fixture():
    """a 10-point cloud with 4 points in the region -> V = 0.4: member
    at tau = 0.4, not at tau = 0.41; region = whole domain -> 1.0."""
    sc = mini_scene([dict(mu=(0, 0, 5))], [dict(fx=100.0, fy=100.0, cx=50.0, cy=50.0, width=100, height=100,
                                                R=np.eye(3), t=np.zeros(3), z_near=0.1, z_far=100.0)])
    pre = {"cam_gu": np.array([0.5], np.float32), "cam_gv": np.array([0.5], np.float32)}
    gu = np.array([0.1, 0.2, 0.3, 0.4, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99], np.float32)
    gv = np.full(10, 0.5, np.float32)
    cl = dict(off=np.array([0, 10], np.int64), gu=gu, gv=gv)
    g = oracle.default_grid(2, 1, delta_v=0.0, delta_h=0.0, tau=0.4)
    a = oracle.assign_points(sc, pre, cl, g)
    assert int(a["n"][0, 0]) == 4 and int(a["member"][0]) & 1
    g = oracle.default_grid(2, 1, delta_v=0.0, delta_h=0.0, tau=0.41)
    assert not int(oracle.assign_points(sc, pre, cl, g)["member"][0]) & 1
    g = oracle.default_grid(1, 1, tau=1.0)
    assert int(oracle.assign_points(sc, pre, cl, g)["member"][0]) == 1


def test_footprint_rotated_cross_term():
    """A Gaussian turned 30 degrees about the optical axis: Sigma' has an
    off-diagonal term, (f/z)^2 R2 diag(sx^2, sy^2) R2^T + 0.3 I on the axis; alpha
    at diagonal offsets follows its inverse (float64 closed form, 1e-5)."""
    z, sx, sy, o = 5.0, 0.04, 0.012, 0.9
    th = np.deg2rad(30.0)
    q = (np.cos(th / 2), 0.0, 0.0, np.sin(th / 2))
    D, W, *_ = _render([dict(mu=(0.0, 0.0, z), s=(sx, sy, 0.01), o=o, q=q)])
    f = 100.0
    R2 = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    S = (f / z) ** 2 * R2 @ np.diag([sx * sx, sy * sy]) @ R2.T + 0.3 * np.eye(2)
    Si = np.linalg.inv(S)
    for (py, px) in [(11, 11), (9, 11), (11, 9), (12, 12), (8, 12)]:
        d = np.array([px + 0.5 - 10.5, py + 0.5 - 10.5])
        p = -0.5 * d @ Si @ d
        want = o * np.exp(p) if p >= -4.5 else 0.0
        assert abs(W[py, px] - want) <= 1e-5 * max(want, 1e-12), (py, px, W[py, px], want)


@pytest.mark.parametrize("turn", [0.0, 0.4])
def test_backproject_moved_camera(turn):
    """Back-projection inverts the camera pose: a camera rotated about y by `turn`
    and translated by t sees a Gaussian on its optical axis at depth 5; the
    centre pixel's cloud point is the ground map of R^T((0, 0, 5) - t)."""
    c, s = np.cos(turn), np.sin(turn)
    R = np.array([[c, 0, -s], [0, 1, 0], [s, 0, c]])
    t = np.array([0.3, -0.2, 1.0])
    world = R.T @ (np.array([0.0, 0.0, 5.0]) - t)
    cam = dict(_cam(), R=R, t=t)
    D, W, pu, pv, sc, fr, pre = _render([dict(mu=tuple(world), s=0.01, o=1.0)], cam=cam, stride=1)
    pix = [(py, px) for py in range(21) for px in range(21) if W[py, px] >= 0.1]
    idx = pix.index((10, 10))
    c0, rho, au, av = (np.asarray(a, np.float64) for a in fr)
    h = (world - c0) / rho
    r = np.linalg.norm(h)
    if r > 1:
        h = (2 - 1 / r) * h / r
    mm = pre["minmax"].astype(np.float64)
    gu = np.clip((h @ au - mm[0]) / (mm[1] - mm[0]), 0, 1)
    gv = np.clip((h @ av - mm[2]) / (mm[3] - mm[2]), 0, 1)
    assert abs(pu[idx] - gu) < 1e-5 and abs(pv[idx] - gv) < 1e-5
