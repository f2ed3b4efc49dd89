"""Pins of the anisotropic (projected-covariance) predicate O6a of the oracle
(ledger L24).

Each pin is independent of the oracle's own code: closed forms of the EWA
footprint for axis-aligned Gaussians on and off the optical axis, a rotation
about the optical axis, and a float64 brute force that builds Sigma from the
quaternion, the Jacobian of the perspective map and numpy's symmetric
eigen-solver.
"""
import numpy as np
import pytest

import oracle
from tests.helpers import mini_scene

CAM = dict(fx=200.0, fy=150.0, cx=80.0, cy=60.0, width=160, height=120,
           R=np.eye(3), t=np.zeros(3), z_near=0.1, z_far=100.0)


def _vis(sc):
    pre = {"gate": (sc.opacity >= np.float32(0.005)).astype(np.uint8)}
    return oracle.visibility_aniso(sc, pre, threads=1), pre


def _r_closed(fx, fy, z, a, sx, sy, sz):
    # axis-aligned Sigma = diag(sx^2, sy^2, sz^2), camera R = I, Gaussian at
    # (a z, 0, z): J = [[fx/z, 0, -fx a/z], [0, fy/z, 0]] ->
    # A = fx^2 (sx^2 + a^2 sz^2) / z^2 + 0.3, B = 0, C = fy^2 sy^2 / z^2 + 0.3
    A = fx * fx * (sx * sx + a * a * sz * sz) / (z * z) + 0.3
    C = fy * fy * sy * sy / (z * z) + 0.3
    return 3.0 * np.sqrt(max(A, C))


def test_cov_closed_form_rotation_about_z():
    """Sigma = R diag(s^2) R^T for a rotation by theta about z (q = (cos t/2, 0, 0, sin t/2))."""
    th = 0.7
    s = (0.3, 0.1, 0.05)
    sc = mini_scene([dict(mu=(0, 0, 5), s=s, q=(np.cos(th / 2), 0, 0, np.sin(th / 2)))], [CAM])
    cv = oracle.cov(sc)[0].astype(np.float64)
    c, si = np.cos(th), np.sin(th)
    R = np.array([[c, -si, 0], [si, c, 0], [0, 0, 1]])
    S = R @ np.diag(np.square(s)) @ R.T
    want = [S[0, 0], S[0, 1], S[0, 2], S[1, 1], S[1, 2], S[2, 2]]
    assert np.allclose(cv, want, rtol=1e-5, atol=1e-9)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_axis_aligned_radius_on_axis(axis):
    """On the optical axis the footprint radius is 3 sqrt(max(fx^2 sx^2, fy^2 sy^2)/z^2 + 0.3):
    a Gaussian whose centre lies just inside / outside the left image edge
    dilated by that radius flips visibility (each scale axis separately)."""
    z = 4.0
    s = [0.002, 0.002, 0.002]
    s[axis] = 0.05
    r = _r_closed(CAM["fx"], CAM["fy"], z, 0.0, *s)
    # on axis the centre projects to cx; shift the camera right instead of the
    # Gaussian so the Gaussian stays on its own optical axis is not possible --
    # use the off-axis closed form with sz's contribution (zero when a is tiny).
    gs = []
    for eps in (-1e-3, 1e-3):
        # find a with fx a + cx + r(a) = eps r(a)  (just inside: eps > 0)
        lo, hi = -10.0, 0.0
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            rr = _r_closed(CAM["fx"], CAM["fy"], z, mid, *s)
            if CAM["fx"] * mid + CAM["cx"] + rr < eps * rr:
                lo = mid
            else:
                hi = mid
        gs.append(dict(mu=(0.5 * (lo + hi) * z, 0.0, z), s=tuple(s)))
    sc = mini_scene(gs, [CAM])
    vis, _ = _vis(sc)
    bits = int(vis["rows"][0, 0])
    assert bits == 0b10, (axis, r, bits)


def test_off_axis_depth_elongation_counts():
    """A needle along the viewing axis (sz >> sx, sy) far off-axis: only the
    j02 = -fx x / z^2 term of the Jacobian makes it wide. The closed form
    A = fx^2 (sx^2 + a^2 sz^2)/z^2 + 0.3 decides visibility at the right edge."""
    z = 5.0
    s = (0.001, 0.001, 0.8)
    gs = []
    for eps in (-1e-3, 1e-3):
        lo, hi = 0.0, 10.0  # fx a + cx - W - r(a) = -eps r  (just inside: eps > 0)
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            rr = _r_closed(CAM["fx"], CAM["fy"], z, mid, *s)
            if CAM["fx"] * mid + CAM["cx"] - CAM["width"] - rr < -eps * rr:
                lo = mid
            else:
                hi = mid
        gs.append(dict(mu=(0.5 * (lo + hi) * z, 0.0, z), s=s))
    # the isotropic bound would call both visible (3 max(s) f / z is huge)
    sc = mini_scene(gs, [CAM])
    vis, _ = _vis(sc)
    assert int(vis["rows"][0, 0]) == 0b10


def test_rotation_about_optical_axis_swaps_extents():
    """On axis, rotating the Gaussian by 90 degrees about the optical axis swaps
    its x / y extents: with fx = fy the radius, hence the decision, is unchanged;
    with the edge test on v instead of u it follows the larger extent."""
    cam = dict(CAM, fx=180.0, fy=180.0)
    s = (0.06, 0.01, 0.01)
    q90 = (np.cos(np.pi / 4), 0.0, 0.0, np.sin(np.pi / 4))
    z = 3.0
    r = 3.0 * np.sqrt(180.0 ** 2 * 0.06 ** 2 / z ** 2 + 0.3)
    # centre just inside the top edge (v = -r (1 - 1e-3)) on the optical axis of a shifted camera
    dy = (-r * (1 - 1e-3) - cam["cy"]) / cam["fy"] * z
    cam2 = dict(cam, t=np.array([0.0, -dy, 0.0]))
    sc = mini_scene([dict(mu=(0, 0, z), s=s), dict(mu=(0, 0, z), s=s, q=q90)], [cam2])
    vis, _ = _vis(sc)
    assert int(vis["rows"][0, 0]) == 0b11


def _brute(sc):
    """float64: Sigma from the quaternion, J W Sigma W^T J^T + 0.3 I, eigvalsh."""
    G, N = sc.G, sc.N
    vis = np.zeros((N, G), bool)
    slack = np.zeros((N, G))
    q = np.stack([sc.qw, sc.qx, sc.qy, sc.qz], 1).astype(np.float64)
    w, x, y, z = q.T
    R = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                  2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                  2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1).reshape(G, 3, 3)
    Sd = np.stack([sc.sx, sc.sy, sc.sz], 1).astype(np.float64)
    M = R * Sd[:, None, :]
    Sig = M @ np.transpose(M, (0, 2, 1))
    P = np.stack([sc.x, sc.y, sc.z], 1).astype(np.float64)
    for c in range(N):
        W = sc.R[c].astype(np.float64)
        t = sc.t[c].astype(np.float64)
        pc = P @ W.T + t
        xc, yc, zc = pc.T
        fx, fy, cx, cy = (float(sc.fx[c]), float(sc.fy[c]), float(sc.cx[c]), float(sc.cy[c]))
        Wd, Hd = float(sc.width[c]), float(sc.height[c])
        ok = (zc > sc.z_near[c]) & (zc < sc.z_far[c]) & (sc.opacity >= np.float32(0.005))
        zs = np.where(ok, zc, 1.0)
        J = np.zeros((G, 2, 3))
        J[:, 0, 0] = fx / zs
        J[:, 0, 2] = -fx * xc / zs ** 2
        J[:, 1, 1] = fy / zs
        J[:, 1, 2] = -fy * yc / zs ** 2
        T = J @ W
        Sp = T @ Sig @ np.transpose(T, (0, 2, 1)) + 0.3 * np.eye(2)
        lam = np.linalg.eigvalsh(Sp)[:, -1]
        r = 3 * np.sqrt(lam)
        u = fx * xc / zs + cx
        v = fy * yc / zs + cy
        conds = np.stack([u + r, Wd + r - u, v + r, Hd + r - v], 1)
        vis[c] = ok & (conds >= 0).all(1)
        scale = np.abs(u) + np.abs(v) + r + Wd + Hd
        sl = np.abs(conds).min(1) / scale
        dz = np.minimum(np.abs(zc - sc.z_near[c]), np.abs(zc - sc.z_far[c])) / np.maximum(np.abs(zc), 1e-30)
        slack[c] = np.minimum(sl, dz)
    return vis, slack


def test_brute_force_float64_agrees(tiny_scene):
    """B1-aniso: the fp32 oracle equals the float64 EWA definition on every pair
    whose decision margin exceeds 1e-4 (relative); tiny config, all cameras."""
    sc = tiny_scene
    vis, pre = _vis(sc)
    bv, slack = _brute(sc)
    G = sc.G
    ob = np.unpackbits(vis["rows"].view(np.uint8), bitorder="little").reshape(sc.N, -1)[:, :G].astype(bool)
    sure = slack > 1e-4
    assert sure.mean() > 0.99
    assert (ob[sure] == bv[sure]).all()
    # the anisotropic footprint is never wider than the isotropic envelope used for culling:
    # 3 sqrt(trace(Sigma) |J|_F^2 + 0.3) -- so an iso-visible superset property holds per pair
    assert ob.sum() > 0


def test_depth_statistic_uses_camera_depth(tiny_scene):
    """D_c in the anisotropic mode is the opacity-weighted mean of zc over the
    visible set: recomputed here in float64 from the rows."""
    sc = tiny_scene
    vis, _ = _vis(sc)
    G = sc.G
    ob = np.unpackbits(vis["rows"].view(np.uint8), bitorder="little").reshape(sc.N, -1)[:, :G].astype(bool)
    P = np.stack([sc.x, sc.y, sc.z], 1).astype(np.float64)
    for c in range(0, sc.N, 7):
        zc = P @ sc.R[c, 2].astype(np.float64) + float(sc.t[c, 2])
        o = sc.opacity.astype(np.float64)
        m = ob[c]
        if m.any():
            want = (o[m] * zc[m]).sum() / o[m].sum()
            assert abs(vis["D"][c] - want) <= 1e-6 * abs(want)
            assert vis["K"][c] == m.sum()
