"""Brute-force float64 evaluation of SPEC's visibility predicate (pin B1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). This is deliberately a
*different formula* from the oracle's pinned fp32 op order (SURVEY.md §8c
O6): it projects with divisions, in float64, exactly as SPEC.md states it:

  SPEC.md:243 visibility.visible_set -- "Gaussian i's center projects with
  depth in (z_near, z_far) and its projected center falls within the image
  rectangle dilated by its 3 sigma screen-space footprint, and opacity >= eps_o";
  SPEC.md:99  project_point -- "pixel = (fx x/z + cx, fy y/z + cy)";
  SPEC.md:299 -- footprint r = 3 max(scale) / depth * max(fx, fy) pixels;
  SPEC.md:298 -- eps_o = 0.005.

`margin` returns, per (camera, Gaussian), the smallest normalised distance
to any of the predicate's decision boundaries, so tests can compare the
oracle with this formula away from the boundary band.
"""
import numpy as np

EPS_O = 0.005


def predicate_f64(scene, cams=None, gidx=None):
    """visible[c, i] and margin[c, i] in float64 for the selected cameras/Gaussians."""
    cams = np.arange(scene.N) if cams is None else np.asarray(cams)
    g = slice(None) if gidx is None else np.asarray(gidx)
    P = np.stack([scene.x[g], scene.y[g], scene.z[g]]).astype(np.float64)          # [3, G]
    smax = np.max(np.stack([scene.sx[g], scene.sy[g], scene.sz[g]]), axis=0).astype(np.float64)
    op = scene.opacity[g].astype(np.float64)
    vis, mar = [], []
    for c in cams:
        R = scene.R[c].astype(np.float64)
        t = scene.t[c].astype(np.float64)
        pc = R @ P + t[:, None]
        xc, yc, zc = pc
        fx, fy = float(scene.fx[c]), float(scene.fy[c])
        cx, cy = float(scene.cx[c]), float(scene.cy[c])
        W, H = float(scene.width[c]), float(scene.height[c])
        zn, zf = float(scene.z_near[c]), float(scene.z_far[c])
        with np.errstate(divide="ignore", invalid="ignore"):
            u = fx * xc / zc + cx
            v = fy * yc / zc + cy
            r = 3.0 * smax * max(fx, fy) / zc
        depth_ok = (zc > zn) & (zc < zf)
        img_ok = (u >= -r) & (u <= W + r) & (v >= -r) & (v <= H + r)
        op_ok = op >= EPS_O
        vis.append(depth_ok & img_ok & op_ok)
        # normalised margins to each boundary (relative to the scale of the quantities)
        with np.errstate(divide="ignore", invalid="ignore"):
            m = np.minimum.reduce([
                np.abs(zc - zn) / max(zn, 1e-30), np.abs(zf - zc) / zf,
                np.abs(u + r) / (np.abs(u) + np.abs(r) + 1.0), np.abs(W + r - u) / (np.abs(u) + W + np.abs(r)),
                np.abs(v + r) / (np.abs(v) + np.abs(r) + 1.0), np.abs(H + r - v) / (np.abs(v) + H + np.abs(r)),
                np.abs(op - EPS_O) / EPS_O,
            ])
        m = np.where(np.isfinite(m), m, 0.0)
        mar.append(m)
    return np.array(vis), np.array(mar)
