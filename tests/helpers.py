"""Small explicit scenes for hand cases (no generator, no method arithmetic)."""
import dataclasses

import numpy as np

from synth.scenes import Scene, SceneConfig

C0_CAM = dict(fx=100.0, fy=100.0, cx=50.0, cy=50.0, width=100, height=100,
              R=np.eye(3), t=np.zeros(3), z_near=0.1, z_far=100.0)


def mini_scene(gaussians, cameras, m=1, n=1):
    """gaussians: list of dicts {mu, s (scalar or 3), o, q (optional)};
    cameras: list of dicts with the CameraView fields."""
    G = len(gaussians)
    f32 = lambda a: np.asarray(a, dtype=np.float32)
    mu = np.array([g["mu"] for g in gaussians], dtype=np.float64)
    s = np.array([np.broadcast_to(np.asarray(g.get("s", 0.1), dtype=np.float64), (3,)) for g in gaussians])
    q = np.array([g.get("q", (1.0, 0.0, 0.0, 0.0)) for g in gaussians], dtype=np.float64)
    o = np.array([g.get("o", 1.0) for g in gaussians], dtype=np.float64)
    N = len(cameras)
    cfg = SceneConfig("mini", G, N, m, n, 100, 100, 90.0, (-1, 1, -1, 1), 1.0, 1, 0.0, 0)
    return Scene(cfg, f32(mu[:, 0]), f32(mu[:, 1]), f32(mu[:, 2]), f32(s[:, 0]), f32(s[:, 1]), f32(s[:, 2]),
                 f32(q[:, 0]), f32(q[:, 1]), f32(q[:, 2]), f32(q[:, 3]), f32(o),
                 cam_id=np.arange(N, dtype=np.int32),
                 fx=f32([c["fx"] for c in cameras]), fy=f32([c["fy"] for c in cameras]),
                 cx=f32([c["cx"] for c in cameras]), cy=f32([c["cy"] for c in cameras]),
                 width=np.array([c["width"] for c in cameras], np.int32),
                 height=np.array([c["height"] for c in cameras], np.int32),
                 R=f32([np.asarray(c["R"]) for c in cameras]), t=f32([np.asarray(c["t"]) for c in cameras]),
                 z_near=f32([c["z_near"] for c in cameras]), z_far=f32([c["z_far"] for c in cameras]))


def bits_of_row(row, G):
    """Set of Gaussian indices whose bit is set in a u32 row (bit i%32 of word i/32)."""
    out = set()
    for w, val in enumerate(row):
        val = int(val)
        while val:
            b = (val & -val).bit_length() - 1
            i = 32 * w + b
            if i < G:
                out.add(i)
            val &= val - 1
    return out


def bits_of_mask64(mask, G):
    out = set()
    for w, val in enumerate(mask):
        val = int(val)
        while val:
            b = (val & -val).bit_length() - 1
            i = 64 * w + b
            if i < G:
                out.add(i)
            val &= val - 1
    return out


def nadir_camera(px, py, pz, f=100.0, W=100, H=100, zn=0.01, zf=100.0):
    """Camera at (px,py,pz) looking down -z: R = diag(1,-1,-1), t = -R p."""
    R = np.diag([1.0, -1.0, -1.0])
    t = -R @ np.array([px, py, pz])
    return dict(fx=f, fy=f, cx=W / 2, cy=H / 2, width=W, height=H, R=R, t=t, z_near=zn, z_far=zf)
