"""Deterministic synthetic Gaussian scenes and aerial camera rigs.

Shapes follow BASELINE.json `configs` and the recipe of SURVEY.md §8(d)
("Configs restated as synthetic inputs", "Value distributions"):

* 70 % clustered structure (log-normal cluster masses, sigma = skew),
  25 % ground plane, 5 % far background on the upper hemisphere;
* per-axis scales exp(N(ln 0.004, 0.5)), background scaled by distance;
* quaternions = normalised N(0,1)^4, opacity = sigmoid(N(0, 1.5));
* cameras: jittered lawnmower grid over 1.1x the footprint, ceil(N/5)
  positions x 5 orientations (nadir + 4 headings at -55 deg pitch),
  pinhole fx = fy = W / (2 tan(hfov/2)), cx = W/2, cy = H/2.

The Gaussians are emitted in a random order (as a trained 3DGS checkpoint
is), so any spatial sort the engine applies is exercised.

Camera convention (SPEC.md:45 CameraView): world_to_cam rotation R (row
major) and translation t, p_cam = R p_world + t, camera looks along +z_cam.

Everything is drawn from numpy's PCG64 stream seeded by the config seed;
fp64 draws are rounded once to fp32. No method arithmetic lives here.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class SceneConfig:
    name: str
    G: int
    N: int
    m: int
    n: int
    width: int
    height: int
    hfov_deg: float
    footprint: tuple          # (xmin, xmax, ymin, ymax)
    altitude: float
    clusters: int
    skew: float
    seed: int
    z_near: float = 0.01
    z_far: float = 8.0
    pitch_deg: float = -55.0


# SURVEY.md §8(d) table "Configs restated as synthetic inputs". Altitudes are
# the tuned values ("Tune the altitude ... until the measured
# median visible fraction falls in the target band, then freeze them"); the
# measured medians are recorded in DESIGN.md "Input recipe".
CONFIGS = {
    "tiny": SceneConfig("tiny", 10_000, 64, 2, 2, 160, 120, 60.0, (-1, 1, -1, 1), 1.5, 16, 1.0, 0x25100001),
    "rubble": SceneConfig("rubble", 2_000_000, 1657, 3, 3, 1152, 864, 60.0, (-1, 1, -1, 1), 0.7, 72, 1.0,
                          0x25100002),
    "building": SceneConfig("building", 3_000_000, 1920, 4, 3, 1152, 864, 60.0, (-1, 1, -0.75, 0.75), 0.45, 96,
                            1.0, 0x25100003),
    "residence": SceneConfig("residence", 4_000_000, 2582, 4, 4, 1368, 912, 60.0, (-1, 1, -1, 1), 0.6, 128,
                             1.0, 0x25100004),
    "matrixcity": SceneConfig("matrixcity", 10_000_000, 5620, 6, 6, 1600, 900, 60.0, (-1, 1, -1, 1), 0.35, 288,
                              1.2, 0x25100005),
}


def make_config(base: str, **over) -> SceneConfig:
    """A config derived from a named one (smaller G/N for tests, other seed...)."""
    return dataclasses.replace(CONFIGS[base], **over)


@dataclasses.dataclass
class Scene:
    cfg: SceneConfig
    # Gaussians, SoA fp32, caller order (SPEC.md:28-33 Gaussian3D)
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    sx: np.ndarray
    sy: np.ndarray
    sz: np.ndarray
    qw: np.ndarray
    qx: np.ndarray
    qy: np.ndarray
    qz: np.ndarray
    opacity: np.ndarray
    # cameras (SPEC.md:44-49 CameraView)
    cam_id: np.ndarray      # int32 [N]
    fx: np.ndarray          # fp32 [N]
    fy: np.ndarray
    cx: np.ndarray
    cy: np.ndarray
    width: np.ndarray       # int32 [N]
    height: np.ndarray
    R: np.ndarray           # fp32 [N,3,3] world->cam, row major
    t: np.ndarray           # fp32 [N,3]
    z_near: np.ndarray      # fp32 [N]
    z_far: np.ndarray

    @property
    def G(self) -> int:
        return int(self.x.shape[0])

    @property
    def N(self) -> int:
        return int(self.fx.shape[0])

    def gaussian_arrays(self):
        return [self.x, self.y, self.z, self.sx, self.sy, self.sz, self.qw, self.qx, self.qy, self.qz,
                self.opacity]

    def subset_cameras(self, idx) -> "Scene":
        idx = np.asarray(idx)
        d = dataclasses.asdict(self) if False else None  # noqa: F841 (keep dataclass shallow)
        return dataclasses.replace(
            self, cam_id=self.cam_id[idx], fx=self.fx[idx], fy=self.fy[idx], cx=self.cx[idx], cy=self.cy[idx],
            width=self.width[idx], height=self.height[idx], R=self.R[idx], t=self.t[idx],
            z_near=self.z_near[idx], z_far=self.z_far[idx])

    def permute_gaussians(self, perm) -> "Scene":
        perm = np.asarray(perm)
        kw = {k: getattr(self, k)[perm] for k in ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz",
                                                   "opacity")}
        return dataclasses.replace(self, **kw)


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))


def _gaussians(cfg: SceneConfig, rng: np.random.Generator):
    G = cfg.G
    xmin, xmax, ymin, ymax = cfg.footprint
    area = (xmax - xmin) * (ymax - ymin)
    n_struct = int(round(0.70 * G))
    n_ground = int(round(0.25 * G))
    n_bg = G - n_struct - n_ground

    # structure: log-normal cluster masses, centres uniform on the footprint
    masses = rng.lognormal(0.0, cfg.skew, size=cfg.clusters)
    masses /= masses.sum()
    counts = rng.multinomial(n_struct, masses)
    ccx = rng.uniform(xmin, xmax, cfg.clusters)
    ccy = rng.uniform(ymin, ymax, cfg.clusters)
    hc = rng.uniform(0.01, 0.15, cfg.clusters)
    cell = math.sqrt(area / cfg.clusters)
    cid = np.repeat(np.arange(cfg.clusters), counts)
    sx_ = rng.normal(0.0, 0.35 * cell, n_struct)
    sy_ = rng.normal(0.0, 0.35 * cell, n_struct)
    px = ccx[cid] + sx_
    py = ccy[cid] + sy_
    pz = np.abs(rng.normal(0.0, 1.0, n_struct)) * hc[cid]

    # ground
    gx = rng.uniform(xmin, xmax, n_ground)
    gy = rng.uniform(ymin, ymax, n_ground)
    gz = rng.normal(0.0, 0.002, n_ground)

    # background: direction uniform on the upper hemisphere, distance 2 e^{U(0, ln 10)}
    v = rng.normal(size=(n_bg, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    v[:, 2] = np.abs(v[:, 2])
    dist = 2.0 * np.exp(rng.uniform(0.0, math.log(10.0), n_bg))
    bx, by, bz = (v * dist[:, None]).T

    x = np.concatenate([px, gx, bx])
    y = np.concatenate([py, gy, by])
    z = np.concatenate([pz, gz, bz])
    scale_mul = np.concatenate([np.ones(n_struct + n_ground), dist])
    s = np.exp(rng.normal(math.log(0.004), 0.5, size=(G, 3))) * scale_mul[:, None]
    q = rng.normal(size=(G, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = 1.0 / (1.0 + np.exp(-rng.normal(0.0, 1.5, G)))

    order = rng.permutation(G)   # checkpoint order: spatially unsorted
    cols = [x, y, z, s[:, 0], s[:, 1], s[:, 2], q[:, 0], q[:, 1], q[:, 2], q[:, 3], op]
    return [_f32(c[order]) for c in cols]


def _look(forward, up=(0.0, 0.0, 1.0)):
    """world->cam rotation rows (x_cam, y_cam, z_cam=forward), right handed."""
    f = np.asarray(forward, dtype=np.float64)
    f = f / np.linalg.norm(f)
    xa = np.cross(f, np.asarray(up, dtype=np.float64))
    if np.linalg.norm(xa) < 1e-9:          # nadir: image x along world +x
        xa = np.array([1.0, 0.0, 0.0])
        xa = xa - f * np.dot(xa, f)
    xa /= np.linalg.norm(xa)
    ya = np.cross(f, xa)
    return np.stack([xa, ya, f])


def _cameras(cfg: SceneConfig, rng: np.random.Generator):
    N = cfg.N
    xmin, xmax, ymin, ymax = cfg.footprint
    cxm, cym = 0.5 * (xmin + xmax), 0.5 * (ymin + ymax)
    hw, hh = 0.55 * (xmax - xmin), 0.55 * (ymax - ymin)      # 1.1x the footprint
    P = -(-N // 5)
    aspect = hw / hh
    nx = max(1, int(math.ceil(math.sqrt(P * aspect))))
    ny = max(1, int(math.ceil(P / nx)))
    pos = []
    for j in range(ny):
        cols = range(nx) if j % 2 == 0 else range(nx - 1, -1, -1)   # lawnmower
        for i in cols:
            pos.append((i, j))
    pos = pos[:P]
    dx, dy = 2 * hw / nx, 2 * hh / ny
    pitch = math.radians(cfg.pitch_deg)
    Rs, ts, cen = [], [], []
    for (i, j) in pos:
        px = cxm - hw + (i + 0.5 + rng.uniform(-0.25, 0.25)) * dx
        py = cym - hh + (j + 0.5 + rng.uniform(-0.25, 0.25)) * dy
        pz = cfg.altitude * (1.0 + rng.uniform(-0.05, 0.05))
        o = np.array([px, py, pz])
        fwds = [(0.0, 0.0, -1.0)]
        for k in range(4):
            th = math.radians(90.0 * k) + rng.uniform(-0.1, 0.1)
            fwds.append((math.cos(pitch) * math.cos(th), math.cos(pitch) * math.sin(th), math.sin(pitch)))
        for f in fwds:
            R = _look(f)
            Rs.append(R)
            ts.append(-R @ o)
            cen.append(o)
    Rs = np.stack(Rs)[:N]
    ts = np.stack(ts)[:N]
    W, H = cfg.width, cfg.height
    f = W / (2.0 * math.tan(math.radians(cfg.hfov_deg) / 2.0))
    return dict(
        cam_id=np.arange(N, dtype=np.int32),
        fx=_f32(np.full(N, f)), fy=_f32(np.full(N, f)),
        cx=_f32(np.full(N, W / 2.0)), cy=_f32(np.full(N, H / 2.0)),
        width=np.full(N, W, dtype=np.int32), height=np.full(N, H, dtype=np.int32),
        R=_f32(Rs), t=_f32(ts),
        z_near=_f32(np.full(N, cfg.z_near)), z_far=_f32(np.full(N, cfg.z_far)),
    )


def make_scene(cfg) -> Scene:
    """Generate the scene for a config (name or SceneConfig); deterministic in cfg.seed."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    g = _gaussians(cfg, rng)
    c = _cameras(cfg, rng)
    return Scene(cfg, *g, **c)


def array_hashes(scene: Scene) -> dict:
    """SHA-256 (first 16 hex digits) of every generated array, for run logs."""
    out = {}
    for k in ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity", "fx", "fy", "cx", "cy",
              "width", "height", "R", "t", "z_near", "z_far"):
        out[k] = hashlib.sha256(np.ascontiguousarray(getattr(scene, k)).tobytes()).hexdigest()[:16]
    return out
