"""CPU oracle for the LoBE-GS visibility engine -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import, call, link or execute anything under
oracle/. The product path (paper_2510_01767_b200) never imports it and must
fail loudly when its CUDA library is missing.

The oracle is a plain scalar C++17 implementation (lobe_oracle.cpp) of
SURVEY.md §8(c) steps O1-O11, plus a float64 brute-force SPEC-formula
checker (brute.py). It shares no code with the CUDA path. This module only
marshals numpy arrays through ctypes and sequences the steps in the order
the paper defines them.

Parity status per function:
  validate / frame / prep / cam_setup / visibility (rows, K, z_min, z_max),
  assign, block_loads, crop: pinned (hand cases, B1 brute force,
  set enumeration, invariants);
  depth mean D_c: "parity partially unpinned" -- pinned only by hand case H7
  and positivity/bounds invariants (no paper values exist, ledger L3/L4).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lobe_oracle.cpp")
_LIB = os.path.join(_HERE, "liblobe_oracle.so")
_lock = threading.Lock()
_lib = None

STATUS = {0: "OK", 1: "INVALID_INPUT", 2: "INVALID_CONFIG", 3: "INVALID_CUTS", 4: "INVALID_INDEX",
          5: "DEGENERATE_SCENE"}
MODE_RATIO, MODE_HOME, MODE_UNION = 0, 1, 2


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle {what}: {STATUS.get(code, code)}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def build(force=False):
    """Compile the oracle with the contract's flags (SURVEY.md §8c 'Build flags')."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread",
               "-o", _LIB + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = ctypes.CDLL(build())
    return _lib


class _Cam(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("R", ctypes.c_float * 9),
                ("t", ctypes.c_float * 3), ("z_near", ctypes.c_float), ("z_far", ctypes.c_float)]


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _cams(scene):
    N = scene.N
    arr = (_Cam * N)()
    for c in range(N):
        k = arr[c]
        k.fx, k.fy, k.cx, k.cy = (float(scene.fx[c]), float(scene.fy[c]), float(scene.cx[c]), float(scene.cy[c]))
        k.width, k.height = int(scene.width[c]), int(scene.height[c])
        k.R[:] = [float(v) for v in scene.R[c].reshape(9)]
        k.t[:] = [float(v) for v in scene.t[c]]
        k.z_near, k.z_far = float(scene.z_near[c]), float(scene.z_far[c])
    return arr


def _chk(code, what):
    if code != 0:
        raise OracleError(code, what)


def nthreads():
    return int(os.environ.get("LOBE_ORACLE_THREADS", os.cpu_count() or 1))


def frame(scene, center=None, radius=None, axis_u=None, axis_v=None):
    """O2: resolved (c0, rho, a_u, a_v); None -> automatic (ledger L12)."""
    L = lib()
    c0 = np.zeros(3, np.float32) if center is None else np.asarray(center, np.float32).copy()
    rho = ctypes.c_float(0.0 if radius is None else float(radius))
    au = np.zeros(3, np.float32) if axis_u is None else np.asarray(axis_u, np.float32).copy()
    av = np.zeros(3, np.float32) if axis_v is None else np.asarray(axis_v, np.float32).copy()
    flags = (1 if center is None else 0) | (2 if radius is None else 0) | (4 if axis_u is None else 0)
    if axis_u is None and axis_v is not None:
        raise ValueError("give both axes or none")
    cams = _cams(scene)
    _chk(L.oracle_frame(ctypes.c_int64(scene.N), cams, ctypes.c_uint32(flags), _p(c0), ctypes.byref(rho),
                        _p(au), _p(av)), "frame")
    return c0, np.float32(rho.value), au, av


def validate(scene):
    L = lib()
    bad = ctypes.c_int64(-1)
    g = [np.ascontiguousarray(a, np.float32) for a in scene.gaussian_arrays()]
    st = L.oracle_validate_gaussians(ctypes.c_int64(scene.G), *[_p(a) for a in g], ctypes.byref(bad))
    if st:
        raise OracleError(st, f"validate gaussians (index {bad.value})")
    st = L.oracle_validate_cameras(ctypes.c_int64(scene.N), _cams(scene), ctypes.byref(bad))
    if st:
        raise OracleError(st, f"validate cameras (index {bad.value})")


def prep(scene, fr):
    """O3 + O4: per-Gaussian k, gate, gu, gv; per-camera setup rows and centre grid coords."""
    L = lib()
    c0, rho, au, av = fr
    G, N = scene.G, scene.N
    k = np.empty(G, np.float32)
    gate = np.empty(G, np.uint8)
    gu = np.empty(G, np.float32)
    gv = np.empty(G, np.float32)
    mm = np.empty(4, np.float32)
    _chk(L.oracle_prep(ctypes.c_int64(G), _p(scene.x), _p(scene.y), _p(scene.z), _p(scene.sx), _p(scene.sy),
                       _p(scene.sz), _p(scene.opacity), _p(c0), ctypes.c_float(rho), _p(au), _p(av), _p(k),
                       _p(gate), _p(gu), _p(gv), _p(mm)), "prep")
    setup = np.empty((N, 16), np.float32)
    cgu = np.empty(N, np.float32)
    cgv = np.empty(N, np.float32)
    _chk(L.oracle_cam_setup(ctypes.c_int64(N), _cams(scene), _p(c0), ctypes.c_float(rho), _p(au), _p(av), _p(mm),
                            _p(setup), _p(cgu), _p(cgv)), "cam_setup")
    return dict(k=k, gate=gate, gu=gu, gv=gv, minmax=mm, setup=setup, cam_gu=cgu, cam_gv=cgv)


def visibility(scene, pre, cams=None, threads=None):
    """O6/O7 for the selected cameras (all by default)."""
    L = lib()
    G = scene.G
    sel = None if cams is None else np.ascontiguousarray(cams, np.int64)
    ns = scene.N if sel is None else int(sel.shape[0])
    words = (G + 31) // 32
    rows = np.empty((ns, words), np.uint32)
    K = np.empty(ns, np.uint32)
    S = np.empty(ns, np.float64)
    Om = np.empty(ns, np.float64)
    zmin = np.empty(ns, np.float32)
    zmax = np.empty(ns, np.float32)
    _chk(L.oracle_visibility(ctypes.c_int64(G), _p(scene.x), _p(scene.y), _p(scene.z), _p(pre["k"]),
                             _p(pre["gate"]), _p(scene.opacity), ctypes.c_int64(ns), _p(sel), _p(pre["setup"]),
                             _p(rows), _p(K), _p(S), _p(Om), _p(zmin), _p(zmax),
                             ctypes.c_int(threads or nthreads())), "visibility")
    with np.errstate(invalid="ignore", divide="ignore"):
        D = np.where(K > 0, S / np.where(Om > 0, Om, 1.0), 0.0)   # O7
    return dict(rows=rows, K=K, S=S, Om=Om, D=D, zmin=zmin, zmax=zmax)


PRED_ISO, PRED_ANISO = 0, 1


def cov(scene):
    """O6a per-Gaussian 3D covariance {S00, S01, S02, S11, S12, S22} (ledger L24)."""
    L = lib()
    out = np.empty((scene.G, 6), np.float32)
    _chk(L.oracle_cov(ctypes.c_int64(scene.G), _p(scene.sx), _p(scene.sy), _p(scene.sz), _p(scene.qw),
                      _p(scene.qx), _p(scene.qy), _p(scene.qz), _p(out)), "cov")
    return out


def visibility_aniso(scene, pre, cams=None, threads=None):
    """O6a/O7 with the projected-covariance footprint (ledger L24)."""
    L = lib()
    G = scene.G
    sel = None if cams is None else np.ascontiguousarray(cams, np.int64)
    ns = scene.N if sel is None else int(sel.shape[0])
    words = (G + 31) // 32
    rows = np.empty((ns, words), np.uint32)
    K = np.empty(ns, np.uint32)
    S = np.empty(ns, np.float64)
    Om = np.empty(ns, np.float64)
    zmin = np.empty(ns, np.float32)
    zmax = np.empty(ns, np.float32)
    cv = pre.get("cov")
    if cv is None:
        cv = pre["cov"] = cov(scene)
    _chk(L.oracle_visibility_aniso(ctypes.c_int64(G), _p(scene.x), _p(scene.y), _p(scene.z), _p(cv),
                                   _p(pre["gate"]), _p(scene.opacity), ctypes.c_int64(ns), _p(sel), _cams(scene),
                                   _p(rows), _p(K), _p(S), _p(Om), _p(zmin), _p(zmax),
                                   ctypes.c_int(threads or nthreads())), "visibility_aniso")
    with np.errstate(invalid="ignore", divide="ignore"):
        D = np.where(K > 0, S / np.where(Om > 0, Om, 1.0), 0.0)   # O7
    return dict(rows=rows, K=K, S=S, Om=Om, D=D, zmin=zmin, zmax=zmax)


def default_grid(m, n, v=None, h=None, delta_v=None, delta_h=None, tau=None):
    """Uniform cuts (v0_i = i/m) and the paper's defaults
    delta = (0.1/m, 0.1/n) in fp32 (ledger L14), tau = 0.15."""
    if v is None:
        v = np.array([np.float32(i / m) for i in range(1, m)], np.float32)
    if h is None:
        h = np.array([np.float32(j / n) for j in range(1, n)], np.float32)
    dv = np.float32(np.float32(0.1) / np.float32(m)) if delta_v is None else np.float32(delta_v)
    dh = np.float32(np.float32(0.1) / np.float32(n)) if delta_h is None else np.float32(delta_h)
    return dict(m=m, n=n, v=np.asarray(v, np.float32), h=np.asarray(h, np.float32), dv=dv, dh=dh,
                tau=0.15 if tau is None else float(tau))


def assign(scene, pre, vis, grid, threads=None):
    L = lib()
    m, n = grid["m"], grid["n"]
    B = m * n
    ns = vis["rows"].shape[0]
    ncb = np.empty((ns, B), np.uint32)
    n0 = np.empty((ns, B), np.uint32)
    member = np.empty(ns, np.uint64)
    home = np.empty(ns, np.int32)
    cgu = pre["cam_gu"] if ns == scene.N else pre["cam_gu_sel"]
    cgv = pre["cam_gv"] if ns == scene.N else pre["cam_gv_sel"]
    _chk(L.oracle_assign(ctypes.c_int64(scene.G), _p(pre["gu"]), _p(pre["gv"]), ctypes.c_int64(ns),
                         _p(vis["rows"]), _p(vis["K"]), _p(cgu), _p(cgv), ctypes.c_int(m), ctypes.c_int(n),
                         _p(grid["v"]), _p(grid["h"]), ctypes.c_float(grid["dv"]), ctypes.c_float(grid["dh"]),
                         ctypes.c_double(grid["tau"]), _p(ncb), _p(n0), _p(member), _p(home),
                         ctypes.c_int(threads or nthreads())), "assign")
    return dict(n=ncb, n0=n0, member=member, home=home)


def block_loads(scene, pre, vis, asg, grid, mode=MODE_RATIO, masks=True):
    L = lib()
    m, n = grid["m"], grid["n"]
    B = m * n
    G = scene.G
    N = vis["rows"].shape[0]
    out = dict(n_cams=np.empty(B, np.uint32), g_blk=np.empty(B, np.uint32), g_vis=np.empty(B, np.uint32),
               incidences=np.empty(B, np.uint64), area=np.empty(B, np.float64), g_avgvis=np.empty(B, np.float64),
               lohi=np.empty((B, 4), np.float32))
    M = np.empty((B, (G + 63) // 64), np.uint64) if masks else None
    obj = ctypes.c_uint32(0)
    _chk(L.oracle_block_loads(ctypes.c_int64(G), _p(pre["gu"]), _p(pre["gv"]), ctypes.c_int64(N), _p(vis["rows"]),
                              _p(asg["member"]), _p(asg["home"]), _p(asg["n0"]), ctypes.c_int(m), ctypes.c_int(n),
                              _p(grid["v"]), _p(grid["h"]), ctypes.c_float(grid["dv"]), ctypes.c_float(grid["dh"]),
                              ctypes.c_int(mode), _p(out["n_cams"]), _p(out["g_blk"]), _p(out["g_vis"]),
                              _p(out["incidences"]), _p(out["area"]), _p(out["g_avgvis"]), _p(out["lohi"]), _p(M),
                              ctypes.byref(obj)), "block_loads")
    out["objective"] = int(obj.value)
    out["M"] = M
    return out


def crop(scene, pre, grid, M):
    L = lib()
    m, n = grid["m"], grid["n"]
    B = m * n
    W = (scene.G + 63) // 64
    c = np.empty((B, W), np.uint64)
    e = np.empty((B, W), np.uint64)
    _chk(L.oracle_crop(ctypes.c_int64(scene.G), _p(pre["gu"]), _p(pre["gv"]), ctypes.c_int(m), ctypes.c_int(n),
                       _p(grid["v"]), _p(grid["h"]), _p(M), _p(c), _p(e)), "crop")
    return c, e


def run(scene, grid=None, mode=MODE_RATIO, frame_args=None, threads=None, masks=True, predicate=PRED_ISO):
    """The whole path in the paper's order: validate, frame, per-Gaussian /
    per-camera setup, visibility (isotropic O6 or anisotropic O6a), assignment,
    block loads, crop."""
    validate(scene)
    cfg = scene.cfg
    if grid is None:
        grid = default_grid(cfg.m, cfg.n)
    fr = frame(scene, **(frame_args or {}))
    pre = prep(scene, fr)
    if predicate == PRED_ANISO:
        vis = visibility_aniso(scene, pre, threads=threads)
    else:
        vis = visibility(scene, pre, threads=threads)
    asg = assign(scene, pre, vis, grid, threads=threads)
    bl = block_loads(scene, pre, vis, asg, grid, mode=mode, masks=masks)
    out = dict(frame=fr, pre=pre, vis=vis, asg=asg, loads=bl, grid=grid)
    if masks:
        out["crop"], out["eligible"] = crop(scene, pre, grid, bl["M"])
    return out


def evaluate_cuts(scene, pre, vis, grid, mode=MODE_RATIO):
    """Objective max_b G_vis for one candidate grid on cached rows (PAPER.md:167,
    :179 'the back-projection is computed once and reused')."""
    asg = assign(scene, pre, vis, grid)
    return block_loads(scene, pre, vis, asg, grid, mode=mode, masks=False)["objective"]


# ------------------------------------------------------------------------------
# NEXT-4 block pipeline (
# ledger L25). Plain list operations over sub-scenes (small cases only); every
# float operation is one numpy float32 op in the order written (no fusion).
SUB_FIELDS = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")


def block_of_points(fr, mm, grid, x, y, z):
    """Delta = 0 cell block p n + q of arbitrary positions (O3 map, clamped, L25)."""
    L = lib()
    c0, rho, au, av = fr
    x, y, z = (np.ascontiguousarray(a, np.float32) for a in (x, y, z))
    out = np.empty(len(x), np.int32)
    _chk(L.oracle_block_of_points(ctypes.c_int64(len(x)), _p(x), _p(y), _p(z), _p(c0), ctypes.c_float(rho), _p(au),
                                  _p(av), _p(np.ascontiguousarray(mm, np.float32)), grid["m"], grid["n"],
                                  _p(grid["v"]), _p(grid["h"]), _p(out)), "block_of_points")
    return out


def subscene(scene, crop_b, elig_b):
    """visibility_crop: the Gaussians of block b's crop mask in
    ascending caller index; origin = that index; in_block = eligible bit."""
    G = scene.G
    idx = [i for i in range(G) if (int(crop_b[i >> 6]) >> (i & 63)) & 1]
    sub = {k: np.array([getattr(scene, k)[i] for i in idx], np.float32) for k in SUB_FIELDS}
    sub["origin"] = np.array(idx, np.int64)
    sub["in_block"] = np.array([(int(elig_b[i >> 6]) >> (i & 63)) & 1 for i in idx], np.uint8)
    return sub


def _rot(qw, qx, qy, qz):
    f = np.float32
    two, one = f(2.0), f(1.0)
    return [one - two * (qy * qy + qz * qz), two * (qx * qy - qw * qz), two * (qx * qz + qw * qy),
            two * (qx * qy + qw * qz), one - two * (qx * qx + qz * qz), two * (qy * qz - qw * qx),
            two * (qx * qz - qw * qy), two * (qy * qz + qw * qx), one - two * (qx * qx + qy * qy)]


def densify_step(sub, grad, normals, tau_grad, scale_split, fr, mm, grid, b):
    """simulate_densify_step (ledger L25). Selected: in_block and
    grad >= tau_grad. Clone (max s < scale_split): two Gaussians at
    mu + (0.1 s) * n_k, k = 1 keeps the origin, k = 2 gets -1. Split: two
    children at mu + R(q) (s * n_k) with scale s / 1.6, origin -1. n_1 =
    normals[i, 0:3], n_2 = normals[i, 3:6]. Moved / new Gaussians get a fresh
    in-block test; everything else is copied field for field, in input order."""
    f = np.float32
    out = {k: [] for k in SUB_FIELDS + ("origin", "in_block")}
    pend = []  # (out position, x, y, z) needing an in-block test

    def put(vals, origin, inb):
        for k in SUB_FIELDS:
            out[k].append(f(vals[k]))
        out["origin"].append(int(origin))
        out["in_block"].append(int(inb))

    for i in range(len(sub["x"])):
        g = {k: f(sub[k][i]) for k in SUB_FIELDS}
        if not (sub["in_block"][i] and f(grad[i]) >= f(tau_grad)):
            put(g, sub["origin"][i], sub["in_block"][i])
            continue
        n = [f(v) for v in normals[i]]
        smax = max(g["sx"], g["sy"], g["sz"])
        for k in range(2):
            nk = n[3 * k:3 * k + 3]
            c = dict(g)
            if smax < f(scale_split):  # clone: jitter by 0.1 s
                c["x"] = g["x"] + (f(0.1) * g["sx"]) * nk[0]
                c["y"] = g["y"] + (f(0.1) * g["sy"]) * nk[1]
                c["z"] = g["z"] + (f(0.1) * g["sz"]) * nk[2]
                origin = sub["origin"][i] if k == 0 else -1
            else:  # split: sample inside the parent footprint, scale / 1.6
                r = _rot(g["qw"], g["qx"], g["qy"], g["qz"])
                t = [g["sx"] * nk[0], g["sy"] * nk[1], g["sz"] * nk[2]]
                d = [(r[3 * a] * t[0] + r[3 * a + 1] * t[1]) + r[3 * a + 2] * t[2] for a in range(3)]
                c["x"], c["y"], c["z"] = g["x"] + d[0], g["y"] + d[1], g["z"] + d[2]
                c["sx"], c["sy"], c["sz"] = g["sx"] / f(1.6), g["sy"] / f(1.6), g["sz"] / f(1.6)
                origin = -1
            pend.append(len(out["x"]))
            put(c, origin, 0)
    res = {k: np.array(v, np.float32) for k, v in out.items() if k in SUB_FIELDS}
    res["origin"] = np.array(out["origin"], np.int64)
    res["in_block"] = np.array(out["in_block"], np.uint8)
    if pend:
        pend = np.array(pend)
        blk = block_of_points(fr, mm, grid, res["x"][pend], res["y"][pend], res["z"][pend])
        res["in_block"][pend] = (blk == b).astype(np.uint8)
    return res


def prune_outside(sub, fr, mm, grid, b):
    """prune_outside: keep the Gaussians whose centre lies in block
    b's delta = 0 cell (fresh test), in order."""
    blk = block_of_points(fr, mm, grid, sub["x"], sub["y"], sub["z"])
    keep = [i for i in range(len(blk)) if blk[i] == b]
    res = {k: np.asarray(v)[keep] for k, v in sub.items()}
    res["in_block"] = np.ones(len(keep), np.uint8)
    return res


def merge_blocks(subs):
    """merge_blocks: concatenation in block order; a non-negative
    origin appearing twice is an integrity error (returns (merged, ok))."""
    res = {k: np.concatenate([np.asarray(s[k]) for s in subs]) for k in subs[0]}
    o = res["origin"][res["origin"] >= 0]
    ok = len(np.unique(o)) == len(o)
    return res, ok


# ------------------------------------------------------------------------------
# NEXT-1 paper-exact camera selection (
# SPEC.md:335-353, :383-387; ledger L26): alpha-blended depth render of each
# camera's visible Gaussians at 1/downscale resolution, back-projection of every
# stride-th pixel with weight >= eps_w, V_{c,b} ratios over the clouds.
def render_camera(scene, pre, fr, c, vis_idx, downscale=4, stride=2, eps_w=0.1):
    """One camera: returns (D map, W map, cloud gu, cloud gv)."""
    L = lib()
    c0, rho, au, av = fr
    cv = pre.get("cov")
    if cv is None:
        cv = pre["cov"] = cov(scene)
    cams = _cams(scene)
    Wd, Hd = int(scene.width[c]) // downscale, int(scene.height[c]) // downscale
    D = np.zeros((Hd, Wd), np.float32)
    W = np.zeros((Hd, Wd), np.float32)
    cap = max(1, -(-Hd // stride) * -(-Wd // stride))
    pu = np.empty(cap, np.float32)
    pv = np.empty(cap, np.float32)
    K = ctypes.c_int64()
    vis_idx = np.ascontiguousarray(vis_idx, np.int64)
    _chk(L.oracle_render_camera(ctypes.c_int64(scene.G), _p(scene.x), _p(scene.y), _p(scene.z), _p(cv),
                                _p(scene.opacity), ctypes.byref(cams[c]), ctypes.c_int64(len(vis_idx)), _p(vis_idx),
                                ctypes.c_int(downscale), ctypes.c_int(stride), ctypes.c_float(eps_w), _p(c0),
                                ctypes.c_float(rho), _p(au), _p(av), _p(np.ascontiguousarray(pre["minmax"])),
                                _p(D), _p(W), _p(pu), _p(pv), ctypes.byref(K)), "render_camera")
    return D, W, pu[:K.value].copy(), pv[:K.value].copy()


def render_clouds(scene, pre, vis, fr, downscale=4, stride=2, eps_w=0.1):
    """All cameras: CSR clouds {off, gu, gv} from the visibility rows' sets."""
    G = scene.G
    rows = vis["rows"]
    bits = np.unpackbits(rows.view(np.uint8), bitorder="little").reshape(rows.shape[0], -1)[:, :G]
    off = [0]
    us, vs = [], []
    for c in range(rows.shape[0]):
        _, _, pu, pv = render_camera(scene, pre, fr, c, np.flatnonzero(bits[c]), downscale, stride, eps_w)
        us.append(pu)
        vs.append(pv)
        off.append(off[-1] + len(pu))
    return dict(off=np.array(off, np.int64), gu=np.concatenate(us) if us else np.zeros(0, np.float32),
                gv=np.concatenate(vs) if vs else np.zeros(0, np.float32))


def assign_points(scene, pre, clouds, grid):
    """O8 over the back-projected clouds: V_{c,b} = n / K >= tau."""
    L = lib()
    m, n = grid["m"], grid["n"]
    B = m * n
    ns = len(clouds["off"]) - 1
    ncb = np.empty((ns, B), np.uint32)
    n0 = np.empty((ns, B), np.uint32)
    member = np.empty(ns, np.uint64)
    home = np.empty(ns, np.int32)
    _chk(L.oracle_assign_points(ctypes.c_int64(ns), _p(clouds["off"]), _p(clouds["gu"]), _p(clouds["gv"]),
                                _p(pre["cam_gu"]), _p(pre["cam_gv"]), ctypes.c_int(m), ctypes.c_int(n),
                                _p(grid["v"]), _p(grid["h"]), ctypes.c_float(grid["dv"]), ctypes.c_float(grid["dh"]),
                                ctypes.c_double(grid["tau"]), _p(ncb), _p(n0), _p(member), _p(home)),
         "assign_points")
    K = np.diff(clouds["off"]).astype(np.uint32)
    return dict(n=ncb, n0=n0, member=member, home=home, K=K)
