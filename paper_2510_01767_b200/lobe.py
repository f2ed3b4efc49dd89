"""ctypes binding of the C ABI in include/lobe.h (argument marshalling only).

Every step of the path runs in csrc/liblobe.so (sm_100a kernels + host
runtime). There is no fallback: if the library is missing or no CUDA device is
present, calls raise. Names follow the C ABI without the `lobe_` prefix.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOBE_LIB", os.path.join(_HERE, "csrc", "liblobe.so"))  # override: tuning builds

STATUS = {0: "OK", 1: "INVALID_INPUT", 2: "INVALID_CONFIG", 3: "INVALID_CUTS", 4: "INVALID_INDEX",
          5: "DEGENERATE_SCENE", 6: "CUDA", 7: "NCCL", 8: "OOM", 9: "STATE", 10: "CAPACITY", 11: "INTEGRITY"}
ASSIGN_RATIO, ASSIGN_HOME, ASSIGN_UNION = 0, 1, 2
FRAME_AUTO_CENTER, FRAME_AUTO_RADIUS, FRAME_AUTO_AXES, FRAME_AUTO_ALL = 1, 2, 4, 7

# symbols include/lobe.h declares (tests check the library exports all of them)
EXPORTS = ["lobe_load_scene", "lobe_free_scene", "lobe_last_error", "lobe_assign_cameras", "lobe_block_loads",
           "lobe_crop_masks", "lobe_balance_partition", "lobe_bo_run", "lobe_mask_words", "lobe_block_partial",
           "lobe_masks_combine", "lobe_block_records", "lobe_crop_from_masks", "lobe_export_rows",
           "lobe_get_stats", "lobe_scene_info", "lobe_version", "lobe_dev_vis_bench", "lobe_block_subscene",
           "lobe_densify_step", "lobe_prune_outside", "lobe_merge_blocks", "lobe_render_select",
           "lobe_camera_clouds", "lobe_render_maps", "lobe_nccl_unique_id", "lobe_release_comms",
           "lobe_xchg_block_loads_host", "lobe_xchg_all_masks_host", "lobe_xchg_gather_cameras_host"]


PREDICATE_ISOTROPIC, PREDICATE_ANISOTROPIC = 0, 1  # lobe_options.predicate (DESIGN.md ledger L24)


class LobeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class Gaussians(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64)] + [(k, ctypes.c_void_p) for k in
                                           ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")] + \
               [("on_device", ctypes.c_int32)]


SUB_FIELDS = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")


class SubScene(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64)] + [(k, ctypes.c_void_p) for k in SUB_FIELDS] + \
               [("origin", ctypes.c_void_p), ("in_block", ctypes.c_void_p)]


def _sub_alloc(cap, device):
    """Device arrays (torch) for a sub-scene of capacity `cap`."""
    import torch
    cap = max(int(cap), 1)
    d = {k: torch.empty(cap, dtype=torch.float32, device=device) for k in SUB_FIELDS}
    d["origin"] = torch.empty(cap, dtype=torch.int64, device=device)
    d["in_block"] = torch.empty(cap, dtype=torch.uint8, device=device)
    return d


def _sub_struct(d, n):
    return SubScene(int(n), *[_ptr(d[k]) for k in SUB_FIELDS], _ptr(d["origin"]), _ptr(d["in_block"]))


def _sub_result(d, st):
    return {k: v[:st.n] for k, v in d.items()}


class Camera(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int32), ("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float),
                ("cy", ctypes.c_float), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("R", ctypes.c_float * 9), ("t", ctypes.c_float * 3), ("z_near", ctypes.c_float),
                ("z_far", ctypes.c_float)]


class Frame(ctypes.Structure):
    _fields_ = [("center", ctypes.c_float * 3), ("radius", ctypes.c_float), ("axis_u", ctypes.c_float * 3),
                ("axis_v", ctypes.c_float * 3), ("auto_flags", ctypes.c_uint32)]


# lobe_host_comm callbacks (include/lobe.h): 0 = success
HC_ALL_GATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)
HC_ALL_REDUCE_U64 = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t)
HC_ALL_TO_ALL_V = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t),
                                   ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t),
                                   ctypes.POINTER(ctypes.c_size_t))


class HostComm(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("all_gather", HC_ALL_GATHER), ("all_reduce_u64", HC_ALL_REDUCE_U64),
                ("all_to_all_v", HC_ALL_TO_ALL_V)]


class Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("assign_mode", ctypes.c_int32), ("predicate", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("host_comm", ctypes.POINTER(HostComm))]


class Grid(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("n", ctypes.c_int32), ("v", ctypes.c_void_p), ("h", ctypes.c_void_p),
                ("delta_v", ctypes.c_float), ("delta_h", ctypes.c_float), ("tau", ctypes.c_double)]


class BlockLoad(ctypes.Structure):
    _fields_ = [("block_id", ctypes.c_int32), ("row", ctypes.c_int32), ("col", ctypes.c_int32),
                ("lo", ctypes.c_float * 2), ("hi", ctypes.c_float * 2), ("area", ctypes.c_double),
                ("n_cams", ctypes.c_uint32), ("g_blk", ctypes.c_uint32), ("g_vis", ctypes.c_uint32),
                ("g_avgvis", ctypes.c_double), ("incidences", ctypes.c_uint64)]


class BalanceOpts(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int32), ("seed", ctypes.c_uint64), ("delta_scale", ctypes.c_float),
                ("tau", ctypes.c_double), ("n_sobol", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("t_prep_ms", "t_vis_ms", "t_hist_ms", "t_loads_ms", "t_comm_ms",
                                               "t_crop_ms")] + \
               [(k, ctypes.c_uint64) for k in ("tests_executed", "bytes_read", "bytes_written", "vis_launches",
                                               "evaluations")] + \
               [(k, ctypes.c_int64) for k in ("n_gaussians", "n_cameras", "n_local_cameras", "cam_begin")] + \
               [("tile_pairs", ctypes.c_uint64), ("dense_tests", ctypes.c_uint64), ("t_cull_ms", ctypes.c_double),
                ("t_depth_ms", ctypes.c_double),
                ("kernel_launches", ctypes.c_uint64),
                ("cub_launches", ctypes.c_uint64), ("kept_tests", ctypes.c_uint64),
                ("accepted_tests", ctypes.c_uint64), ("exact_variant_tests", ctypes.c_uint64 * 6),
                ("decided_tests", ctypes.c_uint64 * 4), ("visible_bits", ctypes.c_uint64 * 2),
                ("exact_pattern_tests", ctypes.c_uint64 * 9), ("render_tests", ctypes.c_uint64),
                ("render_composited", ctypes.c_uint64), ("t_render_kernel_ms", ctypes.c_double)]


OBJECTIVE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                                ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_uint32))

_lib = None


def lib():
    """Load csrc/liblobe.so. Raises if it is missing: there is no CPU path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2510_01767_b200.build` "
                              "(the engine has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.lobe_last_error.restype = ctypes.c_char_p
        L.lobe_version.restype = ctypes.c_char_p
        L.lobe_mask_words.restype = ctypes.c_size_t
        L.lobe_mask_words.argtypes = [vp]
        L.lobe_free_scene.argtypes = [vp]
        L.lobe_free_scene.restype = None
        L.lobe_load_scene.argtypes = [ctypes.POINTER(Gaussians), ctypes.POINTER(Camera), i64,
                                      ctypes.POINTER(Frame), ctypes.POINTER(Options), ctypes.POINTER(vp)]
        L.lobe_assign_cameras.argtypes = [vp, ctypes.POINTER(Grid)] + [vp] * 8
        L.lobe_block_loads.argtypes = [vp, ctypes.POINTER(Grid), vp, vp]
        L.lobe_crop_masks.argtypes = [vp, ctypes.POINTER(Grid), vp, vp]
        L.lobe_balance_partition.argtypes = [vp, i32, i32, ctypes.POINTER(BalanceOpts), vp, vp, vp, vp, vp]
        L.lobe_bo_run.argtypes = [i32, i32, ctypes.POINTER(BalanceOpts), OBJECTIVE_FN, vp, vp, vp, vp, vp]
        L.lobe_block_partial.argtypes = [vp, ctypes.POINTER(Grid), vp, vp, vp]
        L.lobe_scene_info.argtypes = [vp, vp, vp, vp, vp]
        SP = ctypes.POINTER(SubScene)
        L.lobe_block_subscene.argtypes = [vp, ctypes.POINTER(Grid), i32, ctypes.POINTER(Gaussians), SP, i64]
        L.lobe_densify_step.argtypes = [vp, ctypes.POINTER(Grid), i32, SP, vp, vp, ctypes.c_float, ctypes.c_float,
                                        SP, i64]
        L.lobe_prune_outside.argtypes = [vp, ctypes.POINTER(Grid), i32, SP, SP, i64]
        L.lobe_merge_blocks.argtypes = [vp, SP, i32, SP, i64]
        L.lobe_render_select.argtypes = [vp, ctypes.POINTER(Gaussians), i32, i32, ctypes.c_float]
        L.lobe_camera_clouds.argtypes = [vp, vp, vp, vp, i64]
        L.lobe_render_maps.argtypes = [vp, ctypes.POINTER(Gaussians), i64, i32, vp, vp]
        L.lobe_masks_combine.argtypes = [vp, i32, vp, i32, vp, vp]
        L.lobe_block_records.argtypes = [vp, ctypes.POINTER(Grid), vp, vp, vp, vp, vp]
        L.lobe_crop_from_masks.argtypes = [vp, ctypes.POINTER(Grid), vp, vp, vp]
        L.lobe_export_rows.argtypes = [vp, i64, i64, vp]
        L.lobe_get_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.lobe_dev_vis_bench.argtypes = [vp, i32, i32, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]
        L.lobe_nccl_unique_id.argtypes = [vp]
        L.lobe_release_comms.argtypes = []
        L.lobe_release_comms.restype = None
        HCP, sz = ctypes.POINTER(HostComm), ctypes.c_size_t
        L.lobe_xchg_block_loads_host.argtypes = [HCP, i32, i32, i32, sz, vp, vp, vp, vp, vp]
        L.lobe_xchg_all_masks_host.argtypes = [HCP, i32, i32, i32, sz, vp, vp]
        L.lobe_xchg_gather_cameras_host.argtypes = [HCP, i32, i32, i64, sz, vp, vp]
        for name in EXPORTS:
            if name not in ("lobe_last_error", "lobe_version", "lobe_mask_words", "lobe_free_scene",
                            "lobe_release_comms"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise LobeError(code, lib().lobe_last_error().decode())


def _ptr(a):
    """Address of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(type(a))


def version():
    return lib().lobe_version().decode()


def make_cameras(scene):
    N = scene.N
    arr = (Camera * N)()
    R = scene.R.reshape(N, 9)
    for c in range(N):
        k = arr[c]
        k.id = int(scene.cam_id[c])
        k.fx, k.fy, k.cx, k.cy = float(scene.fx[c]), float(scene.fy[c]), float(scene.cx[c]), float(scene.cy[c])
        k.width, k.height = int(scene.width[c]), int(scene.height[c])
        k.R[:] = [float(v) for v in R[c]]
        k.t[:] = [float(v) for v in scene.t[c]]
        k.z_near, k.z_far = float(scene.z_near[c]), float(scene.z_far[c])
    return arr


def make_grid(m, n, v=None, h=None, delta_v=-1.0, delta_h=-1.0, tau=-1.0):
    """Grid struct + the arrays it points to (kept alive in the returned tuple)."""
    v = np.ascontiguousarray(v if v is not None else [np.float32(i / m) for i in range(1, m)], np.float32)
    h = np.ascontiguousarray(h if h is not None else [np.float32(j / n) for j in range(1, n)], np.float32)
    g = Grid(int(m), int(n), v.ctypes.data if v.size else None, h.ctypes.data if h.size else None,
             float(delta_v), float(delta_h), float(tau))
    return g, (v, h)


class Scene:
    """Owning wrapper of a lobe_scene* handle."""

    def __init__(self, gaussians, cameras, frame=None, device=0, rank=0, world=1, stream=None,
                 assign_mode=ASSIGN_RATIO, predicate=0, nccl_id=None, host_comm=None):
        """gaussians: an object with x..opacity attributes (numpy host arrays or
        torch CUDA tensors); cameras: a synth Scene (its camera arrays) or a
        ctypes Camera array. frame: dict(center, radius, axis_u, axis_v) or None
        (automatic, ledger L12). nccl_id (128 bytes from nccl_unique_id(), the
        same on every rank) or host_comm (a HostComm): the scene's communicator --
        every call is then collective and returns global outputs (include/lobe.h)."""
        L = lib()
        self._keep = []
        names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")
        arrs = [getattr(gaussians, k) for k in names]
        on_dev = int(getattr(arrs[0], "is_cuda", False))
        if not on_dev and not isinstance(arrs[0], np.ndarray):
            arrs = [a.numpy() for a in arrs]     # host torch tensors (e.g. pinned) -> numpy views
        if not on_dev:
            arrs = [np.ascontiguousarray(a, np.float32) for a in arrs]
        self._keep.append(arrs)
        g = Gaussians(int(arrs[0].shape[0]), *[_ptr(a) for a in arrs], on_dev)
        cams = cameras if isinstance(cameras, ctypes.Array) else make_cameras(cameras)
        fr = Frame()
        flags = 0
        frame = frame or {}
        if frame.get("center") is None:
            flags |= FRAME_AUTO_CENTER
        else:
            fr.center[:] = [float(v) for v in frame["center"]]
        if frame.get("radius") is None:
            flags |= FRAME_AUTO_RADIUS
        else:
            fr.radius = float(frame["radius"])
        if frame.get("axis_u") is None:
            flags |= FRAME_AUTO_AXES
        else:
            fr.axis_u[:] = [float(v) for v in frame["axis_u"]]
            fr.axis_v[:] = [float(v) for v in frame["axis_v"]]
        fr.auto_flags = flags
        st = stream if (stream is None or isinstance(stream, int)) else stream.cuda_stream
        opt = Options(int(device), int(rank), int(world), st, int(assign_mode), int(predicate), None, None)
        if nccl_id is not None:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            opt.nccl_unique_id = ctypes.addressof(self._nccl_id)
        if host_comm is not None:
            self._host_comm = host_comm  # the callbacks must outlive the scene
            opt.host_comm = ctypes.pointer(host_comm)
        h = ctypes.c_void_p()
        _check(L.lobe_load_scene(ctypes.byref(g), cams, len(cams), ctypes.byref(fr), ctypes.byref(opt),
                                 ctypes.byref(h)))
        self.handle = h
        self.frame = dict(center=np.array(fr.center[:], np.float32), radius=np.float32(fr.radius),
                          axis_u=np.array(fr.axis_u[:], np.float32), axis_v=np.array(fr.axis_v[:], np.float32))
        info = [ctypes.c_int64() for _ in range(4)]
        _check(L.lobe_scene_info(h, *[ctypes.byref(x) for x in info]))  # does not wait for the device
        self.G, self.N, self.n_local, self.cam_begin = [x.value for x in info]
        self.collective = nccl_id is not None or host_comm is not None
        self.n_out = self.N if (self.collective or world == 1) else self.n_local  # per-camera output rows

    def close(self):
        if getattr(self, "handle", None):
            lib().lobe_free_scene(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- calls ----------------------------------------------------------
    def stats(self):
        s = Stats()
        _check(lib().lobe_get_stats(self.handle, ctypes.byref(s)))
        return s

    def assign_cameras(self, m, n, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        NL, B = self.n_out, m * n
        out = dict(K=np.empty(NL, np.uint32), D=np.empty(NL, np.float64), zmin=np.empty(NL, np.float32),
                   zmax=np.empty(NL, np.float32), n=np.empty((NL, B), np.uint32), n0=np.empty((NL, B), np.uint32),
                   member=np.empty(NL, np.uint64), home=np.empty(NL, np.int32))
        _check(lib().lobe_assign_cameras(self.handle, ctypes.byref(g), *[_ptr(out[k]) for k in
                                                                         ("K", "D", "zmin", "zmax", "n", "n0",
                                                                          "member", "home")]))
        return out

    def block_loads(self, m, n, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        recs = (BlockLoad * (m * n))()
        obj = ctypes.c_uint32()
        _check(lib().lobe_block_loads(self.handle, ctypes.byref(g), recs, ctypes.byref(obj)))
        return records_to_dict(recs, int(obj.value))

    def crop_masks(self, m, n, crop=True, eligible=True, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        W = (self.G + 63) // 64
        c = np.empty((m * n, W), np.uint64) if crop else None
        e = np.empty((m * n, W), np.uint64) if eligible else None
        _check(lib().lobe_crop_masks(self.handle, ctypes.byref(g), _ptr(c), _ptr(e)))
        return c, e

    def crop_masks_into(self, m, n, crop_ptr, elig_ptr, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        _check(lib().lobe_crop_masks(self.handle, ctypes.byref(g), _ptr(crop_ptr), _ptr(elig_ptr)))

    def balance_partition(self, m, n, L=100, seed=0, delta_scale=0.1, tau=0.15, n_sobol=8):
        o = BalanceOpts(int(L), int(seed), float(delta_scale), float(tau), int(n_sobol))
        v = np.empty(max(m - 1, 1), np.float32)
        h = np.empty(max(n - 1, 1), np.float32)
        hist = np.empty(L, np.uint32)
        D = (m - 1) + (n - 1)
        ch = np.empty((L, max(D, 1)), np.float32)
        recs = (BlockLoad * (m * n))()
        _check(lib().lobe_balance_partition(self.handle, m, n, ctypes.byref(o), _ptr(v), _ptr(h), _ptr(hist),
                                            _ptr(ch), recs))
        return dict(v=v[:m - 1], h=h[:n - 1], history=hist, cut_history=ch[:, :D], best=records_to_dict(recs, None))

    # ---- block pipeline ----------------------
    def block_subscene(self, m, n, block, coarse, device="cuda", **grid_kw):
        """The crop sub-scene of `block` (dict of device tensors; origin, in_block)."""
        g, keep = make_grid(m, n, **grid_kw)
        arrs = [getattr(coarse, k) for k in SUB_FIELDS]
        cg = Gaussians(int(arrs[0].shape[0]), *[_ptr(a) for a in arrs], 1)
        d = _sub_alloc(self.G, device)
        st = _sub_struct(d, 0)
        _check(lib().lobe_block_subscene(self.handle, ctypes.byref(g), int(block), ctypes.byref(cg),
                                         ctypes.byref(st), int(self.G)))
        return _sub_result(d, st)

    def densify_step(self, m, n, block, sub, grad, normals, tau_grad, scale_split, device="cuda", **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        nin = int(sub["x"].shape[0])
        si = _sub_struct(sub, nin)
        d = _sub_alloc(2 * nin, device)
        so = _sub_struct(d, 0)
        _check(lib().lobe_densify_step(self.handle, ctypes.byref(g), int(block), ctypes.byref(si), _ptr(grad),
                                       _ptr(normals), ctypes.c_float(tau_grad), ctypes.c_float(scale_split),
                                       ctypes.byref(so), int(max(2 * nin, 1))))
        return _sub_result(d, so)

    def prune_outside(self, m, n, block, sub, device="cuda", **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        nin = int(sub["x"].shape[0])
        si = _sub_struct(sub, nin)
        d = _sub_alloc(nin, device)
        so = _sub_struct(d, 0)
        _check(lib().lobe_prune_outside(self.handle, ctypes.byref(g), int(block), ctypes.byref(si),
                                        ctypes.byref(so), int(max(nin, 1))))
        return _sub_result(d, so)

    def merge_blocks(self, subs, device="cuda"):
        """Concatenation in order; raises LobeError(INTEGRITY) on a duplicated origin."""
        arr = (SubScene * max(len(subs), 1))()
        tot = 0
        for k, sb in enumerate(subs):
            nk = int(sb["x"].shape[0])
            arr[k] = _sub_struct(sb, nk)
            tot += nk
        d = _sub_alloc(tot, device)
        so = _sub_struct(d, 0)
        _check(lib().lobe_merge_blocks(self.handle, arr, len(subs), ctypes.byref(so), int(max(tot, 1))))
        return _sub_result(d, so)

    # ---- paper-exact camera selection ---------
    @staticmethod
    def _coarse(coarse):
        arrs = [getattr(coarse, k) for k in SUB_FIELDS]
        return Gaussians(int(arrs[0].shape[0]), *[_ptr(a) for a in arrs], 1), arrs

    def render_select(self, coarse, downscale=4, stride=2, eps_w=0.1):
        """Render every local camera's depth, back-project, and assign cameras by
        their clouds from now on (coarse: the loaded Gaussians, device tensors)."""
        cg, keep = self._coarse(coarse)
        _check(lib().lobe_render_select(self.handle, ctypes.byref(cg), int(downscale), int(stride),
                                        ctypes.c_float(eps_w)))

    def camera_clouds(self):
        off = np.empty(self.n_local + 1, np.int64)
        lib().lobe_camera_clouds(self.handle, _ptr(off), None, None, 0)  # size query (offsets are always filled)
        n = int(off[-1])
        gu = np.empty(max(n, 1), np.float32)
        gv = np.empty(max(n, 1), np.float32)
        _check(lib().lobe_camera_clouds(self.handle, _ptr(off), _ptr(gu), _ptr(gv), max(n, 1)))
        return off, gu[:n], gv[:n]

    def render_maps(self, coarse, camera, downscale, width, height):
        cg, keep = self._coarse(coarse)
        D = np.empty((height // downscale, width // downscale), np.float32)
        W = np.empty_like(D)
        _check(lib().lobe_render_maps(self.handle, ctypes.byref(cg), int(camera), int(downscale), _ptr(D), _ptr(W)))
        return D, W

    def export_rows(self, c0=0, count=None):
        count = self.n_local - c0 if count is None else count
        out = np.empty((count, (self.G + 31) // 32), np.uint32)
        _check(lib().lobe_export_rows(self.handle, int(c0), int(count), _ptr(out)))
        return out

    def dev_vis_bench(self, variant=0, reps=3):
        ms = ctypes.c_float()
        grid = ctypes.c_int32()
        _check(lib().lobe_dev_vis_bench(self.handle, int(variant), int(reps), ctypes.byref(ms), ctypes.byref(grid)))
        return float(ms.value), int(grid.value)

    def mask_words(self):
        return int(lib().lobe_mask_words(self.handle))

    def block_partial(self, m, n, d_masks, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        B = m * n
        nc = np.empty(B, np.uint32)
        inc = np.empty(B, np.uint64)
        _check(lib().lobe_block_partial(self.handle, ctypes.byref(g), _ptr(d_masks), _ptr(nc), _ptr(inc)))
        return nc, inc

    def masks_combine(self, B, d_gathered, W, d_out):
        gv = np.empty(B, np.uint32)
        _check(lib().lobe_masks_combine(self.handle, int(B), _ptr(d_gathered), int(W), _ptr(d_out), _ptr(gv)))
        return gv

    def block_records(self, m, n, n_cams, incid, g_vis, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        recs = (BlockLoad * (m * n))()
        obj = ctypes.c_uint32()
        n_cams = np.ascontiguousarray(n_cams, np.uint32)
        incid = np.ascontiguousarray(incid, np.uint64)
        g_vis = np.ascontiguousarray(g_vis, np.uint32)
        _check(lib().lobe_block_records(self.handle, ctypes.byref(g), _ptr(n_cams), _ptr(incid), _ptr(g_vis), recs,
                                        ctypes.byref(obj)))
        return records_to_dict(recs, int(obj.value))

    def crop_from_masks_into(self, m, n, d_masks, crop_ptr, elig_ptr, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        _check(lib().lobe_crop_from_masks(self.handle, ctypes.byref(g), _ptr(d_masks), _ptr(crop_ptr),
                                          _ptr(elig_ptr)))

    def crop_from_masks(self, m, n, d_masks, crop=True, eligible=True, **grid_kw):
        g, keep = make_grid(m, n, **grid_kw)
        W = (self.G + 63) // 64
        c = np.empty((m * n, W), np.uint64) if crop else None
        e = np.empty((m * n, W), np.uint64) if eligible else None
        _check(lib().lobe_crop_from_masks(self.handle, ctypes.byref(g), _ptr(d_masks), _ptr(c), _ptr(e)))
        return c, e


_BLOCKLOAD_DT = None


def records_to_dict(recs, objective):
    global _BLOCKLOAD_DT
    if _BLOCKLOAD_DT is None:  # numpy view of lobe_block_load (built once: the ctypes -> dtype path is slow)
        _BLOCKLOAD_DT = np.ctypeslib.as_array((BlockLoad * 1)()).dtype
    a = np.frombuffer(recs, dtype=_BLOCKLOAD_DT)  # structured view, no per-record loop
    B = len(recs)
    out = dict(block_id=a["block_id"].astype(np.int32), n_cams=a["n_cams"].astype(np.uint32),
               g_blk=a["g_blk"].astype(np.uint32), g_vis=a["g_vis"].astype(np.uint32),
               incidences=a["incidences"].astype(np.uint64), area=a["area"].astype(np.float64),
               g_avgvis=a["g_avgvis"].astype(np.float64),
               lohi=np.concatenate([a["lo"], a["hi"]], axis=1).astype(np.float32).reshape(B, 4))
    out["objective"] = objective if objective is not None else int(out["g_vis"].max()) if B else 0
    return out


def bo_run(m, n, objective, L=100, seed=0, n_sobol=8):
    """Host BO driver (no GPU needed) with a Python objective(v, h) -> int."""
    D = (m - 1) + (n - 1)
    errs = []

    def cb(ctx, vp, hp, outp):
        try:
            v = np.array([vp[i] for i in range(m - 1)], np.float32)
            h = np.array([hp[i] for i in range(n - 1)], np.float32)
            outp[0] = int(objective(v, h))
            return 0
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            return 1

    fn = OBJECTIVE_FN(cb)
    o = BalanceOpts(int(L), int(seed), 0.1, 0.15, int(n_sobol))
    v = np.empty(max(m - 1, 1), np.float32)
    h = np.empty(max(n - 1, 1), np.float32)
    hist = np.empty(L, np.uint32)
    ch = np.empty((L, max(D, 1)), np.float32)
    code = lib().lobe_bo_run(m, n, ctypes.byref(o), fn, None, _ptr(v), _ptr(h), _ptr(hist), _ptr(ch))
    if errs:
        raise errs[0]
    _check(code)
    return dict(v=v[:m - 1], h=h[:n - 1], history=hist, cut_history=ch[:, :D])


def nccl_unique_id():
    """128-byte ncclUniqueId for Scene(nccl_id=...) (rank 0 creates, every rank uses)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().lobe_nccl_unique_id(buf))
    return buf.raw


def release_comms():
    lib().lobe_release_comms()


def xchg_block_loads_host(comm, rank, world, B, words, partial, counts_local):
    """lobe_xchg_block_loads_host: the library's exchange choreography on host
    buffers (partial: B x words u32, counts_local: 2B u64) -> own, g_vis, counts."""
    partial = np.ascontiguousarray(partial, np.uint32)
    counts_local = np.ascontiguousarray(counts_local, np.uint64)
    nb = (rank + 1) * B // world - rank * B // world
    own = np.zeros((max(nb, 1), words), np.uint32)
    gv = np.zeros(B, np.uint32)
    cg = np.zeros(2 * B, np.uint64)
    _check(lib().lobe_xchg_block_loads_host(ctypes.byref(comm), rank, world, B, words, _ptr(partial),
                                            _ptr(counts_local), _ptr(own), _ptr(gv), _ptr(cg)))
    return own[:nb], gv, cg


def xchg_all_masks_host(comm, rank, world, B, words, own):
    own = np.ascontiguousarray(own, np.uint32)
    out = np.zeros((B, words), np.uint32)
    _check(lib().lobe_xchg_all_masks_host(ctypes.byref(comm), rank, world, B, words,
                                          _ptr(own) if own.size else None, _ptr(out)))
    return out


def xchg_gather_cameras_host(comm, rank, world, N, local):
    """local: this rank's shard rows (numpy, any dtype / trailing shape) -> all N."""
    local = np.ascontiguousarray(local)
    elem = local.itemsize * int(np.prod(local.shape[1:], dtype=np.int64))
    out = np.zeros((N,) + local.shape[1:], local.dtype)
    _check(lib().lobe_xchg_gather_cameras_host(ctypes.byref(comm), rank, world, N, elem,
                                               _ptr(local) if local.size else None, _ptr(out)))
    return out

