"""Process-group setup for the multi-GPU engine.

The exchange itself -- the OR reduce-scatter of the partial block masks by
owned blocks, the popcount, the G_vis all-gather, the |C^(b)| / I_b SUM
all-reduce, the per-camera all-gathers -- runs inside liblobe.so
(csrc/lobe_comm.cpp): every lobe_* call of a scene with a communicator is
collective and returns global outputs on every rank. This module only hands the
library a communicator for a torch.distributed group:

  - NCCL backend (GPUs): rank 0 asks the library for an ncclUniqueId, the group
    broadcasts its 128 bytes once, and the library creates (and caches) its own
    ncclComm on the scene's stream;
  - any other backend (gloo): `TorchHostComm` exposes the group's all_gather /
    all_reduce / all_to_all on host tensors as lobe_host_comm callbacks.

`Engine` keeps the call names the bench and tests use; every method is one
library call.
"""
from __future__ import annotations

import ctypes
import traceback

import numpy as np

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


def _world(group=None):
    if dist is not None and dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard(n_cams, rank, world):
    """Camera range of a rank (same rule as lobe_load_scene)."""
    return rank * n_cams // world, (rank + 1) * n_cams // world


def _u8(addr, nbytes):
    """A uint8 tensor viewing `nbytes` of host memory at `addr` (no copy)."""
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8)
    return torch.frombuffer((ctypes.c_uint8 * nbytes).from_address(addr), dtype=torch.uint8)


class TorchHostComm:
    """lobe_host_comm over a torch.distributed group (host buffers; e.g. gloo).

    The library calls these from inside a lobe_* call on this thread; every rank
    makes the same sequence of calls. Keep the object alive while scenes use it."""

    def __init__(self, group=None):
        from . import lobe
        self.group = group
        self.rank, self.world = _world(group)
        self._fns = (lobe.HC_ALL_GATHER(self._all_gather), lobe.HC_ALL_REDUCE_U64(self._all_reduce_u64),
                     lobe.HC_ALL_TO_ALL_V(self._all_to_all_v))
        self.struct = lobe.HostComm(None, *self._fns)

    def _all_gather(self, ctx, send, recv, nbytes):
        try:
            if nbytes:
                out = torch.empty(self.world * nbytes, dtype=torch.uint8)
                dist.all_gather(list(out.view(self.world, nbytes).unbind(0)), _u8(send, nbytes).clone(),
                                group=self.group)
                ctypes.memmove(recv, out.data_ptr(), self.world * nbytes)
            return 0
        except Exception:  # pragma: no cover - reported to the library as a failed collective
            traceback.print_exc()
            return 1

    def _all_reduce_u64(self, ctx, buf, count):
        try:
            if count:
                a = np.ctypeslib.as_array(buf, shape=(count,))
                t = torch.from_numpy(a.astype(np.int64))  # counts < 2^63
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
                a[:] = t.numpy().astype(np.uint64)
            return 0
        except Exception:  # pragma: no cover
            traceback.print_exc()
            return 1

    def _all_to_all_v(self, ctx, send, sb, so, recv, rb, ro):
        try:
            W = self.world
            sb = [int(sb[j]) for j in range(W)]
            so = [int(so[j]) for j in range(W)]
            rb = [int(rb[j]) for j in range(W)]
            ro = [int(ro[j]) for j in range(W)]
            src = torch.cat([_u8(send + so[j], sb[j]) for j in range(W)]) if sum(sb) else torch.empty(0, dtype=torch.uint8)
            dst = torch.empty(sum(rb), dtype=torch.uint8)
            dist.all_to_all_single(dst, src, output_split_sizes=rb, input_split_sizes=sb, group=self.group)
            off = 0
            for j in range(W):
                if rb[j]:
                    ctypes.memmove(recv + ro[j], dst.data_ptr() + off, rb[j])
                off += rb[j]
            return 0
        except Exception:  # pragma: no cover
            traceback.print_exc()
            return 1


_NCCL_IDS = {}


def communicator(group=None):
    """Scene keyword arguments that give the library this group's communicator
    ({} at world 1). NCCL groups share one unique id per group (the library then
    reuses one ncclComm for every scene of the run)."""
    rank, world = _world(group)
    if world == 1:
        return {}
    backend = dist.get_backend(group)
    if backend == "nccl":
        key = id(group)
        if key not in _NCCL_IDS:
            from . import lobe
            obj = [lobe.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            _NCCL_IDS[key] = obj[0]
        return {"nccl_id": _NCCL_IDS[key]}
    key = ("host", id(group))
    if key not in _NCCL_IDS:
        _NCCL_IDS[key] = TorchHostComm(group)
    return {"host_comm": _NCCL_IDS[key].struct}


class Engine:
    """One rank's view of the collective engine (a lobe.Scene with this group's
    communicator). All ranks call every method with the same arguments."""

    def __init__(self, local, group=None):
        self.local = local
        self.group = group
        self.rank, self.world = _world(group)

    @classmethod
    def from_scene(cls, gaussians, cameras, frame=None, device=None, stream=None, assign_mode=0, group=None,
                   predicate=0):
        from . import lobe
        rank, world = _world(group)
        dev = torch.cuda.current_device() if device is None else device
        sc = lobe.Scene(gaussians, cameras, frame=frame, device=dev, rank=rank, world=world, stream=stream,
                        assign_mode=assign_mode, predicate=predicate, **communicator(group))
        return cls(sc, group)

    def block_loads(self, m, n, **grid_kw):
        return self.local.block_loads(m, n, **grid_kw)

    def crop_masks(self, m, n, **grid_kw):
        return self.local.crop_masks(m, n, **grid_kw)

    def crop_masks_into(self, m, n, crop_out, elig_out, **grid_kw):
        """Crop / eligible masks written straight into (device or host) buffers."""
        return self.local.crop_masks_into(m, n, crop_out, elig_out, **grid_kw)

    def assign_cameras(self, m, n, **grid_kw):
        return self.local.assign_cameras(m, n, **grid_kw)

    def balance_partition(self, m, n, L=100, seed=0, n_sobol=8):
        return self.local.balance_partition(m, n, L=L, seed=seed, n_sobol=n_sobol)

    def render_select(self, coarse, downscale=4, stride=2, eps_w=0.1):
        """Paper-exact camera selection: every rank renders its
        own cameras; assignments stay per camera, so the exchange is unchanged."""
        self.local.render_select(coarse, downscale=downscale, stride=stride, eps_w=eps_w)

    def stats(self):
        return self.local.stats()

    def close(self):
        if hasattr(self.local, "close"):
            self.local.close()
