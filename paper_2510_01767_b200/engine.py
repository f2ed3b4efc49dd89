"""Multi-GPU exchange layer: cameras sharded over ranks,
Gaussians replicated, one exchange per evaluation.

Each rank's `local` backend (a `lobe.Scene` on its GPU) computes everything
for its camera shard [floor(rN/W), floor((r+1)N/W)) -- rows, depth statistic,
histograms, assignment, partial block masks. This module only moves data
between ranks with torch.distributed (NCCL over NVLink on GPUs, gloo in the
CPU tests) and calls back into the library for the OR-combine / popcount
kernel:

  per evaluation   all_to_all(partial masks of each rank's own blocks)
                   ->  lobe_masks_combine (OR of the W partials + popcount, own blocks only)
                   all_gather(combined masks of the own blocks), all_gather(G_vis of the own blocks)
                   all_reduce(SUM, |C^(b)| and I_b)          ->  lobe_block_records
  per-camera data  all_gather (padded to the largest shard)

All ranks call every method collectively with the same grid; results are
identical on every rank (I12). With world == 1 the calls go straight to the
library.
"""
from __future__ import annotations

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


class Engine:
    def __init__(self, local, group=None):
        """local: an object with the lobe.Scene methods for this rank's shard."""
        self.local = local
        self.group = group
        self.rank, self.world = _world(group)
        self.device = getattr(local, "device", None) or ("cuda" if torch.cuda.is_available() else "cpu")
        self._comb_key = None
        self._comb = None
        self._loads = None

    @classmethod
    def from_scene(cls, gaussians, cameras, frame=None, device=None, stream=None, assign_mode=0, group=None,
                   predicate=0):
        from . import lobe
        rank, world = _world(group)
        dev = torch.cuda.current_device() if device is None else device
        sc = lobe.Scene(gaussians, cameras, frame=frame, device=dev, rank=rank, world=world, stream=stream,
                        assign_mode=assign_mode, predicate=predicate)
        sc.device = f"cuda:{dev}"
        return cls(sc, group)

    # ------------------------------------------------------------------ utils
    def _all_gather_flat(self, t):
        """t: 1-D tensor, identical shape on every rank -> world x len, rank-major."""
        out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
        if t.is_cuda:
            dist.all_gather_into_tensor(out, t, group=self.group)
        else:
            parts = list(out.view(self.world, -1).unbind(0))
            dist.all_gather(parts, t, group=self.group)
            out = torch.stack(parts).reshape(-1)
        return out

    def _grid_key(self, m, n, grid_kw):
        return (m, n) + tuple((k, np.asarray(v).tobytes() if v is not None else None) for k, v in
                              sorted(grid_kw.items()))

    # ------------------------------------------------------------------ calls
    def block_loads(self, m, n, **grid_kw):
        if self.world == 1:
            return self.local.block_loads(m, n, **grid_kw)
        key = self._grid_key(m, n, grid_kw)
        if self._comb_key == key and self._loads is not None:
            return self._loads  # this grid was already exchanged (e.g. by crop_masks first)
        B = m * n
        W, r = self.world, self.rank
        words = self.local.mask_words()
        part = torch.zeros(B * words, dtype=torch.int32, device=self.device)
        nc, inc = self.local.block_partial(m, n, part, **grid_kw)
        # OR reduce-scatter by blocks: rank j owns blocks [floor(jB/W), floor((j+1)B/W));
        # each rank sends every other rank the partial masks of that rank's
        # blocks (one all_to_all), then ORs the W partials of its own blocks
        # and popcounts them with lobe_masks_combine
        nb = [shard(B, j, W)[1] - shard(B, j, W)[0] for j in range(W)]
        recv = torch.empty(W * nb[r] * words, dtype=torch.int32, device=self.device)
        dist.all_to_all_single(recv, part, output_split_sizes=[nb[r] * words] * W,
                               input_split_sizes=[k * words for k in nb], group=self.group)
        own = torch.zeros(nb[r] * words, dtype=torch.int32, device=self.device)
        gv_own = self.local.masks_combine(nb[r], recv, W, own) if nb[r] > 0 else np.zeros(0, np.uint32)
        # every rank needs the combined masks of all blocks for the crop: one
        # all_gather of the owned slices, padded to the largest share
        P = max(nb)
        buf = torch.zeros(P * words, dtype=torch.int32, device=self.device)
        buf[:nb[r] * words] = own
        gat = self._all_gather_flat(buf).view(W, P * words)
        comb = torch.cat([gat[j, :nb[j] * words] for j in range(W)])
        gvb = torch.zeros(P, dtype=torch.int64, device=self.device)
        gvb[:nb[r]] = torch.from_numpy(np.asarray(gv_own, np.int64)).to(self.device)
        gva = self._all_gather_flat(gvb).view(W, P).cpu().numpy()
        gv = np.concatenate([gva[j, :nb[j]] for j in range(W)]).astype(np.uint32)
        counts = torch.from_numpy(np.concatenate([nc.astype(np.int64), inc.astype(np.int64)])).to(self.device)
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=self.group)
        counts = counts.cpu().numpy()
        self._comb_key = key
        self._comb = comb
        self._loads = self.local.block_records(m, n, counts[:B].astype(np.uint32), counts[B:].astype(np.uint64),
                                               gv, **grid_kw)
        return self._loads

    def crop_masks(self, m, n, **grid_kw):
        if self.world == 1:
            return self.local.crop_masks(m, n, **grid_kw)
        if self._comb_key != self._grid_key(m, n, grid_kw):
            self.block_loads(m, n, **grid_kw)
        return self.local.crop_from_masks(m, n, self._comb, **grid_kw)

    def crop_masks_into(self, m, n, crop_out, elig_out, **grid_kw):
        """Crop / eligible masks written straight into (device or host) buffers."""
        if self.world == 1:
            return self.local.crop_masks_into(m, n, crop_out, elig_out, **grid_kw)
        if self._comb_key != self._grid_key(m, n, grid_kw):
            self.block_loads(m, n, **grid_kw)
        return self.local.crop_from_masks_into(m, n, self._comb, crop_out, elig_out, **grid_kw)

    def render_select(self, coarse, downscale=4, stride=2, eps_w=0.1):
        """Paper-exact camera selection: every rank renders its
        own cameras; assignments stay per camera, so the exchange is unchanged."""
        self.local.render_select(coarse, downscale=downscale, stride=stride, eps_w=eps_w)
        self._comb_key = None
        self._loads = None

    def close(self):
        self._comb = None
        self._loads = None
        if hasattr(self.local, "close"):
            self.local.close()

    def assign_cameras(self, m, n, **grid_kw):
        loc = self.local.assign_cameras(m, n, **grid_kw)
        if self.world == 1:
            return loc
        N = self.local.N
        nmax = -(-N // self.world) + 1
        out = {}
        for k, a in loc.items():
            a = np.ascontiguousarray(a)
            per = int(np.prod(a.shape[1:])) if a.ndim > 1 else 1
            buf = np.zeros((nmax, per * a.dtype.itemsize), np.uint8)
            buf[:a.shape[0]] = a.reshape(a.shape[0], -1).view(np.uint8)
            t = torch.from_numpy(buf.reshape(-1)).to(self.device)
            g = self._all_gather_flat(t).cpu().numpy().reshape(self.world, nmax, -1)
            rows = [g[r, :shard(N, r, self.world)[1] - shard(N, r, self.world)[0]] for r in range(self.world)]
            cat = np.concatenate(rows).view(a.dtype)
            out[k] = cat.reshape((N,) + a.shape[1:])
        return out

    def balance_partition(self, m, n, L=100, seed=0, n_sobol=8):
        """Every rank runs the same deterministic BO; each evaluation is a
        collective block_loads, so all ranks see the same objective values and
        therefore the same proposals (no broadcast needed)."""
        if self.world == 1:
            return self.local.balance_partition(m, n, L=L, seed=seed, n_sobol=n_sobol)
        from . import lobe

        def f(v, h):
            return self.block_loads(m, n, v=v, h=h)["objective"]

        r = lobe.bo_run(m, n, f, L=L, seed=seed, n_sobol=n_sobol)
        r["best"] = self.block_loads(m, n, v=r["v"], h=r["h"])
        return r
