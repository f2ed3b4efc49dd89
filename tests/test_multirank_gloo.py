"""The multi-rank exchange (paper_2510_01767_b200/engine.py) on
CPU with the gloo backend, world sizes 2, 3 and 5 (5 ranks share the 12
blocks unevenly: the block-sharded OR reduce-scatter pads the gathers).

Each rank's local backend here is the oracle restricted to the rank's camera
shard (test infrastructure); the choreography under test -- shard ranges,
all_to_all of the partial masks by owned blocks, OR-combine, all_gather of
the combined masks and counts, count all_reduce,
per-camera all_gather with padding -- is the engine's own code, the same that
runs over NCCL on GPUs. Results must equal the world = 1 oracle (I12).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2510_01767_b200.engine import Engine, shard
from synth import make_scene, make_config

CFG = dict(base="building", G=12_000, N=23, seed=0xE1)


class OracleLocal:
    """lobe.Scene-shaped local backend backed by the oracle on one camera shard."""

    device = "cpu"

    def __init__(self, sc, rank, world):
        self.sc = sc
        self.N = sc.N
        self.c0, self.c1 = shard(sc.N, rank, world)
        self.sel = np.arange(self.c0, self.c1)
        fr = oracle.frame(sc)
        self.pre = oracle.prep(sc, fr)
        self.pre["cam_gu_sel"] = self.pre["cam_gu"][self.sel]
        self.pre["cam_gv_sel"] = self.pre["cam_gv"][self.sel]
        self.vis = oracle.visibility(sc, self.pre, cams=self.sel, threads=1)
        self.G = sc.G

    def _grid(self, m, n, **kw):
        return oracle.default_grid(m, n, v=kw.get("v"), h=kw.get("h"))

    def mask_words(self):
        return (self.G + 31) // 32

    def assign_cameras(self, m, n, **kw):
        g = self._grid(m, n, **kw)
        a = oracle.assign(self.sc, self.pre, self.vis, g, threads=1)
        return dict(K=self.vis["K"], D=self.vis["D"], zmin=self.vis["zmin"], zmax=self.vis["zmax"], n=a["n"],
                    n0=a["n0"], member=a["member"], home=a["home"])

    def block_partial(self, m, n, d_masks, **kw):
        g = self._grid(m, n, **kw)
        a = oracle.assign(self.sc, self.pre, self.vis, g, threads=1)
        bl = oracle.block_loads(self.sc, self.pre, self.vis, a, g, masks=True)
        B = m * n
        w32 = bl["M"].view(np.uint32).reshape(B, -1)[:, :self.mask_words()]
        d_masks.copy_(torch.from_numpy(w32.reshape(-1).view(np.int32).copy()))
        self._static = bl
        return bl["n_cams"], bl["incidences"]

    def masks_combine(self, B, gathered, W, out):
        g = gathered.numpy().view(np.uint32).reshape(W, B, -1)
        comb = np.bitwise_or.reduce(g, axis=0)
        out.copy_(torch.from_numpy(comb.reshape(-1).view(np.int32).copy()))
        return np.array([int(np.unpackbits(comb[b].view(np.uint8)).sum()) for b in range(B)], np.uint32)

    def block_records(self, m, n, n_cams, incid, g_vis, **kw):
        st = self._static
        rec = dict(n_cams=np.asarray(n_cams, np.uint32), incidences=np.asarray(incid, np.uint64),
                   g_vis=np.asarray(g_vis, np.uint32), g_blk=st["g_blk"], area=st["area"], lohi=st["lohi"])
        rec["g_avgvis"] = np.where(rec["n_cams"] > 0, rec["g_vis"] / np.maximum(rec["n_cams"], 1), 0.0)
        rec["objective"] = int(rec["g_vis"].max())
        return rec

    def crop_from_masks(self, m, n, d_masks, **kw):
        g = self._grid(m, n, **kw)
        B = m * n
        w32 = d_masks.numpy().view(np.uint32).reshape(B, -1)
        W64 = (self.G + 63) // 64
        pad = np.zeros((B, 2 * W64), np.uint32)
        pad[:, :w32.shape[1]] = w32
        return oracle.crop(self.sc, self.pre, g, np.ascontiguousarray(pad).view(np.uint64))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, cfg=None):
    cfg = cfg or CFG
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = make_scene(make_config(cfg["base"], G=cfg["G"], N=cfg["N"], seed=cfg["seed"]))
        eng = Engine(OracleLocal(sc, rank, world))
        m, n = sc.cfg.m, sc.cfg.n
        L = eng.block_loads(m, n)
        A = eng.assign_cameras(m, n)
        c, e = eng.crop_masks(m, n)
        v = np.linspace(0.3, 0.8, m - 1).astype(np.float32)
        L2 = eng.block_loads(m, n, v=v)
        q.put((rank, {k: L[k] for k in ("n_cams", "g_vis", "incidences", "g_blk", "objective")},
               {k: A[k] for k in A}, c, e, int(L2["objective"])))
    finally:
        dist.destroy_process_group()


TINY = dict(base="tiny", G=3_000, N=17, seed=0xE2)  # 2 x 2 = 4 blocks: with 5 ranks one owns none


@pytest.mark.parametrize("world,cfg", [(2, CFG), (3, CFG), (5, CFG), (5, TINY)])
def test_gloo_engine_matches_world1(world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, cfg)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = make_scene(make_config(cfg["base"], G=cfg["G"], N=cfg["N"], seed=cfg["seed"]))
    ref = oracle.run(sc)
    m, n = sc.cfg.m, sc.cfg.n
    g2 = oracle.default_grid(m, n, v=np.linspace(0.3, 0.8, m - 1).astype(np.float32))
    ref2 = oracle.evaluate_cuts(sc, ref["pre"], ref["vis"], g2)
    for rank, L, A, c, e, obj2 in res:
        for k in ("n_cams", "g_vis", "incidences", "g_blk"):
            assert (np.asarray(L[k]) == ref["loads"][k]).all(), (rank, k)
        assert L["objective"] == ref["loads"]["objective"]
        for k, rk in (("K", "K"), ("zmin", "zmin"), ("zmax", "zmax")):
            assert (A[k] == ref["vis"][rk]).all(), k
        assert (A["D"] == ref["vis"]["D"]).all()
        for k in ("n", "n0", "member", "home"):
            assert (A[k] == ref["asg"][k]).all(), k
        assert (c == ref["crop"]).all() and (e == ref["eligible"]).all()
        assert obj2 == ref2
