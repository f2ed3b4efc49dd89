"""The multi-rank exchange on CPU with the gloo backend,
world sizes 2, 3 and 5 (5 ranks share the 12 blocks unevenly, and with 4
blocks one rank owns none).

The choreography under test is the library's own (csrc/lobe_comm.cpp, the code
every collective lobe_* call runs): the OR reduce-scatter of the partial masks
by owned blocks, the popcount, the G_vis all-gather, the |C^(b)| / I_b
all-reduce, the all-gather of the combined masks and the per-camera
all-gathers, driven here through the lobe_xchg_*_host exports with the
engine's TorchHostComm (gloo) as transport. Each rank's partial inputs are the
oracle restricted to the rank's camera shard (test infrastructure). Results
must equal the world = 1 oracle (I12).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2510_01767_b200 import lobe
from paper_2510_01767_b200.engine import TorchHostComm, communicator, shard
from synth import make_scene, make_config

CFG = dict(base="building", G=12_000, N=23, seed=0xE1)
TINY = dict(base="tiny", G=3_000, N=17, seed=0xE2)  # 2 x 2 = 4 blocks: with 5 ranks one owns none


def _rank_partial(sc, pre, vis_loc, g):
    """This rank's evaluation (oracle, local cameras): per-camera outputs, the
    partial masks (B x words u32: OR of the local members' rows) and counts."""
    asg = oracle.assign(sc, pre, vis_loc, g, threads=1)
    bl = oracle.block_loads(sc, pre, vis_loc, asg, g, masks=True)
    B = g["m"] * g["n"]
    words = (sc.G + 31) // 32
    partial = np.ascontiguousarray(bl["M"].view(np.uint32).reshape(B, -1)[:, :words])
    counts = np.concatenate([bl["n_cams"].astype(np.uint64), bl["incidences"].astype(np.uint64)])
    return asg, bl, partial, counts


def _worker(rank, world, port, q, cfg):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kw = communicator()  # gloo -> the library's host-comm transport
        hc = kw["host_comm"]
        sc = make_scene(make_config(cfg["base"], G=cfg["G"], N=cfg["N"], seed=cfg["seed"]))
        m, n = sc.cfg.m, sc.cfg.n
        B, words = m * n, (sc.G + 31) // 32
        c0, c1 = shard(sc.N, rank, world)
        sel = np.arange(c0, c1)
        pre = oracle.prep(sc, oracle.frame(sc))
        pre["cam_gu_sel"], pre["cam_gv_sel"] = pre["cam_gu"][sel], pre["cam_gv"][sel]
        vis = oracle.visibility(sc, pre, cams=sel, threads=1)
        out = {}
        grids = [("uniform", oracle.default_grid(m, n)),
                 ("cuts", oracle.default_grid(m, n, v=np.linspace(0.3, 0.8, m - 1).astype(np.float32)))]
        for name, g in grids:
            asg, bl, partial, counts = _rank_partial(sc, pre, vis, g)
            own, gv, cg = lobe.xchg_block_loads_host(hc, rank, world, B, words, partial, counts)
            allm = lobe.xchg_all_masks_host(hc, rank, world, B, words, own)
            W64 = (sc.G + 63) // 64
            pad = np.zeros((B, 2 * W64), np.uint32)
            pad[:, :words] = allm
            crop, elig = oracle.crop(sc, pre, g, np.ascontiguousarray(pad).view(np.uint64))
            per = {k: lobe.xchg_gather_cameras_host(hc, rank, world, sc.N, np.asarray(v))
                   for k, v in (("K", vis["K"]), ("D", vis["D"]), ("zmin", vis["zmin"]), ("zmax", vis["zmax"]),
                                ("n", asg["n"]), ("n0", asg["n0"]), ("member", asg["member"]),
                                ("home", asg["home"]))}
            out[name] = dict(g_vis=gv, n_cams=cg[:B], incidences=cg[B:], crop=crop, eligible=elig, per=per,
                             own_blocks=shard(B, rank, world))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,cfg", [(2, CFG), (3, CFG), (5, CFG), (5, TINY)])
def test_gloo_exchange_matches_world1(world, cfg):
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
    a2 = oracle.assign(sc, ref["pre"], ref["vis"], g2)
    bl2 = oracle.block_loads(sc, ref["pre"], ref["vis"], a2, g2, masks=True)
    cr2, el2 = oracle.crop(sc, ref["pre"], g2, bl2["M"])
    expect = {"uniform": (ref["asg"], ref["loads"], ref["crop"], ref["eligible"]), "cuts": (a2, bl2, cr2, el2)}
    for rank, out in res:
        for name, (asg, bl, cr, el) in expect.items():
            o = out[name]
            for k in ("g_vis", "n_cams", "incidences"):
                assert (np.asarray(o[k]).astype(np.int64) == np.asarray(bl[k]).astype(np.int64)).all(), (rank, k)
            assert (o["crop"] == cr).all() and (o["eligible"] == el).all(), (rank, name)
            for k in ("K", "zmin", "zmax"):
                assert (o["per"][k] == ref["vis"][k]).all(), k
            assert (o["per"]["D"] == ref["vis"]["D"]).all()
            for k in ("n", "n0", "member", "home"):
                assert (o["per"][k] == asg[k]).all(), (name, k)


def test_host_comm_struct_has_callbacks():
    """TorchHostComm fills every lobe_host_comm callback (the library rejects a
    partial struct with LOBE_E_INVALID_CONFIG)."""
    hc = TorchHostComm.__new__(TorchHostComm)
    hc.group, hc.rank, hc.world = None, 0, 1
    hc._fns = (lobe.HC_ALL_GATHER(lambda *a: 0), lobe.HC_ALL_REDUCE_U64(lambda *a: 0),
               lobe.HC_ALL_TO_ALL_V(lambda *a: 0))
    s = lobe.HostComm(None, *hc._fns)
    assert all(bool(getattr(s, f)) for f in ("all_gather", "all_reduce_u64", "all_to_all_v"))
