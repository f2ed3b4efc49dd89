"""Collective C ABI on the GPU.

- NCCL: a scene with a communicator built from lobe_nccl_unique_id runs every
  call through the library's exchange (ncclSend / ncclRecv all-to-all,
  k_masks_combine, ncclAllGather, ncclAllReduce on the scene's stream). Only one
  GPU is available, so this runs at world = 1 (a real ncclComm of one rank: the
  NCCL code path executes, every collective is an identity) and must give the
  bytes of the communicator-less scene.
- Host comm: W = 2 and 3 processes share the GPU, each loads its camera shard
  with a gloo-backed lobe_host_comm (device buffers staged through host
  memory; no rank's kernel waits on another's), and every collective output --
  per-camera arrays of all N cameras, block records, crop / eligible masks, the
  BO trajectory -- must equal world 1 bit for bit (I12).
"""
import os
import socket

import numpy as np
import pytest

from synth import make_scene, make_config
from tests.test_gpu_parity import _lobe

pytestmark = pytest.mark.gpu

CFG = dict(base="rubble", G=60_000, N=41, seed=0x99)


def _run_all(S, m, n, L=6):
    a = S.assign_cameras(m, n)
    b = S.block_loads(m, n)
    v = np.linspace(0.3, 0.7, m - 1).astype(np.float32)
    b2 = S.block_loads(m, n, v=v, tau=0.3)
    c, e = S.crop_masks(m, n)
    c2, e2 = S.crop_masks(m, n, v=v, tau=0.3)
    bo = S.balance_partition(m, n, L=L, seed=3)
    return dict(a=a, b=b, b2=b2, c=c, e=e, c2=c2, e2=e2, bo=bo)


def _same(x, y):
    for k in x["a"]:
        assert (x["a"][k] == y["a"][k]).all(), k
    for key in ("b", "b2"):
        for k in ("n_cams", "g_blk", "g_vis", "incidences", "area", "g_avgvis", "lohi"):
            assert (x[key][k] == y[key][k]).all(), (key, k)
        assert x[key]["objective"] == y[key]["objective"]
    for key in ("c", "e", "c2", "e2"):
        assert (x[key] == y[key]).all(), key
    assert (x["bo"]["history"] == y["bo"]["history"]).all()
    assert (x["bo"]["cut_history"] == y["bo"]["cut_history"]).all()
    assert (x["bo"]["v"] == y["bo"]["v"]).all() and (x["bo"]["h"] == y["bo"]["h"]).all()


def test_nccl_comm_world1_matches_plain():
    lobe = _lobe()
    sc = make_scene(make_config(CFG["base"], G=CFG["G"], N=CFG["N"], seed=CFG["seed"]))
    m, n = 3, 3
    with lobe.Scene(sc, sc) as S:
        ref = _run_all(S, m, n)
    nid = lobe.nccl_unique_id()
    assert len(nid) == 128
    with lobe.Scene(sc, sc, nccl_id=nid) as S:
        assert S.collective
        got = _run_all(S, m, n)
        st = S.stats()
        assert st.t_comm_ms > 0.0
    _same(got, ref)
    with lobe.Scene(sc, sc, nccl_id=nid) as S:  # the cached ncclComm is reused
        _same(_run_all(S, m, n), ref)
    lobe.release_comms()


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2510_01767_b200 import lobe
    from paper_2510_01767_b200.engine import Engine
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        sc = make_scene(make_config(CFG["base"], G=CFG["G"], N=CFG["N"], seed=CFG["seed"]))
        eng = Engine.from_scene(sc, sc, device=0)
        assert eng.local.collective and eng.local.n_local < sc.N
        out = _run_all(eng.local, 3, 3)
        out["bo"] = {k: out["bo"][k] for k in ("history", "cut_history", "v", "h")}
        out["b"] = dict(out["b"])
        q.put((rank, out))
        eng.close()
    except Exception as ex:  # pragma: no cover
        import traceback
        traceback.print_exc()
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_host_comm_ranks_match_world1(world):
    lobe = _lobe()
    import torch.multiprocessing as mp
    sc = make_scene(make_config(CFG["base"], G=CFG["G"], N=CFG["N"], seed=CFG["seed"]))
    with lobe.Scene(sc, sc) as S:
        ref = _run_all(S, 3, 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, out in res:
        assert not isinstance(out, str), out
        _same(out, ref)
    for p in procs:
        assert p.exitcode == 0


def test_bench_two_ranks_shared_gpu():
    """bench.py's multi-rank path (self-spawn under torch.distributed.run, the
    collective engine, timings max over ranks, rank-0 line) with both ranks on
    the one GPU through the host-callback communicator (LOBE_BENCH_SHARED_GPU):
    the line reports 2 GPUs and the world-1 objective."""
    import json
    import subprocess
    import sys
    _lobe()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    args = [sys.executable, os.path.join(root, "bench.py"), "--config", "tiny", "--steps", "2", "--warmup", "3",
            "--no-bo", "--no-cpu-baseline", "--no-dense-ref", "--e2e-steps", "1", "--render", "0"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    one = subprocess.run(args, cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert one.returncode == 0, one.stderr[-2000:]
    l1 = json.loads(one.stdout.strip().splitlines()[-1])
    env["LOBE_BENCH_SHARED_GPU"] = "1"
    two = subprocess.run(args + ["--gpus", "2"], cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert two.returncode == 0, two.stderr[-3000:]
    l2 = json.loads([l for l in two.stdout.splitlines() if l.startswith("{")][-1])
    assert l2["n_gpus"] == 2 and l2["value"] > 0 and l2["engine_eval_ms"] > 0
    assert l2["objective_uniform"] == l1["objective_uniform"]
    assert l2["visible_incidences"] == l1["visible_incidences"]
    assert "not a measurement" in l2["data"]
