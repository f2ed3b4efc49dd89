"""GPU parity of the block pipeline (
ledger L25): sub-scene extraction, the densification simulator, prune and
merge against the oracle, field for field (floats bit-exact)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _lobe():
    from paper_2510_01767_b200 import lobe
    return lobe


@pytest.fixture(scope="module")
def setup():
    import torch
    from synth import make_config, make_scene
    sc = make_scene(make_config("tiny", G=3000, N=32, seed=0x2510AC))
    m = n = 3
    grid = oracle.default_grid(m, n)
    o = oracle.run(sc, grid=grid)
    fr, pre = o["frame"], o["pre"]

    class DG:
        pass

    dg = DG()
    for k in oracle.SUB_FIELDS:
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
    S = _lobe().Scene(sc, sc)
    yield sc, grid, o, fr, pre, dg, S
    S.close()


def _cmp(gpu, ref):
    assert int(gpu["x"].shape[0]) == len(ref["x"])
    for k in oracle.SUB_FIELDS + ("origin", "in_block"):
        g = gpu[k].cpu().numpy()
        r = np.asarray(ref[k])
        assert g.dtype == r.dtype or k in ("in_block",), k
        assert np.array_equal(g.astype(r.dtype), r), k


def _to_dev(sub):
    import torch
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in sub.items()}


def test_subscene_all_blocks(setup):
    sc, grid, o, fr, pre, dg, S = setup
    for b in range(9):
        gs = S.block_subscene(3, 3, b, dg)
        ref = oracle.subscene(sc, o["crop"][b], o["eligible"][b])
        _cmp(gs, ref)


@pytest.mark.parametrize("split", [0.0, 0.004, 10.0])
def test_densify_prune_merge(setup, split):
    import torch
    sc, grid, o, fr, pre, dg, S = setup
    rng = np.random.default_rng(int(split * 1000) + 7)
    gpu_pruned, ref_pruned = [], []
    for b in range(9):
        ref = oracle.subscene(sc, o["crop"][b], o["eligible"][b])
        gsub = S.block_subscene(3, 3, b, dg)
        for step in range(2):
            nn = len(ref["x"])
            grad = rng.uniform(0, 2, nn).astype(np.float32)
            grad[rng.uniform(size=nn) < 0.1] = 1e30
            nrm = rng.normal(size=(nn, 6)).astype(np.float32)
            ref = oracle.densify_step(ref, grad, nrm, 1.0, split, fr, pre["minmax"], grid, b)
            gsub = S.densify_step(3, 3, b, gsub, torch.from_numpy(grad).cuda(), torch.from_numpy(nrm).cuda(),
                                  1.0, split)
            _cmp(gsub, ref)
        ref = oracle.prune_outside(ref, fr, pre["minmax"], grid, b)
        gsub = S.prune_outside(3, 3, b, gsub)
        _cmp(gsub, ref)
        gpu_pruned.append(gsub)
        ref_pruned.append(ref)
    merged_ref, ok = oracle.merge_blocks(ref_pruned)
    assert ok
    _cmp(S.merge_blocks(gpu_pruned), merged_ref)


def test_merge_integrity_error(setup):
    sc, grid, o, fr, pre, dg, S = setup
    lobe = _lobe()
    a = S.block_subscene(3, 3, 4, dg)
    with pytest.raises(lobe.LobeError) as e:
        S.merge_blocks([a, a])
    assert e.value.status == "INTEGRITY"


def test_identity_pipeline_acceptance_9(setup):
    """Acceptance #9 on the GPU path: crop -> prune -> merge over the 3x3 grid
    recovers exactly the Gaussians visible from an assigned camera of their
    containing block (the oracle's eligible masks), without duplicates."""
    sc, grid, o, fr, pre, dg, S = setup
    subs = [S.prune_outside(3, 3, b, S.block_subscene(3, 3, b, dg)) for b in range(9)]
    merged = S.merge_blocks(subs)
    got = set(merged["origin"].cpu().numpy().tolist())
    want = set()
    for b in range(9):
        e = o["eligible"][b]
        for i in range(sc.G):
            if (int(e[i >> 6]) >> (i & 63)) & 1:
                want.add(i)
    assert got == want and int(merged["x"].shape[0]) == len(want)
