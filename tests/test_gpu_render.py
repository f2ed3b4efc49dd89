"""GPU parity of the paper-exact camera selection (ledger
L26): depth / weight maps, back-projected clouds and the cloud-ratio
assignments and block loads equal the oracle's bit for bit."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    from paper_2510_01767_b200 import lobe
    from synth import make_scene
    sc = make_scene("tiny")
    grid = oracle.default_grid(2, 2)
    o = oracle.run(sc, grid=grid)

    class DG:
        pass

    dg = DG()
    for k in oracle.SUB_FIELDS:
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
    S = lobe.Scene(sc, sc)
    yield sc, grid, o, dg, S
    S.close()


def _vis_idx(o, c, G):
    row = o["vis"]["rows"][c]
    return np.flatnonzero(np.unpackbits(row.view(np.uint8), bitorder="little")[:G])


def test_maps_bit_exact(setup):
    sc, grid, o, dg, S = setup
    for c in (0, 5, 17, 40, 63):
        D, W = S.render_maps(dg, c, 4, int(sc.width[c]), int(sc.height[c]))
        Do, Wo, _, _ = oracle.render_camera(sc, o["pre"], o["frame"], c, _vis_idx(o, c, sc.G), 4, 2, 0.1)
        assert np.array_equal(D, Do) and np.array_equal(W, Wo), c


def test_clouds_and_assignment(setup):
    sc, grid, o, dg, S = setup
    S.render_select(dg)
    off, gu, gv = S.camera_clouds()
    cl = oracle.render_clouds(sc, o["pre"], o["vis"], o["frame"])
    assert np.array_equal(off, cl["off"])
    assert np.array_equal(gu, cl["gu"]) and np.array_equal(gv, cl["gv"])
    for g in (grid, oracle.default_grid(3, 3), oracle.default_grid(2, 2, tau=0.4)):
        ref = oracle.assign_points(sc, o["pre"], cl, g)
        a = S.assign_cameras(g["m"], g["n"], v=g["v"], h=g["h"], delta_v=g["dv"], delta_h=g["dh"], tau=g["tau"])
        assert np.array_equal(a["n"], ref["n"]) and np.array_equal(a["n0"], ref["n0"])
        assert np.array_equal(a["member"], ref["member"]) and np.array_equal(a["home"], ref["home"])
        # visibility-based outputs are unchanged by the selection mode
        assert np.array_equal(a["K"], o["vis"]["K"])
        bl = oracle.block_loads(sc, o["pre"], o["vis"], ref, g)
        L = S.block_loads(g["m"], g["n"], v=g["v"], h=g["h"], delta_v=g["dv"], delta_h=g["dh"], tau=g["tau"])
        for k in ("n_cams", "g_vis", "g_blk", "incidences"):
            assert np.array_equal(L[k], bl[k]), k


def test_mid_size_clouds_and_assignment():
    """A Rubble-shaped scene (40k Gaussians, 12 cameras at 288x216 after the
    1/4 downscale: many 16x16 tiles, deep splat lists): clouds, assignments
    and block loads equal the oracle's bit for bit."""
    import torch
    from paper_2510_01767_b200 import lobe
    from synth import make_scene, make_config
    sc = make_scene(make_config("rubble", G=40_000, N=12, seed=0x4D1))
    g = oracle.default_grid(3, 3)
    o = oracle.run(sc, grid=g)
    cl = oracle.render_clouds(sc, o["pre"], o["vis"], o["frame"])

    class DG:
        pass

    dg = DG()
    for k in oracle.SUB_FIELDS:
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
    with lobe.Scene(sc, sc) as S:
        S.render_select(dg)
        off, gu, gv = S.camera_clouds()
        assert np.array_equal(off, cl["off"])
        assert np.array_equal(gu, cl["gu"]) and np.array_equal(gv, cl["gv"])
        ref = oracle.assign_points(sc, o["pre"], cl, g)
        a = S.assign_cameras(3, 3)
        assert np.array_equal(a["n"], ref["n"]) and np.array_equal(a["member"], ref["member"])
        assert np.array_equal(a["home"], ref["home"])
        bl = oracle.block_loads(sc, o["pre"], o["vis"], ref, g)
        L = S.block_loads(3, 3)
        for k in ("n_cams", "g_vis", "g_blk", "incidences"):
            assert np.array_equal(L[k], bl[k]), k


@pytest.mark.parametrize("cfg,sample", [("rubble", [0, 1, 2, 413, 829, 1243, 1656]),
                                        ("matrixcity", [0, 2, 2811, 5619])])
def test_full_size_render_sampled_cameras(cfg, sample):
    """Full BASELINE sizes (Rubble 2M x 1657; MatrixCity 10M x 5620, 1.16e8
    cloud points): the selection runs over every camera on the GPU; for nadir
    and oblique cameras spread over the flight path, the depth / weight maps and
    the back-projected clouds equal the oracle's (computed for those cameras
    alone from the oracle's own visible sets) bit for bit."""
    import torch
    from paper_2510_01767_b200 import lobe
    from synth import make_scene
    sc = make_scene(cfg)
    fr = oracle.frame(sc)
    pre = oracle.prep(sc, fr)
    vis = oracle.visibility(sc, pre, cams=sample)
    bits = np.unpackbits(vis["rows"].view(np.uint8), bitorder="little").reshape(len(sample), -1)[:, :sc.G]

    class DG:
        pass

    dg = DG()
    for k in oracle.SUB_FIELDS:
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
    with lobe.Scene(sc, sc) as S:
        S.render_select(dg)
        off, gu, gv = S.camera_clouds()
        assert off.shape[0] == sc.N + 1 and off[-1] > 0
        for i, c in enumerate(sample):
            Do, Wo, pu, pv = oracle.render_camera(sc, pre, fr, c, np.flatnonzero(bits[i]), 4, 2, 0.1)
            D, W = S.render_maps(dg, c, 4, int(sc.width[c]), int(sc.height[c]))
            assert np.array_equal(D, Do) and np.array_equal(W, Wo), c
            assert off[c + 1] - off[c] == len(pu), c
            assert np.array_equal(gu[off[c]:off[c + 1]], pu) and np.array_equal(gv[off[c]:off[c + 1]], pv), c
