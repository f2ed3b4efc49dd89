"""Benchmark of the LoBE-GS visibility engine on B200 (contract: see DESIGN.md "Measurement").

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lobe|reference] [--config matrixcity]

--gpus N > 1 without a launcher re-executes itself under torch.distributed.run
(N ranks, one per GPU, 127.0.0.1); under a launcher WORLD_SIZE must equal N.

A step is one pass of the whole hot path over one synthetic scene resident in
HBM (plus the a11 exchange when N > 1): ingest and
per-Gaussian precompute with the spatial sort, camera setup, the Gaussian x
camera visibility pass with the depth statistic, the camera assignment and the
block loads at the paper's uniform cuts, and the crop / densify-eligible masks.
The partition-balancing loop (a10, L = 100 evaluations on the cached rows) is
timed separately and reported under "bo" ("The BO-loop time
... is reported separately").

value  = G * N logical visibility tests / step time (max over ranks, CUDA events)
e2e    = the same metric through the C ABI with pinned HOST buffers, host<->device
         copies inside the timed region
roofline: the visibility kernel (a3), FP32-ALU bound, 22 flop per test.
"""
import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOP_PER_TEST_ISO = 22  # 9 FFMA (w,u,v) + 2 FFMA (edge tests), 2 flop each
# anisotropic predicate (ledger L24): 9 FMA (xc,yc,zc) + 2 mul (a,b) + 2 FMA (upix,vpix) + 4 mul (J)
# + 6 FMA + 6 mul (T) + 2 x 3 x (2 FMA + 1 mul) (V) + 3 x (2 FMA + 1 mul) + 2 add (A, B, C) + 2 add + 2 mul
# (mid, d) + 1 FMA + 1 mul (disc) + 1 add + 1 mul (r) + 2 add (W + r, H + r) = 108 flop; the reciprocal and
# the two square roots are not counted
FLOP_PER_TEST_ANISO = 108
FLOP_PER_TEST = FLOP_PER_TEST_ISO
FP32_LANES_PER_SM = 128
# FFMA issued per exact test by open-condition pattern (k_vis_tiles; lobe_stats.exact_pattern_tests): left / top
# edge u or v (3), right / bottom edge w + u or v + the edge (7), top-left u + v (6), top-right / bottom-left
# w + u + v + one edge (10), the four edges and all six w + u + v + both edges (11); 2 flop per FFMA
PATTERN_NAMES = ("left_edge", "top_edge", "right_edge", "bottom_edge", "top_left", "top_right", "bottom_left",
                 "four_edges", "all_six")
PATTERN_FFMA = (3, 3, 7, 7, 6, 10, 10, 11, 11)


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="lobe", choices=["lobe", "reference"])
    p.add_argument("--config", default="matrixcity")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-bo", action="store_true")
    p.add_argument("--no-dense-ref", action="store_true", help="skip the dense pinned-test reference kernel")
    p.add_argument("--bo-L", type=int, default=100)
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--render", type=int, default=1, help="also time the depth-render camera selection (NEXT-1)")
    p.add_argument("--predicate", default="iso", choices=["iso", "aniso"],
                   help="visibility predicate: iso = SPEC.md:299 bound (the metric's path), aniso = EWA footprint")
    p.add_argument("--spawn-check", action="store_true",
                   help="print each rank's (rank, world) as JSON and exit (launcher test; needs no GPU)")
    return p.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """--gpus N > 1 outside a launcher: run N ranks under torch.distributed.run
    (one per GPU) and return their exit code; None = this process is a rank."""
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but the launcher's WORLD_SIZE is "
                             f"{os.environ['WORLD_SIZE']}\n")
            return 2
        return None
    if args.gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_dict(cfg_name, sc, pred, world):
    """The workload description both arms print (identical keys and values)."""
    return {"workload": f"{cfg_name}-shaped", "G": sc.G, "N": sc.N, "grid": f"{sc.cfg.m}x{sc.cfg.n}",
            "predicate": "anisotropic (EWA, ledger L24)" if pred else "isotropic (SPEC.md:299)",
            "parallelism": f"camera-sharded x{world}", "l2": "inputs larger than L2 (no flush)",
            "step": "a1-a9 (+a11 exchange): load+precompute+sort, visibility, assignment, block loads "
                    "at uniform cuts, crop masks", "seed": hex(sc.cfg.seed)}


def cpu_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_cores": os.cpu_count()}


def scene_hashes(sc):
    """SHA-256 of every generated input array (inputs are logged)."""
    from synth import array_hashes
    h = array_hashes(sc)
    allh = hashlib.sha256("".join(h[k] for k in sorted(h)).encode()).hexdigest()[:16]
    return {"arrays": h, "all": allh}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML samples of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- cpu baseline
def _oracle_sample(sc, pre, sel, threads, pred):
    import oracle
    pre["cam_gu_sel"], pre["cam_gv_sel"] = pre["cam_gu"][sel], pre["cam_gv"][sel]
    if pred:
        vis = oracle.visibility_aniso(sc, pre, cams=sel, threads=threads)
    else:
        vis = oracle.visibility(sc, pre, cams=sel, threads=threads)
    oracle.assign(sc, pre, vis, oracle.default_grid(sc.cfg.m, sc.cfg.n), threads=threads)


def cpu_baseline(sc, target_s=12.0, pred=0):
    """The oracle as it stands, on the host cores, on a bounded sample of the
    same workload: the visibility pass (O6/O7) and camera assignment (O8) of a
    random sample of cameras over all G Gaussians, all threads; plus the same on
    one thread (the single-core rate)."""
    import oracle
    threads = oracle.nthreads()
    t0 = time.perf_counter()
    oracle.validate(sc)
    fr = oracle.frame(sc)
    pre = oracle.prep(sc, fr)
    if pred:
        pre["cov"] = oracle.cov(sc)
    t_prep = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    t_sample, done = 0.0, 0
    while done < sc.N and t_sample < target_s:
        sel = np.sort(rng.choice(sc.N, min(threads, sc.N), replace=False))
        t1 = time.perf_counter()
        _oracle_sample(sc, pre, sel, threads, pred)
        t_sample += time.perf_counter() - t1
        done += len(sel)
    # single core: cameras one at a time on one thread for ~2 s
    t_one, done1 = 0.0, 0
    while done1 < sc.N and t_one < 2.0:
        sel = np.sort(rng.choice(sc.N, 1, replace=False))
        t1 = time.perf_counter()
        _oracle_sample(sc, pre, sel, 1, pred)
        t_one += time.perf_counter() - t1
        done1 += 1
    out = {"value": sc.G * done / t_sample, "unit": "tests/s", "cores": threads, "kind": "oracle",
           "single_core_value": sc.G * done1 / t_one,
           "sample": f"{done} random cameras x all {sc.G} Gaussians: visibility ({'O6a' if pred else 'O6'}/O7) "
                     f"+ assignment (O8), {t_sample:.1f} s on {threads} threads; single core: {done1} cameras, "
                     f"{t_one:.1f} s; per-Gaussian prep (O3, single thread) {t_prep:.1f} s not included",
           "cpu_seconds": t_sample + t_one + t_prep}
    out.update(cpu_info())
    return out


def run_reference(args, cfg_name):
    """--impl reference: the oracle on the host cores, timed as it stands, on
    this arm's config/metric; each step a bounded sample of the workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from synth import make_scene
    pred = 1 if args.predicate == "aniso" else 0
    sc = make_scene(cfg_name)
    threads = oracle.nthreads()
    oracle.validate(sc)
    fr = oracle.frame(sc)
    t0 = time.perf_counter()
    pre = oracle.prep(sc, fr)
    if pred:
        pre["cov"] = oracle.cov(sc)
    t_prep = time.perf_counter() - t0
    rng = np.random.default_rng(1)
    per_step = max(1, threads)

    def step():
        _oracle_sample(sc, pre, np.sort(rng.choice(sc.N, per_step, replace=False)), threads, pred)

    for _ in range(args.warmup):
        step()
    t1 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t1) / args.steps
    # per-camera share of the one-off precompute, so the rate covers the same rows
    t_step = dt + t_prep * per_step / sc.N
    value = sc.G * per_step / t_step
    cpu = {"value": value, "unit": "tests/s", "cores": threads, "kind": "oracle",
           "sample": f"per step {per_step} random cameras x all {sc.G} Gaussians: visibility "
                     f"({'O6a' if pred else 'O6'}/O7) + assignment (O8) + their share of the per-Gaussian prep"}
    cpu.update(cpu_info())
    line = {"metric": "gaussian_camera_visibility_tests_per_s", "value": value, "unit": "tests/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "config": config_dict(cfg_name, sc, pred, args.gpus),
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def load_profile(name, cfg_name, world, pred):
    """A committed ncu summary under profiles/ if it was taken on this config."""
    path = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(path):
        return None
    try:
        tj = json.load(open(path))
    except Exception:
        return None
    if tj.get("config") != cfg_name or tj.get("world", 1) != 1 or pred:
        return None
    return tj


# ----------------------------------------------------------------------------- main arm
def main():
    args = parse()
    cfg_name = args.config
    if args.spawn_check and "WORLD_SIZE" not in os.environ and args.gpus <= 1:
        print(json.dumps({"rank": 0, "world": 1}), flush=True)
        return 0
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    rank, world, local = dist_env()
    if args.spawn_check:
        # one write() per line: the ranks share the launcher's stdout pipe
        os.write(1, (json.dumps({"rank": rank, "world": world, "local_rank": local}) + "\n").encode())
        return 0
    if args.impl == "reference":
        return run_reference(args, cfg_name)
    import torch
    import torch.distributed as dist
    # LOBE_BENCH_SHARED_GPU=1 (tests only): every rank on GPU 0 with a gloo group,
    # so the library's host-callback communicator carries the exchange -- checks
    # the multi-rank plumbing of this script on a one-GPU box; never a bench value
    shared = os.environ.get("LOBE_BENCH_SHARED_GPU") == "1"
    dev = 0 if shared else local
    if not torch.cuda.is_available() or torch.cuda.device_count() <= dev:
        sys.stderr.write(f"bench.py: rank {rank} needs GPU {dev}; {torch.cuda.device_count()} visible\n")
        return 2
    torch.cuda.set_device(dev)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_01767_b200 import lobe
    from paper_2510_01767_b200.engine import Engine, shard
    from synth import make_scene

    global FLOP_PER_TEST
    pred = 1 if args.predicate == "aniso" else 0
    FLOP_PER_TEST = FLOP_PER_TEST_ANISO if pred else FLOP_PER_TEST_ISO
    sc = make_scene(cfg_name)
    G, N, m, n = sc.G, sc.N, sc.cfg.m, sc.cfg.n
    B = m * n
    W64 = (G + 63) // 64
    names = ("x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "opacity")

    class DevG:
        pass

    dg = DevG()
    for k in names:
        setattr(dg, k, torch.from_numpy(getattr(sc, k)).cuda())
    cams = lobe.make_cameras(sc)
    stream = torch.cuda.current_stream()
    crop_d = torch.empty(B * W64, dtype=torch.int64, device="cuda")
    elig_d = torch.empty(B * W64, dtype=torch.int64, device="cuda")
    group = None
    acc = {}

    def reset_acc():
        acc.clear()
        acc.update({"t_vis_ms": [], "t_cull_ms": [], "t_depth_ms": [], "t_eval_ms": [], "t_comm_ms": [],
                    "t_crop_ms": [], "kernels": 0, "cub": 0, "tests": 0})

    reset_acc()

    def step(gsrc, crop_out, elig_out):
        eng = Engine.from_scene(gsrc, cams, stream=stream, group=group, predicate=pred)
        # nothing here waits for the device until block_loads reads the block
        # counts: the evaluation and the crop are enqueued first, so the crop
        # runs while the host builds the records; assign_cameras' copies follow
        eng.crop_masks_into(m, n, crop_out, elig_out)
        L = eng.block_loads(m, n)
        A = eng.assign_cameras(m, n)
        st = eng.stats()
        for k in ("t_vis_ms", "t_cull_ms", "t_depth_ms", "t_comm_ms", "t_crop_ms"):
            acc[k].append(getattr(st, k))
        acc["t_eval_ms"].append(st.t_hist_ms + st.t_loads_ms)
        acc["st"] = st
        acc["kernels"] += st.kernel_launches
        acc["cub"] += st.cub_launches
        acc["tests"] += st.tests_executed
        eng.close()
        return L, A

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(vals):
        if world == 1:
            return list(vals)
        t = torch.tensor(list(vals), dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def timed(nsteps, gsrc, crop_out, elig_out):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = None
        for _ in range(nsteps):
            out = step(gsrc, crop_out, elig_out)
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1) / nsteps
        return max_over_ranks([ms])[0], out

    # ---- warmup + timed (inputs resident in HBM; inputs >> L2 so no flush needed)
    for _ in range(args.warmup):
        step(dg, crop_d, elig_d)
    reset_acc()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, (Lrec, Aout) = timed(args.steps, dg, crop_d, elig_d)
    st = acc["st"]
    mean = {k: statistics.mean(acc[k]) for k in ("t_vis_ms", "t_cull_ms", "t_depth_ms", "t_eval_ms", "t_comm_ms",
                                                 "t_crop_ms")}
    # engine evaluation: a3 + a5-a8 + the combine at the uniform cuts
    engine_eval = mean["t_vis_ms"] + mean["t_eval_ms"] + mean["t_comm_ms"]
    t_vis, t_eval, t_comm, engine_eval_max, t_depth = max_over_ranks(
        [mean["t_vis_ms"], mean["t_eval_ms"], mean["t_comm_ms"], engine_eval, mean["t_depth_ms"]])
    timed_kernels, timed_cub = acc["kernels"], acc["cub"]
    c0, c1 = shard(N, rank, world)
    n_local = c1 - c0
    value = G * N / (ms * 1e-3)

    # ---- e2e: pinned host buffers through the C ABI
    class HostG:
        pass

    hg = HostG()
    for k in names:
        t = torch.empty(G, dtype=torch.float32, pin_memory=True)
        t.numpy()[:] = getattr(sc, k)
        setattr(hg, k, t)
    crop_h = torch.empty(B * W64, dtype=torch.int64, pin_memory=True)
    elig_h = torch.empty(B * W64, dtype=torch.int64, pin_memory=True)
    step(hg, crop_h, elig_h)  # warm
    ms_e2e, _ = timed(args.e2e_steps, hg, crop_h, elig_h)
    h2d = 11 * 4 * G + N * 80
    d2h = 2 * B * W64 * 8 + N * (4 + 8 + 4 + 4 + 2 * B * 4 + 8 + 4) + B * 64

    # ---- isolated stage times: inside the step a4 runs on a side stream next to
    # the evaluation, so their CUDA-event times overlap and each is inflated by
    # the other. Here a4 is deferred (LOBE_A4_STREAM=0) and runs alone after
    # the evaluations: these are the per-kernel numbers the rooflines and the
    # §8(d) scaling quantity use (the step's own numbers are kept as "in_step").
    iso = {"t_vis_ms": [], "t_eval_ms": [], "t_comm_ms": [], "t_depth_ms": []}
    prev_env = os.environ.get("LOBE_A4_STREAM")
    os.environ["LOBE_A4_STREAM"] = "0"
    try:
        for _ in range(3):
            eng = Engine.from_scene(dg, cams, stream=stream, group=group, predicate=pred)
            for _ in range(3):
                eng.block_loads(m, n)
                s1 = eng.stats()
                iso["t_eval_ms"].append(s1.t_hist_ms + s1.t_loads_ms)
                iso["t_comm_ms"].append(s1.t_comm_ms)
            eng.assign_cameras(m, n)  # a4 enqueued now, alone on the scene's stream
            s1 = eng.stats()
            iso["t_vis_ms"].append(s1.t_vis_ms)
            iso["t_depth_ms"].append(s1.t_depth_ms)
            eng.close()
    finally:
        if prev_env is None:
            os.environ.pop("LOBE_A4_STREAM", None)
        else:
            os.environ["LOBE_A4_STREAM"] = prev_env
    iso_mean = {k: statistics.median(v) for k, v in iso.items()}
    iso_engine = iso_mean["t_vis_ms"] + iso_mean["t_eval_ms"] + iso_mean["t_comm_ms"]
    iso_vis, iso_eval, iso_comm, iso_engine_max, iso_depth = max_over_ranks(
        [iso_mean["t_vis_ms"], iso_mean["t_eval_ms"], iso_mean["t_comm_ms"], iso_engine, iso_mean["t_depth_ms"]])

    # ---- dense pinned-test reference (no bounds: every one of the G x N_local tests)
    dense_ref = None
    if not pred and not args.no_dense_ref:
        eng = Engine.from_scene(dg, cams, stream=stream, group=group, predicate=pred)
        dms, dgrid = eng.local.dev_vis_bench(variant=2, reps=2)
        eng.close()
        dense_ref = {"kernel": "k_vis<16,4,dense> (lobe_dev_vis_bench variant 2: the full O6 test, no bounds)",
                     "ms": dms, "tests": G * n_local, "grid": dgrid}

    # ---- BO loop (a10), reported separately
    bo = None
    if not args.no_bo:
        eng = Engine.from_scene(dg, cams, stream=stream, group=group, predicate=pred)
        barrier()
        t0 = time.perf_counter()
        r = eng.balance_partition(m, n, L=args.bo_L, seed=0)
        barrier()
        bo_s = time.perf_counter() - t0
        bst = eng.stats()
        bo = {"L": args.bo_L, "seconds": bo_s, "ms_per_evaluation": bo_s * 1e3 / args.bo_L,
              "gpu_eval_ms": bst.t_hist_ms + bst.t_loads_ms, "comm_ms_last_evaluation": bst.t_comm_ms,
              "objective_uniform": int(r["history"][0]), "objective_best": int(r["history"].min()),
              "improvement": 1.0 - float(r["history"].min()) / max(1, int(r["history"][0])),
              "tests_executed": int(bst.tests_executed)}
        # paper-exact camera selection (ledger L26): depth
        # render + back-projection of every camera, then the BO loop on the clouds
        if args.render and world == 1:
            barrier()
            t0 = time.perf_counter()
            eng.local.render_select(dg)
            barrier()
            rs = time.perf_counter() - t0
            off, _, _ = eng.local.camera_clouds()
            rst = eng.stats()
            rflop = 11.0 * rst.render_tests + 28.0 * rst.render_composited
            t0 = time.perf_counter()
            r2 = eng.balance_partition(m, n, L=args.bo_L, seed=0)
            bo2 = time.perf_counter() - t0
            bo["render_selection"] = {"seconds": rs, "cameras": int(N), "cloud_points": int(off[-1]),
                                      "downscale": 4, "stride": 2, "eps_w": 0.1,
                                      "bo_seconds": bo2, "objective_uniform": int(r2["history"][0]),
                                      "objective_best": int(r2["history"].min()),
                                      # k_render (per-pixel compositing): 11 flop per (pixel, splat) footprint
                                      # test + 28 per composited splat (pinned exp, alpha, weights, depth)
                                      "k_render": {"ms": rst.t_render_kernel_ms, "tests": int(rst.render_tests),
                                                   "composited": int(rst.render_composited), "flop": rflop,
                                                   "achieved_TFLOPs": rflop / max(rst.t_render_kernel_ms, 1e-9)
                                                   * 1e-9,
                                                   "frac_fp32": rflop / max(rst.t_render_kernel_ms, 1e-9) * 1e-9
                                                   / (torch.cuda.get_device_properties(0).multi_processor_count
                                                      * FP32_LANES_PER_SM * 2 * 1.965e9 / 1e12),
                                                   "bound": "alu (compositing loop; splats staged in shared memory)"}}
        eng.close()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(sc, pred=pred)
    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the visibility pass (a3)
    props = torch.cuda.get_device_properties(0)
    sms = props.multi_processor_count
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_max_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak = sms * FP32_LANES_PER_SM * 2 * sm_max_mhz * 1e6 / 1e12  # TFLOP/s
    dense_tests = int(st.dense_tests)
    t_vis0 = mean["t_vis_ms"]  # rank 0's own pass (the counters below are rank 0's)
    # contract convention: 22 flop per EXECUTED exact test; the box
    # bounds decide the rest ("the roofline stays defined on
    # executed tests")
    achieved = FLOP_PER_TEST * dense_tests / (t_vis0 * 1e-3) / 1e12
    pat = [int(x) for x in st.exact_pattern_tests]
    issued_flop = float(sum(2 * f * c for f, c in zip(PATTERN_FFMA, pat))) if not pred else None
    clocks = clk.summary()
    decided = [int(x) for x in st.decided_tests]
    roof = {"bound": "alu",
            "kernel": ("k_cull + k_vis_tiles_aniso (a3)" if pred else "k_cull + k_slice_codes + k_vis_tiles (a3)"),
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "convention": f"SURVEY §8(d) contract: {FLOP_PER_TEST} flop per executed exact test "
                          "(9 FFMA w,u,v + 2 FFMA edges, 2 flop each), whatever the kernel issues",
            "traffic": None,
            "peak_basis": f"{sms} SMs x {FP32_LANES_PER_SM} FP32 lanes x 2 flop x {sm_max_mhz:.0f} MHz "
                          "(sm_max_mhz of MEASURED_PEAKS.json)",
            "kernel_ms": t_vis0, "cull_ms": mean["t_cull_ms"], "kernel_share_of_step": t_vis0 / ms,
            "executed_tests": dense_tests, "logical_tests": int(G * n_local),
            "executed_fraction": dense_tests / float(G * n_local),
            # I16, counted inside k_cull / k_vis_tiles (real Gaussians, padding excluded): sums to G x N_local
            "decided_in_kernels": {"tile_rejected": decided[0], "slice_rejected": decided[1],
                                   "slice_accepted": decided[2], "exact_tested": decided[3],
                                   "sum_equals_G_x_N_local": sum(decided) == G * n_local},
            "logical_tests_per_s_kernel": G * n_local / (t_vis0 * 1e-3),
            "executed_tests_per_s_kernel": dense_tests / (t_vis0 * 1e-3),
            "dense_roofline_ms": FLOP_PER_TEST * G * n_local / (peak * 1e12) * 1e3,
            "logical_frac_of_dense_roofline": (FLOP_PER_TEST * G * n_local / (peak * 1e12) * 1e3) / t_vis0,
            "target_logical_tests_per_s": 0.6 * peak * 1e12 / FLOP_PER_TEST,
            "frac_at_measured_clock": (achieved / (peak * (clocks["sm_mhz"] or sm_max_mhz) / sm_max_mhz))}
    if issued_flop is not None:
        roof["exact_tests_by_open_conditions"] = dict(zip(PATTERN_NAMES, pat))
        roof["issued"] = {"flop": issued_flop, "achieved": issued_flop / (t_vis0 * 1e-3) / 1e12,
                          "frac": issued_flop / (t_vis0 * 1e-3) / 1e12 / peak,
                          "basis": "FFMA the kernel issues per open-condition pattern "
                                   f"{dict(zip(PATTERN_NAMES, PATTERN_FFMA))} x 2 flop x the exact tests run "
                                   "with that pattern (lobe_stats.exact_pattern_tests), over the pass time"}
    if dense_ref is not None:
        dflop = FLOP_PER_TEST * dense_ref["tests"]
        dense_ref["achieved"] = dflop / (dense_ref["ms"] * 1e-3) / 1e12
        dense_ref["frac"] = dense_ref["achieved"] / peak
        dense_ref["basis"] = "22 flop x G x N_local (every test executed) / the kernel's CUDA-event time"
        roof["dense_reference"] = dense_ref
    nc = load_profile("r02_vis_tiles_ncu.json", cfg_name, world, pred)
    if nc:
        # DRAM bytes of one k_vis_tiles launch (the pass's dominant kernel) from the committed
        # ncu --set full capture; algorithmic: 16 B x G_pad read + the kept pairs' row words
        roof["traffic"] = nc.get("dram_bytes_per_launch")
        roof["traffic_kernel"] = "k_vis_tiles (profiles/r02_vis_tiles_ncu.json)"
        roof["ncu"] = {k: nc[k] for k in nc if k not in ("config", "world")}
    # the depth statistic (a4): 9 flop per visible (Gaussian, camera) incidence
    # (w: 3 FMA, o*w: 1 FMA, o: 1 add), the statistic's own work
    vis_inc = int(np.asarray(Aout["K"], np.int64).sum())
    depth_flop = 9.0 * float(np.asarray(Aout["K"][c0:c1], np.int64).sum())  # rank 0's cameras
    t_dep = iso_mean["t_depth_ms"]  # alone on the stream (the in-step time overlaps the evaluation)
    depth_roof = {"bound": "alu", "kernel": "k_depth_pairs + camera order + k_depth_reduce (a4)",
                  "achieved": depth_flop / (t_dep * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                  "frac": depth_flop / (t_dep * 1e-3) / 1e12 / peak, "kernel_ms": t_dep,
                  "in_step_ms": mean["t_depth_ms"],
                  "timing": "kernel_ms: a4 alone on the scene's stream (LOBE_A4_STREAM=0); in_step_ms: on the "
                            "depth side stream inside the timed step, concurrent with the evaluation and crop",
                  "flop_basis": "9 flop per visible (Gaussian, camera) incidence of this rank's cameras"}
    # a5-a8 (one evaluation at the uniform cuts) against HBM
    hbm = float(peaks.get("hbm_gbs", 6468.3))
    logical_bytes = n_local * G / 8.0 + B * G / 8.0
    actual_bytes = 2 * 128.0 * int(st.tile_pairs) + B * G / 8.0  # hist + masks read each non-empty pair's 128 B
    t_ev = iso_mean["t_eval_ms"]
    evaluation = {"kernels": "k_zones + k_gblk + k_hist + k_assign + k_block_masks (a5-a8)", "ms": t_ev,
                  "in_step_ms": mean["t_eval_ms"],
                  "timing": "ms: one evaluation at the uniform cuts with nothing else on the device (median of 9); "
                            "in_step_ms: the step's first evaluation, concurrent with a4 on the side stream",
                  "bound": "hbm", "hbm_peak_GBps": hbm, "hbm_peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy)",
                  "logical_bytes": logical_bytes, "logical_GBps": logical_bytes / (t_ev * 1e-3) / 1e9,
                  "logical_frac_of_hbm": logical_bytes / (t_ev * 1e-3) / 1e9 / hbm,
                  "row_bytes_touched": actual_bytes,
                  "achieved_GBps": actual_bytes / (t_ev * 1e-3) / 1e9,
                  "frac": actual_bytes / (t_ev * 1e-3) / 1e9 / hbm}
    line = {"metric": "gaussian_camera_visibility_tests_per_s", "value": value, "unit": "tests/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic" + (" (LOBE_BENCH_SHARED_GPU test run: all ranks on GPU 0, not a measurement)"
                                   if shared else ""),
            "config": config_dict(cfg_name, sc, pred, world),
            "roofline": roof, "depth_roofline": depth_roof, "evaluation_roofline": evaluation,
            # the scaling quantity (a3 + a5-a8 + combine, max over ranks) and the exchange alone
            # measured with a4 out of the way (see evaluation_roofline.timing); in_step: inside the timed step
            "engine_eval_ms": iso_engine_max, "t_comm_ms": iso_comm, "t_vis_ms_max_over_ranks": iso_vis,
            "t_depth_ms_max_over_ranks": iso_depth, "t_crop_ms": mean["t_crop_ms"],
            "in_step": {"engine_eval_ms": engine_eval_max, "t_comm_ms": t_comm, "t_vis_ms": t_vis,
                        "t_depth_ms": t_depth, "t_eval_ms": t_eval},
            "cpu_baseline": cpu,
            "e2e": {"value": G * N / (ms_e2e * 1e-3), "unit": "tests/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e},
            "gpu_launches": int(timed_kernels),
            "gpu_launches_note": f"own kernels in the timed region ({args.steps} steps, rank 0), "
                                 f"{timed_kernels / args.steps:.0f} per step; plus CUB primitive calls "
                                 f"(radix sort, scan): {timed_cub / args.steps:.0f} per step",
            "clocks": clocks, "bo": bo,
            "objective_uniform": int(Lrec["objective"]),
            "visible_incidences": vis_inc,
            "tile_pairs": int(st.tile_pairs),
            "input_hashes": scene_hashes(sc)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
