"""Time every lobe_dev_vis_bench variant on a config (diagnosis; CUDA events in
the library): 0 = the production tile-major pass, 1.. = camera-inner k_vis
variants (2 = the dense reference the bench reports)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401  (CUDA context)
from paper_2510_01767_b200 import lobe
from synth import make_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "matrixcity"
variants = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(9))
sc = make_scene(cfg)
with lobe.Scene(sc, sc, device=0) as S:
    for v in variants:
        ms, grid = S.dev_vis_bench(v, reps=2)
        frac = 22.0 * sc.G * sc.N / (ms * 1e-3) / 74.45e12
        print(f"variant {v}: {ms:8.3f} ms grid {grid}  dense-frac {frac:.3f}", flush=True)
