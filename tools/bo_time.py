"""Diagnosis only: host time of the BO driver (lobe_bo_run, no GPU) at the
MatrixCity grid (6 x 6, L = 100) with a cheap deterministic objective, and a
hash of its trajectory (history + cut history) to check that a change of the
GP code keeps the trajectory bit-identical. LOBE_TRACE_HOST=1 prints the
phases (fit, candidates, pattern search, objective)."""
import hashlib
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2510_01767_b200 import lobe


def objective(v, h):
    v = np.asarray(v, np.float64)
    h = np.asarray(h, np.float64)
    return int(1e6 * (np.sum(np.sin(7 * v) ** 2) + np.sum((h - 0.4) ** 2)) + 12345)


for rep in range(2):
    t0 = time.perf_counter()
    r = lobe.bo_run(6, 6, objective, L=100, seed=0)
    t = time.perf_counter() - t0
    hsh = hashlib.sha256(r["history"].tobytes() + r["cut_history"].tobytes()).hexdigest()[:16]
    print(f"{t:.3f} s  trajectory {hsh}  best {r['history'].min()}")
