"""Paper-scale SIR particle filter on the B200 (M/pfilter.py:182-226):
N = 2^20 particles, T = 100 steps, Megopolis / C1-128 / Metropolis at B = 16, 32, 64.
Reports RMSE and the resample ratio (stage-2 share of the step, CUDA-event times)."""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2109_13504_b200 import pfilter as pf  # noqa: E402
from paper_2109_13504_b200.rng import derive_seed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--t", type=int, default=100)
ap.add_argument("--trajectories", type=int, default=2)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--rng", default="megores")
a = ap.parse_args()
trajs = [pf.generate_trajectory(a.t, 0.0, derive_seed(1100, i)) for i in range(a.trajectories)]
t0 = time.time()
rows = pf.run_benchmark(pf.FilterConfig(n_particles=a.n, rng=a.rng), trajs, a.runs, [16, 32, 64],
                        [("megopolis", None), ("c1", 128), ("metropolis", None)], derive_seed(1101))
out = {"n": a.n, "t_steps": a.t, "trajectories": a.trajectories, "runs": a.runs, "rng": a.rng,
       "wall_s": round(time.time() - t0, 1), "rows": rows,
       "paper_k40m_megopolis": {"16": {"ratio": 0.603, "rmse": 3.039}, "32": {"ratio": 0.718, "rmse": 2.972},
                                "64": {"ratio": 0.821, "rmse": 2.948}}}
print(json.dumps(out, indent=1))
