"""Golden data for the SIR particle filter (M/pfilter.py) from the UNMODIFIED reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_pf.py
"""

import json
import math
import os

import numpy as np

import megores as m
from megores import pfilter as pf
from megores import rng
from megores.weights import WeightVector

OUT = os.path.dirname(os.path.abspath(__file__))
arrays, meta = {}, {}

# stage-level: init particles, one predict/update, estimate_ratio subsets
cfg = pf.FilterConfig(n_particles=2**12)
st = pf.init_state(cfg, 5)
arrays["init_particles"] = st.particles
traj = m.generate_trajectory(20, 0.0, 7)
arrays["traj_truth"], arrays["traj_obs"] = traj.truth, traj.observations
t = 1
noise = rng.gaussian_at(rng.derive_seed(5, pf._TAG_PROCESS, t), np.arange(cfg.n_particles), 0) * math.sqrt(10.0)
pred = pf.transition(st.particles, t, noise)
w = WeightVector(pf.likelihood(float(traj.observations[0]), pred, 1.0), "single")
arrays["step1_pred"], arrays["step1_w"] = pred, np.asarray(w.values)
ratios = []
for sub, seed in [(4096, 11), (1000, 12), (17, 13)]:
    r = m.estimate_ratio(w, sub, seed)
    ratios.append({"subset": sub, "seed": seed, "ratio": r})
ww = WeightVector(np.asarray(pf.likelihood(3.0, np.linspace(-20, 20, 50000), 1.0)), "single")
arrays["ratio_w2"] = np.asarray(ww.values)
ratios.append({"subset": 4096, "seed": 99, "ratio": m.estimate_ratio(ww, 4096, 99), "w": "ratio_w2"})
meta["ratios"] = ratios

# whole filters: fixed B and the runtime-B policy (M/pfilter.py:136-141)
runs = {}
for name, c in [("megopolis_b8", pf.FilterConfig(n_particles=2**12, resampler="megopolis", b_fixed=8)),
                ("c1_b8", pf.FilterConfig(n_particles=2**12, resampler="c1", partition_bytes=128, b_fixed=8)),
                ("megopolis_runtime_b", pf.FilterConfig(n_particles=2**12, resampler="megopolis", b_fixed=None,
                                                        epsilon=0.1)),
                ("metropolis_b16_double", pf.FilterConfig(n_particles=2**12, resampler="metropolis", b_fixed=16,
                                                          precision="double"))]:
    est, _ = pf.run_filter(c, traj, 42)
    arrays[f"est_{name}"] = est
    runs[name] = {"resampler": c.resampler, "b_fixed": c.b_fixed, "partition_bytes": c.partition_bytes,
                  "precision": c.precision, "epsilon": c.epsilon, "n": c.n_particles}
meta["runs"] = runs

# benchmark rows (RMSE is the paper's filter metric)
trajs = [m.generate_trajectory(30, 0.0, rng.derive_seed(1100, i)) for i in range(2)]
rows = pf.run_benchmark(pf.FilterConfig(n_particles=2**14), trajs, 4, [16, 64],
                        [("megopolis", None), ("c1", 128)], rng.derive_seed(1101))
meta["bench_rows"] = [{k: v for k, v in r.items() if k != "resample_ratio"} for r in rows]

np.savez_compressed(os.path.join(OUT, "pf_golden.npz"), **arrays)
with open(os.path.join(OUT, "pf_golden.json"), "w") as f:
    json.dump(meta, f, indent=1)
print(json.dumps(meta, indent=1)[:1500])
