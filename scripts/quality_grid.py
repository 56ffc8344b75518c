"""Paper-scale resampling quality grid on the B200 (the reference's bench.quality_grid,
M/bench.py:107-149, with the paper's N range).

Per (algorithm, N, y): S weight sequences (Gaussian family, device generator), B from the
eps = 0.01 rule on each, K resampling runs per sequence; MSE/N, variance and bias
contribution from the device QualityAccumulator, averaged over sequences (not pooled).

    python scripts/quality_grid.py [--k 256 --seq 16] [--ns 15,20,22] > profiles/rNN_quality_grid.json
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2109_13504_b200 as mg  # noqa: E402

PAPER = {  # MSE/N
    "megopolis": {0.0: 0.2760, 1.0: 0.3769, 2.0: 0.5213, 3.0: 0.6067, 4.0: 0.6508},
    "metropolis": "0.9994-1.0002 for all y",
    "c1:128": {4.0: 15.3599},
    "c2:128": {0.0: 1.7029},
}

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--seq", type=int, default=8)
ap.add_argument("--ns", default="15,20,22")
ap.add_argument("--ys", default="0,1,2,3,4")
ap.add_argument("--algs", default="megopolis,metropolis,c1:128,c2:128")
ap.add_argument("--rng", default="megores")
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()

rows = []
t0 = time.time()
for token in a.algs.split(","):
    name, _, part = token.partition(":")
    pb = int(part) if part else None
    for lg in (int(x) for x in a.ns.split(",")):
        n = 1 << lg
        for y in (float(x) for x in a.ys.split(",")):
            per_seq, bs = [], []
            for s in range(a.seq):
                w = mg.gen_gaussian_weights(mg.GaussianWeightParams(y, n), mg.derive_seed(a.seed, lg, int(1000 * y), s),
                                            "single")
                b = mg.iterations_for(w, 0.01).b
                bs.append(b)
                acc = mg.QualityAccumulator(n)
                # the K runs in one device pass (mgp_quality_runs): identical to K add() calls
                acc.add_runs(name, w, b, [mg.derive_seed(a.seed, 7, lg, s, k) for k in range(a.k)],
                             partition_bytes=pb, rng=a.rng)
                per_seq.append(acc.finalize())
            row = {"algorithm": token, "n": n, "y": y, "b_mean": float(np.mean(bs)), "k": a.k, "sequences": a.seq,
                   "mse_per_particle": float(np.mean([q.mse_per_particle for q in per_seq])),
                   "variance_per_particle": float(np.mean([q.variance for q in per_seq])) / n,
                   "bias_contribution": float(np.mean([q.bias_contribution for q in per_seq]))}
            rows.append(row)
            print(f"{token:12s} N=2^{lg:<2d} y={y:.0f} B={row['b_mean']:6.1f}  MSE/N={row['mse_per_particle']:.4f}  "
                  f"bias={row['bias_contribution']:.4f}", file=sys.stderr, flush=True)
print(json.dumps({"rng": a.rng, "k": a.k, "sequences": a.seq, "wall_s": round(time.time() - t0, 1), "paper": PAPER,
                  "rows": rows}, indent=1))
