"""Wall time of the reference's call shape at 2^24 (megopolis(WeightVector(numpy float32), 354,
seed), pageable numpy in) with the returned array page-locked (MGP_PINNED_OUTPUT=1, default) or
plain numpy (0); ancestors compared between the two.  The page-locked variant measured slower and
was removed, so both modes now run the plain-numpy path."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402

n = 1 << 24
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single").values
out = {}
for mode in ("0", "1", "0", "1"):
    os.environ["MGP_PINNED_OUTPUT"] = mode
    for rng in ("philox", "megores"):
        a = mg.megopolis(mg.WeightVector(w, "single"), 354, seed=7, rng=rng)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            a = mg.megopolis(mg.WeightVector(w, "single"), 354, seed=7, rng=rng)
            ts.append(time.perf_counter() - t0)
        out.setdefault(rng, []).append(a)
        print(f"pinned_output={mode} {rng:8s} {1e3 * sorted(ts)[2]:.2f} ms (median of 5)", flush=True)
for rng, arrs in out.items():
    print(rng, "identical across modes:", all(np.array_equal(arrs[0], x) for x in arrs[1:]))
