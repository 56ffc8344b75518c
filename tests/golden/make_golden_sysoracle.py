"""Golden vectors of the reference's ``systematic_oracle(w, u)`` (M/resample.py:339-354) and
``estimate_ratio`` (M/weights.py:134-154) from the UNMODIFIED reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_sysoracle.py
"""

import json
import os

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    import megores as m

    rnd = np.random.default_rng(339)
    cases = []
    for trial in range(40):
        n = int(rnd.integers(1, 3000))
        prec = "single" if trial % 2 == 0 else "double"
        w = rnd.uniform(0, 1, n) ** int(rnd.integers(1, 5))
        if trial % 5 == 0:
            w[rnd.random(n) < 0.3] = 0.0
        if not np.any(w > 0):
            w[0] = 1.0
        wv = m.WeightVector(w, prec)
        u = float(rnd.uniform(0, 1))
        anc = m.systematic_oracle(wv, u)
        seed = int(rnd.integers(0, 2**63))
        sub = int(rnd.integers(1, n + 1))
        cases.append({"precision": prec, "w": np.asarray(wv.values).tolist(), "u": u, "anc": anc.tolist(),
                      "ratio_subset": sub, "ratio_seed": seed, "ratio": m.estimate_ratio(wv, sub, seed)})
    with open(os.path.join(OUT, "golden_sysoracle.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_sysoracle.py (unmodified reference megores)",
                   "cases": cases}, f)


if __name__ == "__main__":
    main()
