"""Golden vectors for the prefix-sum resamplers from the UNMODIFIED reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_prefix.py

Calls only the reference's public API: np.cumsum as used by ``_inclusive_prefix``
(M/resample.py:288-291), ``multinomial`` (:295-304) and ``systematic_improved``
(:307-336), plus ``systematic_oracle`` (:339-354) as a cross-check.  Weights are
either stored (small cases) or regenerated from a recipe the tests rebuild
(``weights_for``, also used by tests/test_prefix_*.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def weights_for(recipe: dict, gaussian=None) -> np.ndarray:
    """Rebuild a case's weights from its recipe (numpy only, except "gaussian")."""
    fam, n, prec, seed = recipe["family"], recipe["n"], recipe["precision"], recipe["seed"]
    dt = np.float32 if prec == "single" else np.float64
    r = np.random.default_rng(seed)
    if fam == "gaussian":
        return gaussian(recipe["y"], n, seed, prec)
    if fam == "ones":
        return np.ones(n, dtype=dt)
    if fam == "uniform2":
        return (r.uniform(0, 1, n) ** 2).astype(dt)
    if fam == "sparse":  # mostly zeros, a few heavy particles
        w = np.zeros(n, dtype=dt)
        idx = r.choice(n, size=max(1, n // 50), replace=False)
        w[idx] = r.uniform(0.5, 2.0, len(idx)).astype(dt)
        return w
    if fam == "wide":  # exponents spread over 60 decades
        return (10.0 ** r.uniform(-30, 30, n)).astype(dt)
    if fam == "tiny":  # subnormal-heavy float32 / tiny float64
        base = np.float32(1e-44) if dt == np.float32 else 1e-310
        return (r.integers(0, 50, n) * base).astype(dt)
    if fam == "dyadic":  # exactly representable halves/quarters: rounding ties in the scan
        return (r.integers(1, 8, n) / 4.0).astype(dt)
    raise ValueError(fam)


def main():
    import megores as m
    from megores import rng
    from megores.resample import systematic_oracle

    def gaussian(y, n, seed, prec):
        return np.asarray(m.gen_gaussian_weights(m.GaussianWeightParams(y, n), seed, prec).values)

    cases = []
    arrays = {}
    recipes = []
    for prec in ("single", "double"):
        for y in (0.0, 1.0, 4.0):
            for n in (1, 2, 3, 64, 1000, 4097, 65536, 1 << 20):
                recipes.append({"family": "gaussian", "y": y, "n": n, "precision": prec,
                                "seed": int(rng.derive_seed(700, n, int(y * 10), prec == "single"))})
        for fam, n in (("ones", 64), ("ones", 5000), ("uniform2", 256), ("uniform2", 100000), ("sparse", 4096),
                       ("sparse", 1 << 18), ("wide", 3000), ("wide", 1 << 18), ("tiny", 2048), ("dyadic", 70000),
                       ("dyadic", 1 << 20)):
            recipes.append({"family": fam, "n": n, "precision": prec, "seed": 41 + n})
    # float32 scan past 2^24: every further add of 1.0 is a rounding tie (saturates at 2^24)
    recipes.append({"family": "ones", "n": (1 << 24) + 4096, "precision": "single", "seed": 0})
    recipes.append({"family": "gaussian", "y": 1.0, "n": 1 << 22, "precision": "single",
                    "seed": int(rng.derive_seed(701))})

    for ci, rec in enumerate(recipes):
        w = weights_for(rec, gaussian)
        n = len(w)
        if not np.any(w > 0):
            continue
        wv = m.WeightVector(w, rec["precision"])
        cum = np.cumsum(np.asarray(wv.values))  # _inclusive_prefix (M/resample.py:288-291)
        seeds = [0, 7, int(rng.derive_seed(702, ci))]
        case = {"id": ci, "recipe": rec, "weights_sha": sha(w), "cum_sha": sha(cum),
                "cum_last": float(cum[-1]), "multinomial": [], "systematic": []}
        small = n <= 4097
        if small:
            case["weights"] = f"w{ci}"
            arrays[f"w{ci}"] = w
            case["cum"] = f"c{ci}"
            arrays[f"c{ci}"] = cum
        else:
            pick = np.unique(np.linspace(0, n - 1, 97).astype(np.int64))
            case["cum_sample_idx"] = pick.tolist()
            case["cum_sample"] = [float(v) for v in cum[pick]]
        for s in seeds:
            a = m.multinomial(wv, s)
            ent = {"seed": s, "sha": sha(a)}
            if small:
                ent["anc"] = f"m{ci}_{s}"
                arrays[ent["anc"]] = a
            else:
                ent["first"] = a[:16].tolist()
            case["multinomial"].append(ent)
            if n <= (1 << 20) or rec["family"] == "ones" or rec.get("y", 9) <= 1.0:
                a = m.systematic_improved(wv, s)
                if n <= 4097 and rec["precision"] == "double":
                    # (for "single" the pure-Python oracle compares float32 cum against a weak
                    # Python-float target in float32 under NumPy 2 promotion, while the numba
                    # kernel compares in float64 -- they differ at a few particles)
                    u0 = float(rng.uniform01_at(np.uint64(s), rng.GLOBAL_OFFSET_LANE, 0))
                    assert np.array_equal(a, systematic_oracle(wv, u0))
                ent = {"seed": s, "sha": sha(a)}
                if small:
                    ent["anc"] = f"s{ci}_{s}"
                    arrays[ent["anc"]] = a
                else:
                    ent["first"] = a[:16].tolist()
                case["systematic"].append(ent)
        cases.append(case)
        print(ci, rec["family"], rec["precision"], n, flush=True)
    np.savez_compressed(os.path.join(OUT, "golden_prefix.npz"), **arrays)
    with open(os.path.join(OUT, "golden_prefix.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_prefix.py (unmodified reference megores)",
                   "cases": cases}, f, indent=0)


if __name__ == "__main__":
    sys.exit(main())
