"""Generate golden vectors from the UNMODIFIED reference package (megores).

Run in the build container only (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Everything written here is produced by calling the reference's public API
(pkg/src/megores/*.py); nothing from this repository is imported, so the
fixtures pin the oracle (oracle/) and the CUDA path against the reference
itself.  Small cases store full weights and ancestors; large cases store the
sha256 of the weight bytes (so a regenerated input can be checked) and of the
ancestor bytes, plus a sample of ancestor values.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

import megores as m
from megores import rng
from megores.resample import comparison_indices, megopolis_offsets

OUT = os.path.dirname(os.path.abspath(__file__))
U64 = 2**64 - 1


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def gaussian(y, n, seed, precision):
    return m.gen_gaussian_weights(m.GaussianWeightParams(y, n), seed, precision)


arrays: dict[str, np.ndarray] = {}
meta: dict = {"cases": [], "rng": {}, "b_rule": [], "means": [], "quality": [], "offsets": []}


def put(name, arr):
    assert name not in arrays, name
    arrays[name] = np.ascontiguousarray(arr)
    return name


# ---------------------------------------------------------------------------
# 1. RNG known-answer vectors (M/rng.py:67-191)

seeds = [0, 1, 7, 99, 2**32 - 1, 2**32, 2**63, U64, 0x0123456789ABCDEF]
lanes = [0, 1, 31, 32, 2**20, 2**31 - 1, 2**61, 2**61 + 5, 2**62, 2**62 + 3, U64]
ctrs = [0, 1, 2, 3, 353, 707, 2**32 + 1, U64]
grid = np.array([(s, l, c, salt) for s in seeds for l in lanes for c in ctrs for salt in (0, 1)],
                dtype=np.uint64)
h = rng._hash_np(0, 0, 0, 0)  # warm
hs = np.array([int(rng._hash_np(int(s), int(l), int(c), int(salt))) for s, l, c, salt in grid],
              dtype=np.uint64)
put("rng_grid", grid)
put("rng_hash", hs)
u = np.array([rng.u01(np.uint64(s), np.uint64(l), np.uint64(c)) for s, l, c, salt in grid[::2]])
put("rng_u01", u)
ns = [1, 2, 7, 32, 1000, 2**16, 2**20 + 1, 3 * 2**20, 2**24, 2**28, 2**31 - 1, 2**40 + 3]
ub = np.array([[rng.uint_below(np.uint64(s), np.uint64(l), np.uint64(c), n) for n in ns]
               for s, l, c, salt in grid[::2]], dtype=np.int64)
put("rng_uint_below", ub)
put("rng_uint_below_n", np.array(ns, dtype=np.int64))
ds_parts = [(2002, 0, 0, 0, 0), (1, 1), (5,), (0,), (U64, 3, 9), (1001, 4, 3), (2002, 3, 4, 3, 31)]
meta["rng"]["derive_seed"] = [[list(p), int(rng.derive_seed(p[0], *p[1:]))] for p in ds_parts]
# Box-Muller gaussians (weights generator input, M/rng.py:152-161)
put("rng_gauss", rng.gaussian_at(123, np.arange(257), 0))

# ---------------------------------------------------------------------------
# 2. Offsets (M/resample.py:263-265)

for n, b, s in [(64, 5, 3), (2**20, 8, 77), (128, 6, 17), (33, 9, 0), (2**24, 354, 7),
                (2**28, 64, U64), (1000, 17, 12345), (1, 4, 5)]:
    off = megopolis_offsets(n, b, s)
    meta["offsets"].append({"n": n, "b": b, "seed": s, "name": put(f"off_{n}_{b}_{s}", off)})

# ---------------------------------------------------------------------------
# 3. Resampler cases (M/resample.py:125-282)

cases = []


def add_case(tag, kind, w, b, seed, warp=32, part=None, strict=True, full=True):
    wv = np.asarray(w.values)
    warpcfg = m.WarpConfig(warp_size=warp)
    t0 = time.time()
    if kind == "metropolis":
        anc = m.metropolis(w, b, seed)
    elif kind == "c1":
        anc = m.metropolis_c1(w, b, m.PartitionConfig(part), warpcfg, seed, strict)
    elif kind == "c2":
        anc = m.metropolis_c2(w, b, m.PartitionConfig(part), warpcfg, seed, strict)
    elif kind == "megopolis":
        anc = m.megopolis(w, b, warpcfg, seed, strict)
    else:
        raise ValueError(kind)
    dt = time.time() - t0
    c = {"tag": tag, "kind": kind, "n": len(wv), "precision": w.precision, "b": b,
         "seed": int(seed), "warp": warp, "part": part, "strict": strict,
         "anc_sha": sha(anc.astype(np.int64)), "w_sha": sha(wv), "seconds": round(dt, 3)}
    name = f"case{len(meta['cases'])}"
    if full:
        c["w"] = put(name + "_w", wv)
        c["anc"] = put(name + "_anc", anc.astype(np.int64))
    else:
        pos = np.unique(np.concatenate([np.arange(64), np.random.default_rng(len(wv)).integers(0, len(wv), 192)]))
        c["sample_pos"] = put(name + "_pos", pos.astype(np.int64))
        c["sample_anc"] = put(name + "_sanc", anc[pos].astype(np.int64))
    meta["cases"].append(c)
    print(f"{tag:40s} {kind:10s} n={len(wv):9d} b={b:4d} {dt:7.2f}s", flush=True)


# 3a. survey Appendix A KAT: w=float32(1..64), N=64, B=5, seed=3, PS=128
w64 = m.WeightVector(np.arange(1, 65, dtype=np.float32), "single")
for kind in ("megopolis", "metropolis", "c1", "c2"):
    add_case("kat_1to64", kind, w64, 5, 3, part=128)

# 3b. small grids over y, precision, seeds, algorithms, partitions, warps
for prec in ("single", "double"):
    for y in (0.0, 1.0, 2.0, 3.0, 4.0):
        for n in (32, 96, 1024, 4096):
            w = gaussian(y, n, rng.derive_seed(11, n, int(10 * y)), prec)
            wd = np.asarray(w.values, dtype=np.float64)
            b = m.compute_iterations(0.01, float(wd.mean()), float(wd.max())).b
            s = rng.derive_seed(12, n, int(10 * y), 1 if prec == "single" else 2)
            add_case(f"grid_{prec}_y{y}", "megopolis", w, b, s)
            add_case(f"grid_{prec}_y{y}", "metropolis", w, b, s)
            if n % 32 == 0 and n >= 32:
                add_case(f"grid_{prec}_y{y}", "c1", w, b, s, part=128)
                add_case(f"grid_{prec}_y{y}", "c2", w, b, s, part=128)

# 3c. partition sweep (config 3 shape, reduced N)
w = gaussian(4.0, 2**14, rng.derive_seed(31, 14), "single")
for ps in (128, 256, 512, 1024, 2048):
    for kind in ("c1", "c2"):
        add_case(f"ps{ps}", kind, w, 37, 99, part=ps)

# 3d. logical warp sizes other than 32 (W is semantic, M/resample.py:59-75)
for warp in (1, 4, 16, 64, 7):
    n = 448  # multiple of 1,4,16,64,7
    w = gaussian(2.0, n, rng.derive_seed(41, warp), "single")
    add_case(f"warp{warp}", "megopolis", w, 11, 5, warp=warp)
    add_case(f"warp{warp}", "c1", w, 11, 5, warp=warp, part=64)
    add_case(f"warp{warp}", "c2", w, 11, 5, warp=warp, part=64)

# 3e. permissive mode (N not a multiple of W; M/resample.py:103-108, T/test_resample.py:180-183)
for n in (33, 100, 1000, 4095):
    w = gaussian(1.0, n, rng.derive_seed(51, n), "single")
    add_case("permissive", "megopolis", w, 9, 6, strict=False)
    add_case("permissive_w7", "megopolis", w, 9, 6, warp=7, strict=False)
    add_case("metropolis_oddn", "metropolis", w, 9, 6)

# 3f. zero weights (zero rule M/resample.py:118-122), subnormals, huge values, one-hot
r = np.random.default_rng(61)
for prec in ("single", "double"):
    base = gaussian(2.0, 512, rng.derive_seed(61, 1), prec).values.astype(np.float64)
    wz = base.copy(); wz[r.random(512) < 0.5] = 0.0
    wsub = base.copy(); wsub[::3] = 1e-42 if prec == "single" else 3e-320
    whuge = base * (1e30 if prec == "single" else 1e300)
    onehot = np.zeros(512); onehot[77] = 1.0
    mostly0 = np.zeros(512); mostly0[[3, 100, 300]] = [1.0, 0.5, 0.25]
    for tag, arr in (("zeros", wz), ("subnormal", wsub), ("huge", whuge), ("onehot", onehot),
                     ("mostly_zero", mostly0), ("ones", np.ones(512))):
        w = m.WeightVector(arr, prec)
        for kind in ("megopolis", "metropolis", "c1", "c2"):
            add_case(f"{tag}_{prec}", kind, w, 13, 2024, part=128)
# two-particle zero-never-escapes (T/test_resample.py:26-29), single particle (21-23)
add_case("zero_escape", "metropolis", m.WeightVector(np.array([0.0, 1.0]), "double"), 64, 3)
add_case("single", "metropolis", m.WeightVector(np.array([2.5]), "double"), 5, 0)
add_case("single_f32", "megopolis", m.WeightVector(np.array([2.5]), "single"), 5, 0, warp=1)

# 3g. extreme seeds
for s in (0, 1, 2**63, U64):
    w = gaussian(3.0, 256, 8, "single")
    add_case(f"seed{s}", "megopolis", w, 21, s)
    add_case(f"seed{s}", "metropolis", w, 21, s)

# 3h. weight-scale invariance inputs (T/test_resample.py:329-339)
w = gaussian(1.5, 128, 91, "double")
for c in (1.0, 0.25, 2.0, 1024.0):
    ws = m.WeightVector(np.asarray(w.values) * c, "double")
    for kind in ("megopolis", "metropolis", "c1", "c2"):
        add_case(f"scale{c}", kind, ws, 8, 17, part=128)

# 3i. config 1: N=2^16, y=1, weights seed derive_seed(1,1), f32, run seed 7
w1 = gaussian(1.0, 2**16, rng.derive_seed(1, 1), "single")
wd1 = np.asarray(w1.values, dtype=np.float64)
b1 = m.compute_iterations(0.01, float(wd1.mean()), float(wd1.max())).b
meta["config1"] = {"b": b1, "mean": float(wd1.mean()), "max": float(wd1.max()), "w_sha": sha(w1.values)}
put("config1_w", np.asarray(w1.values))
for kind in ("megopolis", "metropolis", "c1", "c2"):
    add_case("config1", kind, w1, b1, 7, part=128, full=False)

# 3j. config 2/3/4 shapes at full size: sha + samples only
if "--big" in sys.argv:
    for y in (0.0, 1.0, 2.0, 3.0, 4.0):
        w = gaussian(y, 2**20, rng.derive_seed(2, 20, int(1000 * y), 0), "single")
        wd = np.asarray(w.values, dtype=np.float64)
        b = m.compute_iterations(0.01, float(wd.mean()), float(wd.max())).b
        for kind in ("megopolis", "metropolis"):
            add_case(f"config2_y{y}", kind, w, b, 7, full=False)
        if y in (0.0, 4.0):
            for ps in (128, 2048):
                for kind in ("c1", "c2"):
                    add_case(f"config3_y{y}", kind, w, b, 7, part=ps, full=False)
    w = gaussian(4.0, 2**24, rng.derive_seed(2, 24, 4000, 0), "single")
    wd = np.asarray(w.values, dtype=np.float64)
    b = m.compute_iterations(0.01, float(wd.mean()), float(wd.max())).b
    meta["config4"] = {"b": b, "mean": float(wd.mean()), "max": float(wd.max()), "w_sha": sha(w.values)}
    add_case("config4_y4", "megopolis", w, b, 7, full=False)

# ---------------------------------------------------------------------------
# 4. B rule (M/weights.py:114-131; f64 mean/max as M/bench.py:119-120)

for ratio, eps in [(0.5, 0.01), (math.exp(-4.0) / math.sqrt(2.0), 0.01), (1.0, 0.01), (0.3, 0.5),
                   (1e-6, 1e-6), (0.999999, 0.01), (0.114, 0.05)]:
    meta["b_rule"].append({"eps": eps, "mean": ratio, "max": 1.0,
                           "b": m.compute_iterations(eps, ratio, 1.0).b})
for y in (0.0, 1.0, 2.0, 3.0, 4.0):
    for n in (2**10 + 3, 2**14, 2**16 + 7):
        for prec in ("single", "double"):
            w = gaussian(y, n, rng.derive_seed(71, n, int(y)), prec)
            wd = np.asarray(w.values, dtype=np.float64)
            mean, mx = float(wd.mean()), float(wd.max())
            meta["b_rule"].append({"eps": 0.01, "mean": mean, "max": mx, "n": n, "y": y,
                                   "precision": prec, "w_sha": sha(w.values),
                                   "b": m.compute_iterations(0.01, mean, mx).b})
# pairwise-sum (np.mean) bit pins on awkward sizes.  Inputs are built from raw
# PCG64 integers (platform independent): f32 with random exponent in [2^-20, 2^20).


def mean_input(n, seed=81):
    r = np.random.default_rng([seed, n])
    mant = r.integers(0, 2**23, n, dtype=np.uint32)
    expo = r.integers(127 - 20, 127 + 20, n, dtype=np.uint32)
    return ((expo << np.uint32(23)) | mant).view(np.float32)


for n in (1, 7, 8, 9, 127, 128, 129, 1000, 4097, 65536, 65537, 100003, 2**20 + 13):
    a = mean_input(n)
    meta["means"].append({"n": n, "recipe": "mean_input(n, 81)", "a_sha": sha(a),
                          "mean": float(np.asarray(a, dtype=np.float64).mean()),
                          "sum": float(np.asarray(a, dtype=np.float64).sum())})

# ---------------------------------------------------------------------------
# 5. Offspring + quality statistics (M/resample.py:361-368, M/metrics.py:55-110)

for kind, part in (("megopolis", None), ("metropolis", None), ("c1", 128), ("c2", 128)):
    n = 2048
    w = gaussian(2.0, n, rng.derive_seed(91, 1), "double")
    wd = np.asarray(w.values, dtype=np.float64)
    b = m.compute_iterations(0.01, float(wd.mean()), float(wd.max())).b
    fn = m.make_resampler(kind, partition_bytes=part)
    acc = m.QualityAccumulator(n)
    offs = []
    for k in range(6):
        anc = fn(w, b, rng.derive_seed(92, k))
        o = m.ancestors_to_offspring(anc, n)
        offs.append(o)
        acc.add(o, w)
    st = acc.finalize()
    meta["quality"].append({
        "kind": kind, "part": part, "n": n, "b": b, "w": put(f"q_{kind}_w", wd),
        "offspring": put(f"q_{kind}_off", np.array(offs, dtype=np.int64)),
        "se0": m.squared_error(offs[0], w),
        "mse": st.mse, "variance": st.variance, "bias_sq": st.bias_sq,
        "bias_contribution": st.bias_contribution, "mse_per_particle": st.mse_per_particle})

# comparison_indices replay (T/test_resample.py:353-376) for the trace-fidelity pin
for kind in ("metropolis", "c1", "c2", "megopolis"):
    put(f"trace_{kind}", comparison_indices(kind, 256, 6, 77, m.WarpConfig(), 128))

np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
meta["generator"] = {"numpy": np.__version__, "reference": "pkg/src/megores (unmodified)",
                     "big": "--big" in sys.argv}
with open(os.path.join(OUT, "golden.json"), "w") as f:
    json.dump(meta, f, indent=1, sort_keys=True)
print("wrote", len(arrays), "arrays,", len(meta["cases"]), "cases")
