"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the Megopolis hot path.

Python face of ``oracle/mgp_oracle.c`` (a plain-C restatement of the reference
package ``pkg/src/megores``) plus numpy restatements of the reference's
off-kernel arithmetic (quality statistics, B rule, weight generator).

Allowed importers: ``tests/``, ``__graft_entry__.smoke()`` (as checker) and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg.  The product
package ``paper_2109_13504_b200`` never imports this module.

Pinned against the unmodified reference by ``tests/test_oracle_golden.py``
(golden vectors from ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")

M_LANE = np.uint64(0x9E3779B97F4A7C15)  # M/rng.py:45
M_CTR = np.uint64(0xD1B54A32D192ED03)  # M/rng.py:46
M_SALT = np.uint64(0x8CB92BA72F3D8DD7)  # M/rng.py:47
WARP_LANE_BASE = 1 << 61  # M/rng.py:42
GLOBAL_OFFSET_LANE = 1 << 62  # M/rng.py:43
GAUSSIAN_PEAK = 1.0 / math.sqrt(2.0 * math.pi)  # M/weights.py:37

KINDS = {"metropolis": 0, "c1": 1, "c2": 2, "megopolis": 3}
RNGS = {"megores": 0, "philox": 1}

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
            os.path.join(HERE, "mgp_oracle.c")
        ):
            build()
        L = ctypes.CDLL(LIB_PATH)
        u64, i64, i32, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.mgo_mix.argtypes = [u64]
        L.mgo_mix.restype = u64
        L.mgo_hash_u64.argtypes = [u64, u64, u64, u64]
        L.mgo_hash_u64.restype = u64
        L.mgo_u01.argtypes = [u64, u64, u64]
        L.mgo_u01.restype = ctypes.c_double
        L.mgo_uint_below.argtypes = [u64, u64, u64, i64]
        L.mgo_uint_below.restype = i64
        L.mgo_derive_seed.argtypes = [u64, vp, i32]
        L.mgo_derive_seed.restype = u64
        L.mgo_philox4x32_10.argtypes = [vp, vp, vp]
        L.mgo_philox_word.argtypes = [u64, u64, u64]
        L.mgo_philox_word.restype = ctypes.c_uint32
        L.mgo_offsets.argtypes = [i64, i64, u64, i32, vp]
        L.mgo_resample_range.argtypes = [i32, vp, i32, i64, i64, u64, i64, i64, i32, i64, i64, vp, i32]
        L.mgo_resample_range.restype = i32
        L.mgo_pairwise_sum.argtypes = [vp, i32, i64]
        L.mgo_pairwise_sum.restype = ctypes.c_double
        L.mgo_offspring.argtypes = [vp, i64, i64, vp]
        L.mgo_gather.argtypes = [vp, i64, vp, i64, vp]
        L.mgo_num_threads.restype = i32
        L.mgo_cumsum.argtypes = [vp, i32, i64, vp]
        L.mgo_multinomial.argtypes = [vp, i32, i64, u64, vp]
        L.mgo_systematic.argtypes = [vp, i32, i64, u64, vp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _weights(w) -> tuple[np.ndarray, int]:
    values = np.ascontiguousarray(getattr(w, "values", w))
    if values.dtype == np.float32:
        return values, 0
    if values.dtype == np.float64:
        return values, 1
    raise ValueError(f"weights must be float32 or float64, got {values.dtype}")


# ---------------------------------------------------------------------------
# RNG (M/rng.py)


def hash_u64(seed, lane, counter, salt=0) -> int:
    return int(lib().mgo_hash_u64(int(seed), int(lane), int(counter), int(salt)))


def u01(seed, lane, counter) -> float:
    return float(lib().mgo_u01(int(seed), int(lane), int(counter)))


def uint_below(seed, lane, counter, n) -> int:
    return int(lib().mgo_uint_below(int(seed), int(lane), int(counter), int(n)))


def derive_seed(seed, *parts) -> int:
    arr = np.array([int(p) & (2**64 - 1) for p in parts] or [0], dtype=np.uint64)
    return int(lib().mgo_derive_seed(int(seed) & (2**64 - 1), _ptr(arr), len(parts)))


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().mgo_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def philox_word(seed, lane, t) -> int:
    return int(lib().mgo_philox_word(int(seed), int(lane), int(t)))


def _mix_np(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def hash_np(seed, lane, counter, salt=0):
    """Vectorised twin of M/rng.py:73-82."""
    with np.errstate(over="ignore"):
        base = _mix_np(np.uint64(seed) + M_LANE)
        x = (base + np.asarray(lane, dtype=np.uint64) * M_LANE
             + np.asarray(counter, dtype=np.uint64) * M_CTR
             + np.asarray(salt, dtype=np.uint64) * M_SALT)
        return _mix_np(x)


def gaussian_np(seed, lane, counter):
    """Box-Muller on salts 0/1, M/rng.py:152-161."""
    h1 = hash_np(seed, lane, counter, 0)
    h2 = hash_np(seed, lane, counter, 1)
    u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    u2 = (h2 >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def gen_gaussian_weights(y: float, n: int, seed, precision="single") -> np.ndarray:
    """M/weights.py:100-104 (values only)."""
    x = gaussian_np(seed, np.arange(n), 0)
    w = np.exp(-0.5 * (x - y) ** 2) * GAUSSIAN_PEAK
    return w.astype(np.float32 if precision == "single" else np.float64)


# ---------------------------------------------------------------------------
# Resamplers (M/resample.py:96-282) -- same preconditions and messages


def _check(values, b):
    if not np.any(values > 0):  # M/resample.py:96-100
        raise ValueError("all weights are zero")
    if b < 1:  # M/resample.py:204-205
        raise ValueError(f"B must be >= 1, got {b}")


def _check_warp(n, warp, strict, name):  # M/resample.py:103-108
    if strict and n % warp:
        raise ValueError(f"{name} requires N ({n}) to be a multiple of the warp size ({warp}) in strict mode")


def _n_weights(part_bytes, word_bytes=4):  # M/resample.py:84-87
    if part_bytes < 1 or part_bytes % word_bytes:
        raise ValueError("partition_bytes must be a positive multiple of word_bytes")
    return part_bytes // word_bytes


def resample(kind, w, b, seed=0, warp=32, partition_bytes=None, strict=True, rng="megores",
             threads=0, p0=0, p1=None) -> np.ndarray:
    values, dtype = _weights(w)
    n = len(values)
    _check(values, b)
    n_w = 0
    if kind in ("c1", "c2"):
        _check_warp(n, warp, strict, f"metropolis_{kind}")
        n_w = _n_weights(partition_bytes)
        if n % n_w:
            raise ValueError(f"N={n} is not divisible by the partition width {n_w}")
    elif kind == "megopolis":
        _check_warp(n, warp, strict, "megopolis")
    elif kind != "metropolis":
        raise ValueError(f"unknown resampler {kind!r}")
    p1 = n if p1 is None else p1
    anc = np.zeros(n, dtype=np.int64)
    rc = lib().mgo_resample_range(KINDS[kind], _ptr(values), dtype, n, int(b), int(seed) & (2**64 - 1),
                                  int(warp), n_w, RNGS[rng], int(p0), int(p1), _ptr(anc), int(threads))
    if rc:
        raise MemoryError("oracle allocation failed")
    return anc


def megopolis_offsets(n, b, seed, rng="megores") -> np.ndarray:
    out = np.zeros(max(b, 1), dtype=np.int64)
    lib().mgo_offsets(int(n), int(b), int(seed) & (2**64 - 1), RNGS[rng], _ptr(out))
    return out[:b]


def megopolis(w, b, warp=32, seed=0, strict=True, rng="megores", **kw):
    return resample("megopolis", w, b, seed, warp, None, strict, rng, **kw)


def metropolis(w, b, seed, rng="megores", **kw):
    return resample("metropolis", w, b, seed, rng=rng, **kw)


def metropolis_c1(w, b, partition_bytes, warp=32, seed=0, strict=True, rng="megores", **kw):
    return resample("c1", w, b, seed, warp, partition_bytes, strict, rng, **kw)


def metropolis_c2(w, b, partition_bytes, warp=32, seed=0, strict=True, rng="megores", **kw):
    return resample("c2", w, b, seed, warp, partition_bytes, strict, rng, **kw)


# ---------------------------------------------------------------------------
# B rule (M/weights.py:114-131 fed by f64 mean/max as M/bench.py:119-120)


def pairwise_sum(a) -> float:
    values, dtype = _weights(a)
    return float(lib().mgo_pairwise_sum(_ptr(values), dtype, len(values)))


def weight_mean_max(w) -> tuple[float, float]:
    values, _ = _weights(w)
    return pairwise_sum(values) / len(values), float(np.max(values.astype(np.float64)))


def compute_iterations(epsilon, mean_w, max_w) -> int:
    if not (0.0 < epsilon <= 1.0):
        raise ValueError(f"epsilon must be in (0, 1], got {epsilon}")
    if mean_w <= 0 or max_w <= 0:
        raise ValueError("mean_w and max_w must be positive")
    if mean_w > max_w:
        raise ValueError(f"mean_w ({mean_w}) exceeds max_w ({max_w})")
    ratio = mean_w / max_w
    if ratio >= 1.0 or epsilon == 1.0:
        return 1
    return max(math.ceil(math.log(epsilon) / math.log(1.0 - ratio)), 1)


# ---------------------------------------------------------------------------
# Offspring, gather, quality (M/resample.py:361-377, M/metrics.py:55-110)


def ancestors_to_offspring(anc, n=None) -> np.ndarray:
    a = np.ascontiguousarray(anc, dtype=np.int64)
    n = len(a) if n is None else n
    if a.size and (a.min() < 0 or a.max() >= n):
        raise ValueError("ancestor indices out of range")
    out = np.zeros(n, dtype=np.int64)
    lib().mgo_offspring(_ptr(a), len(a), n, _ptr(out))
    return out


def apply_ancestors(states, anc) -> np.ndarray:
    s = np.ascontiguousarray(states)
    a = np.ascontiguousarray(anc, dtype=np.int64)
    if len(s) != len(a):
        raise ValueError(f"length mismatch: {len(s)} states vs {len(a)} ancestors")
    out = np.empty_like(s)
    row = s.strides[0] if s.ndim else s.itemsize
    lib().mgo_gather(_ptr(s), row, _ptr(a), len(a), _ptr(out))
    return out


def expected_offspring(w) -> np.ndarray:
    values = np.asarray(getattr(w, "values", w), dtype=np.float64)
    total = values.sum()
    if total <= 0:
        raise ValueError("total weight must be positive")
    return len(values) * values / total


class QualityAccumulator:
    """Restatement of M/metrics.py:71-110 (float64 streaming sums)."""

    def __init__(self, n):
        self.n, self.k = n, 0
        self.sum = np.zeros(n)
        self.sum_sq = np.zeros(n)
        self.se_total = 0.0
        self.expected = None

    def add(self, offspring, w):
        o = np.asarray(offspring, dtype=np.float64)
        if self.expected is None:
            self.expected = expected_offspring(w)
        self.k += 1
        self.sum += o
        self.sum_sq += o * o
        self.se_total += float(((o - self.expected) ** 2).sum())

    def finalize(self) -> dict:
        if self.k < 2:
            raise ValueError(f"need at least 2 runs to estimate variance, got {self.k}")
        k = self.k
        mean = self.sum / k
        mse = self.se_total / k
        variance = float((self.sum_sq / k - mean * mean).sum())
        bias_sq = float(((mean - self.expected) ** 2).sum())
        return {"mse": mse, "variance": variance, "bias_sq": bias_sq,
                "bias_contribution": bias_sq / mse if mse > 0 else 0.0,
                "mse_per_particle": mse / self.n}


# ---------------------------------------------------------------------------
# Prefix-sum resamplers (M/resample.py:288-336)


def cumsum(w) -> np.ndarray:
    """np.cumsum in the weights' dtype, sequential left to right (M/resample.py:288-291)."""
    values, dt = _weights(w)
    out = np.empty_like(values)
    lib().mgo_cumsum(_ptr(values), dt, len(values), _ptr(out))
    return out


def multinomial(w, seed) -> np.ndarray:
    """M/resample.py:295-304."""
    values, dt = _weights(w)
    _check(values, 1)
    cum = cumsum(values)
    out = np.empty(len(values), dtype=np.int64)
    lib().mgo_multinomial(_ptr(cum), dt, len(values), int(seed) & (2**64 - 1), _ptr(out))
    return out


def systematic(w, seed) -> np.ndarray:
    """systematic_improved, M/resample.py:307-336."""
    values, dt = _weights(w)
    _check(values, 1)
    cum = cumsum(values)
    out = np.empty(len(values), dtype=np.int64)
    lib().mgo_systematic(_ptr(cum), dt, len(values), int(seed) & (2**64 - 1), _ptr(out))
    return out


def num_threads() -> int:
    return int(lib().mgo_num_threads())
