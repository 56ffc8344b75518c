"""Host-side mirror of the reference stream's API (M/rng.py): seeds, lane constants, draws.

The per-draw hash itself runs on the device (csrc/mgp_device.cuh); callers only
need the seed derivation to build per-run seeds exactly like the reference's
harness (M/bench.py:124, T/conftest.py:40).
"""

from __future__ import annotations

WARP_LANE_BASE = 1 << 61  # M/rng.py:42
GLOBAL_OFFSET_LANE = 1 << 62  # M/rng.py:43
_M_LANE = 0x9E3779B97F4A7C15  # M/rng.py:45
_M_CTR = 0xD1B54A32D192ED03  # M/rng.py:46
_M_SALT = 0x8CB92BA72F3D8DD7  # M/rng.py:47
_MASK = (1 << 64) - 1


def _mix(x: int) -> int:  # M/rng.py:85-89
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK
    return x ^ (x >> 31)


def derive_seed(seed, *parts) -> int:
    """Fold experiment coordinates into a fresh 64-bit seed (M/rng.py:180-191)."""
    h = _mix((int(seed) + _M_LANE) & _MASK)
    for p in parts:
        h = _mix(h ^ (((int(p) & _MASK) * _M_CTR + _M_SALT) & _MASK))
    return h


# ---------------------------------------------------------------------------
# Host (numpy) draws for the small host-side sequences of the filter harness
# (trajectory noise, M/pfilter.py:106-126).  The per-particle draws run on the
# device (csrc/mgp_kernels.cuh gaussian_at_dev).


def _hash_np(seed, lane, counter, salt=0):  # M/rng.py:73-82
    import numpy as np

    m1, m2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)

    def mix(x):
        x = (x ^ (x >> np.uint64(30))) * m1
        x = (x ^ (x >> np.uint64(27))) * m2
        return x ^ (x >> np.uint64(31))

    with np.errstate(over="ignore"):
        base = mix(np.uint64(int(seed) & _MASK) + np.uint64(_M_LANE))
        x = (base + np.asarray(lane, dtype=np.uint64) * np.uint64(_M_LANE)
             + np.asarray(counter, dtype=np.uint64) * np.uint64(_M_CTR)
             + np.asarray(salt, dtype=np.uint64) * np.uint64(_M_SALT))
        return mix(x)


def gaussian_at(seed, lane, counter, mean=0.0, stddev=1.0):  # M/rng.py:152-161
    import numpy as np

    if stddev < 0:
        raise ValueError(f"stddev must be >= 0, got {stddev}")
    h1 = _hash_np(seed, lane, counter, 0)
    h2 = _hash_np(seed, lane, counter, 1)
    u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    u2 = (h2 >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return mean + stddev * z


def uniform01_at(seed, lane, counter):  # M/rng.py:128-131
    import numpy as np

    h = _hash_np(seed, lane, counter)
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform_open01_at(seed, lane, counter):  # M/rng.py:134-137
    import numpy as np

    h = _hash_np(seed, lane, counter)
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def uniform_int_at(seed, lane, counter, n):  # M/rng.py:140-149: floor(u * n), clamped
    import numpy as np

    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    v = (uniform01_at(seed, lane, counter) * n).astype(np.int64)
    return np.minimum(v, n - 1)


# ---------------------------------------------------------------------------
# Scalar API (M/rng.py:59-64, 92-121, 164-177): the same values as the array API and as the
# device's per-draw hash (csrc/mgp_device.cuh).

from dataclasses import dataclass  # noqa: E402


@dataclass(frozen=True)
class StreamKey:  # M/rng.py:59-64: coordinates of a single random draw
    seed: int
    lane: int
    counter: int


def hash_u64(seed, lane, counter, salt=0) -> int:  # M/rng.py:92-102
    base = _mix((int(seed) + _M_LANE) & _MASK)
    return _mix((base + int(lane) * _M_LANE + int(counter) * _M_CTR + int(salt) * _M_SALT) & _MASK)


def u01(seed, lane, counter) -> float:  # M/rng.py:105-108
    return float(hash_u64(seed, lane, counter) >> 11) * (1.0 / 9007199254740992.0)


def uint_below(seed, lane, counter, n) -> int:  # M/rng.py:111-121
    v = int(u01(seed, lane, counter) * float(n))
    return n - 1 if v >= n else v


def uniform01(key: StreamKey) -> float:
    return float(uniform01_at(key.seed, key.lane, key.counter))


def uniform_int(key: StreamKey, n: int) -> int:
    return int(uniform_int_at(key.seed, key.lane, key.counter, n))


def gaussian(key: StreamKey, mean: float = 0.0, stddev: float = 1.0) -> float:
    return float(gaussian_at(key.seed, key.lane, key.counter, mean, stddev))
