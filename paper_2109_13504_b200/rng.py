"""Host-side seed helpers and lane constants of the reference stream (M/rng.py).

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
