"""Property-based tests (hypothesis, as the reference's suite uses: T/test_resample.py:144-151,
T/test_weights.py:89-102, T/test_rng.py:103-112) of the product's host-side code, checked
against the CPU oracle.  No GPU needed."""

import ctypes
import math

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2109_13504_b200 as mg
from paper_2109_13504_b200 import _lib
from paper_2109_13504_b200 import rng as prng

U64 = st.integers(0, 2**64 - 1)


@settings(max_examples=200, deadline=None)
@given(data=st.data())
def test_megopolis_index_bijection_property(data):  # T/test_resample.py:144-151
    warp = data.draw(st.sampled_from([1, 4, 7, 16, 32, 64]))
    blocks = data.draw(st.integers(1, 32))
    n = warp * blocks
    o = data.draw(st.integers(0, n - 1))
    start = data.draw(st.integers(0, blocks - 1)) * warp
    W = mg.WarpConfig(warp_size=warp)
    outs = {mg.megopolis_index(i, o, W, n) for i in range(start, start + warp)}
    assert len(outs) == warp and min(outs) % warp == 0


@settings(max_examples=200, deadline=None)
@given(eps=st.floats(1e-6, 1.0, exclude_max=True), eps2=st.floats(1e-6, 1.0, exclude_max=True),
       ratio=st.floats(1e-6, 1.0), ratio2=st.floats(1e-6, 1.0))
def test_compute_iterations_monotone_and_abi_equal(oracle, eps, eps2, ratio, ratio2):  # T/test_weights.py:89-102
    lo_e, hi_e = sorted((eps, eps2))
    lo_r, hi_r = sorted((ratio, ratio2))
    assert mg.compute_iterations(lo_e, hi_r, 1.0).b >= mg.compute_iterations(hi_e, hi_r, 1.0).b
    assert mg.compute_iterations(lo_e, lo_r, 1.0).b >= mg.compute_iterations(lo_e, hi_r, 1.0).b
    b = ctypes.c_int32()
    for e, r in ((lo_e, lo_r), (hi_e, hi_r)):
        rc = _lib.lib().mgp_compute_iterations(e, r, 1.0, ctypes.byref(b))
        expect = oracle.compute_iterations(e, r, 1.0)
        if expect < 2**31 - 1:
            assert rc == 0 and b.value == expect == mg.compute_iterations(e, r, 1.0).b


@settings(max_examples=100, deadline=None)
@given(seed=U64, parts=st.lists(U64, max_size=5))
def test_derive_seed_matches_oracle(oracle, seed, parts):  # M/rng.py:180-191
    assert prng.derive_seed(seed, *parts) == oracle.derive_seed(seed, *parts)


@settings(max_examples=100, deadline=None)
@given(seed=U64, n=st.integers(1, 2**31 - 1), b=st.integers(0, 700), philox=st.booleans())
def test_offsets_host_matches_oracle(oracle, seed, n, b, philox):  # M/resample.py:263-265
    rng = "philox" if philox else "megores"
    got = mg.megopolis_offsets(n, b, seed, rng=rng)
    assert np.array_equal(got, oracle.megopolis_offsets(n, b, seed, rng=rng))
    assert got.size == 0 or (got.min() >= 0 and got.max() < n)


@settings(max_examples=50, deadline=None)
@given(seed=U64, lanes=st.lists(st.integers(0, 2**40), min_size=1, max_size=20))
def test_host_gaussian_matches_oracle(oracle, seed, lanes):  # M/rng.py:152-161
    a = prng.gaussian_at(seed, np.array(lanes), 0)
    b = oracle.gaussian_np(seed, np.array(lanes, dtype=np.uint64), 0)
    assert np.array_equal(a, b)


@settings(max_examples=100, deadline=None)
@given(n=st.integers(1, 10**6), warp=st.integers(1, 64), strict=st.booleans(), b=st.integers(-2, 5))
def test_abi_argument_validation_mirrors_reference(n, warp, strict, b):
    """Host-side validation (no device work): the C ABI rejects exactly what the reference's
    wrappers reject (M/resample.py:103-108, 204-205), with the same message."""
    null = ctypes.c_void_p(0)
    rc = _lib.lib().mgp_megopolis(null, 0, n, b, 0, warp, int(strict), 0, 0, null, null)
    msg = _lib.lib().mgp_last_error().decode()
    if b < 1:
        assert rc == _lib.MGP_EINVAL and msg == f"B must be >= 1, got {b}"
    elif strict and n % warp:
        assert rc == _lib.MGP_EINVAL and msg == (f"megopolis requires N ({n}) to be a multiple of the warp size "
                                                 f"({warp}) in strict mode")
    else:
        assert rc == _lib.MGP_EINVAL and msg == "null pointer"


def test_pw_depth_tree_covers_all(oracle):
    """The numpy pairwise tree is split into a complete top tree of <= 4096-element chunks:
    check the chunk spans tile [0, n) for awkward n (host restatement of pw_chunk_span)."""
    def depth(n):
        sizes, d = {n}, 0
        while max(sizes) > 4096:
            nxt = set()
            for s in sizes:
                n2 = s // 2 - (s // 2) % 8
                nxt |= {n2, s - n2}
            sizes, d = nxt, d + 1
        return d

    def span(n, d, c):
        lo, ln = 0, n
        for k in range(d - 1, -1, -1):
            n2 = ln // 2 - (ln // 2) % 8
            if (c >> k) & 1:
                lo, ln = lo + n2, ln - n2
            else:
                ln = n2
        return lo, ln

    for n in (1, 4096, 4097, 65537, 100003, 2**20 + 13, 3 * 2**21 + 5):
        d = depth(n)
        pos = 0
        for c in range(1 << d):
            lo, ln = span(n, d, c)
            assert lo == pos and 0 < ln <= 4096
            pos += ln
        assert pos == n
        assert math.isfinite(oracle.pairwise_sum(np.ones(n)))


def test_host_weight_validation_matches_numpy():
    """mgp_check_host_weights (WeightVector's host validation, M/weights.py:53-59) against the
    reference's numpy scans on arrays seeded with non-finite, negative, -0.0 and zero values."""
    from paper_2109_13504_b200 import _lib

    rs = np.random.default_rng(8)
    specials = [np.inf, -np.inf, np.nan, -1e-30, -0.0, 0.0, 1e-45, -5.0]
    for dt in (np.float32, np.float64):
        for n in (1, 7, (1 << 18) + 3, 1 << 20):
            for k in range(6):
                x = rs.random(n).astype(dt)
                for _ in range(k):
                    x[rs.integers(0, n)] = rs.choice(specials)
                counts = np.zeros(4, dtype=np.int64)
                _lib.check(_lib.lib().mgp_check_host_weights(x.ctypes.data, 0 if dt == np.float32 else 1, n,
                                                             counts.ctypes.data))
                fin = np.isfinite(x)
                assert counts[0] == int((~fin).sum())
                assert counts[1] == int((x[fin] < 0).sum())
                assert counts[2] == int((x == 0).sum())
                assert counts.sum() == n
