"""ancestors_to_offspring (M/resample.py:361-368) at the sizes that take the queued
shared-memory histogram (n >= 2^20): against np.bincount, the count-matrix bucketed histogram and
the int32 global-atomic histogram of round 1 (mgp_debug_offspring_mode), on uniform, heavy-tailed
(Megopolis at y = 4), one-hot (every queue but one empty, the full one spilling into the overflow
list), index-skewed and ragged inputs, n_anc != n, unaligned ancestor arrays and out-of-range
ancestors."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def mg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_13504_b200 as m

    return m


def all_modes(mg, a, n):
    from paper_2109_13504_b200 import _lib

    out = []
    for mode in (0, 1, 2):
        _lib.check(_lib.lib().mgp_debug_offspring_mode(mode))
        try:
            out.append(mg.ancestors_to_offspring(a, n))
        finally:
            _lib.check(_lib.lib().mgp_debug_offspring_mode(0))
    return out


@pytest.mark.parametrize("n", [1 << 20, (1 << 20) + 77, 3 << 20, 1 << 24])
def test_bucketed_histogram(mg, n):
    rs = np.random.default_rng(n)
    cases = [rs.integers(0, n, n), np.full(n, n - 1), rs.integers(0, 5, n) * (n // 5),
             np.sort(rs.integers(0, n, n)) ** 2 // n,  # index-skewed: the low queues overflow
             (n - 1 - np.sqrt(rs.random(n)) * (n - 1)).astype(np.int64)]  # density grows toward 0
    w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 3, "single", device="cuda")
    cases.append(mg.megopolis(w, 60, seed=1, rng="philox", strict=False).cpu().numpy())
    for a in cases:
        want = np.bincount(a, minlength=n)
        for got in all_modes(mg, torch.from_numpy(a).cuda(), n):
            assert np.array_equal(got.cpu().numpy(), want)


def test_ragged_and_errors(mg):
    rs = np.random.default_rng(1)
    n = (1 << 21) + 5
    a = rs.integers(0, n, n // 3)  # fewer ancestors than bins
    assert np.array_equal(mg.ancestors_to_offspring(a, n), np.bincount(a, minlength=n))
    a = rs.integers(0, 1 << 20, 3 << 20)  # more ancestors than bins
    assert np.array_equal(mg.ancestors_to_offspring(a, 1 << 20), np.bincount(a, minlength=1 << 20))
    a = torch.from_numpy(rs.integers(0, 1 << 20, (1 << 20) + 1)).cuda()[1:]  # 8-byte aligned only
    assert np.array_equal(mg.ancestors_to_offspring(a, 1 << 20).cpu().numpy(),
                          np.bincount(a.cpu().numpy(), minlength=1 << 20))
    bad = rs.integers(0, 1 << 20, 1 << 20)
    bad[12345] = 1 << 20
    with pytest.raises(ValueError):
        mg.ancestors_to_offspring(torch.from_numpy(bad).cuda(), 1 << 20)
    bad[12345] = -3
    with pytest.raises(ValueError):
        mg.ancestors_to_offspring(bad, 1 << 20)


def test_queued_histogram_many_buckets(mg):
    """n > 2^25: more than 2048 buckets (queue reservations stored in shared memory instead of
    registers) and, at n = 2^27, 8192 buckets with the tile still at 8192 ancestors; skewed inputs
    so some queues overflow."""
    rs = np.random.default_rng(99)
    for n in ((1 << 26) + 12345, 1 << 27):
        a = rs.integers(0, n, n)
        a[: n // 4] = rs.integers(0, 1 << 16, n // 4)  # the first 4 buckets take a quarter: overflow
        got = mg.ancestors_to_offspring(torch.from_numpy(a).cuda(), n)
        assert np.array_equal(got.cpu().numpy(), np.bincount(a, minlength=n))
        del got
        torch.cuda.empty_cache()


def test_flag_reset_by_the_call(mg):
    """mgp_offspring zeroes the caller's out-of-range flag itself (the queued path does it in
    k_offq_zero, ahead of the programmatically launched scatter): a flag left at 1 by an earlier
    call reads 0 after a valid call and 1 after an invalid one."""
    from paper_2109_13504_b200 import _device as D
    from paper_2109_13504_b200 import _lib

    n = 1 << 21
    rs = np.random.default_rng(5)
    a = torch.from_numpy(rs.integers(0, n, n)).cuda()
    counts = torch.empty(n, dtype=torch.int64, device="cuda")
    flag = torch.ones(1, dtype=torch.int32, device="cuda")
    L = _lib.lib()
    _lib.check(L.mgp_offspring(D.ptr(a), n, n, D.ptr(counts), D.ptr(flag), D.stream_ptr()))
    assert int(flag.item()) == 0
    assert np.array_equal(counts.cpu().numpy(), np.bincount(a.cpu().numpy(), minlength=n))
    a[777] = n
    _lib.check(L.mgp_offspring(D.ptr(a), n, n, D.ptr(counts), D.ptr(flag), D.stream_ptr()))
    assert int(flag.item()) == 1
    a[777] = 0
    _lib.check(L.mgp_offspring(D.ptr(a), n, n, D.ptr(counts), D.ptr(flag), D.stream_ptr()))
    assert int(flag.item()) == 0
