"""ancestors_to_offspring (M/resample.py:361-368) at the sizes that take the bucketed
shared-memory histogram (n >= 2^20): against np.bincount and against the int32 global-atomic
histogram of round 1 (mgp_debug_offspring_mode), on uniform, heavy-tailed (Megopolis at y = 4),
one-hot and ragged inputs, n_anc != n, and out-of-range ancestors."""

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


def both_modes(mg, a, n):
    from paper_2109_13504_b200 import _lib

    out = []
    for mode in (0, 1):
        _lib.check(_lib.lib().mgp_debug_offspring_mode(mode))
        try:
            out.append(mg.ancestors_to_offspring(a, n))
        finally:
            _lib.check(_lib.lib().mgp_debug_offspring_mode(0))
    return out


@pytest.mark.parametrize("n", [1 << 20, (1 << 20) + 77, 3 << 20, 1 << 24])
def test_bucketed_histogram(mg, n):
    rs = np.random.default_rng(n)
    cases = [rs.integers(0, n, n), np.full(n, n - 1), rs.integers(0, 5, n) * (n // 5)]
    w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 3, "single", device="cuda")
    cases.append(mg.megopolis(w, 60, seed=1, rng="philox", strict=False).cpu().numpy())
    for a in cases:
        want = np.bincount(a, minlength=n)
        got, got_atomic = both_modes(mg, torch.from_numpy(a).cuda(), n)
        assert np.array_equal(got.cpu().numpy(), want)
        assert np.array_equal(got_atomic.cpu().numpy(), want)


def test_ragged_and_errors(mg):
    rs = np.random.default_rng(1)
    n = (1 << 21) + 5
    a = rs.integers(0, n, n // 3)  # fewer ancestors than bins
    assert np.array_equal(mg.ancestors_to_offspring(a, n), np.bincount(a, minlength=n))
    a = rs.integers(0, 1 << 20, 3 << 20)  # more ancestors than bins
    assert np.array_equal(mg.ancestors_to_offspring(a, 1 << 20), np.bincount(a, minlength=1 << 20))
    bad = rs.integers(0, 1 << 20, 1 << 20)
    bad[12345] = 1 << 20
    with pytest.raises(ValueError):
        mg.ancestors_to_offspring(torch.from_numpy(bad).cuda(), 1 << 20)
    bad[12345] = -3
    with pytest.raises(ValueError):
        mg.ancestors_to_offspring(bad, 1 << 20)
