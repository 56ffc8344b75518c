"""The float32 bracket of the megores stream (k_megopolis_megores_f32 and the Metropolis-C1/C2
bracket path, mgp_kernels.cuh) where its accept bound is tight: weights that are small integer
multiples of the smallest subnormal 2^-149.  There hi = lo + 2^-149 and the partner weight equals
hi on a large share of the rounds; the bound hi >= u * wk holds only up to one spacing, so the
accept test is strict and those rounds go to the exact float64 re-run.  Ancestors against the CPU
oracle (the reference's float64 rule, M/resample.py:118-122), and the re-run must have fired."""

import ctypes

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


def subnormal_weights(n, seed):
    rs = np.random.default_rng(seed)
    w = rs.integers(1, 17, n).astype(np.float32) * np.float32(2.0 ** -149)
    assert (w > 0).all() and (w < np.float32(2.0 ** -126)).all()
    return w


def fallbacks():
    from paper_2109_13504_b200 import _lib

    c = ctypes.c_int64(0)
    _lib.check(_lib.lib().mgp_debug_megores_fallbacks(ctypes.byref(c), 1))
    return c.value


@pytest.mark.parametrize("n", [1 << 16, 1 << 20])
def test_megopolis_subnormal_bracket(mg, n):
    from oracle import oracle as ora

    w = subnormal_weights(n, n)
    fallbacks()
    got = mg.megopolis(mg.WeightVector(torch.from_numpy(w).cuda(), "single"), 48, seed=11)
    torch.cuda.synchronize()
    assert fallbacks() > 0
    assert np.array_equal(got.cpu().numpy(), ora.megopolis(w, 48, seed=11))


@pytest.mark.parametrize("kind", ["c1", "c2"])
def test_c12_subnormal_bracket(mg, kind):
    from oracle import oracle as ora

    n = 1 << 18
    w = subnormal_weights(n, 7)
    fn = mg.metropolis_c1 if kind == "c1" else mg.metropolis_c2
    ofn = ora.metropolis_c1 if kind == "c1" else ora.metropolis_c2
    fallbacks()
    got = fn(mg.WeightVector(torch.from_numpy(w).cuda(), "single"), 48, mg.PartitionConfig(128), seed=5)
    torch.cuda.synchronize()
    assert fallbacks() > 0
    assert np.array_equal(got.cpu().numpy(), ofn(w, 48, 128, seed=5))


def adversarial_pair(u):
    """Subnormal state / partner weights (k, m multiples of 2^-149) for which the bracket's accept
    bound is exactly the partner weight while the reference rejects: with u23 = floor(u 2^23) 2^-23,
    lo = floor(u23 k) and hi = lo + 1 spacing; m = hi and u k > m, so fl64(u wk) > wj."""
    h53 = int(u * 2.0 ** 53)
    assert h53 / 2.0 ** 53 == u
    top = h53 >> 30  # u23 * 2^23
    for k in range(1 << 21, 1 << 22):
        m = (top * k >> 23) + 1
        if h53 * k > m << 53:  # u k > m exactly
            wk, wj = k * 2.0 ** -149, m * 2.0 ** -149
            if u * wk > wj:  # the reference's float64 product rejects
                return np.float32(wk), np.float32(wj)
    raise AssertionError("no adversarial pair")


@pytest.mark.parametrize("kind", ["megopolis", "c1", "c2"])
def test_bracket_accept_bound_is_strict(mg, kind):
    """One round (B = 1) of particle i against its partner j with the adversarial pair: the reference
    keeps i; an accept test of hi <= wj would move it to j."""
    from oracle import oracle as ora

    n, i, seed = 1 << 16, 4101, 23
    def run(w):
        wv = mg.WeightVector(torch.from_numpy(w).cuda(), "single")
        if kind == "megopolis":
            return mg.megopolis(wv, 1, seed=seed).cpu().numpy()
        fn = mg.metropolis_c1 if kind == "c1" else mg.metropolis_c2
        return fn(wv, 1, mg.PartitionConfig(128), seed=seed).cpu().numpy()

    def oracle_run(w):
        if kind == "megopolis":
            return ora.megopolis(w, 1, seed=seed)
        fn = ora.metropolis_c1 if kind == "c1" else ora.metropolis_c2
        return fn(w, 1, 128, seed=seed)

    w = np.ones(n, dtype=np.float32)
    w[i] = np.float32(2.0 ** -140)  # every partner outweighs it: the first round accepts j
    j = int(run(w)[i])
    assert j != i
    wk, wj = adversarial_pair(ora.u01(seed, i, 0))  # u of round 0 (counter 0 of lane i)
    w[i], w[j] = wk, wj
    fallbacks()
    got = run(w)
    want = oracle_run(w)
    assert want[i] == i
    assert got[i] == i and np.array_equal(got, want)
    assert fallbacks() > 0


@pytest.mark.parametrize("kind", ["megopolis", "c1", "c2"])
def test_bracket_multi_launch(mg, kind):
    """B > 1024: the bracket paths across several launches (the carried ancestor state, the round
    counters of each launch's exact re-run), on weights with a tight bracket (subnormal multiples)
    and on ordinary ones, device and host entries."""
    from oracle import oracle as ora

    n = 1 << 12
    for w in (subnormal_weights(n, 5), (np.random.default_rng(6).random(n) ** 4 + 1e-3).astype(np.float32)):
        for b in (1025, 2049):
            if kind == "megopolis":
                want = ora.megopolis(w, b, seed=b)
                got_h = mg.megopolis(w, b, seed=b)
                got_d = mg.megopolis(mg.WeightVector(torch.from_numpy(w).cuda(), "single"), b, seed=b)
            else:
                fn = mg.metropolis_c1 if kind == "c1" else mg.metropolis_c2
                ofn = ora.metropolis_c1 if kind == "c1" else ora.metropolis_c2
                want = ofn(w, b, 128, seed=b)
                got_h = fn(w, b, mg.PartitionConfig(128), seed=b)
                got_d = fn(mg.WeightVector(torch.from_numpy(w).cuda(), "single"), b, mg.PartitionConfig(128), seed=b)
            assert np.array_equal(got_h, want), (kind, b, "host")
            assert np.array_equal(got_d.cpu().numpy(), want), (kind, b, "device")
