"""Pin the CPU oracle (oracle/) against golden vectors from the unmodified reference.

These run without a GPU.  The golden vectors were produced by
tests/golden/make_golden.py calling pkg/src/megores directly.
"""

import hashlib

import numpy as np
import pytest

U64 = 2**64 - 1


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def test_rng_hash_grid(golden, oracle):
    meta, z = golden
    grid, hs = z["rng_grid"], z["rng_hash"]
    got = np.array([oracle.hash_u64(*map(int, g)) for g in grid], dtype=np.uint64)
    assert np.array_equal(got, hs)
    # vectorised numpy twin as well (M/rng.py:73-82)
    assert np.array_equal(oracle.hash_np(0, 0, 0, 0), np.uint64(0x48218226FF3CD4BF))


def test_rng_u01_uint_below(golden, oracle):
    meta, z = golden
    grid = z["rng_grid"][::2]
    u = np.array([oracle.u01(s, l, c) for s, l, c, _ in grid])
    assert np.array_equal(u, z["rng_u01"])  # bit-exact doubles
    ns = z["rng_uint_below_n"]
    got = np.array([[oracle.uint_below(s, l, c, int(n)) for n in ns] for s, l, c, _ in grid])
    assert np.array_equal(got, z["rng_uint_below"])


def test_rng_uint_below_pow2_is_shift(golden, oracle):
    # uint_below(2^k) == h >> (64-k), used by the CUDA fast paths
    for k in (5, 10, 20, 24, 28):
        for lane in range(50):
            h = oracle.hash_u64(99, lane, 3)
            assert oracle.uint_below(99, lane, 3, 2**k) == h >> (64 - k)


def test_derive_seed(golden, oracle):
    meta, _ = golden
    for parts, expect in meta["rng"]["derive_seed"]:
        assert oracle.derive_seed(parts[0], *parts[1:]) == expect


def test_box_muller_numpy(golden, oracle):
    meta, z = golden
    assert np.allclose(oracle.gaussian_np(123, np.arange(257), 0), z["rng_gauss"], rtol=0, atol=1e-14)


def test_offsets(golden, oracle):
    meta, z = golden
    for o in meta["offsets"]:
        got = oracle.megopolis_offsets(o["n"], o["b"], o["seed"])
        assert np.array_equal(got, z[o["name"]]), o


def _run_case(oracle, c, w):
    kind = c["kind"]
    if kind == "megopolis":
        return oracle.megopolis(w, c["b"], c["warp"], c["seed"], c["strict"])
    if kind == "metropolis":
        return oracle.metropolis(w, c["b"], c["seed"])
    fn = oracle.metropolis_c1 if kind == "c1" else oracle.metropolis_c2
    return fn(w, c["b"], c["part"], c["warp"], c["seed"], c["strict"])


def test_all_small_cases_bit_exact(golden, oracle):
    meta, z = golden
    n_full = 0
    for c in meta["cases"]:
        if "w" not in c:
            continue
        w = z[c["w"]]
        anc = _run_case(oracle, c, w)
        assert np.array_equal(anc, z[c["anc"]]), c["tag"] + "/" + c["kind"]
        n_full += 1
    assert n_full > 250


def test_config1_and_big_cases(golden, oracle):
    """Config 1 (N=2^16 y=1) and, when present, the 2^20 / 2^24 cases."""
    meta, z = golden
    w1 = z["config1_w"]
    assert sha(w1) == meta["config1"]["w_sha"]
    mean, mx = oracle.weight_mean_max(w1)
    assert mean == meta["config1"]["mean"] and mx == meta["config1"]["max"]
    assert oracle.compute_iterations(0.01, mean, mx) == meta["config1"]["b"] == 6
    for c in meta["cases"]:
        if c["tag"] != "config1":
            continue
        anc = _run_case(oracle, c, w1)
        assert sha(anc) == c["anc_sha"], c["kind"]
    # the regenerated config-1 weights must equal the reference's bytes on this CPU
    regen = oracle.gen_gaussian_weights(1.0, 2**16, oracle.derive_seed(1, 1), "single")
    assert sha(regen) == meta["config1"]["w_sha"]


@pytest.mark.slow
def test_config2_regenerated(golden, oracle):
    meta, z = golden
    for c in meta["cases"]:
        if not c["tag"].startswith("config2_y") and not c["tag"].startswith("config3_y"):
            continue
        y = float(c["tag"].split("_y")[1])
        w = oracle.gen_gaussian_weights(y, 2**20, oracle.derive_seed(2, 20, int(1000 * y), 0), "single")
        if sha(w) != c["w_sha"]:
            pytest.skip("weight generator not bit-identical on this CPU (libm differences)")
        anc = _run_case(oracle, c, w)
        assert sha(anc) == c["anc_sha"], c["tag"] + c["kind"]


def test_b_rule(golden, oracle):
    meta, z = golden
    for r in meta["b_rule"]:
        assert oracle.compute_iterations(r["eps"], r["mean"], r["max"]) == r["b"]
        if "n" in r:
            w = oracle.gen_gaussian_weights(r["y"], r["n"], oracle.derive_seed(71, r["n"], int(r["y"])),
                                            r["precision"])
            if sha(w) == r["w_sha"]:
                mean, mx = oracle.weight_mean_max(w)
                assert mean == r["mean"] and mx == r["max"]


def mean_input(n, seed=81):
    r = np.random.default_rng([seed, n])
    mant = r.integers(0, 2**23, n, dtype=np.uint32)
    expo = r.integers(127 - 20, 127 + 20, n, dtype=np.uint32)
    return ((expo << np.uint32(23)) | mant).view(np.float32)


def test_pairwise_mean_bits(golden, oracle):
    meta, _ = golden
    for r in meta["means"]:
        a = mean_input(r["n"])
        assert sha(a) == r["a_sha"]
        s = oracle.pairwise_sum(a)
        assert s == r["sum"] and s / r["n"] == r["mean"], r["n"]


def test_quality_and_offspring(golden, oracle):
    meta, z = golden
    for q in meta["quality"]:
        w = z[q["w"]]
        offs = z[q["offspring"]]
        acc = oracle.QualityAccumulator(q["n"])
        for o in offs:
            acc.add(o, w)
        st = acc.finalize()
        for key in ("mse", "variance", "bias_sq", "bias_contribution", "mse_per_particle"):
            assert st[key] == q[key], key
        # offspring of a re-run equal the stored ones
        b = q["b"]
        for k, o in enumerate(offs):
            seed = oracle.derive_seed(92, k)
            anc = oracle.resample(q["kind"], w, b, seed, partition_bytes=q["part"])
            assert np.array_equal(oracle.ancestors_to_offspring(anc, q["n"]), o)


def test_offspring_gather_examples(oracle):
    # T/test_resample.py:278-300
    assert list(oracle.ancestors_to_offspring(np.arange(5))) == [1] * 5
    assert list(oracle.ancestors_to_offspring(np.array([2, 2, 0, 5, 5, 5]))) == [1, 0, 2, 0, 0, 3]
    with pytest.raises(ValueError):
        oracle.ancestors_to_offspring(np.array([0, 7]), 4)
    s = np.array([10.0, 11.0, 12.0, 13.0])
    assert list(oracle.apply_ancestors(s, np.full(4, 3))) == [13.0] * 4
    with pytest.raises(ValueError):
        oracle.apply_ancestors(s, np.arange(3))


def test_precondition_errors(oracle):
    with pytest.raises(ValueError, match="all weights are zero"):
        oracle.metropolis(np.zeros(4), 4, 0)
    with pytest.raises(ValueError):
        oracle.metropolis(np.ones(4), 0, 0)
    with pytest.raises(ValueError):
        oracle.megopolis(np.ones(33), 4)
    with pytest.raises(ValueError):
        oracle.metropolis_c1(np.ones(64), 4, 130)
    with pytest.raises(ValueError):
        oracle.metropolis_c1(np.ones(64), 4, 3 * 128)


# Philox4x32-10 known-answer vectors (Salmon et al. SC'11, Random123 kat_vectors)
PHILOX_KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox_kat(oracle):
    for ctr, key, expect in PHILOX_KAT:
        assert tuple(int(x) for x in oracle.philox4x32_10(ctr, key)) == expect


def test_philox_stream_properties(oracle):
    w = np.arange(1, 65, dtype=np.float32)
    a = oracle.megopolis(w, 5, seed=3, rng="philox")
    b = oracle.megopolis(w, 5, seed=3, rng="philox")
    assert np.array_equal(a, b) and a.min() >= 0 and a.max() < 64
    # the uniform weights map property holds for the philox stream too
    ones = np.ones(128)
    anc = oracle.megopolis(ones, 6, seed=17, rng="philox")
    last = int(oracle.megopolis_offsets(128, 6, 17, rng="philox")[-1])
    expect = [((i - i % 32) + (last - last % 32) + (i + last) % 32) % 128 for i in range(128)]
    assert list(anc) == expect


def test_threads_do_not_change_results(oracle):
    w = oracle.gen_gaussian_weights(3.0, 4096, 5)
    a1 = oracle.megopolis(w, 40, seed=9, threads=1)
    a8 = oracle.megopolis(w, 40, seed=9, threads=8)
    assert np.array_equal(a1, a8)
