"""The reference's own resampler tests and quality acceptance criteria, run against
the B200 implementation through its public API.

Mirrors pkg/tests/test_resample.py (T/test_resample.py) and the acceptance criteria of
pkg/tests/test_acceptance.py (criteria 1-12) with the same fixtures (T/conftest.py:15-44),
thresholds and seeds.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def m():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_13504_b200 as mg

    return mg


def gaussian_w(m, y, n, seed, precision="double"):
    from oracle import oracle  # reference-equivalent host generator (bit-identical here)

    return m.WeightVector(oracle.gen_gaussian_weights(y, n, seed, precision), precision)


# --------------------------------------------------------------------------- metropolis
def test_metropolis_single_particle(m):  # T/test_resample.py:21-23
    assert list(m.metropolis(m.WeightVector(np.array([2.5]), "double"), 5, seed=0)) == [0]


def test_metropolis_zero_weight_never_escapes(m):  # :26-29
    anc = m.metropolis(m.WeightVector(np.array([0.0, 1.0]), "double"), 64, seed=3)
    assert np.all(anc == 1)


def test_metropolis_rejects(m):  # :32-39
    with pytest.raises(ValueError):
        m.metropolis(m.WeightVector(np.zeros(4), "double"), 4, seed=0)
    with pytest.raises(ValueError):
        m.metropolis(m.WeightVector(np.ones(4), "double"), 0, seed=0)


def test_metropolis_uniform_weights_multinomial_uniform(m):  # :42-53
    n, runs = 8, 10**5 // 8
    counts = np.zeros(n)
    w = m.WeightVector(torch.ones(n, dtype=torch.float64, device="cuda"), "double")
    for k in range(runs):
        counts += m.ancestors_to_offspring(m.metropolis(w, 3, seed=k), n).cpu().numpy()
    total = runs * n
    freq = counts / total
    stderr = np.sqrt((1 / n) * (1 - 1 / n) / total)
    assert np.all(np.abs(freq - 1 / n) < 4 * stderr)


def test_one_hot_attraction_monotone_in_b(m):  # :56-68
    n = 64
    w = m.WeightVector(torch.from_numpy(np.eye(1, n, 7)[0]).cuda(), "double")
    fracs = []
    for b in (1, 4, 16, 64, 256):
        hits = 0
        for k in range(50):
            hits += int((m.metropolis(w, b, seed=k) == 7).sum())
        fracs.append(hits / (50 * n))
    assert all(a <= b + 0.02 for a, b in zip(fracs, fracs[1:]))
    assert fracs[-1] > 0.95


# --------------------------------------------------------------------------- c1 / c2
def test_c1_in_range(m):  # :75-84
    w = gaussian_w(m, 1.0, 64, 5)
    anc = m.metropolis_c1(w, 16, m.PartitionConfig(128), seed=3)
    assert anc.min() >= 0 and anc.max() < 64


def test_single_partition_c1_c2_match_metropolis_distribution(m):  # :104-119
    n, runs, b = 64, 3000, 8
    w = m.WeightVector(torch.from_numpy(gaussian_w(m, 1.0, n, 21).values).cuda(), "double")
    part = m.PartitionConfig(n * 4)
    sums = {"metropolis": np.zeros(n), "c1": np.zeros(n), "c2": np.zeros(n)}
    for k in range(runs):
        sums["metropolis"] += m.ancestors_to_offspring(m.metropolis(w, b, seed=k), n).cpu().numpy()
        sums["c1"] += m.ancestors_to_offspring(m.metropolis_c1(w, b, part, seed=k + 7 * runs), n).cpu().numpy()
        sums["c2"] += m.ancestors_to_offspring(m.metropolis_c2(w, b, part, seed=k + 9 * runs), n).cpu().numpy()
    means = {k: v / runs for k, v in sums.items()}
    tol = 6 * 2.5 / np.sqrt(runs)
    assert np.all(np.abs(means["c1"] - means["metropolis"]) < tol)
    assert np.all(np.abs(means["c2"] - means["metropolis"]) < tol)


# --------------------------------------------------------------------------- megopolis
def test_megopolis_uniform_weights_permutation(m):  # :154-162
    n = 1024
    w = m.WeightVector(np.ones(n), "double")
    for b in (1, 7):
        anc = m.megopolis(w, b, seed=5)
        assert sorted(anc) == list(range(n))
        off = m.ancestors_to_offspring(anc, n)
        assert np.all(off == 1)
        assert m.squared_error(off, w) == 0.0


def test_megopolis_uniform_equals_last_offset_map(m):  # :165-171
    n, b = 128, 6
    w = m.WeightVector(np.ones(n), "double")
    anc = m.megopolis(w, b, seed=17)
    last = m.megopolis_offsets(n, b, 17)[-1]
    assert list(anc) == [m.megopolis_index(i, int(last), m.WarpConfig(), n) for i in range(n)]


def test_megopolis_strict_and_permissive(m):  # :174-183
    w = m.WeightVector(np.ones(33), "double")
    with pytest.raises(ValueError):
        m.megopolis(w, 4, seed=0)
    anc = m.megopolis(w, 4, seed=0, strict=False)
    assert anc.min() >= 0 and anc.max() < 33


def test_megopolis_offspring_bound_sharp_form(m):  # :186-197
    rnd = np.random.default_rng(4)
    for trial in range(300):
        n = 32 * int(rnd.integers(1, 9))
        b = int(rnd.integers(1, 17))
        w = gaussian_w(m, float(rnd.uniform(0, 3)), n, m.derive_seed(50, trial))
        anc = m.megopolis(w, b, seed=m.derive_seed(51, trial))
        counts = m.ancestors_to_offspring(anc, n)
        adopters = counts - (anc == np.arange(n))
        assert adopters.max() <= b


# --------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("kind", ["metropolis", "c1", "c2", "megopolis"])
def test_conservation(m, kind):  # :319-326
    n = 128
    fn = m.make_resampler(kind, partition_bytes=128)
    for trial in range(20):
        w = gaussian_w(m, float(trial % 4), n, m.derive_seed(70, trial))
        off = m.ancestors_to_offspring(fn(w, 6, m.derive_seed(71, trial)), n)
        assert off.sum() == n


@pytest.mark.parametrize("kind", ["metropolis", "c1", "c2", "megopolis"])
def test_weight_scale_invariance_metropolis_family(m, kind):  # :329-339
    n = 128
    fn = m.make_resampler(kind, partition_bytes=128)
    w = gaussian_w(m, 1.5, n, 91)
    base = fn(w, 8, 17)
    for c in (0.25, 2.0, 1024.0):
        assert np.array_equal(fn(m.WeightVector(np.asarray(w.values) * c, "double"), 8, 17), base)


# --------------------------------------------------------------------------- acceptance
QUALITY_N, QUALITY_K, QUALITY_SEQ, EPS = 2**14, 32, 4, 0.01
ALGS = (("megopolis", None), ("metropolis", None), ("c1", 128), ("c2", 128))
YS = (0.0, 1.0, 2.0, 3.0, 4.0)
MEGOPOLIS_TARGETS = {0.0: 0.276, 1.0: 0.377, 2.0: 0.521, 3.0: 0.607, 4.0: 0.651}


@pytest.fixture(scope="module")
def quality_grid(m):
    """T/conftest.py:15-44 on the GPU (weights, B rule, K runs, accumulator all on device)."""
    grid, weights = {}, {}
    for yi, y in enumerate(YS):
        for s in range(QUALITY_SEQ):
            w = gaussian_w(m, y, QUALITY_N, m.derive_seed(1001, yi, s), "double")
            wd = m.WeightVector(torch.from_numpy(w.values).cuda(), "double")
            weights[(yi, s)] = (wd, m.iterations_for(wd, EPS).b)
    for ai, (name, part) in enumerate(ALGS):
        fn = m.make_resampler(name, partition_bytes=part)
        for yi, y in enumerate(YS):
            per_seq = []
            for s in range(QUALITY_SEQ):
                w, b = weights[(yi, s)]
                acc = m.QualityAccumulator(QUALITY_N)
                for k in range(QUALITY_K):
                    anc = fn(w, b, m.derive_seed(2002, ai, yi, s, k))
                    acc.add(m.ancestors_to_offspring(anc, QUALITY_N), w)
                per_seq.append(acc.finalize())
            grid[(name, part, y)] = per_seq
    return grid


def gmean(ps, f):
    return float(np.mean([getattr(s, f) for s in ps]))


def gstderr(ps, f):
    v = np.array([getattr(s, f) for s in ps])
    return float(v.std(ddof=1) / np.sqrt(len(v)))


def test_criterion_01_metropolis_normalized_mse(quality_grid):
    vals = [gmean(quality_grid[("metropolis", None, y)], "mse_per_particle") for y in YS]
    assert all(abs(v - 1.0) <= 0.10 for v in vals), vals


def test_criterion_02_megopolis_mse_targets(quality_grid):
    for y in YS:
        meg = gmean(quality_grid[("megopolis", None, y)], "mse_per_particle")
        met = gmean(quality_grid[("metropolis", None, y)], "mse_per_particle")
        assert abs(meg - MEGOPOLIS_TARGETS[y]) <= 0.10 * MEGOPOLIS_TARGETS[y] and meg < met, (y, meg)


def test_criterion_03_c1_degradation(quality_grid):
    c1 = [gmean(quality_grid[("c1", 128, y)], "mse_per_particle") for y in YS]
    c2_y0 = gmean(quality_grid[("c2", 128, 0.0)], "mse_per_particle")
    assert abs(c1[-1] - 15.35) <= 0.15 * 15.35 and all(a < b for a, b in zip(c1, c1[1:]))
    assert abs(c2_y0 - 1.70) <= 0.10 * 1.70


def test_criterion_04_bias_parity(quality_grid):
    for y in YS:
        st = {k: (gmean(quality_grid[(k[0], k[1], y)], "bias_contribution"),
                  gstderr(quality_grid[(k[0], k[1], y)], "bias_contribution")) for k in ALGS}
        meg_m, meg_s = st[("megopolis", None)]
        for other in (("metropolis", None), ("c2", 128)):
            o_m, o_s = st[other]
            assert abs(meg_m - o_m) <= max(2.0 * float(np.hypot(meg_s, o_s)), 0.1 / QUALITY_K)
        if y >= 3.0:
            assert st[("c1", 128)][0] > meg_m


def test_criterion_07_proposition_oracle(m):
    n, heavy, trials = 64, 7, 10**4
    vals = np.ones(n)
    vals[heavy] = 10.0
    w = m.WeightVector(torch.from_numpy(vals).cuda(), "double")
    budget = m.compute_iterations(0.05, float(vals.mean()), float(vals.max()))
    ratio = vals.mean() / vals.max()
    p = 0.0  # proposition_recurrence (M/weights.py:157-172)
    for _ in range(budget.b):
        p = 1.0 / n + p * (1.0 - ratio)
    hits = np.empty(trials)
    for t in range(trials):
        hits[t] = float(int(m.megopolis(w, budget.b, seed=m.derive_seed(700, t))[0]) == heavy)
    emp = hits.mean()
    stderr = hits.std(ddof=1) / np.sqrt(trials)
    assert abs(emp - p) <= 3 * stderr and emp >= vals[heavy] / vals.sum() - 0.05


def test_criterion_08_traffic_model_exactness(m):  # T/test_acceptance.py:205-229
    from paper_2109_13504_b200.warpsim import count_transactions, trace_algorithm, traffic_report

    warp = m.WarpConfig()
    trace = trace_algorithm("megopolis", m.WeightVector(np.ones(2**12), "double"), 8, warp, None, 81)
    grouped = trace.indices.reshape(8, -1, 32)
    rep = traffic_report(trace)  # every (round, warp) group needs exactly 4 segments
    assert rep.per_warp_max == 4 and rep.total_transactions == 4 * 8 * (2**12 // 32)
    worked = (count_transactions(np.arange(32), warp), count_transactions(np.arange(0, 64, 2), warp),
              count_transactions(np.arange(1, 33), warp), count_transactions(grouped[0, 0], warp))
    assert worked == (4, 8, 5, 4)
    w20 = m.WeightVector(np.ones(2**20), "double")
    means = {kind: traffic_report(trace_algorithm(kind, w20, 2, warp, part, 82)).per_iteration_mean
             for kind, part in (("megopolis", None), ("c1", 2048), ("c2", 2048), ("metropolis", None))}
    assert means["megopolis"] < means["c1"] < means["metropolis"]
    assert means["megopolis"] < means["c2"] < means["metropolis"]


def test_criterion_09_megopolis_structural_invariants(m):
    rnd = np.random.default_rng(90)
    for trial in range(1000):
        n = 32 * int(rnd.integers(1, 17))
        y = float(rnd.uniform(0, 4))
        w = gaussian_w(m, y, n, m.derive_seed(900, trial))
        b = m.iterations_for(w, 0.01).b
        off = m.ancestors_to_offspring(m.megopolis(w, b, seed=m.derive_seed(901, trial)), n)
        assert off.sum() == n and off.max() <= b
    for trial in range(100):
        n = 32 * int(rnd.integers(1, 9))
        anc = m.megopolis(m.WeightVector(np.ones(n), "double"), int(rnd.integers(1, 9)), seed=m.derive_seed(902, trial))
        assert sorted(anc) == list(range(n))


def test_criterion_05_unbiased_baselines_and_ordering(m):  # T/test_acceptance.py:84-106
    n, k = 2**12, 64
    w = gaussian_w(m, 1.0, n, m.derive_seed(500), "double")
    wd = np.asarray(w.values)
    b = m.compute_iterations(0.01, float(wd.mean()), float(wd.max())).b
    wdev = m.WeightVector(torch.from_numpy(wd).cuda(), "double")
    expect = n * wd / wd.sum()
    mse, unbiased_ok = {}, True
    for kind in ("multinomial", "systematic", "megopolis"):
        fn = m.make_resampler(kind)
        runs = np.stack([m.ancestors_to_offspring(fn(wdev, b, m.derive_seed(501, i)), n).cpu().numpy()
                         for i in range(k)]).astype(np.float64)
        mse[kind] = m.quality_stats(runs, wdev).mse
        if kind != "megopolis":
            mean, std = runs.mean(axis=0), runs.std(axis=0, ddof=1)
            live = std > 0
            z = (mean[live] - expect[live]) / (std[live] / np.sqrt(k))
            unbiased_ok = unbiased_ok and (np.abs(z) > 3).mean() <= 0.01
            unbiased_ok = unbiased_ok and np.all(np.abs(mean[~live] - expect[~live]) <= 1.0)
    assert unbiased_ok and mse["systematic"] < mse["megopolis"] < mse["multinomial"], mse


def test_criterion_06_prefix_sum_instability(m):  # T/test_acceptance.py:109-176
    ns, k_mse, k_meg, sequences = (2**12, 2**16, 2**20), 8, 32, 2

    def exact_bias_sq(values):  # the kernels' float32 prefix vs the float64 reference
        c = np.asarray(m.inclusive_prefix(values), dtype=np.float64)
        e32 = len(c) * np.diff(np.concatenate(([0.0], c))) / c[-1]
        v64 = np.asarray(values, dtype=np.float64)
        return float(np.sum((e32 - n64(v64)) ** 2))

    def n64(v):
        return len(v) * v / v.sum()

    bc = {}
    for n in ns:
        per = {kind: [] for kind in ("multinomial", "systematic")}
        for s in range(sequences):
            w = gaussian_w(m, 1.0, n, m.derive_seed(600, n, s), "single")
            wdev = m.WeightVector(torch.from_numpy(w.values).cuda(), "single")
            bias_sq = exact_bias_sq(w.values)
            for kind in per:
                fn = m.make_resampler(kind)
                acc = m.QualityAccumulator(n)
                for i in range(k_mse):
                    acc.add(m.ancestors_to_offspring(fn(wdev, 1, m.derive_seed(601, n, s, i)), n), wdev)
                per[kind].append(bias_sq / acc.finalize().mse)
        for kind in per:
            bc[(kind, n)] = float(np.mean(per[kind]))
    for kind in ("multinomial", "systematic"):
        seq = [bc[(kind, n)] for n in ns]
        assert seq[0] < seq[1] < seq[2], (kind, seq)
    fn = m.make_resampler("megopolis")
    meg = {}
    for n in (ns[0], ns[-1]):
        per = []
        for s in range(sequences):
            w = gaussian_w(m, 1.0, n, m.derive_seed(600, n, s), "single")
            wdev = m.WeightVector(torch.from_numpy(w.values).cuda(), "single")
            b = m.iterations_for(wdev, 0.01).b
            acc = m.QualityAccumulator(n)
            for i in range(k_meg):
                acc.add(m.ancestors_to_offspring(fn(wdev, b, m.derive_seed(601, n, s, i)), n), wdev)
            per.append(acc.finalize().bias_contribution)
        meg[n] = float(np.mean(per))
    floor = 1.0 / k_meg
    assert abs(meg[ns[-1]] - meg[ns[0]]) <= 0.1 * floor
    assert all(0.8 * floor <= v <= 1.2 * floor for v in meg.values()), meg


def test_criterion_10_systematic_oracle_equivalence(m):  # T/test_acceptance.py:253-262
    from oracle import oracle  # the sequential stratified restatement (M/resample.py:339-354)

    rnd = np.random.default_rng(100)
    for trial in range(500):
        n = int(rnd.integers(1, 257))
        w = rnd.uniform(0, 1, n) ** 3 + 1e-9
        seed = m.derive_seed(1000, trial)
        assert np.array_equal(m.systematic_improved(m.WeightVector(w, "double"), seed), oracle.systematic(w, seed))


def test_criterion_11_end_to_end_orderings(m):  # T/test_acceptance.py:265-287
    from paper_2109_13504_b200 import pfilter as pf

    trajectories = [pf.generate_trajectory(100, 0.0, m.derive_seed(1100, i)) for i in range(4)]
    cfg = pf.FilterConfig(n_particles=2**16, precision="single")
    rows = pf.run_benchmark(cfg, trajectories, 10, [16, 32, 64],
                            [("megopolis", None), ("c1", 128), ("systematic", None)], m.derive_seed(1101))
    rmse = {(r["algorithm"], r["b"]): r["rmse"] for r in rows}
    meg = [rmse[("megopolis", b)] for b in (16, 32, 64)]
    c1 = [rmse[("c1", b)] for b in (16, 32, 64)]
    sys_r = rmse[("systematic", 0)]
    assert all(a <= c - 0.05 for a, c in zip(meg, c1)), (meg, c1)
    assert abs(meg[2] - sys_r) <= 0.03 * sys_r and meg[2] <= meg[0] + 0.05 and meg[2] <= meg[1] + 0.05, (meg, sys_r)


def test_criterion_12_cli_determinism(m, tmp_path):  # T/test_acceptance.py:290-308 (quality, pf)
    from paper_2109_13504_b200.cli import main

    commands = {
        "quality": ["quality", "--algorithms", "megopolis,c2:128", "--n-grid", "1024", "--params", "0,1",
                    "--k-runs", "4", "--sequences", "2", "--seed", "12"],
        "pf": ["pf", "--algorithms", "megopolis", "--n", "1024", "--b-grid", "4", "--trajectories", "1",
               "--runs", "2", "--t-steps", "5", "--seed", "12"],
    }
    for name, args in commands.items():
        payloads = []
        for rep in range(2):
            out = tmp_path / f"{name}-{rep}.csv"
            assert main(args + ["--out", str(out)]) == 0
            payloads.append(out.read_bytes())
        assert payloads[0] == payloads[1], name

