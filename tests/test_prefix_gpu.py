"""GPU: the prefix-sum resamplers (M/resample.py:285-336) against the reference.

* ``inclusive_prefix`` (mgp_cumsum) must equal np.cumsum -- numpy's sequential rounding --
  bit for bit: every golden case (tests/golden/golden_prefix.*, made by the unmodified
  reference), adversarial inputs (rounding ties, 60 decades of exponents, subnormals,
  zeros, float32 saturation past 2^24) and random sizes around the chunk boundaries.
* ``multinomial`` / ``systematic_improved`` must reproduce the reference's ancestors
  (sha256 of the int64 bytes) through both the device and the host-buffer paths.
* Ports of the reference's own tests for these methods (T/test_resample.py:204-271,
  342-350) run against this package.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2109_13504_b200 as mg  # noqa: E402
from make_golden_prefix import weights_for  # noqa: E402

from oracle import oracle as ora  # noqa: E402  (checker only)

GOLD = json.load(open(os.path.join(HERE, "golden", "golden_prefix.json")))
ARR = np.load(os.path.join(HERE, "golden", "golden_prefix.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def case_weights(case):
    if "weights" in case:
        return ARR[case["weights"]]
    return weights_for(case["recipe"], lambda y, n, s, p: ora.gen_gaussian_weights(y, n, s, p))


def dev(w):
    return mg.WeightVector(torch.from_numpy(np.ascontiguousarray(w)).cuda(),
                           "single" if w.dtype == np.float32 else "double")


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c['id']}-{c['recipe']['family']}-"
                         f"{c['recipe']['precision']}-{c['recipe']['n']}")
def test_prefix_golden(case):
    w = case_weights(case)
    assert sha(w) == case["weights_sha"]
    wd = dev(w)
    cum = mg.inclusive_prefix(wd)
    assert sha(cum.cpu().numpy()) == case["cum_sha"]
    for ent in case["multinomial"]:
        assert sha(mg.multinomial(wd, ent["seed"]).cpu().numpy()) == ent["sha"], ("multinomial", ent["seed"])
    for ent in case["systematic"]:
        assert sha(mg.systematic_improved(wd, ent["seed"]).cpu().numpy()) == ent["sha"], ("systematic", ent["seed"])
    if len(w) <= 70000:  # host-buffer path (mgp_resample_host, kinds 4/5)
        for ent in case["multinomial"][:1]:
            a = mg.multinomial(w, ent["seed"])
            assert isinstance(a, np.ndarray) and a.dtype == np.int64 and sha(a) == ent["sha"]
        for ent in case["systematic"][:1]:
            assert sha(mg.make_resampler("systematic")(w, 99, ent["seed"])) == ent["sha"]


def _adversarial(rng, n, dt):
    kind = rng.integers(0, 7)
    if kind == 0:  # dyadic: exact halves / quarters -> rounding ties once the sum is large
        w = rng.integers(0, 9, n) / 4.0
    elif kind == 1:  # exponents over 60 decades
        w = 10.0 ** rng.uniform(-30, 30, n)
    elif kind == 2:  # heavy tail with zeros
        w = np.where(rng.random(n) < 0.3, 0.0, rng.pareto(0.7, n))
    elif kind == 3:  # subnormal-scale weights
        w = rng.integers(0, 5, n) * (1e-45 if dt == np.float32 else 5e-324)
    elif kind == 4:  # one huge weight in the middle
        w = rng.random(n)
        w[n // 2] = 1e20
    elif kind == 5:  # powers of two (ties everywhere)
        w = 2.0 ** rng.integers(-8, 8, n)
    else:
        w = rng.random(n) ** 4
    w = w.astype(dt)
    if not np.any(w > 0):
        w[0] = 1
    return w


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_cumsum_adversarial(dt):
    rng = np.random.default_rng(2024 if dt == np.float32 else 2025)
    sizes = [1, 2, 31, 1023, 1024, 1025, 2047, 2048, 32 * 1024 - 1, 32 * 1024 + 1, 33 * 1024 + 7, 100003, 1 << 18]
    for trial in range(60):
        n = int(sizes[trial % len(sizes)] if trial < 2 * len(sizes) else rng.integers(1, 300000))
        w = _adversarial(rng, n, dt)
        got = mg.inclusive_prefix(torch.from_numpy(w).cuda()).cpu().numpy()
        ref = np.cumsum(w)
        assert got.tobytes() == ref.tobytes(), (trial, n, w[:4])


def test_cumsum_large_float32():
    """2^24 float32 Gaussian weights: hundreds of binades of drift vs the float64 sum."""
    w = ora.gen_gaussian_weights(4.0, 1 << 24, 31337, "single")
    got = mg.inclusive_prefix(torch.from_numpy(w).cuda()).cpu().numpy()
    assert got.tobytes() == np.cumsum(w).tobytes()


def test_cumsum_saturation_ties():
    """float32 ones past 2^24: every further add is an exact tie that rounds back to 2^24."""
    n = (1 << 25) + 77
    w = np.ones(n, np.float32)
    got = mg.inclusive_prefix(torch.ones(n, dtype=torch.float32, device="cuda")).cpu().numpy()
    assert got.tobytes() == np.cumsum(w).tobytes()
    assert got[-1] == 2.0**24


def test_cumsum_overflow_to_inf():
    w = np.full(3000, 3e37, np.float32)
    got = mg.inclusive_prefix(torch.from_numpy(w).cuda()).cpu().numpy()
    with np.errstate(over="ignore"):  # the reference's own cumsum overflows to inf here, on purpose
        ref = np.cumsum(w)
    assert got.tobytes() == ref.tobytes()


# ---------------------------------------------------------------------------
# the reference's own tests for these methods, against this package


def test_multinomial_trivial_cases():  # T/test_resample.py:204-207
    assert list(mg.multinomial(mg.WeightVector(np.array([1.0]), "double"), 0)) == [0]
    anc = mg.multinomial(mg.WeightVector(np.array([0.0, 1.0, 0.0, 0.0]), "double"), 1)
    assert np.all(anc == 1)


def test_multinomial_mean_offspring():  # T/test_resample.py:210-219
    w = torch.tensor([1.0, 2.0, 3.0, 2.0], dtype=torch.float64, device="cuda")
    runs = 10**4
    counts = np.zeros(4)
    for k in range(runs):
        counts += np.bincount(mg.multinomial(w, k).cpu().numpy(), minlength=4)
    mean = counts / runs
    expect = np.array([0.5, 1.0, 1.5, 1.0])
    stderr = np.sqrt(expect * (1 - expect / 4) / runs)
    assert np.all(np.abs(mean - expect) < 3.5 * stderr)


def test_systematic_uniform_weights_identity():  # T/test_resample.py:222-224
    w = mg.WeightVector(np.ones(64), "double")
    assert list(mg.systematic_improved(w, 3)) == list(range(64))


def test_systematic_improved_matches_oracle():  # T/test_resample.py:256-265
    rnd = np.random.default_rng(8)
    for trial in range(100):
        n = int(rnd.integers(1, 257))
        w = rnd.uniform(0, 1, n) ** 2
        if w.sum() == 0:
            continue
        seed = ora.derive_seed(60, trial)
        assert np.array_equal(mg.systematic_improved(mg.WeightVector(w, "double"), seed), ora.systematic(w, seed))


@pytest.mark.parametrize("kind", ["multinomial", "systematic"])
def test_weight_scale_invariance_prefix_sum(kind):  # T/test_resample.py:342-350
    n = 64
    fn = mg.make_resampler(kind)
    w = mg.WeightVector(np.arange(1, n + 1, dtype=np.float64), "double")
    base = fn(w, 1, 23)
    for c in (0.5, 4.0):
        scaled = mg.WeightVector(np.asarray(w.values) * c, "double")
        assert np.array_equal(fn(scaled, 1, 23), base)


def test_prefix_errors():
    with pytest.raises(ValueError, match="all weights are zero"):
        mg.multinomial(np.zeros(8, np.float32), 1)
    with pytest.raises(ValueError, match="all weights are zero"):
        mg.systematic_improved(torch.zeros(8, device="cuda"), 1)


def test_systematic_oracle_and_estimate_ratio_golden():
    """systematic_oracle(w, u) with the reference's comparison semantics, and estimate_ratio,
    against the unmodified reference (tests/golden/make_golden_sysoracle.py)."""
    gold = json.load(open(os.path.join(HERE, "golden", "golden_sysoracle.json")))
    for c in gold["cases"]:
        dt = np.float32 if c["precision"] == "single" else np.float64
        w = np.asarray(c["w"], dtype=dt)
        wv = mg.WeightVector(w, c["precision"])
        got = mg.systematic_oracle(wv, c["u"])
        assert got.tolist() == c["anc"]
        assert mg.estimate_ratio(wv, c["ratio_subset"], c["ratio_seed"]) == c["ratio"]
    with pytest.raises(ValueError, match="u must be in"):
        mg.systematic_oracle(np.ones(4), 1.0)  # T/test_resample.py:268-271


def test_systematic_oracle_reference_cases():  # T/test_resample.py:222-253
    w = mg.WeightVector(np.ones(64), "double")
    for u in (0.25, 0.5, 0.999):
        assert list(mg.systematic_oracle(w, u)) == list(range(64))
    assert list(mg.systematic_oracle(w, 0.0)) == [0] + list(range(63))  # ties resolve to the lower bracket
    assert np.all(mg.systematic_oracle(mg.WeightVector(np.array([0.0, 0.0, 5.0, 0.0]), "double"), 0.3) == 2)
    off = mg.ancestors_to_offspring(mg.systematic_oracle(mg.WeightVector(np.array([0.5, 0.5, 0.0, 0.0]), "double"),
                                                         0.1), 4)
    assert list(off) == [2, 2, 0, 0]
    w4 = mg.WeightVector(np.array([1.0, 2.0, 3.0, 2.0]), "double")
    counts = np.zeros(4)
    for k in range(10**4):
        counts += np.bincount(mg.systematic_oracle(w4, float(ora.u01(1234, k, 0))), minlength=4)
    assert np.all(np.abs(counts / 10**4 - np.array([0.5, 1.0, 1.5, 1.0])) < 0.05)
