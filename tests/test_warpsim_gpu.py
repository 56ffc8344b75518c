"""GPU: the warp transaction model (M/warpsim.py) and the comparison-index replay
(M/resample.py:384-428) on the device, against the unmodified reference.

* golden traces (tests/golden/golden_traffic.json, made by make_golden_traffic.py from the
  reference): sha256 of every (B, N) index matrix and the TrafficReport fields, all four
  algorithms, W in {7, 8, 16, 32}, partitions 64-2048 B, the full 64-bit seed range;
* the reference's own tests (T/test_warpsim.py) ported to this package;
* the replayed indices are the partners the resampling kernels actually use: a Megopolis run
  with uniform weights accepts every proposal, so its ancestors are the last round's indices.
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
sys.path.insert(0, os.path.dirname(HERE))

import paper_2109_13504_b200 as m  # noqa: E402
from paper_2109_13504_b200.warpsim import (  # noqa: E402
    count_transactions,
    rng_draws_per_iteration,
    trace_algorithm,
    traffic_report,
)

WARP = m.WarpConfig()
GOLD = json.load(open(os.path.join(HERE, "golden", "golden_traffic.json")))


def uniform_w(n):
    return m.WeightVector(np.ones(n), "double")


@pytest.mark.parametrize("c", GOLD["cases"], ids=lambda c: f"{c['kind']}-{c['n']}-W{c['warp']}-{c['partition_bytes']}")
def test_comparison_indices_golden(c):
    warp = m.WarpConfig(c["warp"])
    idx = m.comparison_indices(c["kind"], c["n"], c["b"], c["seed"], warp, c["partition_bytes"])
    assert isinstance(idx, np.ndarray) and idx.dtype == np.int64 and idx.shape == (c["b"], c["n"])
    assert idx[0, :8].tolist() == c["first"]
    assert hashlib.sha256(idx.tobytes()).hexdigest()[:32] == c["sha"]
    if "report" in c:
        rep = traffic_report(m.AccessTrace(idx, warp))
        assert [rep.total_transactions, rep.per_iteration_mean, rep.per_warp_max, rep.unnecessary_words] == c["report"]
        dev = traffic_report(trace_algorithm(c["kind"], uniform_w(c["n"]), c["b"], warp, c["partition_bytes"],
                                             c["seed"]))
        assert dev == rep


def test_trace_matches_the_kernels_partners():
    """Uniform weights accept every proposal (u * 1 <= 1), so a Megopolis / Metropolis run's
    ancestors are the replayed indices of its last round."""
    n, b = 4096, 5
    for kind in ("megopolis", "metropolis"):
        fn = m.make_resampler(kind)
        anc = fn(uniform_w(n), b, 77)
        idx = m.comparison_indices(kind, n, b, 77)
        assert np.array_equal(anc, idx[-1])


# ---------------------------------------------------------------------------
# the reference's own tests (T/test_warpsim.py) against this package


def test_aligned_consecutive_is_four():
    assert count_transactions(np.arange(32), WARP) == 4
    assert count_transactions(np.arange(64, 96), WARP) == 4


def test_stride_two_is_eight():
    assert count_transactions(np.arange(0, 64, 2), WARP) == 8


def test_misaligned_consecutive_is_five():
    assert count_transactions(np.arange(1, 33), WARP) == 5


def test_single_segment_is_one():
    assert count_transactions([3] * 32, WARP) == 1
    assert count_transactions(np.arange(8), WARP) == 1


def test_count_transactions_permutation_invariant():
    rr = np.random.default_rng(4)
    for _ in range(30):
        idx = rr.integers(0, 1024, int(rr.integers(1, 33)))
        perm = rr.permutation(idx)
        assert count_transactions(idx, WARP) == count_transactions(perm, WARP)
        assert count_transactions(np.concatenate([idx, idx]), WARP) == count_transactions(idx, WARP)
        assert count_transactions(idx, WARP) == len(np.unique(idx * 4 // 32))


def test_megopolis_trace_exactly_one_block():
    trace = trace_algorithm("megopolis", uniform_w(2**12), 6, WARP, None, 5)
    grouped = trace.indices.reshape(6, -1, 32).cpu().numpy()
    for it in range(6):
        for wi in range(0, grouped.shape[1], 7):
            row = grouped[it, wi]
            assert count_transactions(row, WARP) == 4
            assert len(set(row.tolist())) == 32  # bijection within the block
            assert row.min() % 32 == 0


def test_megopolis_report_mean_four_no_waste():
    rep = traffic_report(trace_algorithm("megopolis", uniform_w(2**12), 8, WARP, None, 1))
    assert rep.per_iteration_mean == 4.0
    assert rep.per_warp_max == 4
    assert rep.unnecessary_words == 0


def test_metropolis_small_n_transaction_range():
    trace = trace_algorithm("metropolis", uniform_w(64), 32, WARP, None, 3)
    grouped = trace.indices.reshape(32, -1, 32).cpu().numpy()
    counts = [count_transactions(grouped[it, wi], WARP) for it in range(32) for wi in range(grouped.shape[1])]
    assert min(counts) >= 1 and max(counts) <= 8


def test_metropolis_max_32_achievable():
    rep = traffic_report(trace_algorithm("metropolis", uniform_w(2**16), 4, WARP, None, 11))
    assert rep.per_warp_max == 32


def test_c1_ps128_at_most_four():
    rep = traffic_report(trace_algorithm("c1", uniform_w(2**12), 8, WARP, 128, 7))
    assert rep.per_warp_max <= 4


def test_stride_example_unnecessary_words():
    rep = traffic_report(m.AccessTrace(np.arange(0, 64, 2)[None, :], WARP))
    assert rep.total_transactions == 8
    assert rep.unnecessary_words == 32


def test_traffic_lower_bound_invariant():
    for kind, part in [("metropolis", None), ("c1", 2048), ("c2", 2048), ("megopolis", None)]:
        rep = traffic_report(trace_algorithm(kind, uniform_w(2**10), 4, WARP, part, 9))
        assert rep.total_transactions >= 4 * (2**10 // 32) * 4


def test_traffic_ordering_at_n_2_10():
    w = uniform_w(2**10)
    mean = {k: traffic_report(trace_algorithm(name, w, 8, WARP, p, 13)).per_iteration_mean
            for k, (name, p) in {"megopolis": ("megopolis", None), "c1_128": ("c1", 128),
                                 "c1_2048": ("c1", 2048), "metropolis": ("metropolis", None)}.items()}
    assert mean["megopolis"] <= mean["c1_128"] <= mean["c1_2048"] <= mean["metropolis"]
    assert mean["megopolis"] == 4.0


def test_rng_draws_and_errors():
    assert [rng_draws_per_iteration(k) for k in ("metropolis", "c1", "c2", "megopolis")] == [2.0, 2.0, 3.0, 1.0]
    with pytest.raises(ValueError, match="no access trace defined"):
        trace_algorithm("systematic", uniform_w(64), 2)
    with pytest.raises(ValueError, match="requires a partition size"):
        m.comparison_indices("c1", 64, 2, 0)
    with pytest.raises(ValueError, match="not a multiple of the warp size"):
        traffic_report(m.AccessTrace(np.zeros((2, 40), np.int64), WARP))
    with pytest.raises(ValueError, match="trace must have shape"):
        m.AccessTrace(np.zeros(4), WARP)
    assert count_transactions([], WARP) == 0
