"""Resampling quality statistics on the B200 (mirrors M/metrics.py:33-121).

The offspring bias / MSE metric of the paper (and of BASELINE.json).  All
accumulators live in HBM as float64 and every reduction uses numpy's pairwise
summation order, so the statistics are bit-identical to the reference's
``QualityAccumulator`` for the same offspring vectors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .weights import _as_weight_vector


@dataclass(frozen=True)
class QualityStats:  # M/metrics.py:33-39
    mse: float
    variance: float
    bias_sq: float
    bias_contribution: float
    mse_per_particle: float


@dataclass(frozen=True)
class RunTimings:  # M/metrics.py:42-52: seconds in predict+update, resample, estimate
    stage1: float
    stage2: float
    stage3: float

    def __post_init__(self):
        if min(self.stage1, self.stage2, self.stage3) < 0:
            raise ValueError("stage timings must be non-negative")


def rmse(truth, estimates) -> float:  # M/metrics.py:124-136 (host: T filter estimates)
    truth = np.asarray(truth, dtype=np.float64)
    estimates = np.asarray(estimates, dtype=np.float64)
    if estimates.ndim != 2 or estimates.shape[1] != truth.shape[0]:
        raise ValueError(f"estimates shape {estimates.shape} does not match truth length {truth.shape}")
    return float(np.sqrt(np.mean((estimates - truth[None, :]) ** 2, axis=0)).mean())


def resample_ratio(timings: RunTimings) -> float:  # M/metrics.py:139-144
    total = timings.stage1 + timings.stage2 + timings.stage3
    if total <= 0:
        raise ValueError("total stage time must be positive")
    return timings.stage2 / total


def _dev_weights(w):
    t = D.torch()
    wv = _as_weight_vector(w)
    vals = wv.values if wv.on_device else t.from_numpy(np.ascontiguousarray(wv.values)).cuda()
    return vals


def _dev_counts(offspring, device):
    t = D.torch()
    if D.is_tensor(offspring):
        return offspring.to(device=device, dtype=t.int64).contiguous()
    return t.from_numpy(np.ascontiguousarray(offspring, dtype=np.int64)).to(device)


def _expected(vals):
    t = D.torch()
    e = t.empty(vals.numel(), dtype=t.float64, device=vals.device)
    total = t.empty(1, dtype=t.float64, device=vals.device)
    with t.cuda.device(vals.device):
        _lib.check(_lib.lib().mgp_expected_offspring(D.ptr(vals), D.wdtype(vals), vals.numel(), D.ptr(e),
                                                     D.ptr(total), D.stream_ptr()))
    if not float(total.item()) > 0:  # M/metrics.py:57-59
        raise ValueError("total weight must be positive")
    return e


def squared_error(offspring, w) -> float:
    """Sum of squared deviations from the expected offspring counts (M/metrics.py:63-68)."""
    D.require_cuda()
    t = D.torch()
    vals = _dev_weights(w)
    n_off = offspring.shape[0] if D.is_tensor(offspring) else len(offspring)
    if n_off != vals.numel():
        raise ValueError(f"length mismatch: {n_off} offspring vs {vals.numel()} weights")
    e = _expected(vals)
    o = _dev_counts(offspring, vals.device)
    out = t.empty(1, dtype=t.float64, device=vals.device)
    with t.cuda.device(vals.device):
        _lib.check(_lib.lib().mgp_squared_error(D.ptr(o), D.ptr(e), o.numel(), D.ptr(out), D.stream_ptr()))
    return float(out.item())


class QualityAccumulator:
    """Streaming mean/variance over K offspring vectors (M/metrics.py:71-110), in HBM."""

    def __init__(self, n: int, device=None):
        D.require_cuda()
        t = D.torch()
        self.n = n
        self.k = 0
        self.device = t.device("cuda") if device is None else t.device(device)
        self._sum = t.zeros(n, dtype=t.float64, device=self.device)
        self._sum_sq = t.zeros(n, dtype=t.float64, device=self.device)
        self._se = t.zeros(2, dtype=t.float64, device=self.device)  # [se_total, se_last_run]
        self._expected = None

    def _check_len(self, what: str, m: int) -> None:
        # the reference fails these as numpy broadcast ValueErrors (M/metrics.py:86-93); the
        # device kernels read self.n elements, so the lengths are checked before any launch
        if m != self.n:
            raise ValueError(f"length mismatch: {m} {what} vs accumulator length {self.n}")

    def add(self, offspring, w) -> None:
        t = D.torch()
        self._check_len("offspring", offspring.shape[0] if D.is_tensor(offspring) else len(offspring))
        if self._expected is None:
            wd = _dev_weights(w).to(self.device)
            self._check_len("weights", wd.numel())
            self._expected = _expected(wd)
        o = _dev_counts(offspring, self.device)
        self._check_len("offspring", o.numel())
        self.k += 1
        with t.cuda.device(self.device):
            _lib.check(_lib.lib().mgp_quality_add(D.ptr(o), D.ptr(self._expected), self.n, D.ptr(self._sum),
                                                  D.ptr(self._sum_sq), D.ptr(self._se),
                                                  D.ptr(self._se[1:]), D.stream_ptr()))

    def add_runs(self, kind: str, w, b: int, seeds, warp_size: int = 32, partition_bytes: int | None = None,
                 strict: bool = True, rng: str = "megores") -> None:
        """K runs of resampler ``kind`` (one per seed) added in one device pass -- the same as
        ``for s in seeds: self.add(ancestors_to_offspring(make_resampler(kind, ...)(w, b, s)), w)``
        (M/bench.py:121-126) without a host round trip per run."""
        import ctypes

        t = D.torch()
        wd = _dev_weights(w).to(self.device)
        self._check_len("weights", wd.numel())
        if self._expected is None:
            self._expected = _expected(wd)
        from .weights import device_stats

        st = device_stats(wd)
        if st.n_pos == 0:
            raise ValueError("all weights are zero")
        seeds = [int(s) & (2**64 - 1) for s in seeds]
        arr = (ctypes.c_uint64 * max(1, len(seeds)))(*seeds)
        flags = _lib.FLAG_NONZERO if st.n_zero == 0 else 0
        with t.cuda.device(self.device):
            _lib.check(_lib.lib().mgp_quality_runs(
                _lib.KIND[kind], D.ptr(wd), D.wdtype(wd), self.n, int(b), ctypes.cast(arr, ctypes.c_void_p),
                len(seeds), int(warp_size), int(partition_bytes or 0), int(bool(strict)), _lib.RNG[rng], flags,
                D.ptr(self._expected), D.ptr(self._sum), D.ptr(self._sum_sq), D.ptr(self._se), D.stream_ptr()))
        self.k += len(seeds)

    @property
    def _se_total(self) -> float:
        return float(self._se[0].item())

    def finalize(self) -> QualityStats:
        if self.k < 2:
            raise ValueError(f"need at least 2 runs to estimate variance, got {self.k}")
        t = D.torch()
        out = t.empty(2, dtype=t.float64, device=self.device)
        with t.cuda.device(self.device):
            _lib.check(_lib.lib().mgp_quality_finalize(D.ptr(self._sum), D.ptr(self._sum_sq), D.ptr(self._expected),
                                                       self.n, self.k, D.ptr(out), D.ptr(out[1:]), D.stream_ptr()))
        variance, bias_sq = (float(x) for x in out.cpu().numpy())
        mse = self._se_total / self.k
        contribution = bias_sq / mse if mse > 0 else 0.0
        return QualityStats(mse=mse, variance=variance, bias_sq=bias_sq, bias_contribution=contribution,
                            mse_per_particle=mse / self.n)


def quality_stats(runs, w) -> QualityStats:
    """MSE / variance / squared-bias over a (K, N) stack of offspring vectors (M/metrics.py:113-121)."""
    if D.is_tensor(runs):
        shape = tuple(runs.shape)
    else:
        runs = np.asarray(runs)
        shape = runs.shape
    if len(shape) != 2:
        raise ValueError("runs must have shape (K, N)")
    acc = QualityAccumulator(shape[1])
    for row in runs:
        acc.add(row, w)
    return acc.finalize()
