"""Weight vectors and the iteration budget (the B rule) on the B200.

Mirrors pkg/src/megores/weights.py (M/weights.py):
  * ``WeightVector``        M/weights.py:42-62 (same validation and errors; values may
                            also be a CUDA tensor, validated by one fused device pass)
  * ``compute_iterations``  M/weights.py:114-131 (host arithmetic, identical)
  * ``iterations_for``      the f64 mean/max of M/bench.py:119-120 computed on the
                            device (numpy-exact pairwise sum) then ``compute_iterations``
  * ``gen_gaussian_weights`` M/weights.py:100-104 evaluated on the device
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib

GAUSSIAN_PEAK = 1.0 / math.sqrt(2.0 * math.pi)  # M/weights.py:37
_DTYPES = {"single": np.float32, "double": np.float64}
_TORCH_DTYPES = {"single": "float32", "double": "float64"}


class _StatsStruct(ctypes.Structure):  # mgp_weight_stats_t
    _fields_ = [("sum", ctypes.c_double), ("mean", ctypes.c_double), ("max", ctypes.c_double),
                ("n_pos", ctypes.c_int64), ("n_zero", ctypes.c_int64), ("n_neg", ctypes.c_int64),
                ("n_nonfinite", ctypes.c_int64), ("n_notnormal", ctypes.c_int64)]


@dataclass(frozen=True)
class WeightStats:
    """One fused device pass over the weights (mgp_weight_stats)."""

    n: int
    sum: float
    mean: float
    max: float
    n_pos: int
    n_zero: int
    n_neg: int
    n_nonfinite: int
    n_notnormal: int

    @property
    def positive_normal(self) -> bool:
        return self.n_notnormal == 0


def device_stats(values) -> WeightStats:
    """Weight statistics of a CUDA tensor (synchronises to read 64 bytes back)."""
    t = D.torch()
    values = values.contiguous()
    out = t.empty(8, dtype=t.float64, device=values.device)
    with t.cuda.device(values.device):
        _lib.check(_lib.lib().mgp_weight_stats(D.ptr(values), D.wdtype(values), values.numel(),
                                               D.ptr(out), D.stream_ptr()))
        host = out.cpu().numpy()
    s = _StatsStruct.from_buffer_copy(host.tobytes())
    return WeightStats(values.numel(), s.sum, s.mean, s.max, s.n_pos, s.n_zero, s.n_neg, s.n_nonfinite,
                       s.n_notnormal)


def _host_flags(values: np.ndarray):
    """(any non-finite, any negative) of a host float array: one parallel pass in libmgp
    (mgp_check_host_weights, host threads only) -- the reference's two numpy scans
    (M/weights.py:56-59) cost ~16 ms at 2^24."""
    if values.size >= 1 << 16 and values.flags.c_contiguous:
        counts = np.zeros(4, dtype=np.int64)
        _lib.check(_lib.lib().mgp_check_host_weights(values.ctypes.data, 0 if values.dtype == np.float32 else 1,
                                                     values.size, counts.ctypes.data))
        return bool(counts[0]), bool(counts[1])
    return (not np.all(np.isfinite(values))), bool(np.any(values < 0))


class WeightVector:
    """Non-negative particle weights; normalisation is not required (M/weights.py:42-62).

    ``values`` may be anything numpy accepts (validated on the host exactly like the
    reference) or a CUDA tensor (kept in HBM, validated by one device pass).
    """

    def __init__(self, values, precision: str = "single"):
        if precision not in _DTYPES:
            raise ValueError(f"precision must be 'single' or 'double', got {precision!r}")
        self.precision = precision
        self._stats = None
        self._ver = None
        if D.is_cuda_tensor(values):
            t = D.torch()
            values = values.to(getattr(t, _TORCH_DTYPES[precision])).contiguous()
            if values.dim() != 1 or values.numel() < 1:
                raise ValueError("weights must be a non-empty 1-d sequence")
            self.values = values
            self.stats()  # validates: finite, non-negative
            return
        if D.is_tensor(values):
            values = values.detach().cpu().numpy()
        values = np.asarray(values, dtype=_DTYPES[precision])
        if values.ndim != 1 or len(values) < 1:
            raise ValueError("weights must be a non-empty 1-d sequence")
        nonfinite, negative = _host_flags(values)
        if nonfinite:
            raise ValueError("weights must be finite")
        if negative:
            raise ValueError("weights must be non-negative")
        self.values = values

    def __len__(self) -> int:
        return int(self.values.shape[0])

    @property
    def on_device(self) -> bool:
        return D.is_cuda_tensor(self.values)

    def stats(self) -> WeightStats:
        """Device statistics of the current values, re-validated like the reference's per-call
        ``_check_weights`` (M/resample.py:96-100, M/weights.py:53-61).  For device-resident
        weights the pass is cached against the tensor's version counter, so an in-place update
        of the caller's tensor (``values`` aliases it) invalidates it; host arrays are re-read
        every call."""
        ver = self.values._version if self.on_device else None
        if self._stats is None or not self.on_device or ver != self._ver:
            D.require_cuda()
            t = D.torch()
            vals = self.values if self.on_device else t.from_numpy(np.ascontiguousarray(self.values)).cuda()
            st = device_stats(vals)
            if st.n_nonfinite:
                raise ValueError("weights must be finite")
            if st.n_neg:
                raise ValueError("weights must be non-negative")
            self._stats, self._ver = st, ver
        return self._stats


@dataclass(frozen=True)
class GaussianWeightParams:  # M/weights.py:65-74
    y: float
    n: int

    def __post_init__(self):
        if self.y < 0:
            raise ValueError(f"y must be >= 0, got {self.y}")
        if self.n < 1:
            raise ValueError(f"n must be >= 1, got {self.n}")


@dataclass(frozen=True)
class IterationBudget:  # M/weights.py:90-97
    b: int
    epsilon: float

    def __post_init__(self):
        if self.b < 1:
            raise ValueError(f"B must be >= 1, got {self.b}")


def compute_iterations(epsilon: float, mean_w: float, max_w: float) -> IterationBudget:
    """B = ceil(ln(eps) / ln(1 - mean_w / max_w)), clamped to >= 1 (M/weights.py:114-131)."""
    if not (0.0 < epsilon <= 1.0):
        raise ValueError(f"epsilon must be in (0, 1], got {epsilon}")
    if mean_w <= 0 or max_w <= 0:
        raise ValueError("mean_w and max_w must be positive")
    if mean_w > max_w:
        raise ValueError(f"mean_w ({mean_w}) exceeds max_w ({max_w})")
    ratio = mean_w / max_w
    if ratio >= 1.0 or epsilon == 1.0:
        return IterationBudget(1, epsilon)
    b = math.ceil(math.log(epsilon) / math.log(1.0 - ratio))
    return IterationBudget(max(b, 1), epsilon)


def _as_weight_vector(w) -> WeightVector:
    if isinstance(w, WeightVector):
        return w
    if hasattr(w, "values") and hasattr(w, "precision"):  # the reference's WeightVector
        return WeightVector(w.values, w.precision)
    if D.is_tensor(w) or isinstance(w, np.ndarray):
        prec = "double" if str(w.dtype).endswith("float64") else "single"
        return WeightVector(w, prec)
    return WeightVector(w)


def iterations_for(w, epsilon: float = 0.01) -> IterationBudget:
    """The benchmark's B rule: f64 mean and max of the weights (M/bench.py:119-120),
    computed on the device with numpy's pairwise summation order, then
    ``compute_iterations``.  Bit-identical to the reference's B."""
    st = _as_weight_vector(w).stats()
    if st.n_pos == 0:
        raise ValueError("mean_w and max_w must be positive")
    return compute_iterations(epsilon, st.mean, st.max)


def gen_gaussian_weights(params: GaussianWeightParams, seed, precision="single", device=None) -> WeightVector:
    """w_i = exp(-(x_i - y)^2 / 2) / sqrt(2 pi), x_i ~ N(0,1) by Box-Muller on the reference's
    stream (M/weights.py:100-104, M/rng.py:152-161).

    Default (``device=None``): the reference's own bytes -- a host numpy WeightVector
    identical to ``megores.gen_gaussian_weights`` (same formula, same numpy libm), so B and
    every ancestor downstream match the reference exactly.

    ``device="cuda"`` (or a device index): generated in HBM by one kernel
    (``mgp_gen_gaussian``) and returned as a CUDA-tensor WeightVector -- for populations too
    large for a host detour (2^28).  NOT bit-exact: the device libm may round
    log/cos/exp differently from the host's in the last float64 bit, which moves a small
    fraction of float32 weights by one ulp."""
    if precision not in _DTYPES:
        raise ValueError(f"precision must be 'single' or 'double', got {precision!r}")
    if device is None:
        return gen_gaussian_weights_host(params, seed, precision)
    D.require_cuda()
    t = D.torch()
    dev = t.device(device) if not isinstance(device, int) else t.device("cuda", device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {device!r}")
    out = t.empty(params.n, dtype=getattr(t, _TORCH_DTYPES[precision]), device=dev)
    with t.cuda.device(dev):
        _lib.check(_lib.lib().mgp_gen_gaussian(float(params.y), params.n, int(seed) & (2**64 - 1),
                                               D.wdtype(out), D.ptr(out), D.stream_ptr()))
    return WeightVector(out, precision)


# ---------------------------------------------------------------------------
# Host generators: the reference's own formulas in numpy (input synthesis for the CLI's
# experiment grids, so the weights -- and every downstream result -- match the reference
# bit for bit).  The hot path never calls these.


@dataclass(frozen=True)
class GammaWeightParams:  # M/weights.py:77-86
    alpha: float
    beta: float
    n: int

    def __post_init__(self):
        if self.alpha <= 0 or self.beta <= 0:
            raise ValueError(f"alpha and beta must be > 0, got {self.alpha}, {self.beta}")
        if self.n < 1:
            raise ValueError(f"n must be >= 1, got {self.n}")


def gen_gaussian_weights_host(params: GaussianWeightParams, seed, precision="single") -> WeightVector:
    """M/weights.py:100-104 in numpy: w = exp(-(x - y)^2 / 2) / sqrt(2 pi), x = gaussian_at(seed, i, 0)."""
    from .rng import gaussian_at

    x = gaussian_at(seed, np.arange(params.n), 0)
    return WeightVector(np.exp(-0.5 * (x - params.y) ** 2) * GAUSSIAN_PEAK, precision)


def gen_gamma_weights(params: GammaWeightParams, seed, precision="single", device=None) -> WeightVector:
    """I.i.d. gamma(alpha, rate=beta) weights by inverse-CDF sampling (M/weights.py:107-111).

    Default: the reference's own bytes -- ``scipy.stats.gamma.ppf`` of
    ``uniform_open01_at(seed, i, 0)`` on the host.  ``device="cuda"`` (or an index): the same
    inverse CDF evaluated in HBM by ``mgp_gen_gamma`` (float64 incomplete-gamma inversion,
    ~1e-14 relative to scipy for alpha <= 1000; tests/test_gamma_gpu.py), returned as a
    CUDA-tensor WeightVector -- the 2^28-population route without a host detour."""
    if precision not in _DTYPES:
        raise ValueError(f"precision must be 'single' or 'double', got {precision!r}")
    if device is None:
        from scipy import stats

        from .rng import uniform_open01_at

        u = uniform_open01_at(seed, np.arange(params.n), 0)
        return WeightVector(stats.gamma.ppf(u, a=params.alpha, scale=1.0 / params.beta), precision)
    D.require_cuda()
    t = D.torch()
    dev = t.device(device) if not isinstance(device, int) else t.device("cuda", device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {device!r}")
    out = t.empty(params.n, dtype=getattr(t, _TORCH_DTYPES[precision]), device=dev)
    with t.cuda.device(dev):
        _lib.check(_lib.lib().mgp_gen_gamma(float(params.alpha), float(params.beta), params.n,
                                            int(seed) & (2**64 - 1), D.wdtype(out), D.ptr(out), D.stream_ptr()))
    return WeightVector(out, precision)


def estimate_ratio(w, subset_size: int, seed) -> float:
    """mean(w) / max(w) over the first ``subset_size`` entries of the seed's stable permutation
    (M/weights.py:134-154), on the device (radix sort of the 53-bit keys, numpy-exact mean)."""
    t = D.torch()
    wv = _as_weight_vector(w)
    n = len(wv)
    if not (1 <= subset_size <= n):
        raise ValueError(f"subset_size must be in [1, {n}], got {subset_size}")
    vals = wv.values if wv.on_device else t.from_numpy(np.ascontiguousarray(wv.values)).cuda()
    out = t.empty(2, dtype=t.float64, device=vals.device)
    with t.cuda.device(vals.device):
        _lib.check(_lib.lib().mgp_estimate_ratio_stats(D.ptr(vals), D.wdtype(vals), n, int(subset_size),
                                                       int(seed) & (2**64 - 1), D.ptr(out), D.stream_ptr()))
    mean, mx = (float(v) for v in out.cpu().numpy())
    if mx == 0.0:
        raise ValueError("subset contains only zero weights")
    return mean / mx


def proposition_recurrence(mean_w: float, max_w: float, n: int, b: int) -> float:
    """P_k = 1/N + P_{k-1} (1 - mean/max), P_0 = 0, after b steps (M/weights.py:157-172)."""
    if b < 0:
        raise ValueError(f"B must be >= 0, got {b}")
    if mean_w <= 0 or max_w <= 0 or mean_w > max_w:
        raise ValueError("need 0 < mean_w <= max_w")
    ratio = mean_w / max_w
    p = 0.0
    for _ in range(b):
        p = 1.0 / n + p * (1.0 - ratio)
    return p
