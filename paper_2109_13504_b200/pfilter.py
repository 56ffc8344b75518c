"""Bootstrap (SIR) particle filter on the B200 -- mirrors pkg/src/megores/pfilter.py.

The filter is the paper's end-to-end application (PAPER.md Alg. "Modified SIR
Particle Filter"; M/pfilter.py:1-226): scalar growth model
x' = x/2 + 25x/(1+x^2) + 8cos(1.2 t) + v, v ~ N(0, 10); z = x^2/20 + n, n ~ N(0, 1).

Every stage runs on the device with the particle cloud resident in HBM:
  stage 1  predict + update   one fused kernel (mgp_pf_predict_update)
  stage 2  B rule + resample + gather   (mgp_estimate_ratio_stats or b_fixed,
           the Metropolis-family kernels, mgp_gather)
  stage 3  estimate = numpy-exact mean  (mgp_mean)
Stage times are CUDA-event times on the filter's stream (the reference uses
perf_counter around its numpy stages, M/pfilter.py:148-163).

Parity: the float64 arithmetic follows the reference operation by operation
(no FMA contraction).  exp/log/cos come from CUDA's libdevice instead of the
host libm, so values can differ in the last bit; the filter is therefore
checked against the reference within tolerance and statistically (RMSE).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _device as D
from . import _lib
from .metrics import QualityStats, RunTimings, resample_ratio, rmse  # noqa: F401  (M/metrics.py names)
from .resample import METROPOLIS_FAMILY, WarpConfig, abi_partition_bytes
from .rng import derive_seed, gaussian_at
from .weights import compute_iterations

_TAG_INIT, _TAG_PROCESS, _TAG_RESAMPLE, _TAG_TRUTH, _TAG_OBS = 1, 2, 3, 4, 5  # M/pfilter.py:40-45
_RATIO_SUBSET = 4096  # M/pfilter.py:47


@dataclass(frozen=True)
class FilterConfig:  # M/pfilter.py:50-65
    n_particles: int
    process_var: float = 10.0
    obs_var: float = 1.0
    resampler: str = "megopolis"
    partition_bytes: int | None = None
    warp: WarpConfig = field(default_factory=WarpConfig)
    b_fixed: int | None = None
    epsilon: float = 0.1
    precision: str = "single"
    rng: str = "megores"

    def __post_init__(self):
        if self.n_particles < 1:
            raise ValueError("n_particles must be positive")
        if self.process_var <= 0 or self.obs_var <= 0:
            raise ValueError("noise variances must be positive")


@dataclass(frozen=True)
class Trajectory:  # M/pfilter.py:68-75
    truth: np.ndarray
    observations: np.ndarray

    def __post_init__(self):
        if len(self.truth) != len(self.observations) or len(self.truth) < 1:
            raise ValueError("truth and observations must have equal positive length")


@dataclass
class FilterState:  # M/pfilter.py:78-83 (particles: CUDA float64 tensor)
    particles: object
    estimate: float
    t: int
    timings: RunTimings


def transition(x, t: int, noise=0.0):
    """Host form of the growth map (M/pfilter.py:86-89)."""
    x = np.asarray(x, dtype=np.float64)
    return x / 2.0 + 25.0 * x / (1.0 + x * x) + 8.0 * math.cos(1.2 * t) + noise


def likelihood(z: float, x, obs_var: float = 1.0):
    """Host form of the observation density (M/pfilter.py:92-103)."""
    if obs_var <= 0:
        raise ValueError("obs_var must be positive")
    x = np.asarray(x, dtype=np.float64)
    residual = z - x * x / 20.0
    dens = np.exp(-0.5 * residual * residual / obs_var) / math.sqrt(2.0 * math.pi * obs_var)
    return np.maximum(dens, np.finfo(np.float64).tiny)


def generate_trajectory(t_steps: int, x0: float = 0.0, seed=0, process_var: float = 10.0,
                        obs_var: float = 1.0) -> Trajectory:
    """Ground truth and observations for t = 1..T (M/pfilter.py:106-126); host, T values."""
    if t_steps < 1:
        raise ValueError("t_steps must be >= 1")
    v = gaussian_at(derive_seed(seed, _TAG_TRUTH), np.arange(t_steps), 0) * math.sqrt(process_var)
    n = gaussian_at(derive_seed(seed, _TAG_OBS), np.arange(t_steps), 0) * math.sqrt(obs_var)
    truth = np.empty(t_steps, dtype=np.float64)
    x = x0
    for t in range(1, t_steps + 1):
        x = float(transition(x, t, v[t - 1]))
        truth[t - 1] = x
    return Trajectory(truth, truth * truth / 20.0 + n)


class _Events:
    def __init__(self, t):
        self.ev = [t.cuda.Event(enable_timing=True) for _ in range(4)]

    def record(self, k, stream):
        self.ev[k].record(stream)

    def timings(self) -> RunTimings:
        self.ev[3].synchronize()
        ms = [self.ev[k].elapsed_time(self.ev[k + 1]) for k in range(3)]
        return RunTimings(*(max(m, 0.0) * 1e-3 for m in ms))


def init_state(cfg: FilterConfig, seed, device=None) -> FilterState:  # M/pfilter.py:129-133
    D.require_cuda()
    t = D.torch()
    dev = t.device("cuda") if device is None else t.device(device)
    x = t.empty(cfg.n_particles, dtype=t.float64, device=dev)
    est = t.empty(1, dtype=t.float64, device=dev)
    with t.cuda.device(dev):
        s = D.stream_ptr()
        _lib.check(_lib.lib().mgp_pf_init(cfg.n_particles, derive_seed(seed, _TAG_INIT), math.sqrt(cfg.process_var),
                                          D.ptr(x), s))
        _lib.check(_lib.lib().mgp_mean(D.ptr(x), _lib.MGP_F64, cfg.n_particles, D.ptr(est), s))
    return FilterState(x, float(est.item()), 0, RunTimings(0.0, 0.0, 0.0))


def _iteration_budget(cfg: FilterConfig, w, step_seed) -> int:  # M/pfilter.py:136-141
    if cfg.b_fixed is not None:
        return cfg.b_fixed
    t = D.torch()
    subset = min(_RATIO_SUBSET, w.numel())
    out = t.empty(2, dtype=t.float64, device=w.device)
    _lib.check(_lib.lib().mgp_estimate_ratio_stats(D.ptr(w), D.wdtype(w), w.numel(), subset, step_seed, D.ptr(out),
                                                   D.stream_ptr()))
    mean, mx = (float(v) for v in out.cpu().numpy())
    if mx == 0.0:
        raise ValueError("subset contains only zero weights")
    return compute_iterations(cfg.epsilon, mean / mx, 1.0).b


def _resample_device(cfg: FilterConfig, w, b: int, seed):
    """Device resample of the step's weights (finite and non-negative by construction; the
    all-zero check is the predict/update kernel's any-positive flag, checked by the caller)."""
    t = D.torch()
    n = w.numel()
    anc = t.empty(n, dtype=t.int64, device=w.device)
    kind = cfg.resampler
    if kind not in _lib.KIND:
        raise ValueError(f"unknown resampler {kind!r}")
    prefix = kind not in METROPOLIS_FAMILY  # multinomial / systematic ignore b (M/resample.py:450-454)
    flags = _lib.FLAG_NONZERO if cfg.precision == "double" else 0  # float32 cast can underflow to 0
    _lib.check(_lib.lib().mgp_resample_range(
        _lib.KIND[kind], D.ptr(w), D.wdtype(w), n, 1 if prefix else int(b), int(seed) & (2**64 - 1),
        cfg.warp.warp_size, abi_partition_bytes(cfg.partition_bytes, cfg.warp), 1, _lib.RNG["megores" if prefix else cfg.rng], flags, 0, n,
        D.ptr(anc), D.stream_ptr()))
    return anc


def _step(x, t: int, z: float, cfg: FilterConfig, seed, est_out, any_pos, ev):
    """One SIR step (M/pfilter.py:143-165) queued on the current stream without host round trips
    (except the estimate_ratio B rule when ``b_fixed`` is None, which the reference also derives
    on the host): the estimate lands in ``est_out`` (device float64), the any-positive flag of the
    step's weights in ``any_pos`` (device int32, zeroed by the caller), stage events in ``ev``."""
    tch = D.torch()
    n = cfg.n_particles
    dev = x.device
    stream = tch.cuda.current_stream(dev)
    s = D.stream_ptr(dev)
    ev.record(0, stream)
    xp = tch.empty_like(x)
    w = tch.empty(n, dtype=tch.float32 if cfg.precision == "single" else tch.float64, device=dev)
    _lib.check(_lib.lib().mgp_pf_predict_update(
        D.ptr(x), n, 8.0 * math.cos(1.2 * t), math.sqrt(cfg.process_var), derive_seed(seed, _TAG_PROCESS, t),
        float(z), cfg.obs_var, D.wdtype(w), D.ptr(xp), D.ptr(w), D.ptr(any_pos), s))
    ev.record(1, stream)
    step_seed = derive_seed(seed, _TAG_RESAMPLE, t)
    b = _iteration_budget(cfg, w, step_seed)
    if b < 1:
        raise ValueError(f"B must be >= 1, got {b}")
    anc = _resample_device(cfg, w, b, step_seed)
    resampled = tch.empty_like(xp)
    _lib.check(_lib.lib().mgp_gather(D.ptr(xp), 8, D.ptr(anc), n, D.ptr(resampled), s))
    ev.record(2, stream)
    _lib.check(_lib.lib().mgp_mean(D.ptr(resampled), _lib.MGP_F64, n, D.ptr(est_out), s))
    ev.record(3, stream)
    return resampled


def sir_step(state: FilterState, z: float, cfg: FilterConfig, seed) -> FilterState:  # M/pfilter.py:143-165
    """Predict/update, resample, estimate on the device; per-stage CUDA-event times."""
    tch = D.torch()
    t = state.t + 1
    dev = state.particles.device
    with tch.cuda.device(dev):
        est = tch.empty(1, dtype=tch.float64, device=dev)
        any_pos = tch.zeros(1, dtype=tch.int32, device=dev)
        ev = _Events(tch)
        resampled = _step(state.particles, t, z, cfg, seed, est, any_pos, ev)
        timings = ev.timings()
        if int(any_pos.item()) == 0:
            raise ValueError("all weights are zero")  # _check_weights (M/resample.py:96-100)
    return FilterState(resampled, float(est.item()), t, timings)


def run_filter(cfg: FilterConfig, trajectory: Trajectory, seed):  # M/pfilter.py:168-179
    """All T steps queued back to back on the device; estimates, the any-positive flags and the
    stage events are read once at the end."""
    tch = D.torch()
    state = init_state(cfg, seed)
    t_steps = len(trajectory.truth)
    dev = state.particles.device
    with tch.cuda.device(dev):
        ests = tch.empty(t_steps, dtype=tch.float64, device=dev)
        any_pos = tch.zeros(t_steps, dtype=tch.int32, device=dev)
        evs = [_Events(tch) for _ in range(t_steps)]
        x = state.particles
        for k in range(t_steps):
            x = _step(x, k + 1, float(trajectory.observations[k]), cfg, seed, ests[k:k + 1], any_pos[k:k + 1], evs[k])
        flags = any_pos.cpu().numpy()
        if not flags.all():
            raise ValueError("all weights are zero")  # _check_weights (M/resample.py:96-100)
        estimates = ests.cpu().numpy()
        stages = np.zeros(3, dtype=np.float64)
        for ev in evs:
            tm = ev.timings()
            stages += (tm.stage1, tm.stage2, tm.stage3)
    stages /= t_steps
    return estimates, RunTimings(*stages)


def run_benchmark(base_cfg: FilterConfig, trajectories, runs_per_trajectory: int, b_values, algorithms, seed=0):
    """RMSE and mean resample ratio per (algorithm, B) (M/pfilter.py:182-226)."""
    rows = []
    for name, part_bytes in algorithms:
        # prefix-sum resamplers ignore B and report b = 0 (M/pfilter.py:191-196)
        for b in (list(b_values) if name in METROPOLIS_FAMILY else [0]):
            cfg = replace(base_cfg, resampler=name, partition_bytes=part_bytes, b_fixed=b if b > 0 else None)
            per_traj, ratios = [], []
            for ti, traj in enumerate(trajectories):
                est = np.empty((runs_per_trajectory, len(traj.truth)))
                for k in range(runs_per_trajectory):
                    e, tm = run_filter(cfg, traj, derive_seed(seed, ti, k))
                    est[k] = e
                    ratios.append(resample_ratio(tm))
                per_traj.append(rmse(traj.truth, est))
            rows.append({"algorithm": name, "partition_bytes": part_bytes, "b": b, "n": cfg.n_particles,
                         "rmse": float(np.mean(per_traj)), "resample_ratio": float(np.mean(ratios))})
    return rows
