"""Metropolis-family resamplers on the B200 -- drop-in for pkg/src/megores/resample.py.

Same names, signatures, defaults, return types and errors as the reference
(M/ = pkg/src/megores/):
  metropolis      M/resample.py:201-206     metropolis_c1  :209-225
  metropolis_c2   :228-244                  megopolis      :268-282
  make_resampler  :431-455                  megopolis_offsets :263-265
  ancestors_to_offspring :361-368           apply_ancestors   :371-377
  multinomial     :295-304                  systematic_improved :307-336
  WarpConfig :59-75, PartitionConfig :78-93, METROPOLIS_FAMILY / ALGORITHMS :55-56

Inputs: a WeightVector (this package's or the reference's), a numpy array, or a
CUDA tensor.  Host inputs go through the host-buffer C-ABI entry
(``mgp_resample_host``: upload, validate, resample, overlapped download) and
return ``np.int64`` arrays like the reference.  CUDA-tensor inputs stay in HBM,
run asynchronously on the current torch stream after one validation pass, and
return an int64 CUDA tensor.

Extra keyword ``rng``: "megores" (default; the reference's stream, bit-exact with
the reference) or "philox" (Philox4x32-10).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .weights import WeightVector, _as_weight_vector

METROPOLIS_FAMILY = ("metropolis", "c1", "c2", "megopolis")
ALGORITHMS = METROPOLIS_FAMILY + ("multinomial", "systematic")


@dataclass(frozen=True)
class WarpConfig:
    """Logical warp geometry (M/resample.py:59-75).  W is semantic: it fixes the
    Megopolis partner index and the C1/C2 partition owner, independent of hardware."""

    warp_size: int = 32
    word_bytes: int = 4
    segment_bytes: int = 32

    def __post_init__(self):
        if self.warp_size < 1:
            raise ValueError(f"warp_size must be positive, got {self.warp_size}")
        if self.word_bytes < 1 or self.segment_bytes % self.word_bytes:
            raise ValueError("segment_bytes must be a positive multiple of word_bytes")

    @property
    def words_per_segment(self) -> int:
        return self.segment_bytes // self.word_bytes


@dataclass(frozen=True)
class PartitionConfig:
    """Partition geometry for the c1/c2 variants (M/resample.py:78-93)."""

    partition_bytes: int

    def n_weights(self, warp: WarpConfig) -> int:
        if self.partition_bytes < 1 or self.partition_bytes % warp.word_bytes:
            raise ValueError("partition_bytes must be a positive multiple of word_bytes")
        return self.partition_bytes // warp.word_bytes

    def n_partitions(self, n: int, warp: WarpConfig) -> int:
        n_w = self.n_weights(warp)
        if n % n_w:
            raise ValueError(f"N={n} is not divisible by the partition width {n_w}")
        return n // n_w


def abi_partition_bytes(partition_bytes, warp: WarpConfig) -> int:
    """The C-ABI's ``partition_bytes`` counts 4-byte words (n_w = partition_bytes / 4,
    include/megopolis_b200.h).  The reference sizes a partition as
    partition_bytes // warp.word_bytes (M/resample.py:84-87), so a WarpConfig with another
    word size is translated here to the same n_w (0 = no partition)."""
    if partition_bytes is None or partition_bytes == 0:
        return 0
    return PartitionConfig(int(partition_bytes)).n_weights(warp) * 4


def _seed(seed) -> int:
    return int(np.uint64(seed)) if not isinstance(seed, int) else seed & (2**64 - 1)


def _rng(rng: str) -> int:
    try:
        return _lib.RNG[rng]
    except KeyError:
        raise ValueError(f"unknown rng stream {rng!r} (choose 'megores' or 'philox')") from None


def _validate(w: WeightVector, b, warp, strict, part, name):
    """Argument checks in the reference's order (M/resample.py:96-108, 84-93); the
    all-zero check needs the data, so it is consulted only when deciding which
    error the reference would raise first or on the device path."""
    n = len(w)
    errs = []
    if b < 1:
        errs.append(f"B must be >= 1, got {b}")
    elif warp is not None and strict and n % warp.warp_size:
        errs.append(f"{name} requires N ({n}) to be a multiple of the warp size "
                    f"({warp.warp_size}) in strict mode")
    elif part is not None:
        try:
            part.n_partitions(n, warp)
        except ValueError as e:
            errs.append(str(e))
    if errs:
        if not w.on_device and not np.any(w.values > 0):
            raise ValueError("all weights are zero")
        if w.on_device and w.stats().n_pos == 0:
            raise ValueError("all weights are zero")
        raise ValueError(errs[0])


def _resample(kind, w, b, seed, warp, part, strict, rng, name):
    w = _as_weight_vector(w)
    b = int(b)
    if kind in ("multinomial", "systematic"):
        b = 1  # the prefix-sum methods take no iteration budget (M/resample.py:450-454)
    _validate(w, b, warp, strict, part, name)
    L = _lib.lib()
    ws = warp.warp_size if warp is not None else 32
    pb = abi_partition_bytes(part.partition_bytes, warp) if part is not None else 0
    if w.on_device:
        t = D.torch()
        vals = w.values
        st = w.stats()
        if st.n_pos == 0:
            raise ValueError("all weights are zero")
        flags = _lib.FLAG_NONZERO if st.n_zero == 0 else 0
        out = t.empty(len(w), dtype=t.int64, device=vals.device)
        with t.cuda.device(vals.device):
            s = D.stream_ptr()
            args = (D.ptr(vals), D.wdtype(vals), len(w), b, _seed(seed))
            if kind == "megopolis":
                rc = L.mgp_megopolis(*args, ws, int(bool(strict)), _rng(rng), flags, D.ptr(out), s)
            elif kind == "metropolis":
                rc = L.mgp_metropolis(*args, _rng(rng), flags, D.ptr(out), s)
            elif kind == "multinomial":
                rc = L.mgp_multinomial(D.ptr(vals), D.wdtype(vals), len(w), _seed(seed), D.ptr(out), s)
            elif kind == "systematic":
                rc = L.mgp_systematic(D.ptr(vals), D.wdtype(vals), len(w), _seed(seed), D.ptr(out), s)
            elif kind == "c1":
                rc = L.mgp_metropolis_c1(*args, ws, pb, int(bool(strict)), _rng(rng), flags, D.ptr(out), s)
            else:
                rc = L.mgp_metropolis_c2(*args, ws, pb, int(bool(strict)), _rng(rng), flags, D.ptr(out), s)
        _lib.check(rc)
        return out
    D.require_cuda()
    vals = np.ascontiguousarray(w.values)
    out = np.empty(len(vals), dtype=np.int64)
    b_used = ctypes.c_int32(0)
    rc = L.mgp_resample_host(_lib.KIND[kind], D.ptr(vals), D.wdtype(vals), len(vals), b, 0.0, _seed(seed), ws, pb,
                             int(bool(strict)), _rng(rng), D.ptr(out), ctypes.byref(b_used), -1)
    _lib.check(rc)
    return out


def resample_batch(kind: str, weights, b: int, seeds, warp: WarpConfig = WarpConfig(), part=None,
                   strict: bool = True, *, rng: str = "megores", epsilon: float = 0.01, out=None):
    """Independent host-buffer resamples (the reference's call shape repeated over a batch, e.g. the
    repetitions of a quality grid point), pipelined on the device: job k+1's upload and job k-1's
    download overlap job k's kernel (mgp_resample_host_batch).  ``weights``: numpy arrays of one
    length and dtype (page-locked ones give the overlap); ``b <= 0`` derives each job's B from
    ``epsilon``.  Returns (ancestor arrays, B per job); the same ancestors as one
    ``make_resampler(kind)`` call per job.  ``out``: optional output arrays (may repeat every other
    job)."""
    D.require_cuda()
    kind = {"metropolis_c1": "c1", "metropolis_c2": "c2", "systematic_improved": "systematic"}.get(kind, kind)
    vals = [np.ascontiguousarray(getattr(w, "values", w)) for w in weights]
    seeds = [int(s) & (2**64 - 1) for s in seeds]
    if len(seeds) != len(vals):
        raise ValueError(f"{len(vals)} weight vectors but {len(seeds)} seeds")
    if not vals:
        return [], []
    n, dt = len(vals[0]), vals[0].dtype
    if any(len(v) != n or v.dtype != dt for v in vals):
        raise ValueError("every weight vector of a batch must have the same length and dtype")
    outs = list(out) if out is not None else [np.empty(n, dtype=np.int64) for _ in vals]
    if len(outs) != len(vals) or any(o.dtype != np.int64 or len(o) != n or not o.flags.c_contiguous for o in outs):
        raise ValueError("out must hold one contiguous int64 array of N elements per job")
    pb = abi_partition_bytes(part.partition_bytes, warp) if part is not None else 0
    k = len(vals)
    hw = (ctypes.c_void_p * k)(*[v.ctypes.data for v in vals])
    ha = (ctypes.c_void_p * k)(*[o.ctypes.data for o in outs])
    sd = (ctypes.c_uint64 * k)(*seeds)
    bu = (ctypes.c_int32 * k)()
    _lib.check(_lib.lib().mgp_resample_host_batch(_lib.KIND[kind], hw, D.wdtype(vals[0]), n, k, int(b), float(epsilon),
                                                  sd, warp.warp_size, pb, int(bool(strict)), _rng(rng), ha, bu, -1))
    return outs, [int(x) for x in bu]


def metropolis(w, b: int, seed, *, rng: str = "megores"):
    """Independent per-particle random comparisons; fully random access (M/resample.py:201-206)."""
    return _resample("metropolis", w, b, seed, None, None, False, rng, "metropolis")


def metropolis_c1(w, b: int, part: PartitionConfig, warp: WarpConfig = WarpConfig(), seed=0, strict: bool = True,
                  *, rng: str = "megores"):
    """One shared partition per warp for all B rounds (M/resample.py:209-225)."""
    return _resample("c1", w, b, seed, warp, part, strict, rng, "metropolis_c1")


def metropolis_c2(w, b: int, part: PartitionConfig, warp: WarpConfig = WarpConfig(), seed=0, strict: bool = True,
                  *, rng: str = "megores"):
    """A fresh shared partition per warp at every round (M/resample.py:228-244)."""
    return _resample("c2", w, b, seed, warp, part, strict, rng, "metropolis_c2")


def megopolis(w, b: int, warp: WarpConfig = WarpConfig(), seed=0, strict: bool = True, *, rng: str = "megores"):
    """Shared global offsets with warp-aligned wrapped-sequential reads (M/resample.py:268-282)."""
    return _resample("megopolis", w, b, seed, warp, None, strict, rng, "megopolis")


def multinomial(w, seed):
    """Per-particle uniform draw located in the prefix sum by binary search (M/resample.py:295-304).

    The prefix sum is numpy's sequential float32/float64 ``np.cumsum`` order, reproduced
    bit for bit on the device (``inclusive_prefix``)."""
    return _resample("multinomial", w, 1, seed, None, None, False, "megores", "multinomial")


def systematic_improved(w, seed, warp: WarpConfig = WarpConfig()):
    """Stratified selection with one shared u (M/resample.py:307-336); each particle's
    bracket is found by a binary search of the exact prefix sum (same result as the
    reference's lockstep forward/backward scans)."""
    return _resample("systematic", w, 1, seed, None, None, False, "megores", "systematic_improved")


def systematic_oracle(w, u: float):
    """Sequential single-pass stratified reference for a given u in [0, 1) (M/resample.py:339-354),
    with the reference's comparison semantics (float32 weights: float32 comparison against
    float32(target), NumPy 2 weak-scalar promotion).  numpy in -> numpy out."""
    u = float(u)
    if not (0.0 <= u < 1.0):
        raise ValueError(f"u must be in [0, 1), got {u}")
    D.require_cuda()
    t = D.torch()
    w = _as_weight_vector(w)
    host = not w.on_device
    vals = t.from_numpy(np.ascontiguousarray(w.values)).cuda() if host else w.values.contiguous()
    if (w.stats().n_pos if not host else int(np.any(w.values > 0))) == 0:
        raise ValueError("all weights are zero")
    out = t.empty(vals.numel(), dtype=t.int64, device=vals.device)
    with t.cuda.device(vals.device):
        _lib.check(_lib.lib().mgp_systematic_oracle(D.ptr(vals), D.wdtype(vals), vals.numel(), u, D.ptr(out),
                                                    D.stream_ptr()))
    return out.cpu().numpy() if host else out


def inclusive_prefix(w):
    """``np.cumsum(values)`` in the weights' dtype, bit-identical to numpy's sequential
    scan (M/resample.py:288-291).  numpy in -> numpy out; CUDA tensor in -> CUDA tensor out."""
    D.require_cuda()
    t = D.torch()
    w = _as_weight_vector(w)
    host = not w.on_device
    vals = t.from_numpy(np.ascontiguousarray(w.values)).cuda() if host else w.values.contiguous()
    out = t.empty_like(vals)
    with t.cuda.device(vals.device):
        _lib.check(_lib.lib().mgp_cumsum(D.ptr(vals), D.wdtype(vals), vals.numel(), D.ptr(out), D.stream_ptr()))
    return out.cpu().numpy() if host else out


def megopolis_index(i: int, o_b: int, warp: WarpConfig, n: int) -> int:
    """Wrapped-sequential comparison index (M/resample.py:247-260); host helper."""
    if not (0 <= i < n) or not (0 <= o_b < n):
        raise ValueError("i and o_b must lie in [0, N)")
    ws = warp.warp_size
    return (i - i % ws + o_b - o_b % ws + (i + o_b) % ws) % n


def megopolis_offsets(n: int, b: int, seed, *, rng: str = "megores") -> np.ndarray:
    """The shared offset list: B uniform integers on the reserved global lane (M/resample.py:263-265)."""
    out = np.empty(max(int(b), 1), dtype=np.int64)
    _lib.check(_lib.lib().mgp_offsets_host(_seed(seed), int(n), int(b), _rng(rng), D.ptr(out)))
    return out[: int(b)]


def make_resampler(kind: str, warp: WarpConfig = WarpConfig(), partition_bytes: int | None = None,
                   strict: bool = True, *, rng: str = "megores"):
    """Bind an algorithm id to a uniform ``fn(w, b, seed) -> ancestors`` (M/resample.py:431-455)."""
    if kind == "metropolis":
        return lambda w, b, seed: metropolis(w, b, seed, rng=rng)
    if kind in ("c1", "c2"):
        if partition_bytes is None:
            raise ValueError(f"{kind} requires a partition size")
        part = PartitionConfig(partition_bytes)
        fn = metropolis_c1 if kind == "c1" else metropolis_c2
        return lambda w, b, seed: fn(w, b, part, warp, seed, strict, rng=rng)
    if kind == "megopolis":
        return lambda w, b, seed: megopolis(w, b, warp, seed, strict, rng=rng)
    if kind == "multinomial":  # the prefix-sum methods ignore b (M/resample.py:450-454)
        return lambda w, b, seed: multinomial(w, seed)
    if kind == "systematic":
        return lambda w, b, seed: systematic_improved(w, seed, warp)
    raise ValueError(f"unknown resampler {kind!r}")


def ancestors_to_offspring(ancestors, n: int | None = None):
    """Count how many particles chose each index as their ancestor (M/resample.py:361-368).

    Device histogram with warp-aggregated atomics.  numpy in -> numpy out;
    CUDA tensor in -> CUDA tensor out."""
    D.require_cuda()
    t = D.torch()
    host = not D.is_cuda_tensor(ancestors)
    dev = t.device("cuda") if host else ancestors.device
    a = D.as_index_tensor(ancestors, dev)
    n = a.numel() if n is None else int(n)
    counts = t.empty(max(n, 1), dtype=t.int64, device=dev)
    bad = t.zeros(1, dtype=t.int32, device=dev)
    with t.cuda.device(dev):
        _lib.check(_lib.lib().mgp_offspring(D.ptr(a), a.numel(), n, D.ptr(counts), D.ptr(bad), D.stream_ptr()))
        if a.numel() and int(bad.item()):
            raise ValueError("ancestor indices out of range")
    counts = counts[:n]
    return counts.cpu().numpy() if host else counts


def apply_ancestors(states, ancestors):
    """Gather states by ancestor index into a fresh array (M/resample.py:371-377).

    Rows of any dtype/shape (states[N, ...]); numpy in -> numpy out."""
    D.require_cuda()
    t = D.torch()
    host = not D.is_cuda_tensor(states)
    if host:
        s_np = np.ascontiguousarray(np.asarray(states))
        n_states = len(s_np)
    else:
        n_states = states.shape[0]
    n_anc = len(ancestors) if not D.is_tensor(ancestors) else ancestors.shape[0]
    if n_states != n_anc:
        raise ValueError(f"length mismatch: {n_states} states vs {n_anc} ancestors")
    dev = t.device("cuda") if host else states.device
    a = D.as_index_tensor(ancestors, dev)
    if a.numel() and (int(a.min()) < 0 or int(a.max()) >= n_states):
        raise IndexError("ancestor index out of range")
    if host:
        src = t.from_numpy(s_np.view(np.uint8).reshape(n_states, -1) if s_np.size else
                           np.zeros((n_states, 0), np.uint8)).to(dev)
    else:
        src = states.contiguous()
    out = t.empty_like(src)
    row_bytes = (src.numel() * src.element_size()) // max(n_states, 1)
    with t.cuda.device(dev):
        _lib.check(_lib.lib().mgp_gather(D.ptr(src), row_bytes, D.ptr(a), n_states, D.ptr(out), D.stream_ptr()))
    if host:
        return out.cpu().numpy().view(s_np.dtype).reshape(s_np.shape)
    return out


def comparison_indices(kind: str, n: int, b: int, seed, warp: WarpConfig = WarpConfig(),
                       partition_bytes: int | None = None, device: bool = False):
    """The (B, N) matrix of weight indices each resampler reads, per round (M/resample.py:384-428).

    Entry [r, i] is the index particle i compares against at round r, from the kernels' own
    draw conventions (reference stream), computed on the device (mgp_comparison_indices).
    Returns ``np.int64`` like the reference, or the CUDA tensor with ``device=True``."""
    D.require_cuda()
    t = D.torch()
    if kind not in METROPOLIS_FAMILY:
        raise ValueError(f"unknown Metropolis-family resampler {kind!r}")
    if kind in ("c1", "c2"):
        if partition_bytes is None:
            raise ValueError(f"{kind} requires a partition size")
        PartitionConfig(partition_bytes).n_partitions(n, warp)
    out = t.empty((int(b), int(n)), dtype=t.int64, device="cuda")
    _lib.check(_lib.lib().mgp_comparison_indices(_lib.KIND[kind], int(n), int(b), int(np.uint64(seed)),
                                                 int(warp.warp_size), int(partition_bytes or 0),
                                                 int(warp.word_bytes), D.ptr(out), D.stream_ptr()))
    return out if device else out.cpu().numpy()
