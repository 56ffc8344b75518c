"""Sharded resampling across GPUs (one process per GPU, torch.distributed over NCCL).

Layout: rank r owns particles [r*n_local, (r+1)*n_local) of a global
population of N = world * n_local.  Each particle's ancestor depends on the FULL
weight vector, the shared offsets and the seed only (M/resample.py:185-197), so:

  1. weights: the per-rank slices are all-gathered into a replicated f32[N]
     (the one real exchange of the path; 4N bytes over NVLink),
  2. B rule: numpy's pairwise tree (np.asarray(w, f64).mean(), M/bench.py:119) splits an
     array of N = 2^g * n_local elements exactly at the rank boundaries when world = 2^g
     and n_local % 8 == 0, n_local > 64 (each split is n2 = len/2 - (len/2) % 8); every
     rank's slice sum is then a node of the global tree, so each rank reduces only its
     own slice and the world slice sums are combined in the tree's order after a tiny
     all-gather -- bit-identical to the single-GPU B, and overlapped with the weight
     all-gather.  Other shapes reduce the replicated array with the same tree,
  3. offsets: derived from the seed on every rank (no collective),
  4. resample: each rank runs the kernel on its particle slice (global indices),
  5. states: apply_ancestors needs rows owned by other ranks -- exchanged with
     all-to-all (bucketed by owner) or read directly from peer memory
     (``gather_from_peers`` / mgp_gather_peers, or fused into the resampling kernel by
     ``ShardedResampler.resample_gather``) through CUDA IPC mappings (``PeerRows``).

The concatenation of every rank's ancestors equals the single-GPU result, which
equals the reference's, bit for bit.

Compute goes through ``ops`` (default: libmgp.so on the current CUDA device).  The
multi-process tests inject a CPU implementation to exercise the protocol with the
gloo backend on machines without GPUs; the product path has no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _device as D
from . import _lib
from .resample import PartitionConfig, WarpConfig, abi_partition_bytes
from .weights import WeightStats, compute_iterations, device_stats


PREFIX_KINDS = ("multinomial", "systematic")


def slice_tree_aligned(world: int, n_local: int) -> bool:
    """True when numpy's pairwise summation tree over world * n_local elements has every
    rank slice as a subtree (see module docstring)."""
    return world >= 1 and (world & (world - 1)) == 0 and n_local % 8 == 0 and n_local > 64


def tree_sum(values):
    """Combine float64 partial sums of consecutive, equally sized tree-aligned pieces in the
    order of numpy's pairwise tree above them (adjacent pairs, level by level)."""
    vals = [float(v) for v in values]
    if len(vals) & (len(vals) - 1):
        raise ValueError("tree_sum needs a power-of-two number of pieces")
    while len(vals) > 1:
        vals = [vals[2 * i] + vals[2 * i + 1] for i in range(len(vals) // 2)]
    return vals[0]


def combine_slice_stats(parts) -> WeightStats:
    """Global WeightStats from per-rank slice stats in rank order, combining the slice sums
    pairwise exactly like numpy's tree above the slices (requires a power-of-two count)."""
    sums = [p.sum for p in parts]
    while len(sums) > 1:
        sums = [sums[2 * i] + sums[2 * i + 1] for i in range(len(sums) // 2)]
    n = sum(p.n for p in parts)
    total = sums[0]
    return WeightStats(n, total, total / n, max(p.max for p in parts), sum(p.n_pos for p in parts),
                       sum(p.n_zero for p in parts), sum(p.n_neg for p in parts),
                       sum(p.n_nonfinite for p in parts), sum(p.n_notnormal for p in parts))


def _pack(st):
    return [float(st.n), float(st.sum), float(st.max), float(st.n_pos), float(st.n_zero), float(st.n_neg),
            float(st.n_nonfinite), float(st.n_notnormal)]


def _unpack(row):
    v = [float(x) for x in row]
    return WeightStats(int(v[0]), v[1], v[1] / v[0] if v[0] else 0.0, v[2], int(v[3]), int(v[4]), int(v[5]),
                       int(v[6]), int(v[7]))


class CudaOps:
    """libmgp.so on the calling rank's current CUDA device."""

    def stats(self, w_full):
        return device_stats(w_full)

    def resample_range(self, kind, w_full, b, seed, warp, partition_bytes, strict, rng, nonzero, p0, p1):
        t = D.torch()
        out = t.empty(p1 - p0, dtype=t.int64, device=w_full.device)
        flags = _lib.FLAG_NONZERO if nonzero else 0
        _lib.check(_lib.lib().mgp_resample_range(
            _lib.KIND[kind], D.ptr(w_full), D.wdtype(w_full), w_full.numel(), int(b), int(seed) & (2**64 - 1),
            int(warp), int(partition_bytes or 0), int(bool(strict)), _lib.RNG[rng], flags, int(p0), int(p1),
            D.ptr(out), D.stream_ptr()))
        return out

    def resample_stripes(self, kind, w_full, b, seed, warp, partition_bytes, strict, rng, nonzero, lo0, lo1):
        t = D.torch()
        out = t.empty(2 * (lo1 - lo0), dtype=t.int64, device=w_full.device)
        flags = _lib.FLAG_NONZERO if nonzero else 0
        _lib.check(_lib.lib().mgp_resample_stripes(
            _lib.KIND[kind], D.ptr(w_full), D.wdtype(w_full), w_full.numel(), int(b), int(seed) & (2**64 - 1),
            int(warp), int(partition_bytes or 0), int(bool(strict)), _lib.RNG[rng], flags, int(lo0), int(lo1),
            D.ptr(out), D.stream_ptr()))
        return out

    def resample_gather(self, kind, w_full, b, seed, warp, partition_bytes, strict, rng, nonzero, layout, p0, p1,
                        peer_states):
        """mgp_resample_gather: ancestors plus the resampled state rows in one kernel."""
        t = D.torch()
        table, ref = _peer_table(peer_states)
        count = (p1 - p0) * (2 if layout == "stripes" else 1)
        anc = t.empty(count, dtype=t.int64, device=w_full.device)
        out = t.empty((count,) + tuple(ref.shape[1:]), dtype=ref.dtype, device=w_full.device)
        ptrs = (ctypes.c_void_p * len(table))(*table)
        row_bytes = ref[0].numel() * ref.element_size() if ref.shape[0] else 0
        flags = _lib.FLAG_NONZERO if nonzero else 0
        _lib.check(_lib.lib().mgp_resample_gather(
            _lib.KIND[kind], D.ptr(w_full), D.wdtype(w_full), w_full.numel(), int(b), int(seed) & (2**64 - 1),
            int(warp), int(partition_bytes or 0), int(bool(strict)), _lib.RNG[rng], flags,
            1 if layout == "stripes" else 0, int(p0), int(p1), ctypes.cast(ptrs, ctypes.c_void_p), len(table),
            int(ref.shape[0]), row_bytes, D.ptr(anc), D.ptr(out), D.stream_ptr()))
        return anc, out

    def offspring(self, local_idx, n_local):
        """counts[r] = #{i: local_idx[i] == r} (ancestors_to_offspring over this rank's rows)."""
        t = D.torch()
        counts = t.empty(n_local, dtype=t.int64, device=local_idx.device)
        idx = local_idx.to(t.int64).contiguous()
        _lib.check(_lib.lib().mgp_offspring(D.ptr(idx), idx.numel(), n_local, D.ptr(counts), None, D.stream_ptr()))
        return counts

    def expected_slice(self, w_slice, n_all, total):
        t = D.torch()
        e = t.empty(w_slice.numel(), dtype=t.float64, device=w_slice.device)
        _lib.check(_lib.lib().mgp_expected_offspring_slice(D.ptr(w_slice), D.wdtype(w_slice), w_slice.numel(),
                                                           int(n_all), float(total), D.ptr(e), D.stream_ptr()))
        return e

    def quality_add(self, counts, e, acc_sum, acc_sumsq):
        """sum += o, sum_sq += o*o over one segment; returns the segment's pairwise sum((o - e)^2)."""
        t = D.torch()
        se = t.zeros(2, dtype=t.float64, device=counts.device)
        _lib.check(_lib.lib().mgp_quality_add(D.ptr(counts), D.ptr(e), counts.numel(), D.ptr(acc_sum),
                                              D.ptr(acc_sumsq), D.ptr(se), D.ptr(se[1:]), D.stream_ptr()))
        return float(se[1].item())

    def quality_finalize(self, acc_sum, acc_sumsq, e, k):
        """The segment's pairwise sum(sum_sq/k - mean^2) and sum((mean - e)^2)."""
        t = D.torch()
        out = t.empty(2, dtype=t.float64, device=acc_sum.device)
        _lib.check(_lib.lib().mgp_quality_finalize(D.ptr(acc_sum), D.ptr(acc_sumsq), D.ptr(e), acc_sum.numel(), int(k),
                                                   D.ptr(out), D.ptr(out[1:]), D.stream_ptr()))
        v, bsq = out.cpu().tolist()
        return v, bsq

    def gather_rows(self, states, idx):
        t = D.torch()
        src = states.contiguous()
        out = t.empty((idx.numel(),) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 0
        _lib.check(_lib.lib().mgp_gather(D.ptr(src), row_bytes, D.ptr(idx.contiguous()), idx.numel(), D.ptr(out),
                                         D.stream_ptr()))
        return out


@dataclass
class ShardedResampler:
    """A resampler over particles sharded across ranks: the Metropolis family, or the prefix-sum
    methods (every rank scans the replicated weights -- numpy's sequential cumsum, bit-exact --
    and searches for its own particles only)."""

    kind: str = "megopolis"
    warp: WarpConfig = WarpConfig()
    partition_bytes: int | None = None
    strict: bool = True
    rng: str = "megores"
    group: object = None
    ops: object = None
    layout: str = "contiguous"  # or "stripes": rank r owns stripe r of each half of the population
    # run the exchange collectives even at world size 1 (instead of local copies): exercises
    # the NCCL data plane on a single GPU (tests/test_nccl_gpu.py)
    force_collectives: bool = False

    def __post_init__(self):
        import torch.distributed as dist

        self._dist = dist
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        if self.ops is None:
            self.ops = CudaOps()
        if self.kind in ("c1", "c2") and self.partition_bytes is None:
            raise ValueError(f"{self.kind} requires a partition size")
        if self.layout not in ("contiguous", "stripes"):
            raise ValueError(f"unknown layout {self.layout!r}")
        if self.kind in PREFIX_KINDS and self.rng != "megores":
            raise ValueError(f"{self.kind} draws from the reference stream only (rng='megores')")

    # -- ownership --------------------------------------------------------------
    def owned(self, n_local: int):
        """Global particle ranges of this rank's local rows, in local order."""
        r = self.rank
        if self.layout == "contiguous":
            return [(r * n_local, (r + 1) * n_local)]
        h, half = n_local // 2, n_local // 2 * self.world
        return [(r * h, (r + 1) * h), (half + r * h, half + (r + 1) * h)]

    def _owner_local(self, g, n_local):
        """(owner rank, local row) of global particle indices g (tensor)."""
        t = D.torch()
        if self.layout == "contiguous":
            owner = t.div(g, n_local, rounding_mode="floor")
            return owner, g - owner * n_local
        h = n_local // 2
        half = h * self.world
        upper = g >= half
        gl = t.where(upper, g - half, g)
        owner = t.div(gl, h, rounding_mode="floor")
        return owner, gl - owner * h + upper.to(g.dtype) * h

    # -- 1. replicated weights ---------------------------------------------
    def _gather_into(self, out, part):
        if self.world == 1 and not self.force_collectives:
            out.copy_(part)
            return
        try:
            self._dist.all_gather_into_tensor(out, part.contiguous(), group=self.group)
        except (RuntimeError, AttributeError, NotImplementedError):
            self._dist.all_gather(list(out.chunk(self.world)), part.contiguous(), group=self.group)

    def replicate_weights(self, w_local):
        """All-gather the per-rank weight slices (or stripes) into the full replicated vector."""
        t = D.torch()
        n_local = w_local.numel()
        if self.layout == "stripes" and n_local % 2:
            raise ValueError(f"the stripes layout needs an even number of particles per rank, got {n_local}")
        full = t.empty(n_local * self.world, dtype=w_local.dtype, device=w_local.device)
        if self.layout == "contiguous":
            self._gather_into(full, w_local)
        else:
            h, half = n_local // 2, n_local // 2 * self.world
            self._gather_into(full[:half], w_local[:h])
            self._gather_into(full[half:], w_local[h:])
        return full

    # -- 2. weight statistics ---------------------------------------------------
    def global_stats(self, w_local, full=None):
        """Statistics of the global weight vector, bit-identical to one device's pass over it.
        Slice-aligned shapes reduce only the local slice plus a world-sized all-gather of
        8 numbers (float64 carries the counts exactly up to 2^53)."""
        t = D.torch()
        n_local = w_local.numel()
        stripes = self.layout == "stripes"
        unit = n_local // 2 if stripes else n_local  # the tree-aligned piece each rank reduces
        if not slice_tree_aligned(self.world, unit) or (stripes and n_local % 2):
            return self.ops.stats(full if full is not None else self.replicate_weights(w_local))
        pieces = [w_local[:unit], w_local[unit:]] if stripes else [w_local]
        mine = t.tensor(sum((_pack(self.ops.stats(pc)) for pc in pieces), []), dtype=t.float64,
                        device=w_local.device)
        rows = t.empty(self.world * mine.numel(), dtype=t.float64, device=w_local.device)
        self._gather_into(rows, mine)
        per = [_unpack(r) for r in rows.view(self.world * len(pieces), 8).cpu().tolist()]
        if not stripes:
            return combine_slice_stats(per)
        lower = combine_slice_stats(per[0::2])  # root of numpy's tree: lower half + upper half
        upper = combine_slice_stats(per[1::2])
        return combine_slice_stats([lower, upper])

    def _checked_b(self, full, w_local, b, epsilon):
        """The reference's validation (M/weights.py:49-59, M/resample.py:96-108, 84-93) and B."""
        n = full.numel()
        st = self.global_stats(w_local, full)
        self._last_stats = st
        if st.n_nonfinite:
            raise ValueError("weights must be finite")
        if st.n_neg:
            raise ValueError("weights must be non-negative")
        if st.n_pos == 0:
            raise ValueError("all weights are zero")
        if self.kind in PREFIX_KINDS:  # multinomial / systematic take no B (M/resample.py:295-336)
            return 1
        if b is None:
            b = compute_iterations(epsilon, st.mean, st.max).b
        if b < 1:
            raise ValueError(f"B must be >= 1, got {b}")
        if self.kind in ("megopolis", "c1", "c2") and self.strict and n % self.warp.warp_size:
            raise ValueError(f"{self.kind} requires N ({n}) to be a multiple of the warp size "
                             f"({self.warp.warp_size}) in strict mode")
        if self.kind in ("c1", "c2"):
            PartitionConfig(self.partition_bytes).n_partitions(n, self.warp)
        return b

    # -- 2-4. B rule + per-slice resample --------------------------------------
    def resample(self, w_local, b: int | None = None, seed=0, epsilon: float = 0.01):
        """Ancestors (global indices) for this rank's particle slice, and the B used."""
        n_local = w_local.numel()
        full = self.replicate_weights(w_local)
        b = self._checked_b(full, w_local, b, epsilon)
        st = self._last_stats
        args = (self.kind, full, b, seed, self.warp.warp_size, abi_partition_bytes(self.partition_bytes, self.warp),
                self.strict, self.rng,
                st.n_zero == 0)
        if self.layout == "stripes":
            (lo0, lo1), _ = self.owned(n_local)
            return self.ops.resample_stripes(*args, lo0, lo1), b
        p0 = self.rank * n_local
        return self.ops.resample_range(*args, p0, p0 + n_local), b

    def resample_gather(self, w_local, peer_states, b: int | None = None, seed=0, epsilon: float = 0.01):
        """resample + apply_ancestors in one kernel.  ``peer_states``: a PeerRows (every rank's
        state array mapped here by CUDA IPC), or a list whose entry r is rank r's local state
        array as addressable from this device (rank order, this rank's own array included).
        Returns (ancestors, resampled local states, B)."""
        n_local = w_local.numel()
        full = self.replicate_weights(w_local)
        b = self._checked_b(full, w_local, b, epsilon)
        st = self._last_stats
        (p0, p1) = self.owned(n_local)[0]
        anc, rows = self.ops.resample_gather(self.kind, full, b, seed, self.warp.warp_size,
                                             abi_partition_bytes(self.partition_bytes, self.warp),
                                             self.strict, self.rng, st.n_zero == 0, self.layout, p0, p1,
                                             peer_states)
        return anc, rows, b

    def _send_to_owners(self, anc, n_local):
        """Bucket global indices by owner rank and deliver each owner its local row indices
        (one all-to-all of counts, one of indices).  Returns (order, send sizes, receive
        sizes, received local indices)."""
        t = D.torch()
        owner, local = self._owner_local(anc, n_local)
        order = t.argsort(owner, stable=True)
        send_idx = local[order].contiguous()
        send_counts = t.bincount(owner, minlength=self.world).to(t.int64)
        recv_counts = t.empty_like(send_counts)
        self._dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        recv_idx = t.empty(sum(rc), dtype=t.int64, device=anc.device)
        self._dist.all_to_all_single(recv_idx, send_idx, output_split_sizes=rc, input_split_sizes=sc,
                                     group=self.group)
        return order, sc, rc, recv_idx

    # -- 6. offspring counts and quality ----------------------
    def offspring(self, anc_local, n_local: int | None = None):
        """ancestors_to_offspring (M/resample.py:361-368) of the whole population, sharded: the
        counts of this rank's own particles (local order).  Ancestors travel to their owners
        (owner-bucketed all-to-all of local indices, 8 bytes per particle) and each owner
        histograms what it received; the counts equal the single-device histogram's slice."""
        t = D.torch()
        n_local = anc_local.numel() if n_local is None else n_local
        anc = anc_local.to(t.int64)
        n_all = n_local * self.world
        if anc.numel() and (int(anc.min()) < 0 or int(anc.max()) >= n_all):
            raise ValueError("ancestor indices out of range")
        if self.world == 1 and not self.force_collectives:
            return self.ops.offspring(anc, n_local)
        _, _, _, recv_idx = self._send_to_owners(anc, n_local)
        return self.ops.offspring(recv_idx, n_local)

    def quality(self, w_local):
        """A QualityAccumulator over the sharded population (see ShardedQuality)."""
        return ShardedQuality(self, w_local)

    # -- 5. particle states ---------------------------------------------------
    def exchange(self, states_local, anc_local):
        """apply_ancestors across ranks: rows anc_local[i] (global) into a fresh local array.

        Requests are bucketed by owner rank and exchanged with two all-to-alls
        (indices out, rows back)."""
        t = D.torch()
        dist = self._dist
        n_local = states_local.shape[0]
        dev = states_local.device
        anc = anc_local.to(device=dev, dtype=t.int64)
        if self.world == 1 and not self.force_collectives:
            return self.ops.gather_rows(states_local, self._owner_local(anc, n_local)[1])
        order, sc, rc, recv_idx = self._send_to_owners(anc, n_local)
        rows = self.ops.gather_rows(states_local, recv_idx)
        reply = t.empty((sum(sc),) + tuple(states_local.shape[1:]), dtype=states_local.dtype, device=dev)
        dist.all_to_all_single(reply, rows.contiguous(), output_split_sizes=sc, input_split_sizes=rc,
                               group=self.group)
        out = t.empty_like(reply)
        out[order] = reply
        return out


class ShardedQuality:
    """QualityAccumulator (M/metrics.py:71-110) over a population sharded like ``sr``.

    Every rank keeps sum / sum_sq / expected offspring for its own particles only.  The
    reductions over all N particles (the per-run squared error, the final variance and
    squared bias) are numpy pairwise sums; when the ownership pieces are nodes of numpy's
    tree (``slice_tree_aligned``, as for the B rule) each rank reduces its pieces and the
    world's partial sums are combined in the tree's order -- bit-identical to one device's
    accumulator over the whole population.  Other shapes all-gather the counts and run the
    full accumulator on every rank."""

    def __init__(self, sr: ShardedResampler, w_local):
        t = D.torch()
        self.sr = sr
        self.n_local = w_local.numel()
        self.n = self.n_local * sr.world
        self.k = 0
        self._se_total = 0.0
        st = sr.global_stats(w_local)
        if not st.sum > 0:  # M/metrics.py:57-59
            raise ValueError("total weight must be positive")
        stripes = sr.layout == "stripes"
        unit = self.n_local // 2 if stripes else self.n_local
        self.aligned = slice_tree_aligned(sr.world, unit) and not (stripes and self.n_local % 2)
        self.segments = [(0, unit), (unit, self.n_local)] if stripes else [(0, self.n_local)]
        if self.aligned:
            self._e = sr.ops.expected_slice(w_local.contiguous(), self.n, st.sum)
            self._sum = t.zeros(self.n_local, dtype=t.float64, device=w_local.device)
            self._sum_sq = t.zeros_like(self._sum)
        else:
            full = sr.replicate_weights(w_local)
            self._e = sr.ops.expected_slice(full, self.n, st.sum)
            self._sum = t.zeros(self.n, dtype=t.float64, device=w_local.device)
            self._sum_sq = t.zeros_like(self._sum)

    def _combine(self, parts):
        """Partial sums, one per (rank, segment), into numpy's whole-array sum."""
        t = D.torch()
        mine = t.tensor(parts, dtype=t.float64, device=self._sum.device).reshape(-1)
        rows = t.empty(self.sr.world * mine.numel(), dtype=t.float64, device=mine.device)
        self.sr._gather_into(rows, mine)
        per = rows.view(self.sr.world, len(parts), -1).cpu().numpy()
        if len(self.segments) == 1:
            return [tree_sum(per[:, 0, c]) for c in range(per.shape[2])]
        return [tree_sum([tree_sum(per[:, 0, c]), tree_sum(per[:, 1, c])]) for c in range(per.shape[2])]

    def _global_counts(self, counts_local):
        """Counts of the whole population in global particle order (unaligned shapes)."""
        t = D.torch()
        every = t.empty(self.n, dtype=t.int64, device=counts_local.device)
        if self.sr.layout == "contiguous":
            self.sr._gather_into(every, counts_local.contiguous())
            return every
        h, half = self.n_local // 2, self.n // 2
        self.sr._gather_into(every[:half], counts_local[:h].contiguous())
        self.sr._gather_into(every[half:], counts_local[h:].contiguous())
        return every

    def add(self, counts_local) -> None:
        """One run: ``counts_local`` = this rank's slice of the offspring vector (e.g. from
        ``ShardedResampler.offspring``)."""
        t = D.torch()
        o = counts_local.to(device=self._sum.device, dtype=t.int64).contiguous()
        if o.numel() != self.n_local:
            raise ValueError(f"length mismatch: {o.numel()} offspring vs {self.n_local} local weights")
        ops = self.sr.ops
        if self.aligned:
            se = [ops.quality_add(o[a:b], self._e[a:b], self._sum[a:b], self._sum_sq[a:b]) for a, b in self.segments]
            run = self._combine([[v] for v in se])[0]
        else:
            run = ops.quality_add(self._global_counts(o), self._e, self._sum, self._sum_sq)
        self.k += 1
        self._se_total += float(run)

    def finalize(self):
        from .metrics import QualityStats

        if self.k < 2:
            raise ValueError(f"need at least 2 runs to estimate variance, got {self.k}")
        ops = self.sr.ops
        if self.aligned:
            parts = [list(ops.quality_finalize(self._sum[a:b], self._sum_sq[a:b], self._e[a:b], self.k))
                     for a, b in self.segments]
            variance, bias_sq = self._combine(parts)
        else:
            variance, bias_sq = ops.quality_finalize(self._sum, self._sum_sq, self._e, self.k)
        mse = self._se_total / self.k
        contribution = bias_sq / mse if mse > 0 else 0.0
        return QualityStats(mse=mse, variance=float(variance), bias_sq=float(bias_sq),
                            bias_contribution=contribution, mse_per_particle=mse / self.n)


class PeerRows:
    """Every rank's particle-state array, addressable from this device (CUDA IPC mappings).

    Collective: each rank passes its own ``states_local`` (same row shape and dtype on every
    rank, allocated on its GPU); the handles travel by one all_gather_object and each rank
    maps its peers' arrays (mgp_ipc_open; peer access over NVLink is enabled lazily).
    ``ptrs[r]`` is rank r's array as seen here (this rank's own pointer unmapped).  The
    arrays must stay alive and in place while mapped; ``close()`` unmaps.  Pass the
    object to ``ShardedResampler.resample_gather`` or ``gather_from_peers``."""

    def __init__(self, states_local, group=None):
        import torch.distributed as dist

        t = D.torch()
        if not states_local.is_cuda or not states_local.is_contiguous():
            raise ValueError("states_local must be a contiguous CUDA tensor")
        self.template = states_local
        self.rows_local = states_local.shape[0]
        L = _lib.lib()
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64(0)
        _lib.check(L.mgp_ipc_export(ctypes.c_void_p(states_local.data_ptr()), h, ctypes.byref(off)))
        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        mine = (bytes(h.raw), int(off.value), tuple(states_local.shape), str(states_local.dtype),
                t.cuda.current_device())
        every = [None] * world
        dist.all_gather_object(every, mine, group=group)
        self.ptrs, self._opened = [], []
        for r, (hr, offr, shape, dtype, _) in enumerate(every):
            if shape != mine[2] or dtype != mine[3]:
                raise ValueError(f"rank {r} holds states {shape} {dtype}, this rank {mine[2]} {mine[3]}")
            if r == rank:
                self.ptrs.append(states_local.data_ptr())
                continue
            p = ctypes.c_void_p(0)
            _lib.check(L.mgp_ipc_open(ctypes.create_string_buffer(hr, 64), offr, ctypes.byref(p)))
            self.ptrs.append(p.value)
            self._opened.append((p.value, offr))

    def __len__(self):
        return len(self.ptrs)

    def close(self):
        for p, off in self._opened:
            _lib.check(_lib.lib().mgp_ipc_close(ctypes.c_void_p(p), off))
        self._opened = []


def _peer_table(peer_states):
    """(pointers, template tensor) from a PeerRows or a list of tensors / raw pointers."""
    if isinstance(peer_states, PeerRows):
        return list(peer_states.ptrs), peer_states.template
    ptrs, ref = [], None
    for p in peer_states:
        if D.is_tensor(p):
            ref = p if ref is None else ref
            ptrs.append(p.data_ptr())
        else:
            ptrs.append(int(p))
    if ref is None:
        raise ValueError("at least one peer must be given as a tensor (shape/dtype template)")
    return ptrs, ref


def gather_from_peers(peer_states, n_local: int, anc, out=None):
    """out[i] = row anc[i] read directly from its owner's memory (mgp_gather_peers).

    ``peer_states``: one CUDA tensor (or raw device pointer) per rank, each holding
    that rank's n_local rows and addressable from this device (NVLink P2P /
    symmetric memory).  Single-kernel sharded gather: no staging, no all-to-all."""
    t = D.torch()
    ptrs, ref = _peer_table(peer_states)
    anc = anc.to(device=ref.device, dtype=t.int64).contiguous()
    if out is None:
        out = t.empty((anc.numel(),) + tuple(ref.shape[1:]), dtype=ref.dtype, device=ref.device)
    row_bytes = ref[0].numel() * ref.element_size()
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    _lib.check(_lib.lib().mgp_gather_peers(ctypes.cast(arr, ctypes.c_void_p), len(ptrs), int(n_local), row_bytes,
                                           D.ptr(anc), anc.numel(), D.ptr(out), D.stream_ptr()))
    return out


def resample_on_devices(kind: str, w, b: int | None = None, seed=0, devices=None, epsilon: float = 0.01,
                        warp: WarpConfig = WarpConfig(), partition_bytes: int | None = None, strict: bool = True,
                        rng: str = "megores"):
    """One process driving several GPUs (mgp_resample_multi): host weights in, ``np.int64``
    ancestors out, bit-identical to the single-device resampler.  ``devices`` defaults to every
    visible GPU; B follows the epsilon rule when ``b`` is None.  Returns (ancestors, B)."""
    import numpy as np

    from .weights import _as_weight_vector

    D.require_cuda()
    t = D.torch()
    wv = _as_weight_vector(w)
    vals = wv.values.cpu().numpy() if D.is_tensor(wv.values) else np.ascontiguousarray(wv.values)
    devs = list(range(t.cuda.device_count())) if devices is None else [int(d) for d in devices]
    arr = (ctypes.c_int * len(devs))(*devs)
    anc = np.empty(len(vals), dtype=np.int64)
    bu = ctypes.c_int32(0)
    _lib.check(_lib.lib().mgp_resample_multi(
        _lib.KIND[kind], vals.ctypes.data, 0 if vals.dtype == np.float32 else 1, len(vals), int(b or 0),
        float(epsilon), int(seed) & (2**64 - 1), int(warp.warp_size), abi_partition_bytes(partition_bytes, warp),
        int(bool(strict)), _lib.RNG[rng], len(devs), ctypes.cast(arr, ctypes.c_void_p), anc.ctypes.data, ctypes.byref(bu)))
    return anc, int(bu.value)
