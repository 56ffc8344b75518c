"""Multi-process (world sizes 2-4, gloo, CPU) tests of the sharded protocol: weight
all-gather, per-slice resampling with global indices, the B rule (slice tree or replicated
array), the cross-rank state exchange (all-to-all and the fused resample + gather), sharded
offspring counts and quality statistics, and the prefix-sum kinds.

The CUDA kernels are replaced by the CPU oracle through ShardedResampler's ``ops``
hook (test infrastructure only); the GPU path is covered by tests/test_parity_gpu.py
and, with real CUDA IPC mappings between processes, by tests/test_ipc_gpu.py.  The cases of a
test run in one process group per world size (spawning costs seconds per group).
"""

import os
import queue
import socket
import sys
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Stats:
    def __init__(self, w):
        from oracle import oracle

        v = w.numpy()
        self.n_nonfinite = int((~np.isfinite(v)).sum())
        self.n_neg = int((v < 0).sum())
        self.n_pos = int((v > 0).sum())
        self.n_zero = int((v == 0).sum())
        self.n_notnormal = int((~np.isfinite(v) | (v <= 0) | (np.abs(v) < np.finfo(v.dtype).tiny)).sum())
        self.n = len(v)
        self.mean, self.max = oracle.weight_mean_max(v)
        self.sum = oracle.pairwise_sum(np.asarray(v, dtype=np.float64))


class OracleOps:
    """CPU stand-in for CudaOps (test infrastructure)."""

    def stats(self, w_full):
        return _Stats(w_full)

    @staticmethod
    def _full(kind, w, b, seed, warp, partition_bytes, strict, rng, **kw):
        from oracle import oracle

        if kind in ("multinomial", "systematic"):
            return getattr(oracle, kind)(w, seed)
        return oracle.resample(kind, w, b, seed, warp, partition_bytes, strict, rng, **kw)

    def resample_range(self, kind, w_full, b, seed, warp, partition_bytes, strict, rng, nonzero, p0, p1):
        anc = self._full(kind, w_full.numpy(), b, seed, warp, partition_bytes, strict, rng)
        return torch.from_numpy(anc[p0:p1].copy())

    def resample_stripes(self, kind, w_full, b, seed, warp, partition_bytes, strict, rng, nonzero, lo0, lo1):
        half = w_full.numel() // 2
        anc = self._full(kind, w_full.numpy(), b, seed, warp, partition_bytes, strict, rng)
        return torch.from_numpy(np.concatenate([anc[lo0:lo1], anc[half + lo0:half + lo1]]))

    def resample_gather(self, kind, w_full, b, seed, warp, partition_bytes, strict, rng, nonzero, layout, p0, p1,
                        peer_states):
        """ancestors as above, then each row read from its owner's array (the fused kernel's
        owner mapping, mgp_kernels.cuh store_result / k_gather_peers)."""
        args = (kind, w_full, b, seed, warp, partition_bytes, strict, rng, nonzero, p0, p1)
        anc = (self.resample_stripes if layout == "stripes" else self.resample_range)(*args)
        n_local, half = peer_states[0].shape[0], w_full.numel() // 2
        rows = []
        for a in anc.tolist():
            if layout == "stripes":
                up = a >= half
                k = a - up * half
                owner, local = k // (n_local // 2), k % (n_local // 2) + up * (n_local // 2)
            else:
                owner, local = divmod(a, n_local)
            rows.append(peer_states[owner][local])
        return anc, torch.stack(rows)

    def offspring(self, local_idx, n_local):
        return torch.from_numpy(np.bincount(local_idx.numpy(), minlength=n_local).astype(np.int64))

    def expected_slice(self, w_slice, n_all, total):  # M/metrics.py:55-60 on a slice
        return torch.from_numpy(n_all * np.asarray(w_slice.numpy(), dtype=np.float64) / total)

    def quality_add(self, counts, e, acc_sum, acc_sumsq):  # M/metrics.py:86-93 on a segment
        o = counts.numpy().astype(np.float64)
        acc_sum += torch.from_numpy(o)
        acc_sumsq += torch.from_numpy(o * o)
        return float(((o - e.numpy()) ** 2).sum())

    def quality_finalize(self, acc_sum, acc_sumsq, e, k):  # M/metrics.py:95-110 on a segment
        mean = acc_sum.numpy() / k
        return float((acc_sumsq.numpy() / k - mean * mean).sum()), float(((mean - e.numpy()) ** 2).sum())

    def gather_rows(self, states, idx):
        return states[idx]


def _worker_stripes(rank, world, case, q):
    from oracle import oracle
    from paper_2109_13504_b200.distributed import ShardedResampler

    kind, n_local, y, prec, rng, b = case
    n, h = n_local * world, n_local // 2
    w_full = oracle.gen_gaussian_weights(y, n, 4343, prec)
    sr = ShardedResampler(kind=kind, partition_bytes=128 if kind in ("c1", "c2") else None, rng=rng,
                          ops=OracleOps(), layout="stripes")
    (a0, a1), (b0, b1) = sr.owned(n_local)
    w_local = torch.from_numpy(np.concatenate([w_full[a0:a1], w_full[b0:b1]]))
    anc_local, b_used = sr.resample(w_local, b=b, seed=77)
    states_full = np.stack([np.arange(n, dtype=np.float64) * 1.5, np.arange(n, dtype=np.float64)], axis=1)
    s_local = torch.from_numpy(np.concatenate([states_full[a0:a1], states_full[b0:b1]]))
    new_local = sr.exchange(s_local, anc_local)
    # the fused path: every rank's state array addressable here (peer mappings, emulated)
    peers = [torch.zeros_like(s_local) for _ in range(world)]
    dist.all_gather(peers, s_local)
    anc_f, rows_f, b_f = sr.resample_gather(w_local, peers, b=b, seed=77)
    assert b_f == b_used and torch.equal(anc_f, anc_local) and torch.equal(rows_f, new_local)
    parts = [torch.zeros(n_local, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, anc_local)
    news = [torch.zeros_like(new_local) for _ in range(world)]
    dist.all_gather(news, new_local)
    if rank == 0:  # back to global particle order
        anc = np.concatenate([p[:h].numpy() for p in parts] + [p[h:].numpy() for p in parts])
        st = np.concatenate([x[:h].numpy() for x in news] + [x[h:].numpy() for x in news])
        q.put((int(b_used), anc, st))


def _worker(rank, world, case, q):
    from oracle import oracle
    from paper_2109_13504_b200.distributed import ShardedResampler
    from paper_2109_13504_b200.resample import WarpConfig

    kind, n_local, y, prec, rng, b = case
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(y, n, 4242, prec)
    w_local = torch.from_numpy(w_full[rank * n_local:(rank + 1) * n_local].copy())
    sr = ShardedResampler(kind=kind, warp=WarpConfig(), partition_bytes=128 if kind in ("c1", "c2") else None,
                          rng=rng, ops=OracleOps())
    anc_local, b_used = sr.resample(w_local, b=b, seed=99)
    # every rank derived the same B
    bt = torch.tensor([b_used])
    bs = [torch.zeros(1, dtype=bt.dtype) for _ in range(world)]
    dist.all_gather(bs, bt)
    parts = [torch.zeros(n_local, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, anc_local)
    # state exchange: states are (value, index) rows
    states_full = np.stack([np.arange(n, dtype=np.float64) * 1.5, np.arange(n, dtype=np.float64)], axis=1)
    s_local = torch.from_numpy(states_full[rank * n_local:(rank + 1) * n_local].copy())
    new_local = sr.exchange(s_local, anc_local)
    peers = [torch.zeros_like(s_local) for _ in range(world)]
    dist.all_gather(peers, s_local)
    anc_f, rows_f, b_f = sr.resample_gather(w_local, peers, b=b, seed=99)
    assert b_f == b_used and torch.equal(anc_f, anc_local) and torch.equal(rows_f, new_local)
    news = [torch.zeros_like(new_local) for _ in range(world)]
    dist.all_gather(news, new_local)
    if rank == 0:
        q.put((int(b_used), [int(x) for x in bs], torch.cat(parts).numpy(), torch.cat(news).numpy()))


def _worker_quality(rank, world, case, q):
    """K runs of the sharded resampler -> sharded offspring -> ShardedQuality, against the
    reference's own single-process QualityAccumulator arithmetic (numpy) on the same runs."""
    from oracle import oracle
    from paper_2109_13504_b200.distributed import ShardedResampler

    layout, n_local, y, rng, runs = case
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(y, n, 4545, "single")
    sr = ShardedResampler(rng=rng, ops=OracleOps(), layout=layout)
    idx = np.concatenate([np.arange(lo, hi) for lo, hi in sr.owned(n_local)])
    w_local = torch.from_numpy(w_full[idx].copy())
    acc = sr.quality(w_local)
    for k in range(runs):
        anc_local, _ = sr.resample(w_local, b=7, seed=1000 + k)
        counts = sr.offspring(anc_local)
        acc.add(counts)
    st = acc.finalize()
    if rank == 0:
        q.put((acc.aligned, st))


class _Collect:
    def __init__(self):
        self.items = []

    def put(self, x):
        self.items.append(x)


def _batch(rank, world, port, fn, cases, q):
    """One process group, every case of a test in turn (spawning per case costs seconds)."""
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for case in cases:
            c = _Collect()
            fn(rank, world, case, c)
            out.append(c.items[0] if c.items else None)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _run(world, cases, target=None):
    """Run ``target`` (default _worker) for every case on ``world`` gloo ranks; rank 0's results."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_batch, args=(r, world, port, target or _worker, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, t0 = None, time.time()
    try:
        while res is None and time.time() - t0 < 600:
            try:
                res = q.get(timeout=1)
            except queue.Empty:
                if any(p.exitcode not in (None, 0) for p in procs):
                    break
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return res


SHARDED_CASES = [
    ("megopolis", 512, 3.0, "single", "megores", None),
    ("megopolis", 256, 1.0, "double", "philox", 9),
    ("metropolis", 320, 2.0, "single", "megores", 7),
    ("c1", 256, 4.0, "single", "megores", None),
    ("c2", 256, 0.0, "single", "philox", 5),
]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_single_process(oracle, world):
    for case, got in zip(SHARDED_CASES, _run(world, SHARDED_CASES)):
        _check_sharded(oracle, world, case, got)


def _check_sharded(oracle, world, case, got):
    kind, n_local, y, prec, rng, b = case
    b_used, bs, anc, states = got
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(y, n, 4242, prec)
    if b is None:
        mean, mx = oracle.weight_mean_max(w_full)
        assert b_used == oracle.compute_iterations(0.01, mean, mx)
    assert bs == [b_used] * world
    ref = oracle.resample(kind, w_full, b_used, 99, 32, 128 if kind in ("c1", "c2") else None, True, rng)
    assert np.array_equal(anc, ref)
    states_full = np.stack([np.arange(n) * 1.5, np.arange(n)], axis=1)
    assert np.array_equal(states, states_full[ref])


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("n_local", [72, 1000, 4096, 3 * 1024 + 8])
def test_slice_stats_combine_bit_exact(oracle, world, n_local):
    """Per-rank slice sums combined in numpy's tree order == the pairwise sum of the whole
    array, bit for bit (the B rule of the sharded path without reducing the replicated array)."""
    from paper_2109_13504_b200.distributed import combine_slice_stats, slice_tree_aligned

    assert slice_tree_aligned(world, n_local)
    w = oracle.gen_gaussian_weights(2.5, world * n_local, 77 + n_local, "single")
    parts = [_Stats(torch.from_numpy(w[r * n_local:(r + 1) * n_local])) for r in range(world)]
    for p in parts:
        p.n_neg, p.n_nonfinite = 0, 0
    g = combine_slice_stats(parts)
    total = oracle.pairwise_sum(np.asarray(w, dtype=np.float64))
    mean, mx = oracle.weight_mean_max(w)
    assert g.sum == total and g.mean == mean and g.max == mx and g.n == world * n_local
    assert not slice_tree_aligned(3, 1024) and not slice_tree_aligned(2, 60) and not slice_tree_aligned(2, 1001)


STRIPES_CASES = [
    ("megopolis", 512, 4.0, "single", "philox", None),
    ("megopolis", 192, 2.0, "double", "megores", 5),
    ("c2", 256, 1.0, "single", "megores", 4),
]


@pytest.mark.parametrize("world", [2, 4])
def test_stripes_layout_equals_single_process(oracle, world):
    """layout="stripes": rank r owns stripe r of each half (the half-split kernel's pairing);
    ancestors, the slice-statistics B and the exchanged states equal the single process's."""
    for case, got in zip(STRIPES_CASES, _run(world, STRIPES_CASES, _worker_stripes)):
        _check_stripes(oracle, world, case, got)


def _check_stripes(oracle, world, case, got):
    kind, n_local, y, prec, rng, b = case
    b_used, anc, states = got
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(y, n, 4343, prec)
    if b is None:
        mean, mx = oracle.weight_mean_max(w_full)
        assert b_used == oracle.compute_iterations(0.01, mean, mx)
    ref = oracle.resample(kind, w_full, b_used, 77, 32, 128 if kind in ("c1", "c2") else None, True, rng)
    assert np.array_equal(anc, ref)
    states_full = np.stack([np.arange(n) * 1.5, np.arange(n)], axis=1)
    assert np.array_equal(states, states_full[ref])



QUALITY_CASES = {
    2: [("contiguous", 256, 2.0, "philox", 3), ("stripes", 512, 1.0, "philox", 2),
        ("contiguous", 48, 2.0, "megores", 3)],  # the last is not tree-aligned: the all-gather route
    4: [("stripes", 256, 3.0, "megores", 3)],
}


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_offspring_quality(oracle, world):
    """ShardedResampler.offspring + ShardedQuality equal the reference's QualityAccumulator
    (M/metrics.py:71-110, numpy) over the same K runs of the whole population, bit for bit."""
    cases = QUALITY_CASES[world]
    for case, got in zip(cases, _run(world, cases, _worker_quality)):
        _check_quality(oracle, world, case, got)


def _check_quality(oracle, world, case, got):
    layout, n_local, y, rng, runs = case
    aligned, st = got
    assert aligned == (n_local >= 128 or (layout == "contiguous" and n_local > 64))
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(y, n, 4545, "single")
    v = w_full.astype(np.float64)
    e = len(v) * v / v.sum()
    s1, s2, se = np.zeros(n), np.zeros(n), 0.0
    for k in range(runs):
        o = np.bincount(oracle.resample("megopolis", w_full, 7, 1000 + k, 32, None, True, rng),
                        minlength=n).astype(np.float64)
        s1 += o
        s2 += o * o
        se += float(((o - e) ** 2).sum())
    mean = s1 / runs
    assert st.mse == se / runs
    assert st.variance == float((s2 / runs - mean * mean).sum())
    assert st.bias_sq == float(((mean - e) ** 2).sum())
    assert st.mse_per_particle == st.mse / n


PREFIX_CASES = {2: [("multinomial", "contiguous", 200, "double")], 4: [("systematic", "stripes", 256, "single")],
                3: [("systematic", "contiguous", 100, "single")]}


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_prefix_resamplers(oracle, world):
    """Sharded multinomial / systematic (every rank scans the replicated weights, searches its own
    particles): the ancestors in global order equal the single-process prefix-sum resampler."""
    cases = PREFIX_CASES[world]
    for case, got in zip(cases, _run(world, cases, _worker_prefix)):
        _check_prefix(oracle, world, case, got)


def _check_prefix(oracle, world, case, got):
    kind, layout, n_local, prec = case
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(2.0, n, 4646, prec)
    assert np.array_equal(got, getattr(oracle, kind)(w_full, 321))


def _worker_prefix(rank, world, case, q):
    from oracle import oracle
    from paper_2109_13504_b200.distributed import ShardedResampler

    kind, layout, n_local, prec = case
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(2.0, n, 4646, prec)
    sr = ShardedResampler(kind=kind, ops=OracleOps(), layout=layout)
    idx = np.concatenate([np.arange(lo, hi) for lo, hi in sr.owned(n_local)])
    anc_local, b = sr.resample(torch.from_numpy(w_full[idx].copy()), seed=321)
    parts = [torch.zeros(n_local, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, anc_local)
    if rank == 0:
        if layout == "stripes":
            h = n_local // 2
            q.put(np.concatenate([p[:h].numpy() for p in parts] + [p[h:].numpy() for p in parts]))
        else:
            q.put(torch.cat(parts).numpy())
