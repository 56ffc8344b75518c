"""GPU, multi-process: the sharded state exchange through real peer mappings.

Two (or four) processes share cuda:0 -- the one GPU this run has -- with gloo collectives.
Each rank allocates its own particle-state array; ``PeerRows`` exchanges CUDA IPC handles
and maps the other ranks' arrays (mgp_ipc_export / mgp_ipc_open: the same mechanism that
maps NVLink peer memory on a multi-GPU node).  Then, per rank:

* ``ShardedResampler.resample_gather`` (mgp_resample_gather: resample and read every
  ancestor's state row from its owner's mapped array inside the resampling kernel), both
  ownership layouts, must equal the oracle's ancestors and ``states_full[ancestors]``;
* ``gather_from_peers`` (mgp_gather_peers) must agree with it;
* the all-to-all ``exchange`` must agree with both;
* ``ShardedResampler.offspring`` + ``ShardedQuality`` over two runs must equal the reference's
  QualityAccumulator arithmetic on the whole population, bit for bit.
"""

from __future__ import annotations

import os
import queue
import socket
import sys
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2109_13504_b200.distributed import PeerRows, ShardedResampler, gather_from_peers

        kind, layout, n_local, rng, b = case
        n = n_local * world
        w_full = oracle.gen_gaussian_weights(3.0, n, 777, "single")
        sr = ShardedResampler(kind=kind, rng=rng, layout=layout,
                              partition_bytes=256 if kind in ("c1", "c2") else None)
        idx = np.concatenate([np.arange(lo, hi) for lo, hi in sr.owned(n_local)])
        w_local = torch.from_numpy(w_full[idx].copy()).cuda()
        states_full = torch.stack([torch.arange(n, dtype=torch.float64) * 0.5,
                                   -torch.arange(n, dtype=torch.float64)], 1)
        # a slack allocation so the array is an interior pointer of its block (exercises the offset)
        block = torch.zeros(n_local * 2 + 64, dtype=torch.float64, device="cuda")
        s_local = block[64:].view(n_local, 2)
        s_local.copy_(states_full[torch.from_numpy(idx)].cuda())
        peers = PeerRows(s_local)
        dist.barrier()
        anc, rows, b_used = sr.resample_gather(w_local, peers, b=b, seed=2021)
        torch.cuda.synchronize()
        anc_sep, _ = sr.resample(w_local, b=b, seed=2021)
        assert torch.equal(anc, anc_sep)
        if layout == "contiguous":
            assert torch.equal(gather_from_peers(peers, n_local, anc), rows)
        assert torch.equal(sr.exchange(s_local, anc), rows)
        # sharded offspring counts and quality over two runs (seeds 2021, 2022)
        acc = sr.quality(w_local)
        acc.add(sr.offspring(anc))
        anc2, _ = sr.resample(w_local, b=b, seed=2022)
        acc.add(sr.offspring(anc2))
        qst = acc.finalize()
        torch.cuda.synchronize()
        dist.barrier()  # every rank done reading before anyone unmaps / frees
        peers.close()
        parts = [torch.zeros(n_local, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, anc.cpu())
        news = [torch.zeros(n_local, 2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(news, rows.cpu())
        if rank == 0:
            if layout == "stripes":  # back to global particle order
                h = n_local // 2
                a = np.concatenate([p[:h].numpy() for p in parts] + [p[h:].numpy() for p in parts])
                st = np.concatenate([x[:h].numpy() for x in news] + [x[h:].numpy() for x in news])
            else:
                a = torch.cat(parts).numpy()
                st = torch.cat(news).numpy()
            q.put((int(b_used), a, st, qst))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, ("megopolis", "contiguous", 1 << 14, "philox", None)),
    (2, ("megopolis", "stripes", 1 << 14, "philox", None)),
    (4, ("megopolis", "stripes", 4096, "megores", 7)),
    (2, ("c2", "contiguous", 4096, "megores", 5)),
    (2, ("metropolis", "stripes", 2048, "philox", 4)),
    (2, ("megopolis", "stripes", 1 << 23, "philox", None)),  # N = 2^24 (config 4), B from the rule
    (2, ("multinomial", "contiguous", 4096, "megores", None)),  # prefix-sum kinds: replicated scan
    (2, ("systematic", "stripes", 1 << 16, "megores", None)),
])
def test_peer_rows_resample_gather(oracle, world, case):
    import torch.multiprocessing as mp

    kind, layout, n_local, rng, b = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, t0 = None, time.time()
    try:
        while res is None and time.time() - t0 < 300:
            try:
                res = q.get(timeout=2)
            except queue.Empty:
                if any(p.exitcode not in (None, 0) for p in procs):
                    break
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    b_used, anc, st, qst = res
    n = n_local * world
    w_full = oracle.gen_gaussian_weights(3.0, n, 777, "single")
    if b is None and kind not in ("multinomial", "systematic"):
        mean, mx = oracle.weight_mean_max(w_full)
        assert b_used == oracle.compute_iterations(0.01, mean, mx)
    def full_ref(seed):
        if kind in ("multinomial", "systematic"):
            return getattr(oracle, kind)(w_full, seed)
        return oracle.resample(kind, w_full, b_used, seed, 32, 256 if kind in ("c1", "c2") else None, True, rng)

    ref = full_ref(2021)
    assert np.array_equal(anc, ref)
    states_full = np.stack([np.arange(n) * 0.5, -np.arange(n, dtype=np.float64)], 1)
    assert np.array_equal(st, states_full[ref])
    # ShardedQuality == the reference's QualityAccumulator arithmetic (M/metrics.py:71-110)
    ref2 = full_ref(2022)
    v = w_full.astype(np.float64)
    e = n * v / v.sum()
    o1, o2 = (np.bincount(r, minlength=n).astype(np.float64) for r in (ref, ref2))
    mean = (o1 + o2) / 2
    assert qst.mse == (float(((o1 - e) ** 2).sum()) + float(((o2 - e) ** 2).sum())) / 2
    assert qst.variance == float(((o1 * o1 + o2 * o2) / 2 - mean * mean).sum())
    assert qst.bias_sq == float(((mean - e) ** 2).sum())
