"""Worker for tests/test_nccl_gpu.py, launched by torchrun (one process per GPU; world size 1
on the single-GPU box).  Runs the sharded data plane over NCCL -- the weight all-gathers, the
stats all-gather behind the bit-exact global B, the owner-bucketed all-to-alls of the
offspring counts and of apply_ancestors -- with ``force_collectives`` so that every exchange
is a real NCCL collective even at world size 1, and checks each result bit for bit against
one device's public API on the same global population.  Prints one JSON line (rank 0)."""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2109_13504_b200 as mg
    from paper_2109_13504_b200.distributed import ShardedResampler
    from oracle import oracle  # checker: the reference's weight bytes

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    assert dist.get_backend() == "nccl"
    n = 1 << 20
    w = oracle.gen_gaussian_weights(4.0, n, 4242, "single")
    wd = torch.from_numpy(w).to(dev)
    b = mg.iterations_for(mg.WeightVector(wd, "single"), 0.01).b
    checks = []
    for layout in ("stripes", "contiguous"):
        n_local = n // world
        if layout == "contiguous":
            w_local = wd[rank * n_local:(rank + 1) * n_local]
        else:
            h, half = n_local // 2, n // 2
            w_local = torch.cat([wd[rank * h:(rank + 1) * h], wd[half + rank * h:half + (rank + 1) * h]])
        for kind, rng, part in (("megopolis", "philox", None), ("megopolis", "megores", None),
                                ("metropolis", "megores", None), ("c2", "philox", 256), ("systematic", "megores", None)):
            sr = ShardedResampler(kind=kind, rng=rng, layout=layout, partition_bytes=part, force_collectives=True)
            a_loc, b_used = sr.resample(w_local, seed=99)
            assert b_used == (1 if kind == "systematic" else b)
            full = torch.empty(n, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(full, a_loc.contiguous())  # rank-major [lower | upper] per rank
            got = full.view(world, -1)
            if layout == "stripes":
                hh = n_local // 2
                got = torch.cat([got[:, :hh].reshape(-1), got[:, hh:].reshape(-1)])
            else:
                got = got.reshape(-1)
            fn = mg.make_resampler(kind, partition_bytes=part, rng=rng)
            want = fn(mg.WeightVector(wd, "single"), b, 99)
            ok_anc = bool(torch.equal(got, want))
            # offspring counts through the owner-bucketed all-to-all
            off_loc = sr.offspring(a_loc)
            off_full = torch.empty(n, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(off_full, off_loc.contiguous())
            og = off_full.view(world, -1)
            if layout == "stripes":
                og = torch.cat([og[:, :hh].reshape(-1), og[:, hh:].reshape(-1)])
            else:
                og = og.reshape(-1)
            ok_off = bool(torch.equal(og, mg.ancestors_to_offspring(want, n)))
            checks.append({"layout": layout, "kind": kind, "rng": rng, "ancestors": ok_anc, "offspring": ok_off})
    # quality accumulator over the sharded population vs one device's
    sr = ShardedResampler(kind="megopolis", rng="philox", layout="stripes", force_collectives=True)
    n_local = n // world
    h, half = n_local // 2, n // 2
    w_local = torch.cat([wd[rank * h:(rank + 1) * h], wd[half + rank * h:half + (rank + 1) * h]])
    acc = sr.quality(w_local)
    ref = mg.QualityAccumulator(n)
    for k in range(3):
        a_loc, _ = sr.resample(w_local, b=b, seed=k)
        acc.add(sr.offspring(a_loc))
        ref.add(mg.ancestors_to_offspring(mg.megopolis(mg.WeightVector(wd, "single"), b, seed=k, rng="philox"), n),
                mg.WeightVector(wd, "single"))
    qa, qr = acc.finalize(), ref.finalize()
    ok_q = all(getattr(qa, f) == getattr(qr, f) for f in ("mse", "variance", "bias_sq", "mse_per_particle"))
    # apply_ancestors across ranks through the all-to-all exchange
    states = torch.arange(n, dtype=torch.float64, device=dev) * 0.5
    st_loc = torch.cat([states[rank * h:(rank + 1) * h], states[half + rank * h:half + (rank + 1) * h]])
    a_loc, _ = sr.resample(w_local, b=b, seed=5)
    moved = sr.exchange(st_loc, a_loc)
    ok_x = bool(torch.equal(moved, states[a_loc]))
    dist.barrier()
    if rank == 0:
        print(json.dumps({"world": world, "backend": dist.get_backend(), "n": n, "b": b, "checks": checks,
                          "quality": ok_q, "exchange": ok_x}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
