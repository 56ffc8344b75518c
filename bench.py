#!/usr/bin/env python3
"""Headline benchmark: Megopolis particles resampled per second on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload (BASELINE.json config 4 / metric): Megopolis resampling of N = 2^24
particles per GPU, Gaussian-family float32 weights with y = 4 (high variance),
B from the epsilon = 0.01 rule (B = 354), the reference's megores random stream
(bit-exact with the reference).  One step = one pass of the hot path over one
batch: weight statistics -> B (host, like the reference) -> Megopolis kernel.
Inputs are resident in HBM for ``value``; ``e2e`` runs the same step through the
host-buffer C-ABI entry (pinned host weights in, pinned host ancestors out).

Multi-GPU (weak scaling): a global population of 2^24 * G particles; rank r owns stripe r
of each half ([r*h, (r+1)*h) and N/2 + [r*h, (r+1)*h), h = 2^23: the "stripes" layout of
distributed.ShardedResampler, under which every rank runs the half-split kernel).  Each
step all-gathers the weight stripes over NCCL (the replicated-weights exchange of SURVEY
8e), derives the global B bit-exactly from per-stripe statistics (an all-gather of 16
words, overlapped with the weight all-gather) and resamples the rank's stripes.

The L2 (126 MB) would hold the 64 MiB weight array across steps, so a 256 MiB
buffer is written between timed steps (outside the CUDA-event windows).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Megopolis particles resampled/sec (N=2^24, 1/2/4/8 B200); % roofline; offspring MSE"
N_PER_GPU = 1 << 24
Y = 4.0
EPS = 0.01
RUN_SEED = 7
WEIGHT_SEED = 20240
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--particles", dest="n", type=int, default=N_PER_GPU, help="particles per GPU")
    ap.add_argument("--rng", default="philox", choices=["megores", "philox"],
                    help="headline stream; the other one is measured too and reported under 'streams'")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quality-runs", type=int, default=32)  # K >= 32
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML clock / throttle-reason sampling during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle port (oracle/), all host threads


def cpu_rate(oracle, w, b, budget_s, nthreads, rng):
    """Particles/s of the oracle on a bounded prefix sample of the workload."""
    n = len(w)
    p = 16384
    t0 = time.perf_counter()
    oracle.megopolis(w, b, seed=RUN_SEED, threads=nthreads, p0=0, p1=p, rng=rng)
    dt = time.perf_counter() - t0
    for _ in range(3):  # the small calibration run under-states the threaded rate: re-aim
        if dt >= 0.5 * budget_s or p >= n:
            break
        p = int(min(n, max(4096, p / max(dt, 1e-6) * budget_s)))
        p -= p % 32
        t0 = time.perf_counter()
        oracle.megopolis(w, b, seed=RUN_SEED, threads=nthreads, p0=0, p1=p, rng=rng)
        dt = time.perf_counter() - t0
    return p / dt, p, dt


def host_weights(n_global, rank_slice=None):
    """Synthetic Gaussian-family weights (M/weights.py:100-104) via the device generator."""
    import paper_2109_13504_b200 as mg

    return mg.gen_gaussian_weights(mg.GaussianWeightParams(Y, n_global), WEIGHT_SEED, "single").values


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle

    import torch

    n = args.n
    if torch.cuda.is_available():
        w = host_weights(n).cpu().numpy()
    else:
        w = oracle.gen_gaussian_weights(Y, n, WEIGHT_SEED, "single")
    mean, mx = oracle.weight_mean_max(w)
    b = oracle.compute_iterations(EPS, mean, mx)
    threads = oracle.num_threads()
    per_step_budget = max(2.0, min(15.0, 150.0 / max(1, args.steps + args.warmup)))
    rate, p, dt = cpu_rate(oracle, w, b, per_step_budget, threads, args.rng)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.megopolis(w, b, seed=RUN_SEED, threads=threads, p0=0, p1=p, rng=args.rng)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = p / t
    sample = f"particles [0, {p}) of N={n} (y=4, B={b}), {args.steps} steps of {t:.2f}s"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3 * n / p,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"megopolis N=2^{int(math.log2(n))} y=4 f32 weights B={b} eps=0.01 {args.rng} stream",
                   "N": n, "B": b},
        "cpu_baseline": {"value": value, "unit": "particles/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2109_13504_b200 as mg
    from paper_2109_13504_b200 import _lib
    from paper_2109_13504_b200 import _device as D

    rank, world, local = dist_env()
    # MGP_BENCH_LOOPBACK=1 (test plumbing only): every rank on cuda:0 with gloo collectives, to
    # exercise the sharded step's logic on a one-GPU machine; never used for a reported number
    loopback = os.environ.get("MGP_BENCH_LOOPBACK") == "1"
    if loopback:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if loopback:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()
    n_loc = args.n
    n_glob = n_loc * world

    # weights: rank r owns stripe r of each half of the global population ("stripes" layout of
    # distributed.ShardedResampler: particles [r*h, (r+1)*h) and N/2 + [r*h, (r+1)*h), h = n/2),
    # so every rank runs the half-split Megopolis kernel.  Each rank produces its stripes
    # (device generator, same per-particle stream as the reference generator) and the two
    # halves are all-gathered.
    full = host_weights(n_glob) if world == 1 else None
    h, half = n_loc // 2, n_glob // 2
    lo0, lo1 = rank * h, (rank + 1) * h
    if world > 1:
        gen_full = host_weights(n_glob)  # deterministic; sliced to emulate per-rank production
        local_w = torch.cat([gen_full[lo0:lo1], gen_full[half + lo0:half + lo1]])
        del gen_full
        full = torch.empty(n_glob, dtype=torch.float32, device=dev)
    else:
        local_w = full
    stats = torch.empty(16, dtype=torch.float64, device=dev)
    from paper_2109_13504_b200.distributed import combine_slice_stats, slice_tree_aligned
    from paper_2109_13504_b200.weights import WeightStats

    aligned = n_loc % 2 == 0 and slice_tree_aligned(world, h)
    stats_all = torch.empty(world * 16, dtype=torch.int64, device=dev)
    anc = torch.empty(n_loc, dtype=torch.int64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)

    def gather_weights(async_op=False):
        if world > 1:
            w1 = dist.all_gather_into_tensor(full[:half], local_w[:h], async_op=async_op)
            w2 = dist.all_gather_into_tensor(full[half:], local_w[h:], async_op=async_op)
            return (w1, w2)
        return ()

    def measure(rng_id):
        """W warm-up + K timed steps of the hot path for one random stream."""
        nonlocal_b = [0]

        def step(ev=None):
            """One hot-path pass: (all-gather) -> stats -> B -> megopolis(slice)."""
            if world > 1 and aligned:
                # stripe statistics + a 16-word all-gather give the global B bit for bit
                # (numpy's tree: lower half + upper half, each the rank stripes in order;
                # distributed.combine_slice_stats); the host derives B while the weight
                # all-gathers are still in flight
                _lib.check(L.mgp_weight_stats(D.ptr(local_w), 0, h, D.ptr(stats), sp))
                _lib.check(L.mgp_weight_stats(D.ptr(local_w[h:]), 0, h, D.ptr(stats[8:]), sp))
                ws = dist.all_gather_into_tensor(stats_all, stats.view(torch.int64), async_op=True)
                wws = gather_weights(async_op=True)
                ws.wait()
                rows = stats_all.view(world * 2, 8).cpu().numpy()
                per = [WeightStats(h, *r.view(np.float64)[:3], *r[3:]) for r in rows]
                g = combine_slice_stats([combine_slice_stats(per[0::2]), combine_slice_stats(per[1::2])])
                b = mg.compute_iterations(EPS, g.mean, g.max).b
                flags = _lib.FLAG_NONZERO if g.n_zero == 0 else 0
                for wk in wws:
                    wk.wait()
            else:
                gather_weights()
                _lib.check(L.mgp_weight_stats(D.ptr(full), 0, n_glob, D.ptr(stats), sp))
                host = stats.cpu().numpy()  # 64 B; the reference also derives B on the host
                mean, mx = float(host[1]), float(host[2])
                b = mg.compute_iterations(EPS, mean, mx).b
                flags = _lib.FLAG_NONZERO if host.view(np.int64)[4] == 0 else 0
            if ev is not None:
                ev[0].record(stream)
            if world > 1:
                _lib.check(L.mgp_resample_stripes(_lib.KIND["megopolis"], D.ptr(full), 0, n_glob, b, RUN_SEED, 32, 0,
                                                  1, rng_id, flags, lo0, lo1, D.ptr(anc), sp))
            else:
                _lib.check(L.mgp_resample_range(_lib.KIND["megopolis"], D.ptr(full), 0, n_glob, b, RUN_SEED, 32, 0,
                                                 1, rng_id, flags, 0, n_loc, D.ptr(anc), sp))
            if ev is not None:
                ev[1].record(stream)
            nonlocal_b[0] = b

        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        import gc

        gc.collect()
        gc.disable()
        with ClockSampler(local) as clk:
            for s in range(args.steps):
                flush.fill_(float(s))
                starts[s].record(stream)
                step(kev[s])
                ends[s].record(stream)
            torch.cuda.synchronize()
        gc.enable()
        if world > 1:
            dist.barrier()
        step_ms = [starts[s].elapsed_time(ends[s]) for s in range(args.steps)]
        kern_ms = [kev[s][0].elapsed_time(kev[s][1]) for s in range(args.steps)]
        t_total = sum(step_ms)
        if world > 1:
            tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_total = float(tt.item())
        return {"b": nonlocal_b[0], "ms_per_step": t_total / args.steps, "step_ms": step_ms, "kern_ms": kern_ms,
                "clocks": clk.summary()}

    res = {}
    other = "megores" if args.rng == "philox" else "philox"
    for name in (args.rng, other):
        res[name] = measure(_lib.RNG[name])
    head = res[args.rng]
    b = head["b"]
    ms_per_step = head["ms_per_step"]
    value = n_glob / (ms_per_step / 1e3)  # all ranks' particles per second
    # stats (2 kernels, per stripe when sharded) + megopolis launches
    launches = args.steps * ((4 if world > 1 and aligned else 2) + math.ceil(b / 1024))

    # roofline: algorithmic bytes of one Megopolis launch: N*B*4 + N*4 + N*8 + 8*B
    alg_bytes = n_loc * b * 4 + n_loc * 4 + n_loc * 8 + 8 * b
    peak, peak_src = load_peaks()

    def roof(r):
        kavg = statistics.mean(r["kern_ms"]) / 1e3
        ach = alg_bytes / kavg / 1e9
        return ach, kavg

    achieved, kern_avg = roof(head)
    # Philox launches (full range, or a rank's stripes) take the half-split kernel
    if args.rng == "philox":
        mego_kernel = "k_megopolis_philox_half (half-split, 4 particles/thread)"
    else:
        mego_kernel = "k_megopolis_w32<megores, 1 particle/thread>"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "megopolis_traffic.json")) as f:
            traffic = json.load(f).get(args.rng, {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    # e2e through the host-buffer C-ABI entry (pinned buffers), rank-local population
    e2e = None
    if not args.no_e2e:
        h_w = local_w.cpu().pin_memory() if world > 1 else full.cpu().pin_memory()
        h_anc = torch.empty(n_loc, dtype=torch.int64).pin_memory()
        bu = ctypes.c_int32(0)

        def e2e_time(rid):
            def e2e_step():
                _lib.check(L.mgp_resample_host(_lib.KIND["megopolis"], D.ptr(h_w), 0, n_loc, 0, EPS, RUN_SEED, 32, 0,
                                               1, rid, D.ptr(h_anc), ctypes.byref(bu), local))

            for _ in range(3):
                e2e_step()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = max(3, min(args.steps, 10))
            for _ in range(reps):
                e2e_step()
            te = (time.perf_counter() - t0) / reps
            if world > 1:
                tt = torch.tensor([te], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                te = float(tt.item())
            return te

        te = e2e_time(_lib.RNG[args.rng])
        e2e = {"value": n_loc * world / te, "unit": "particles/s", "h2d_bytes_per_step": 4 * n_loc,
               "d2h_bytes_per_step": 8 * n_loc, "ms_per_step": te * 1e3, "B": int(bu.value),
               "path": "mgp_resample_host (pinned host weights -> device -> pinned host ancestors)"}
        te_o = e2e_time(_lib.RNG[other])
        res[other]["e2e"] = {"value": n_loc * world / te_o, "ms_per_step": te_o * 1e3}

        # the B-rule reduction, H2D (4N B) and D2H (8N B) reported separately
        # (CUDA events, outside the timed region, median of 5)
        def ev_ms(fn, reps=5):
            out = []
            for _ in range(reps):
                a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                z.record(stream)
                z.synchronize()
                out.append(a.elapsed_time(z))
            return statistics.median(out)

        d_w = torch.empty(n_loc, dtype=torch.float32, device=dev)
        h2d = ev_ms(lambda: d_w.copy_(h_w, non_blocking=True))
        d2h = ev_ms(lambda: h_anc.copy_(anc, non_blocking=True))
        brule = ev_ms(lambda: _lib.check(L.mgp_weight_stats(D.ptr(d_w), 0, n_loc, D.ptr(stats), sp)))
        e2e["transfers"] = {"h2d_ms": h2d, "h2d_GBps": 4 * n_loc / h2d / 1e6, "d2h_ms": d2h,
                            "d2h_GBps": 8 * n_loc / d2h / 1e6, "b_rule_ms": brule}
        del d_w

    # quality (offspring MSE / bias, M/metrics.py) outside the timed region.  N > 1: the sharded
    # path (stripes-layout resample -> owner-bucketed offspring -> ShardedQuality), which equals
    # one device's QualityAccumulator over the whole population bit for bit.
    quality = None
    if args.quality_runs >= 2:
        qs = {}
        for kind in ("megopolis", "metropolis"):
            if world == 1:
                wv = mg.WeightVector(full, "single")
                acc = mg.QualityAccumulator(n_glob)
                fn = mg.make_resampler(kind, rng=args.rng)
                for k in range(args.quality_runs):
                    acc.add(mg.ancestors_to_offspring(fn(wv, b, mg.derive_seed(2002, k)), n_glob), wv)
            else:
                from paper_2109_13504_b200.distributed import ShardedResampler

                sr = ShardedResampler(kind=kind, rng=args.rng, layout="stripes")
                acc = sr.quality(local_w)
                for k in range(args.quality_runs):
                    a_loc, _ = sr.resample(local_w, b=b, seed=mg.derive_seed(2002, k))
                    acc.add(sr.offspring(a_loc))
            st = acc.finalize()
            qs[kind] = {"mse_per_particle": st.mse_per_particle, "bias_contribution": st.bias_contribution}
        quality = {"runs": args.quality_runs, **qs, "paper_megopolis_y4": 0.6508, "paper_metropolis": 1.0}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle

        w_np = full[:n_loc].cpu().numpy() if world == 1 else local_w.cpu().numpy()
        rate, p, dt = cpu_rate(oracle, w_np, b, 12.0, oracle.num_threads(), args.rng)
        cpu = {"value": rate, "unit": "particles/s", "cores": oracle.num_threads(), "kind": "port",
               "sample": f"oracle/mgp_oracle.c megopolis ({args.rng} stream), particles [0, {p}) of the same "
                         f"N=2^24 y=4 B={b} workload, {dt:.1f}s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": f"megopolis N=2^{int(math.log2(n_loc))}/GPU y=4 f32 Gaussian weights, B={b} "
                            f"(eps=0.01 rule), {args.rng} stream",
                "N_per_gpu": n_loc, "N_global": n_glob, "B": b, "rng": args.rng,
                "step": "weight stats -> B (host) -> megopolis" + (" (+ NCCL all-gather)" if world > 1 else ""),
                "l2": "flushed between timed steps (256 MiB write, outside the event windows)",
                "parallelism": f"dp{world} weak (replicated weights, particle slices)",
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": mego_kernel, "kernel_ms": kern_avg * 1e3,
                         "alg_bytes_per_launch": alg_bytes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "step_breakdown_ms": {"step": [round(x, 3) for x in head["step_ms"]],
                                  "kernel": [round(x, 3) for x in head["kern_ms"]]},
            "clocks": head["clocks"],
            "streams": {k: {"value": n_glob / (r["ms_per_step"] / 1e3), "ms_per_step": r["ms_per_step"],
                            "kernel_ms": roof(r)[1] * 1e3, "roofline_frac": roof(r)[0] / peak,
                            "e2e": r.get("e2e"), "clocks": r["clocks"],
                            "parity": ("bit-exact vs the unmodified reference (golden vectors)" if k == "megores"
                                       else "bit-exact vs the reference-side CPU harness (oracle/, Philox)")}
                        for k, r in res.items()},
            "quality": quality,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
