#!/usr/bin/env python3
"""Headline benchmark: Megopolis particles resampled per second on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload (BASELINE.json metric / config 4): Megopolis resampling of a global population of
N = 2^24 particles, Gaussian-family float32 weights with y = 4 (high variance) -- the
reference's own weight bytes (M/weights.py:100-104, seed 20240), identical in both arms --
B from the epsilon = 0.01 rule (B = 354), the Philox stream (north star: bit-exact for a
shared Philox stream; the reference's megores stream is measured too, under "streams").
One step = one pass of the hot path over the batch: (NCCL all-gather of the weight stripes)
-> weight statistics -> B (host, like the reference) -> Megopolis kernel.

Multi-GPU is STRONG scaling at the metric's N = 2^24 (2^24 / G particles per GPU): rank r owns
stripe r of each half of the population ([r*h, (r+1)*h) and N/2 + [r*h, (r+1)*h), h = N/2G,
the "stripes" layout of distributed.ShardedResampler, under which every rank runs the
half-split kernel).  Each step all-gathers the weight stripes over NCCL,
derives the global B bit-exactly from per-stripe statistics and resamples the rank's
stripes.  ``config5`` (nested in the same line) is BASELINE config 5: N = 2^28 global, weights
generated in HBM (labelled: not the reference's bytes), the same step.

``value``: device-timed (CUDA events, max over ranks) with the weights resident in HBM; the
L2 (126 MB) would hold the 64 MiB weights across steps, so a 256 MiB buffer is written
between timed steps (outside the timed windows).  ``e2e``: the same metric through the
reference-facing C-ABI host entry (mgp_resample_host: pinned host weights in, pinned host
ancestors out; N > 1: per-rank pinned stripe upload + the sharded step + ancestor download),
wall clock; ``e2e.batched``: independent jobs through the pipelined batch entry
(mgp_resample_host_batch; each job's copies overlap the neighbouring jobs' kernels).
``e2e_dropin``: the reference's Python call shape,
``megopolis(WeightVector(numpy), B, seed=...)`` with pageable numpy in and out.
``parity``: the timed ancestors against the CPU oracle (oracle/) on the same inputs.
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
N_GLOBAL = 1 << 24
N_CONFIG5 = 1 << 28
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
    ap.add_argument("--n", "--particles", dest="n", type=int, default=N_GLOBAL, help="global particles")
    ap.add_argument("--rng", default="philox", choices=["megores", "philox"],
                    help="headline stream; the other one is measured too and reported under 'streams'")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    ap.add_argument("--no-probe", action="store_true", help="skip the L2 read-bandwidth probe")
    ap.add_argument("--quality-runs", type=int, default=32)  # K >= 32
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded NCCL step even at one rank (torchrun --nproc-per-node 1)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(n, b, rng, world):
    """The ``config`` dict both arms print (identical for the same n / B / stream / world)."""
    return {
        "workload": f"megopolis N=2^{int(math.log2(n))} (global) y=4 float32 Gaussian weights (the reference's "
                    f"bytes, M/weights.py:100-104, seed {WEIGHT_SEED}), B={b} (eps=0.01 rule), {rng} stream, "
                    f"run seed {RUN_SEED}",
        "N": n, "B": b, "y": Y, "rng": rng,
        "parallelism": f"dp{world} strong (replicated weights, particle stripes)",
        "l2": "flushed between timed steps (256 MiB write outside the timed windows)",
    }


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML clock / throttle-reason / board-power sampling during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz, self.power_mw = [], set(), None, []
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
                self.power_mw.append(self.nv.nvmlDeviceGetPowerUsage(self.h))
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
        out = {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power_mw:
            out["power_w"] = round(statistics.median(self.power_mw) / 1000.0, 1)
        return out


# ---------------------------------------------------------------------------
# CPU legs: the oracle port of the path (oracle/, test infrastructure) on the host's cores


def calibrate(oracle, w, b, budget_s, nthreads, rng, p_max):
    """A particle-prefix sample [0, p) that takes about ``budget_s`` on ``nthreads`` threads."""
    p = min(p_max, 16384)
    t0 = time.perf_counter()
    oracle.megopolis(w, b, seed=RUN_SEED, threads=nthreads, p0=0, p1=p, rng=rng)
    dt = time.perf_counter() - t0
    for _ in range(3):  # the small calibration run under-states the threaded rate: re-aim
        if dt >= 0.5 * budget_s or p >= p_max:
            break
        p = int(min(p_max, max(4096, p / max(dt, 1e-6) * budget_s)))
        p -= p % 32
        t0 = time.perf_counter()
        oracle.megopolis(w, b, seed=RUN_SEED, threads=nthreads, p0=0, p1=p, rng=rng)
        dt = time.perf_counter() - t0
    return p, dt


def cpu_leg(oracle, w, b, rng, budget_s=8.0, reps=3):
    """cpu_baseline: all host threads (min / median of ``reps``) and one thread, on particle-prefix
    samples of the workload; returns (dict, ancestors of the all-thread sample [0, p))."""
    threads = oracle.num_threads()
    p, _ = calibrate(oracle, w, b, budget_s, threads, rng, len(w))
    times, anc = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        anc = oracle.megopolis(w, b, seed=RUN_SEED, threads=threads, p0=0, p1=p, rng=rng)
        times.append(time.perf_counter() - t0)
    p1, _ = calibrate(oracle, w, b, budget_s / 2, 1, rng, len(w))
    t0 = time.perf_counter()
    oracle.megopolis(w, b, seed=RUN_SEED, threads=1, p0=0, p1=p1, rng=rng)
    t1 = time.perf_counter() - t0
    med = statistics.median(times)
    d = {"value": p / med, "unit": "particles/s", "cores": threads, "kind": "port",
         "sample": f"oracle/mgp_oracle.c megopolis ({rng} stream) over particles [0, {p}) of the same "
                   f"N={len(w)} y=4 B={b} workload; {reps} reps, median {med:.2f}s",
         "cpu_model": cpu_model(), "nproc": os.cpu_count(),
         "min_s": min(times), "median_s": med, "value_best": p / min(times),
         "value_1thread": p1 / t1, "sample_1thread": f"particles [0, {p1}), {t1:.2f}s"}
    return d, p, anc


def reference_numba(n, b, rng):
    """The UNMODIFIED reference (numba, staged under baseline/_ref by scripts/stage_reference.sh):
    megores.megopolis on the same weights at the full N, all host threads, one call after a
    JIT warm-up.  megores stream only (the reference has no Philox)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if rng != "megores" or not os.path.isfile(os.path.join(ref_dir, "megores", "resample.py")):
        return None
    try:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
        sys.path.insert(0, ref_dir)
        import megores as m

        w = m.gen_gaussian_weights(m.GaussianWeightParams(Y, n), WEIGHT_SEED, "single")
        m.megopolis(m.WeightVector(w.values[:1024], "single"), 2, seed=1)  # JIT
        t0 = time.perf_counter()
        m.megopolis(w, b, seed=RUN_SEED)
        dt = time.perf_counter() - t0
        import numba

        return {"value": n / dt, "unit": "particles/s", "threads": numba.get_num_threads(), "seconds": dt,
                "kind": "reference", "sample": f"megores.megopolis (numba, unmodified) full N={n}, B={b}, 1 call"}
    except Exception as e:  # reported, never fatal
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle  # the reference arm: the CPU port of the path (no libmgp.so)

    n = args.n
    w = oracle.gen_gaussian_weights(Y, n, WEIGHT_SEED, "single")
    mean, mx = oracle.weight_mean_max(w)
    b = oracle.compute_iterations(EPS, mean, mx)
    threads = oracle.num_threads()
    per_step_budget = max(2.0, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    p, _ = calibrate(oracle, w, b, per_step_budget, threads, args.rng, n)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.megopolis(w, b, seed=RUN_SEED, threads=threads, p0=0, p1=p, rng=args.rng)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = p / t
    sample = f"oracle/mgp_oracle.c megopolis ({args.rng} stream) over particles [0, {p}) of N={n} (y=4, B={b}); " \
             f"{args.steps} steps, median {t:.2f}s"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3 * n / p,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(n, b, args.rng, world),
        "cpu_baseline": {"value": value, "unit": "particles/s", "cores": threads, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count(), "min_s": min(times), "median_s": t},
        "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if n <= N_GLOBAL:
        line["reference_numba_megores"] = reference_numba(n, b, "megores")
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def l2_probe(probe, w, off_dev, b, stream):
    """Read bandwidth the Megopolis kernel is bounded by, measured on this GPU now:
    (1) an ld.global.cg float4 read stream over the 64 MiB weight array itself (L2-resident),
    (2) the Megopolis load stream alone (texture fetches of the rotated lines, no arithmetic),
    both timed with CUDA events on ``stream``, median of 5."""
    import torch

    sink = torch.empty(1 << 22, dtype=torch.float32, device=w.device)
    sp = ctypes.c_void_p(stream.cuda_stream)
    nbytes = w.numel() * 4
    out = {}

    def timed(fn, reps=5):
        ts = []
        for _ in range(reps):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            z.record(stream)
            z.synchronize()
            ts.append(a.elapsed_time(z) / 1e3)
        return statistics.median(ts)

    passes = 20
    for blocks_per_sm in (4,):
        blocks = 148 * blocks_per_sm
        probe.mgpp_read_stream(ctypes.c_void_p(w.data_ptr()), nbytes, 1, blocks, ctypes.c_void_p(sink.data_ptr()), sp)
        t = timed(lambda: probe.mgpp_read_stream(ctypes.c_void_p(w.data_ptr()), nbytes, passes, blocks,
                                                 ctypes.c_void_p(sink.data_ptr()), sp))
        out["l2_read_gbs"] = nbytes * passes / t / 1e9
    out["l2_read_desc"] = (f"ld.global.cg float4 read stream, {passes} passes over the {nbytes >> 20} MiB weight "
                           f"array (L2-resident), 148x4 CTAs of 512 threads, median of 5 (libmgp_probe.so)")
    n = w.numel()
    if n & (n - 1) == 0:
        t = timed(lambda: probe.mgpp_megopolis_read(ctypes.c_void_p(w.data_ptr()), n, ctypes.c_void_p(off_dev.data_ptr()),
                                                    b, 148 * 8, ctypes.c_void_p(sink.data_ptr()), sp), reps=3)
        out["megopolis_loads_only_ms"] = t * 1e3
        out["megopolis_loads_only_gbs"] = (n * b * 4) / t / 1e9
    return out


def issue_block(rng, n):
    """The committed ncu summary of the kernel at this stream and size (profiles/megopolis_issue.json,
    made by scripts/issue_block.py from an ncu --set full capture of the same launch)."""
    try:
        with open(os.path.join(ROOT, "profiles", "megopolis_issue.json")) as f:
            d = json.load(f)
        return dict(d[f"{rng}@{n}"], file="profiles/megopolis_issue.json")
    except Exception:
        return None


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
    sharded = world > 1 or args.sharded  # the stripes layout + NCCL exchange (also at world 1)
    if sharded:
        if loopback:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    from paper_2109_13504_b200.distributed import combine_slice_stats, slice_tree_aligned
    from paper_2109_13504_b200.weights import WeightStats

    class Population:
        """One global population sharded over the ranks (stripes layout) plus the step."""

        def __init__(self, n, w_host=None, w_dev_full=None):
            self.n = n
            self.h, self.half = n // 2 // world, n // 2
            self.lo0, self.lo1 = rank * self.h, (rank + 1) * self.h
            self.n_loc = 2 * self.h if sharded else n
            if sharded and (n % (2 * world) or self.h % 32):
                raise SystemExit(f"N={n} does not split into 32-aligned stripes over {world} ranks")
            if w_dev_full is None:
                w_dev_full = torch.from_numpy(w_host).to(dev)
            if sharded:
                self.local_w = torch.cat([w_dev_full[self.lo0:self.lo1], w_dev_full[self.half + self.lo0:self.half + self.lo1]])
                self.full = torch.empty(n, dtype=torch.float32, device=dev)
                del w_dev_full
            else:
                self.full = w_dev_full
                self.local_w = w_dev_full
            self.aligned = sharded and slice_tree_aligned(world, self.h)
            self.stats = torch.empty(16, dtype=torch.float64, device=dev)
            self.stats_all = torch.empty(world * 16, dtype=torch.int64, device=dev)
            self.anc = torch.empty(self.n_loc, dtype=torch.int64, device=dev)
            self.b = None

        def gather_weights(self, async_op=False):
            if sharded:
                h, half = self.h, self.half
                w1 = dist.all_gather_into_tensor(self.full[:half], self.local_w[:h], async_op=async_op)
                w2 = dist.all_gather_into_tensor(self.full[half:], self.local_w[h:], async_op=async_op)
                return (w1, w2)
            return ()

        def step(self, rng_id, ev=None):
            """(all-gather) -> stats -> B -> megopolis over this rank's particles."""
            h = self.h
            if sharded and self.aligned:
                # stripe statistics + a 16-word all-gather give the global B bit for bit (numpy's
                # tree: lower half + upper half, each the rank stripes in order;
                # distributed.combine_slice_stats); B is derived while the weights are in flight
                _lib.check(L.mgp_weight_stats(D.ptr(self.local_w), 0, h, D.ptr(self.stats), sp))
                _lib.check(L.mgp_weight_stats(D.ptr(self.local_w[h:]), 0, h, D.ptr(self.stats[8:]), sp))
                ws = dist.all_gather_into_tensor(self.stats_all, self.stats.view(torch.int64), async_op=True)
                wws = self.gather_weights(async_op=True)
                ws.wait()
                rows = self.stats_all.view(world * 2, 8).cpu().numpy()
                per = [WeightStats(h, *r.view(np.float64)[:3], *r[3:]) for r in rows]
                g = combine_slice_stats([combine_slice_stats(per[0::2]), combine_slice_stats(per[1::2])])
                b = mg.compute_iterations(EPS, g.mean, g.max).b
                flags = _lib.FLAG_NONZERO if g.n_zero == 0 else 0
                for wk in wws:
                    wk.wait()
            else:
                self.gather_weights()
                _lib.check(L.mgp_weight_stats(D.ptr(self.full), 0, self.n, D.ptr(self.stats), sp))
                host = self.stats.cpu().numpy()  # 64 B; the reference also derives B on the host
                b = mg.compute_iterations(EPS, float(host[1]), float(host[2])).b
                flags = _lib.FLAG_NONZERO if host.view(np.int64)[4] == 0 else 0
            if ev is not None:
                ev[0].record(stream)
            if sharded:
                _lib.check(L.mgp_resample_stripes(_lib.KIND["megopolis"], D.ptr(self.full), 0, self.n, b, RUN_SEED, 32,
                                                  0, 1, rng_id, flags, self.lo0, self.lo1, D.ptr(self.anc), sp))
            else:
                _lib.check(L.mgp_resample_range(_lib.KIND["megopolis"], D.ptr(self.full), 0, self.n, b, RUN_SEED, 32,
                                                0, 1, rng_id, flags, 0, self.n, D.ptr(self.anc), sp))
            if ev is not None:
                ev[1].record(stream)
            self.b = b

        def measure(self, rng_id, steps, warmup):
            """W warm-up + K timed steps; per-step and kernel-only CUDA-event times, max over ranks."""
            for _ in range(max(warmup, 3)):
                self.step(rng_id)
            torch.cuda.synchronize()
            starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
            ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
            kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            if sharded:
                dist.barrier()
            torch.cuda.synchronize()
            import gc

            gc.collect()
            gc.disable()
            with ClockSampler(local) as clk:
                for s in range(steps):
                    flush.fill_(float(s))
                    starts[s].record(stream)
                    self.step(rng_id, kev[s])
                    ends[s].record(stream)
                torch.cuda.synchronize()
            gc.enable()
            if sharded:
                dist.barrier()
            step_ms = [starts[s].elapsed_time(ends[s]) for s in range(steps)]
            kern_ms = [kev[s][0].elapsed_time(kev[s][1]) for s in range(steps)]
            t_total = sum(step_ms)
            if sharded:
                tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_total = float(tt.item())
            return {"b": self.b, "ms_per_step": t_total / steps, "step_ms": step_ms, "kern_ms": kern_ms,
                    "clocks": clk.summary(), "anc": self.anc.clone()}

        def owned_ranges(self):
            """(global range, offset into anc) pairs of this rank's particles."""
            if not sharded:
                return [((0, self.n), 0)]
            return [((self.lo0, self.lo1), 0), ((self.half + self.lo0, self.half + self.lo1), self.h)]

    n_glob = args.n
    # the reference's own weight bytes (host numpy, M/weights.py:100-104), identical to the
    # reference arm's input; every rank generates the population and keeps its stripes
    w_host = mg.gen_gaussian_weights(mg.GaussianWeightParams(Y, n_glob), WEIGHT_SEED, "single").values
    pop = Population(n_glob, w_host=w_host)

    res = {}
    other = "megores" if args.rng == "philox" else "philox"
    for name in (args.rng, other):
        res[name] = pop.measure(_lib.RNG[name], args.steps, args.warmup)
    head = res[args.rng]
    b = head["b"]
    ms_per_step = head["ms_per_step"]
    value = n_glob / (ms_per_step / 1e3)  # all ranks' particles per second
    # stats (2 kernels, per stripe when sharded) + megopolis launches
    launches = args.steps * ((4 if pop.aligned else 2) + math.ceil(b / 1024))

    # roofline: algorithmic bytes of one Megopolis launch: N*B*4 + N*4 + N*8 + 8*B
    n_loc = pop.n_loc
    alg_bytes = n_loc * b * 4 + n_loc * 4 + n_loc * 8 + 8 * b
    hbm_peak, hbm_src = load_peaks()

    def kern_avg(r):
        return statistics.mean(r["kern_ms"]) / 1e3

    achieved = alg_bytes / kern_avg(head) / 1e9
    mego_kernel = ("k_megopolis_philox_half (half-split, 4 particles/thread)" if args.rng == "philox"
                   else "k_megopolis_megores_f32 (float32 decision bracket, exact float64 fallback)")
    ib = issue_block(args.rng, n_loc)
    traffic = ib.get("dram_bytes_per_launch") if ib else None
    probe_res = None
    if not args.no_probe:
        try:
            from paper_2109_13504_b200 import build as _b

            probe = ctypes.CDLL(_b.PROBE_OUT)
            probe.mgpp_read_stream.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_void_p, ctypes.c_void_p]
            probe.mgpp_megopolis_read.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
            offs = mg.megopolis_offsets(n_glob, b, RUN_SEED, rng=args.rng)
            off_dev = torch.from_numpy(np.asarray(offs, dtype=np.int64).astype(np.uint32)).to(dev)
            probe_res = l2_probe(probe, pop.full, off_dev, b, stream)
        except Exception as e:
            probe_res = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    l2_peak = probe_res.get("l2_read_gbs") if probe_res else None
    if l2_peak:
        roofline = {"bound": "l2", "achieved": achieved, "peak": l2_peak, "unit": "GB/s", "frac": achieved / l2_peak,
                    "traffic": traffic, "peak_source": "measured in this run: " + probe_res["l2_read_desc"]}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": hbm_src}
    roofline.update({"kernel": mego_kernel, "kernel_ms": kern_avg(head) * 1e3, "alg_bytes_per_launch": alg_bytes,
                     "hbm": {"peak": hbm_peak, "frac": achieved / hbm_peak, "peak_source": hbm_src},
                     "probe": probe_res, "issue": ib})

    # parity of what was timed: rank 0's timed ancestors vs the oracle on the same inputs
    parity = None
    cpu = None
    if rank == 0:
        from oracle import oracle

        anc_head = head["anc"].cpu().numpy()
        (g0, g1), off0 = pop.owned_ranges()[0]
        if world == 1 and not args.no_cpu_baseline:
            cpu, p, ref = cpu_leg(oracle, w_host, b, args.rng)
            checked = p
            mism = int(np.count_nonzero(anc_head[:p] != ref[:p]))
        else:
            p = min(g1 - g0, 1 << 20)
            ref = oracle.megopolis(w_host, b, seed=RUN_SEED, threads=oracle.num_threads(), p0=g0, p1=g0 + p, rng=args.rng)
            checked = p
            mism = int(np.count_nonzero(anc_head[off0:off0 + p] != ref[g0:g0 + p]))
        parity = {"checked": checked, "mismatches": mism, "stream": args.rng,
                  "against": "oracle/mgp_oracle.c (CPU port, pinned to the reference's golden vectors)",
                  "particles": f"[{g0}, {g0 + checked}) of the timed step's ancestors"}
        # the other stream: a 2^20 prefix of its timed ancestors
        q = min(g1 - g0, 1 << 20)
        anc_o = res[other]["anc"].cpu().numpy()
        ref_o = oracle.megopolis(w_host, b, seed=RUN_SEED, threads=oracle.num_threads(), p0=g0, p1=g0 + q, rng=other)
        parity["other_stream"] = {"stream": other, "checked": q,
                                  "mismatches": int(np.count_nonzero(anc_o[off0:off0 + q] != ref_o[g0:g0 + q]))}

    # e2e through the reference-facing host entry
    e2e = None
    e2e_dropin = None
    if not args.no_e2e:
        bu = ctypes.c_int32(0)
        if world == 1:
            h_w = torch.from_numpy(w_host).pin_memory()
            h_anc = torch.empty(n_glob, dtype=torch.int64).pin_memory()

            def e2e_time(rid):
                def e2e_step():
                    _lib.check(L.mgp_resample_host(_lib.KIND["megopolis"], D.ptr(h_w), 0, n_glob, 0, EPS, RUN_SEED, 32,
                                                   0, 1, rid, D.ptr(h_anc), ctypes.byref(bu), local))

                for _ in range(3):
                    e2e_step()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                reps = max(3, min(args.steps, 10))
                for _ in range(reps):
                    e2e_step()
                return (time.perf_counter() - t0) / reps

            te = e2e_time(_lib.RNG[args.rng])
            e2e = {"value": n_glob / te, "unit": "particles/s", "h2d_bytes_per_step": 4 * n_glob,
                   "d2h_bytes_per_step": 8 * n_glob, "ms_per_step": te * 1e3, "B": int(bu.value),
                   "path": "mgp_resample_host (pinned host weights -> device -> pinned host ancestors)"}
            te_o = e2e_time(_lib.RNG[other])
            res[other]["e2e"] = {"value": n_glob / te_o, "ms_per_step": te_o * 1e3}
            # e2e of the headline stream, re-run once to compare with the device-timed ancestors
            _lib.check(L.mgp_resample_host(_lib.KIND["megopolis"], D.ptr(h_w), 0, n_glob, 0, EPS, RUN_SEED, 32, 0, 1,
                                           _lib.RNG[args.rng], D.ptr(h_anc), ctypes.byref(bu), local))
            e2e["parity"] = {"checked": n_glob, "vs": "the device-timed ancestors",
                             "mismatches": int(np.count_nonzero(h_anc.numpy() != head["anc"].cpu().numpy()))}

            # independent jobs through the pipelined batch entry (mgp_resample_host_batch): job k+1's
            # upload and job k-1's download overlap job k's kernel; every job still uploads its
            # 4N bytes and downloads its 8N bytes inside the timed region
            def e2e_batched(rid, count=8):
                outs = [torch.empty(n_glob, dtype=torch.int64).pin_memory() for _ in range(2)]
                hw = (ctypes.c_void_p * count)(*([D.ptr(h_w)] * count))
                ha = (ctypes.c_void_p * count)(*[D.ptr(outs[k & 1]) for k in range(count)])
                sd = (ctypes.c_uint64 * count)(*([RUN_SEED] * count))
                bu = (ctypes.c_int32 * count)()

                def batch():
                    _lib.check(L.mgp_resample_host_batch(_lib.KIND["megopolis"], hw, 0, n_glob, count, 0, EPS, sd, 32,
                                                         0, 1, rid, ha, bu, local))

                batch()
                ts = []
                for _ in range(3):
                    t0 = time.perf_counter()
                    batch()
                    ts.append(time.perf_counter() - t0)
                tb = statistics.median(ts)
                mism = sum(int(np.count_nonzero(o.numpy() != head["anc"].cpu().numpy())) for o in outs)
                return {"value": count * n_glob / tb, "unit": "particles/s", "jobs": count,
                        "ms_per_job": tb / count * 1e3, "h2d_bytes_per_step": 4 * n_glob, "d2h_bytes_per_step": 8 * n_glob,
                        "path": f"mgp_resample_host_batch: {count} independent jobs (pinned host weights in, pinned "
                                "ancestors out), uploads/downloads overlapped with the neighbouring jobs' kernels; "
                                "wall clock over the batch, median of 3",
                        "parity": {"checked": 2 * n_glob, "vs": "the device-timed ancestors", "mismatches": mism}}

            e2e["batched"] = e2e_batched(_lib.RNG[args.rng])

            # the B-rule reduction, H2D (4N B) and D2H (8N B) reported separately
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

            d_w = torch.empty(n_glob, dtype=torch.float32, device=dev)
            h2d = ev_ms(lambda: d_w.copy_(h_w, non_blocking=True))
            d2h = ev_ms(lambda: h_anc.copy_(pop.anc, non_blocking=True))
            brule = ev_ms(lambda: _lib.check(L.mgp_weight_stats(D.ptr(d_w), 0, n_glob, D.ptr(pop.stats), sp)))
            e2e["transfers"] = {"h2d_ms": h2d, "h2d_GBps": 4 * n_glob / h2d / 1e6, "d2h_ms": d2h,
                                "d2h_GBps": 8 * n_glob / d2h / 1e6, "b_rule_ms": brule}
            del d_w

            # the drop-in call shape of the reference's users, WeightVector construction (host
            # validation) included: pageable numpy in, a fresh np.int64 array out
            def dropin():
                return mg.megopolis(mg.WeightVector(w_host, "single"), b, seed=RUN_SEED, rng=args.rng)

            a_np = dropin()
            # wall clock per call; the host side varies from call to call (page faults of the fresh
            # output, host-thread scheduling), so the median of 9 calls is reported with min / mean
            tds = []
            for _ in range(9):
                t0 = time.perf_counter()
                a_np = dropin()
                tds.append(time.perf_counter() - t0)
            td = statistics.median(tds)
            e2e_dropin = {"value": n_glob / td, "unit": "particles/s", "ms_per_step": td * 1e3,
                          "min_ms": min(tds) * 1e3, "mean_ms": statistics.mean(tds) * 1e3, "calls": len(tds),
                          "h2d_bytes_per_step": 4 * n_glob, "d2h_bytes_per_step": 8 * n_glob,
                          "path": "paper_2109_13504_b200.megopolis(WeightVector(np.ndarray float32), B, seed, rng) "
                                  "-- WeightVector construction, pageable numpy in, fresh np.int64 out (the "
                                  "reference's call shape); the host entry stages pageable buffers through "
                                  "page-locked slots with parallel host copies",
                          "parity": {"checked": n_glob, "vs": "the device-timed ancestors",
                                     "mismatches": int(np.count_nonzero(a_np != head["anc"].cpu().numpy()))}}
        else:
            # per rank: pinned stripe upload -> the sharded step -> pinned ancestor download
            h_w = pop.local_w.cpu().pin_memory()
            h_anc = torch.empty(pop.n_loc, dtype=torch.int64).pin_memory()
            rid = _lib.RNG[args.rng]

            def e2e_step():
                pop.local_w.copy_(h_w, non_blocking=True)
                pop.step(rid)
                h_anc.copy_(pop.anc, non_blocking=True)
                torch.cuda.current_stream().synchronize()

            for _ in range(3):
                e2e_step()
            dist.barrier()
            t0 = time.perf_counter()
            reps = max(3, min(args.steps, 10))
            for _ in range(reps):
                e2e_step()
            te = (time.perf_counter() - t0) / reps
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
            e2e = {"value": n_glob / te, "unit": "particles/s", "h2d_bytes_per_step": 4 * pop.n_loc,
                   "d2h_bytes_per_step": 8 * pop.n_loc, "ms_per_step": te * 1e3,
                   "path": "per rank: pinned stripe H2D -> NCCL all-gather -> stats/B -> mgp_resample_stripes -> "
                           "pinned D2H (bytes per rank)"}

    # BASELINE config 5: N = 2^28 global, weights generated in HBM (labelled), same step
    config5 = None
    if not args.no_config5 and args.n == N_GLOBAL:
        free, _ = torch.cuda.mem_get_info()
        if free > 6 * N_CONFIG5 * 4:
            del pop.anc
            w5 = mg.gen_gaussian_weights(mg.GaussianWeightParams(Y, N_CONFIG5), WEIGHT_SEED, "single",
                                         device=dev).values
            pop5 = Population(N_CONFIG5, w_dev_full=w5)
            del w5
            r5 = pop5.measure(_lib.RNG[args.rng], max(3, min(args.steps, 5)), 2)
            b5 = r5["b"]
            nl5 = pop5.n_loc
            alg5 = nl5 * b5 * 4 + nl5 * 4 + nl5 * 8 + 8 * b5
            ach5 = alg5 / kern_avg(r5) / 1e9
            config5 = {"workload": f"megopolis N=2^28 (global) y=4 float32 Gaussian weights generated in HBM "
                                   f"(mgp_gen_gaussian: the reference's formula and stream, not its bytes), B={b5}, "
                                   f"{args.rng} stream",
                       "N": N_CONFIG5, "B": b5, "value": N_CONFIG5 / (r5["ms_per_step"] / 1e3), "unit": "particles/s",
                       "ms_per_step": r5["ms_per_step"], "kernel_ms": kern_avg(r5) * 1e3,
                       "roofline": {"bound": "hbm", "achieved": ach5, "peak": hbm_peak, "unit": "GB/s",
                                    "frac": ach5 / hbm_peak, "alg_bytes_per_launch": alg5,
                                    "traffic": (issue_block(args.rng, nl5) or {}).get("dram_bytes_per_launch"),
                                    "issue": issue_block(args.rng, nl5)},
                       "clocks": r5["clocks"]}
            if rank == 0:
                from oracle import oracle

                wnp = pop5.full.cpu().numpy() if world == 1 else None
                if wnp is not None:
                    a5 = r5["anc"].cpu().numpy()
                    mism, checked = 0, 0
                    for p0 in (0, N_CONFIG5 // 2 - 4096, N_CONFIG5 - 8192):
                        ref = oracle.megopolis(wnp, b5, seed=RUN_SEED, threads=oracle.num_threads(), p0=p0,
                                               p1=p0 + 8192, rng=args.rng)
                        mism += int(np.count_nonzero(a5[p0:p0 + 8192] != ref[p0:p0 + 8192]))
                        checked += 8192
                    config5["parity"] = {"checked": checked, "mismatches": mism,
                                         "particles": "windows of 8192 at the start, middle and end"}
            del pop5, r5
            torch.cuda.empty_cache()

    # quality (offspring MSE / bias, M/metrics.py) outside the timed region.  N > 1: the sharded
    # path (stripes-layout resample -> owner-bucketed offspring -> ShardedQuality), which equals
    # one device's QualityAccumulator over the whole population bit for bit.
    quality = None
    if args.quality_runs >= 2:
        qs = {}
        for kind in ("megopolis", "metropolis"):
            if not sharded:
                wv = mg.WeightVector(pop.full, "single")
                acc = mg.QualityAccumulator(n_glob)
                fn = mg.make_resampler(kind, rng=args.rng)
                for k in range(args.quality_runs):
                    acc.add(mg.ancestors_to_offspring(fn(wv, b, mg.derive_seed(2002, k)), n_glob), wv)
            else:
                from paper_2109_13504_b200.distributed import ShardedResampler

                sr = ShardedResampler(kind=kind, rng=args.rng, layout="stripes", force_collectives=True)
                acc = sr.quality(pop.local_w)
                for k in range(args.quality_runs):
                    a_loc, _ = sr.resample(pop.local_w, b=b, seed=mg.derive_seed(2002, k))
                    acc.add(sr.offspring(a_loc))
            st = acc.finalize()
            qs[kind] = {"mse_per_particle": st.mse_per_particle, "bias_contribution": st.bias_contribution}
        quality = {"runs": args.quality_runs, **qs, "paper_megopolis_y4": 0.6508, "paper_metropolis": 1.0}

    if rank == 0:
        config = workload_config(n_glob, b, args.rng, world)
        line = {
            "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_dropin": e2e_dropin, "parity": parity,
            "gpu_launches": launches,
            "step_breakdown_ms": {"step": [round(x, 3) for x in head["step_ms"]],
                                  "kernel": [round(x, 3) for x in head["kern_ms"]],
                                  "what": "weight stats -> B (host) -> megopolis" +
                                          (" (sharded: + NCCL all-gather of the weight stripes)" if sharded else "")},
            "clocks": head["clocks"],
            "streams": {k: {"value": n_glob / (r["ms_per_step"] / 1e3), "ms_per_step": r["ms_per_step"],
                            "kernel_ms": kern_avg(r) * 1e3,
                            "alg_GBps": alg_bytes / kern_avg(r) / 1e9, "e2e": r.get("e2e"), "clocks": r["clocks"],
                            "parity": ("bit-exact vs the unmodified reference (golden vectors)" if k == "megores"
                                       else "bit-exact vs the reference-side CPU harness (oracle/, Philox)")}
                        for k, r in res.items()},
            "config5": config5,
            "quality": quality,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
