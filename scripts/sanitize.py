"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck / initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import pfilter as pf  # noqa: E402
from paper_2109_13504_b200.distributed import gather_from_peers  # noqa: E402

rr = np.random.default_rng(0)
for n, prec in [(4096, "single"), (3 * 1024, "double"), (96, "single"), (33, "single")]:
    w = rr.random(n).astype(np.float32 if prec == "single" else np.float64)
    w[::7] = 0
    wd = mg.WeightVector(torch.from_numpy(w).cuda(), prec)
    for rng in ("megores", "philox"):
        if n % 32 == 0:
            mg.megopolis(wd, 1030, seed=3, rng=rng)
            mg.metropolis_c1(wd, 9, mg.PartitionConfig(128), seed=3, rng=rng)
            mg.metropolis_c2(wd, 40, mg.PartitionConfig(256 if n % 64 == 0 else 128), seed=3, rng=rng)
        mg.megopolis(wd, 9, mg.WarpConfig(7), seed=3, strict=False, rng=rng)
        anc = mg.metropolis(wd, 9, 3, rng=rng)
        mg.ancestors_to_offspring(anc, n)
        mg.apply_ancestors(torch.arange(n * 3, dtype=torch.float32, device="cuda").reshape(n, 3), anc)
    mg.iterations_for(wd)
    acc = mg.QualityAccumulator(n)
    for k in range(2):
        acc.add(mg.ancestors_to_offspring(mg.megopolis(wd, 5, mg.WarpConfig(1), seed=k), n), wd)
    acc.finalize()
    mg.megopolis(w, 5, mg.WarpConfig(1), seed=1)  # host-buffer path
# prefix sums: binade crossings (ones), rounding ties (dyadic), f64, partial chunks
for w in (np.ones(40000, np.float32), (rr.integers(1, 8, 70001) / 4.0).astype(np.float32), rr.random(5000),
          rr.random(1025).astype(np.float32)):
    wd = torch.from_numpy(w).cuda()
    mg.inclusive_prefix(wd)
    mg.multinomial(wd, 3)
    mg.systematic_improved(wd, 3)
mg.multinomial(np.ones(3000, np.float32), 1)  # host path
# half-split Megopolis through the chunked host path (Philox, N = 2^k)
mg.megopolis(rr.random(1 << 12).astype(np.float32), 7, seed=5, rng="philox")
shards = [torch.rand(100, 2, device="cuda") for _ in range(4)]
gather_from_peers(shards, 100, torch.from_numpy(rr.integers(0, 400, 300)))
# fused resample + peer-row gather: contiguous / stripes owner mappings, fused (W = 32, 4-byte
# rows) and two-kernel (metropolis, 3-byte rows) routes
import ctypes  # noqa: E402

from paper_2109_13504_b200 import _lib  # noqa: E402

wq = torch.from_numpy(rr.random(4096).astype(np.float32)).cuda()
for kind, layout, cols, dt in (("megopolis", 0, 2, torch.float32), ("megopolis", 1, 2, torch.float32),
                               ("megopolis", 1, 3, torch.uint8), ("metropolis", 1, 2, torch.float32),
                               ("metropolis", 0, 2, torch.float32)):
    own = [torch.zeros(1024, cols, dtype=dt, device="cuda") for _ in range(4)]
    tab = (ctypes.c_void_p * 4)(*[o.data_ptr() for o in own])
    lo, hi = (256, 512) if layout else (1024, 2048)
    cnt = (hi - lo) * (2 if layout else 1)
    anc = torch.empty(cnt, dtype=torch.int64, device="cuda")
    out = torch.empty(cnt, cols, dtype=dt, device="cuda")
    _lib.check(_lib.lib().mgp_resample_gather(
        _lib.KIND[kind], wq.data_ptr(), 0, 4096, 9, 3, 32, 0, 1, _lib.RNG["philox"], 0, layout, lo, hi,
        ctypes.cast(tab, ctypes.c_void_p), 4, 1024, cols * own[0].element_size(), anc.data_ptr(), out.data_ptr(),
        torch.cuda.current_stream().cuda_stream))
# single-process multi-device entry (the one GPU listed twice)
wm = rr.random(4096).astype(np.float32)
am = np.empty(4096, dtype=np.int64)
devs = (ctypes.c_int * 2)(0, 0)
_lib.check(_lib.lib().mgp_resample_multi(3, wm.ctypes.data, 0, 4096, 0, 0.01, 5, 32, 0, 1, 1, 2,
                                         ctypes.cast(devs, ctypes.c_void_p), am.ctypes.data, None))
acc = mg.QualityAccumulator(4096)
acc.add_runs("megopolis", mg.WeightVector(wq, "single"), 5, [1, 2, 3])
mg.estimate_ratio(mg.WeightVector(wq, "single"), 1000, 7)
mg.systematic_oracle(mg.WeightVector(wq, "single"), 0.25)
# transaction model: comparison-index replay (all kinds, W 32 and 7) and segment counting
from paper_2109_13504_b200.warpsim import count_transactions, trace_algorithm, traffic_report  # noqa: E402

for kind, part in (("megopolis", None), ("metropolis", None), ("c1", 128), ("c2", 256)):
    traffic_report(trace_algorithm(kind, mg.WeightVector(np.ones(2048), "double"), 5, mg.WarpConfig(), part, 3))
mg.comparison_indices("megopolis", 700, 3, 1, mg.WarpConfig(7))
count_transactions(np.arange(-5, 60, 3))
traj = pf.generate_trajectory(3, 0.0, 1)
pf.run_filter(pf.FilterConfig(n_particles=8192, b_fixed=None), traj, 2)
# round 2: gamma generator, pageable host buffers through the staging slots (>= 4 MiB), the
# texture LRU past its capacity, C1/C2 over ranges whose end is not warp-aligned
mg.gen_gamma_weights(mg.GammaWeightParams(2.0, 1.0, 5000), 3, "single", device="cuda")
mg.gen_gamma_weights(mg.GammaWeightParams(0.5, 2.0, 777), 4, "double", device="cuda")
wp = rr.random(1 << 20).astype(np.float32)
mg.megopolis(mg.WeightVector(wp, "single"), 3, seed=2, rng="philox")  # half-split, staged in and out
mg.metropolis_c1(mg.WeightVector(wp[:1 << 19], "single"), 3, mg.PartitionConfig(256), seed=2)
# the megores float32 brackets and their exact re-runs (subnormal multiples of 2^-149: frequent)
ws = torch.from_numpy(rr.integers(1, 17, 1 << 16).astype(np.float32) * np.float32(2.0 ** -149)).cuda()
mg.megopolis(mg.WeightVector(ws, "single"), 24, seed=3)
mg.metropolis_c1(mg.WeightVector(ws, "single"), 24, mg.PartitionConfig(128), seed=3)
mg.metropolis_c2(mg.WeightVector(ws, "single"), 24, mg.PartitionConfig(128), seed=3)
for k in range(70):
    mg.megopolis(mg.WeightVector(torch.rand(512, device="cuda"), "single"), 2, seed=k)
for kind, part in (("c1", 256), ("c2", 128)):
    out = torch.empty(61 - 32, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().mgp_resample_range(_lib.KIND[kind], wq.data_ptr(), 0, 4096, 7, 3, 32, part, 1,
                                             _lib.RNG["megores"], 0, 32, 61, out.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream))
# queued offspring histogram (n >= 2^20), incl. a ragged n, a one-hot input (queue overflow list),
# the count-matrix and atomic modes, and an out-of-range ancestor
for nn in (1 << 20, (1 << 20) + 77):
    aa = torch.from_numpy(rr.integers(0, nn, nn)).cuda()
    mg.ancestors_to_offspring(aa, nn)
mg.ancestors_to_offspring(torch.full((1 << 20,), 12345, dtype=torch.int64, device="cuda"), 1 << 20)
for mode in (1, 2):
    _lib.check(_lib.lib().mgp_debug_offspring_mode(mode))
    mg.ancestors_to_offspring(aa, nn)
_lib.check(_lib.lib().mgp_debug_offspring_mode(0))
try:
    aa[5] = nn
    mg.ancestors_to_offspring(aa, nn)
except ValueError:
    pass
torch.cuda.synchronize()
print("sanitize workload done")
