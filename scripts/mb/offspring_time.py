"""CUDA-event time of mgp_offspring at 2^24 (Megopolis ancestors, y = 4) per histogram mode
(0 = queued, 1 = int32 global atomics, 2 = count-matrix bucketed), through the C ABI (no Python-side sync)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

n = 1 << 24
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single", device="cuda")
a = mg.megopolis(w, 354, seed=7, rng="philox")
c = torch.empty(n, dtype=torch.int64, device="cuda")
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
for mode in (0, 1, 2, 0, 1, 2):
    L.mgp_debug_offspring_mode(mode)
    for _ in range(3):
        _lib.check(L.mgp_offspring(a.data_ptr(), n, n, c.data_ptr(), bad.data_ptr(), s))
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.mgp_offspring(a.data_ptr(), n, n, c.data_ptr(), bad.data_ptr(), s))
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[5]
    print(f"mode {mode}: {t:.4f} ms  alg {16 * n / t / 1e6:.0f} GB/s")
