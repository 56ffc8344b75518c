"""Minimal driver for ncu: a few hot-path steps (stats -> B -> resample) at the bench config.

    ncu --set full -k regex:k_megopolis -s 2 -c 1 -o prof python scripts/prof_step.py
"""

import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--y", type=float, default=4.0)
ap.add_argument("--kind", default="megopolis")
ap.add_argument("--rng", default="megores")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--part", type=int, default=128)
ap.add_argument("--dtype", default="single")
a = ap.parse_args()

L = _lib.lib()
# the reference's weight bytes (bench.py's input) up to 2^24; device-generated above (config 5)
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(a.y, a.n), 20240, a.dtype, device="cuda" if a.n > 1 << 24 else None)
if not w.on_device:
    w = mg.WeightVector(torch.from_numpy(w.values).cuda(), a.dtype)
stats = torch.empty(8, dtype=torch.float64, device="cuda")
anc = torch.empty(a.n, dtype=torch.int64, device="cuda")
sp = D.stream_ptr()
dt = D.wdtype(w.values)
for _ in range(a.steps):
    _lib.check(L.mgp_weight_stats(D.ptr(w.values), dt, a.n, D.ptr(stats), sp))
    h = stats.cpu().numpy()
    b = mg.compute_iterations(0.01, float(h[1]), float(h[2])).b
    flags = 1 if h.view("int64")[4] == 0 else 0
    pb = a.part if a.kind in ("c1", "c2") else 0
    _lib.check(L.mgp_resample_range(_lib.KIND[a.kind], D.ptr(w.values), dt, a.n, b, 7, 32, pb, 1,
                                    _lib.RNG[a.rng], flags, 0, a.n, D.ptr(anc), sp))
torch.cuda.synchronize()
print("B", b, "flags", flags)
