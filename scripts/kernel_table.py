"""Time every libmgp kernel family at N=2^24 (y=4, B from the eps rule) with CUDA events.

    python scripts/kernel_table.py [--n 16777216] > profiles/rNN_kernel_table.json
"""

import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--y", type=float, default=4.0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
L = _lib.lib()
n = a.n
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(a.y, n), 20240, "single", device="cuda").values
st = mg.WeightVector(w, "single").stats()
b = mg.compute_iterations(0.01, st.mean, st.max).b
anc = torch.empty(n, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sp = D.stream_ptr()
stream = torch.cuda.current_stream()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0


def timeit(fn):
    ts = []
    for r in range(a.reps + 1):
        flush.fill_(float(r))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


rows = []


def add(name, ms, alg_bytes, note=""):
    gbs = alg_bytes / (ms * 1e-3) / 1e9
    rows.append({"kernel": name, "ms": round(ms, 4), "alg_bytes": alg_bytes, "alg_GBps": round(gbs, 1),
                 "frac_of_hbm": round(gbs / peak, 3), "note": note})


resample_bytes = n * b * 4 + n * 4 + n * 8 + 8 * b
for kind, part in [("megopolis", 0), ("metropolis", 0), ("c1", 128), ("c1", 2048), ("c2", 128), ("c2", 2048)]:
    for rng in ("megores", "philox"):
        def go(kind=kind, part=part, rng=rng):
            _lib.check(L.mgp_resample_range(_lib.KIND[kind], D.ptr(w), 0, n, b, 7, 32, part, 1, _lib.RNG[rng],
                                            _lib.FLAG_NONZERO, 0, n, D.ptr(anc), sp))
        ms = timeit(go)
        add(f"{kind}{':' + str(part) if part else ''} {rng}", ms, resample_bytes,
            f"{n * b / (ms * 1e-3):.3e} comparisons/s, {n / (ms * 1e-3):.3e} particles/s")

# float64 weights (the reference's "double"): 128 MiB of weights, beyond L2's reach
w64 = w.double()
for rng in ("megores", "philox"):
    def go64(rng=rng):
        _lib.check(L.mgp_resample_range(_lib.KIND["megopolis"], D.ptr(w64), 1, n, b, 7, 32, 0, 1, _lib.RNG[rng],
                                        _lib.FLAG_NONZERO, 0, n, D.ptr(anc), sp))
    ms = timeit(go64)
    add(f"megopolis f64 {rng}", ms, n * b * 8 + n * 8 + n * 8 + 8 * b,
        f"{n * b / (ms * 1e-3):.3e} comparisons/s, {n / (ms * 1e-3):.3e} particles/s (8 B per comparison)")

stats = torch.empty(8, dtype=torch.float64, device="cuda")
add("weight_stats (pairwise sum+max+flags)", timeit(lambda: _lib.check(L.mgp_weight_stats(D.ptr(w), 0, n, D.ptr(stats), sp))), 4 * n)
counts = torch.empty(n, dtype=torch.int64, device="cuda")
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
_lib.check(L.mgp_megopolis(D.ptr(w), 0, n, b, 7, 32, 1, 0, 1, D.ptr(anc), sp))
add("offspring histogram", timeit(lambda: _lib.check(L.mgp_offspring(D.ptr(anc), n, n, D.ptr(counts), D.ptr(bad), sp))),
    8 * n + 8 * n, "memset + warp-aggregated atomics (y=4 megopolis ancestors)")
e = torch.empty(n, dtype=torch.float64, device="cuda")
tot = torch.empty(1, dtype=torch.float64, device="cuda")
add("expected offspring (sum + N*w/sum)", timeit(lambda: _lib.check(L.mgp_expected_offspring(D.ptr(w), 0, n, D.ptr(e), D.ptr(tot), sp))), 4 * n + 4 * n + 8 * n)
s1 = torch.zeros(n, dtype=torch.float64, device="cuda")
s2 = torch.zeros(n, dtype=torch.float64, device="cuda")
se = torch.zeros(2, dtype=torch.float64, device="cuda")
add("quality add (sum, sum_sq, SE pairwise)", timeit(lambda: _lib.check(L.mgp_quality_add(D.ptr(counts), D.ptr(e), n, D.ptr(s1), D.ptr(s2), D.ptr(se), D.ptr(se[1:]), sp))), 8 * n + 32 * n + 8 * n + 8 * n)
for row_bytes in (8, 32):
    states = torch.empty(n * row_bytes // 8, dtype=torch.float64, device="cuda")
    out = torch.empty_like(states)
    add(f"gather rows of {row_bytes} B", timeit(lambda: _lib.check(L.mgp_gather(D.ptr(states), row_bytes, D.ptr(anc), n, D.ptr(out), sp))),
        8 * n + 2 * row_bytes * n)
# prefix-sum resamplers (M/resample.py:285-336): exact sequential-order np.cumsum + searches
cum = torch.empty(n, dtype=torch.float32, device="cuda")
add("cumsum f32 (np.cumsum order, exact)", timeit(lambda: _lib.check(L.mgp_cumsum(D.ptr(w), 0, n, D.ptr(cum), sp))),
    8 * n, "read w + write prefix (the pipeline reads w three times)")
w64 = w.double()
cum64 = torch.empty(n, dtype=torch.float64, device="cuda")
add("cumsum f64 (np.cumsum order, exact)", timeit(lambda: _lib.check(L.mgp_cumsum(D.ptr(w64), 1, n, D.ptr(cum64), sp))),
    16 * n)
for kind in ("multinomial", "systematic"):
    fn = L.mgp_multinomial if kind == "multinomial" else L.mgp_systematic
    ms = timeit(lambda fn=fn: _lib.check(fn(D.ptr(w), 0, n, 7, D.ptr(anc), sp)))
    add(f"{kind} f32 (cumsum + binary search)", ms, 8 * n + 8 * n, f"{n / (ms * 1e-3):.3e} particles/s")
print(json.dumps({"n": n, "y": a.y, "B": b, "peak_hbm_gbs": peak, "rows": rows}, indent=1))
