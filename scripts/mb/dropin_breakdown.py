"""Where the drop-in call's time goes at 2^24 / B = 354 (Philox): WeightVector construction, the
host entry with a fresh (untouched) np.int64 output, with a reused (already faulted-in) output,
and the host entry on page-locked buffers; median of 7 wall-clock timings each."""
import ctypes
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

n, b = 1 << 24, 354
L = _lib.lib()
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single").values


def med(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts), min(ts)


def host(win, out):
    bu = ctypes.c_int32(0)
    _lib.check(L.mgp_resample_host(_lib.KIND["megopolis"], win.ctypes.data if isinstance(win, np.ndarray) else win.data_ptr(),
                                   0, n, b, 0.0, 7, 32, 0, 1, _lib.RNG["philox"],
                                   out.ctypes.data if isinstance(out, np.ndarray) else out.data_ptr(), ctypes.byref(bu), -1))


reused = np.empty(n, dtype=np.int64)
reused.fill(0)
pin_w = torch.from_numpy(w).pin_memory()
pin_a = torch.empty(n, dtype=torch.int64).pin_memory()
rows = {
    "WeightVector(numpy)": lambda: mg.WeightVector(w, "single"),
    "np.empty + fill (first touch of 128 MiB)": lambda: np.empty(n, dtype=np.int64).fill(0),
    "host entry, pageable in, fresh out": lambda: host(w, np.empty(n, dtype=np.int64)),
    "host entry, pageable in, reused out": lambda: host(w, reused),
    "host entry, pinned in/out": lambda: host(pin_w, pin_a),
    "drop-in megopolis(WeightVector(w))": lambda: mg.megopolis(mg.WeightVector(w, "single"), b, seed=7, rng="philox"),
}
for k, fn in rows.items():
    m, lo = med(fn)
    print(f"{k:45s} median {m:7.2f} ms  min {lo:7.2f}", flush=True)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
