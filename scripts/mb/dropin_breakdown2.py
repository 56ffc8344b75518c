"""Why a reused (resident) pageable output is slower than a fresh one in mgp_resample_host at 2^24
(scripts/mb/dropin_breakdown.py): host-entry wall time only, per output/input kind, median of 7."""
import ctypes
import mmap
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

n, b = 1 << 24, 354
L = _lib.lib()
libc = ctypes.CDLL(None)
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single").values
pin_w = torch.from_numpy(w).pin_memory()
pin_a = torch.empty(n, dtype=torch.int64).pin_memory()


def ptr(x):
    return x.ctypes.data if isinstance(x, np.ndarray) else x.data_ptr()


def host(win, out):
    bu = ctypes.c_int32(0)
    t0 = time.perf_counter()
    _lib.check(L.mgp_resample_host(_lib.KIND["megopolis"], ptr(win), 0, n, b, 0.0, 7, 32, 0, 1, _lib.RNG["philox"],
                                   ptr(out), ctypes.byref(bu), -1))
    return 1e3 * (time.perf_counter() - t0)


def run(name, mk_in, mk_out, reps=7):
    ts = [host(mk_in(), mk_out()) for _ in range(reps + 1)][1:]
    print(f"{name:50s} median {statistics.median(ts):7.2f} ms  min {min(ts):7.2f}  max {max(ts):7.2f}", flush=True)


reused = np.empty(n, dtype=np.int64)
reused.fill(1)
mm = mmap.mmap(-1, 8 * n)
mm_arr = np.frombuffer(mm, dtype=np.int64)


def dontneed():
    libc.madvise(ctypes.c_void_p(ptr(mm_arr)), ctypes.c_size_t(8 * n), 4)  # MADV_DONTNEED
    return mm_arr


def fresh_resident():
    a = np.empty(n, dtype=np.int64)
    a.fill(1)
    return a


for rnd in range(2):
    run("pageable in, fresh out", lambda: w, lambda: np.empty(n, dtype=np.int64))
    run("pageable in, reused out", lambda: w, lambda: reused)
    run("pageable in, fresh out pre-touched", lambda: w, fresh_resident)
    run("pageable in, mmap out after MADV_DONTNEED", lambda: w, dontneed)
    run("pageable in, mmap out resident", lambda: w, lambda: mm_arr)
    run("pinned in, reused pageable out", lambda: pin_w, lambda: reused)
    run("pinned in, fresh pageable out", lambda: pin_w, lambda: np.empty(n, dtype=np.int64))
    run("pageable in, pinned out", lambda: w, lambda: pin_a)
    run("pinned in, pinned out", lambda: pin_w, lambda: pin_a)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
