"""Where the drop-in call's time goes (pageable numpy in and out, mgp_resample_host):
fresh output array per call vs a reused (already faulted-in) one, pinned vs pageable input."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

n = 1 << 24
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single").values
L = _lib.lib()
bu = ctypes.c_int32(0)


def call(hw, ha, rng="philox"):
    _lib.check(L.mgp_resample_host(_lib.KIND["megopolis"], hw.ctypes.data if isinstance(hw, np.ndarray) else hw.data_ptr(),
                                   0, n, 354, 0.0, 7, 32, 0, 1, _lib.RNG[rng],
                                   ha.ctypes.data if isinstance(ha, np.ndarray) else ha.data_ptr(), ctypes.byref(bu), -1))


def t(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * sorted(ts)[len(ts) // 2]


res = {}
pin_w = torch.from_numpy(w).pin_memory()
pin_a = torch.empty(n, dtype=torch.int64).pin_memory()
reused = np.empty(n, dtype=np.int64)
reused[:] = 0
res["pinned_in_pinned_out"] = t(lambda: call(pin_w, pin_a))
res["pageable_in_pinned_out"] = t(lambda: call(w, pin_a))
res["pinned_in_pageable_reused_out"] = t(lambda: call(pin_w, reused))
res["pageable_in_pageable_reused_out"] = t(lambda: call(w, reused))
res["pageable_in_fresh_out"] = t(lambda: call(w, np.empty(n, dtype=np.int64)))
res["np_empty_plus_touch"] = t(lambda: np.empty(n, dtype=np.int64).fill(0))
res["public_api_megopolis"] = t(lambda: mg.megopolis(mg.WeightVector(w, "single"), 354, seed=7, rng="philox"))
print(json.dumps(res))
