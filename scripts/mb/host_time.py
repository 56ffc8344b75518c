"""Wall time of mgp_resample_host at 2^24 (pinned host weights in, pinned ancestors out) for every
Metropolis-family kind and both streams, plus the prefix-sum kinds; ancestors sha for A/B."""
import ctypes
import hashlib
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

n = 1 << 24
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single").values
hw = torch.from_numpy(w).pin_memory()
ha = torch.empty(n, dtype=torch.int64).pin_memory()
L = _lib.lib()
bu = ctypes.c_int32(0)
for kind, part in (("megopolis", 0), ("c1", 128), ("c2", 128), ("metropolis", 0), ("multinomial", 0)):
    for rng in (("megores", "philox") if kind != "multinomial" else ("megores",)):
        def call():
            _lib.check(L.mgp_resample_host(_lib.KIND[kind], hw.data_ptr(), 0, n, 354, 0.0, 7, 32, part, 1,
                                           _lib.RNG[rng], ha.data_ptr(), ctypes.byref(bu), -1))
        call()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        sha = hashlib.sha256(ha.numpy().tobytes()).hexdigest()[:16]
        print(f"{kind:12s} {rng:8s} {1e3 * sorted(ts)[2]:8.3f} ms  sha {sha}", flush=True)
