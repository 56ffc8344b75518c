"""CUDA-event time of Metropolis-C1 / C2 (megores and philox streams) at 2^24, y = 4, B = 354 through
the C ABI, L2 flushed between repetitions; ancestors sha for A/B parity between builds and the
float64 fallback count of the float32-bracket path."""
import ctypes
import hashlib
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

n, b = 1 << 24, 354
L = _lib.lib()
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single", device="cuda").values
anc = torch.empty(n, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sp = D.stream_ptr()
for kind, part in (("c1", 128), ("c1", 2048), ("c2", 128), ("c2", 2048)):
    for rng in ("megores", "philox"):
        def go():
            _lib.check(L.mgp_resample_range(_lib.KIND[kind], D.ptr(w), 0, n, b, 7, 32, part, 1, _lib.RNG[rng],
                                            _lib.FLAG_NONZERO, 0, n, D.ptr(anc), sp))
        ts = []
        for r in range(6):
            flush.fill_(float(r))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            go()
            e1.record()
            torch.cuda.synchronize()
            if r >= 1:
                ts.append(e0.elapsed_time(e1))
        sha = hashlib.sha256(anc.cpu().numpy().tobytes()).hexdigest()[:16]
        cnt = ctypes.c_int64(0)
        _lib.check(L.mgp_debug_megores_fallbacks(ctypes.byref(cnt), 1))
        print(f"{kind}:{part:<5d} {rng:8s} {statistics.median(ts):.4f} ms  sha {sha}  fallbacks/run {cnt.value / 6:.1f}",
              flush=True)
