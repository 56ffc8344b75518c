"""CUDA-event time of the Megopolis launch (both streams, float32 and float64 weights) at 2^24, y = 4, B = 354 through the C ABI,
L2 flushed between repetitions; prints a sha of the ancestors for A/B parity between builds."""
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
w64 = w.double()
for rng, ww, dt in (("megores", w, 0), ("philox", w, 0), ("megores", w64, 1), ("philox", w64, 1)):
    def go():
        _lib.check(L.mgp_resample_range(_lib.KIND["megopolis"], D.ptr(ww), dt, n, b, 7, 32, 0, 1, _lib.RNG[rng],
                                        _lib.FLAG_NONZERO, 0, n, D.ptr(anc), sp))
    ts = []
    for r in range(8):
        flush.fill_(float(r))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        go()
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    sha = hashlib.sha256(anc.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"{rng:8s} f{32 * (dt + 1)} {statistics.median(ts):.4f} ms  min {min(ts):.4f}  sha {sha}", flush=True)
