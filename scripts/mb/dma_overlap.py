"""Megopolis kernel time at 2^24 (Philox, CUDA events on its stream) alone and with a concurrent
128 MiB device->pinned-host copy plus a 64 MiB pinned-host->device copy on other streams (the
batched host entry's overlap): does the copy traffic slow the L2-resident kernel?"""
import os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D, _lib  # noqa: E402
n, b = 1 << 24, 354
L = _lib.lib()
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single", device="cuda").values
anc = torch.empty(n, dtype=torch.int64, device="cuda")
d_src = torch.empty(n, dtype=torch.int64, device="cuda")
h_dst = torch.empty(n, dtype=torch.int64).pin_memory()
h_src = torch.empty(n, dtype=torch.float32).pin_memory()
d_dst = torch.empty(n, dtype=torch.float32, device="cuda")
ks, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def kern():
    _lib.check(L.mgp_resample_range(_lib.KIND["megopolis"], D.ptr(w), 0, n, b, 7, 32, 0, 1, _lib.RNG["philox"],
                                    _lib.FLAG_NONZERO, 0, n, D.ptr(anc), ks.cuda_stream))
for mode in ("alone", "with copies", "alone", "with copies"):
    ts = []
    for r in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ks)
        kern()
        e1.record(ks)
        if mode == "with copies":
            with torch.cuda.stream(s1):
                h_dst.copy_(d_src, non_blocking=True)
            with torch.cuda.stream(s2):
                d_dst.copy_(h_src, non_blocking=True)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    print(f"{mode:12s} kernel {statistics.median(ts):.4f} ms", flush=True)
