"""CUDA-event time of mgp_multinomial / mgp_systematic at 2^24 (f32, L2 flushed), ancestors sha."""
import hashlib, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D, _lib  # noqa: E402
n = 1 << 24
L = _lib.lib()
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single", device="cuda").values
anc = torch.empty(n, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sp = D.stream_ptr()
for kind in ("multinomial", "systematic"):
    fn = L.mgp_multinomial if kind == "multinomial" else L.mgp_systematic
    ts = []
    for r in range(12):
        flush.fill_(float(r))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(fn(D.ptr(w), 0, n, 7, D.ptr(anc), sp))
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    print(f"{kind:12s} {statistics.median(ts):.4f} ms  sha {hashlib.sha256(anc.cpu().numpy().tobytes()).hexdigest()[:16]}", flush=True)
