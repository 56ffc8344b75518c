"""Time the prefix-sum resamplers at 2^24 (f32, y=4) through the C-ABI: cumsum alone, multinomial
and systematic (cumsum + search); the search time is the difference.  Checks multinomial /
systematic against the oracle on a particle subsample."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2109_13504_b200 as mg
from paper_2109_13504_b200 import _lib, _device as D
from oracle import oracle

L = _lib.lib()
n = 1 << 24
w_np = oracle.gen_gaussian_weights(4.0, n, 31337, "single")
w = torch.from_numpy(w_np).cuda()
cum = torch.empty_like(w)
anc = torch.empty(n, dtype=torch.int64, device="cuda")
sp = D.stream_ptr()

def timeit(f, reps=20):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]

tc = timeit(lambda: _lib.check(L.mgp_cumsum(D.ptr(w), 0, n, D.ptr(cum), sp)))
tm = timeit(lambda: _lib.check(L.mgp_multinomial(D.ptr(w), 0, n, 7, D.ptr(anc), sp)))
am = anc.cpu().numpy()
ts_ = timeit(lambda: _lib.check(L.mgp_systematic(D.ptr(w), 0, n, 7, D.ptr(anc), sp)))
a_s = anc.cpu().numpy()
print(f"cumsum {tc*1e3:.1f} us  multinomial {tm*1e3:.1f} us (search {1e3*(tm-tc):.1f})  systematic {ts_*1e3:.1f} us (search {1e3*(ts_-tc):.1f})")
import hashlib
print("multinomial sha", hashlib.sha256(am.tobytes()).hexdigest()[:16], "systematic sha", hashlib.sha256(a_s.tobytes()).hexdigest()[:16])
