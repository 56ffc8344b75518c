"""Time the exact cumsum (np.cumsum order) at 2^24 through the C-ABI (mgp_cumsum) with CUDA
events, L2 warm (the in-pipeline case), and check it bit for bit against numpy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2109_13504_b200 as mg
from paper_2109_13504_b200 import _lib, _device as D
from oracle import oracle

L = _lib.lib()
for prec, dt in (("single", 0), ("double", 1)):
    w_np = oracle.gen_gaussian_weights(4.0, 1 << 24, 31337, prec)
    w = torch.from_numpy(w_np).cuda()
    out = torch.empty_like(w)
    call = lambda: _lib.check(L.mgp_cumsum(D.ptr(w), dt, w.numel(), D.ptr(out), D.stream_ptr()))
    call(); torch.cuda.synchronize()
    ok = out.cpu().numpy().tobytes() == np.cumsum(w_np).tobytes()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); call(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    nb = w_np.nbytes * 2
    print(f"cumsum {prec}: median {ts[15]*1e3:.1f} us  min {ts[0]*1e3:.1f} us  {nb/ts[15]/1e6:.0f} GB/s  exact={ok}")
