import torch, time, ctypes, sys
sys.path.insert(0, '.')
import paper_2109_13504_b200 as mg
from paper_2109_13504_b200 import _lib
n = 1 << 24
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device='cuda')
ha = torch.empty(n, dtype=torch.int64).pin_memory()
da = torch.empty(n, dtype=torch.int64, device='cuda')
for name, fn in (("h2d 64MiB", lambda: d.copy_(h, non_blocking=True)), ("d2h 128MiB", lambda: ha.copy_(da, non_blocking=True))):
    for r in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for r in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(name, ms, "ms", (h.numel()*h.element_size() if 'h2d' in name else ha.numel()*8) / ms / 1e6, "GB/s")
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single", device="cuda").values
hw = w.cpu().pin_memory()
L = _lib.lib()
bu = ctypes.c_int32(0)
for r in range(3):
    _lib.check(L.mgp_resample_host(3, hw.data_ptr(), 0, n, 0, 0.01, 7, 32, 0, 1, 1, ha.data_ptr(), ctypes.byref(bu), -1))
ts = []
for r in range(10):
    t0 = time.perf_counter()
    _lib.check(L.mgp_resample_host(3, hw.data_ptr(), 0, n, 0, 0.01, 7, 32, 0, 1, 1, ha.data_ptr(), ctypes.byref(bu), -1))
    ts.append(time.perf_counter() - t0)
print("host path", sorted(ts)[5] * 1e3, "ms")
