"""Wall time per job of mgp_resample_host_batch (8 Megopolis jobs at 2^24, Philox and megores,
pinned in/out, B from epsilon) as in bench.py's e2e.batched; ancestors sha."""
import ctypes, hashlib, os, statistics, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402
n, count = 1 << 24, 8
L = _lib.lib()
w = torch.from_numpy(mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single").values).pin_memory()
outs = [torch.empty(n, dtype=torch.int64).pin_memory() for _ in range(2)]
hw = (ctypes.c_void_p * count)(*([w.data_ptr()] * count))
ha = (ctypes.c_void_p * count)(*[outs[k & 1].data_ptr() for k in range(count)])
sd = (ctypes.c_uint64 * count)(*([7] * count))
bu = (ctypes.c_int32 * count)()
for rng in ("philox", "megores"):
    def batch():
        _lib.check(L.mgp_resample_host_batch(_lib.KIND["megopolis"], hw, 0, n, count, 0, 0.01, sd, 32, 0, 1,
                                             _lib.RNG[rng], ha, bu, -1))
    batch()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        batch()
        ts.append(time.perf_counter() - t0)
    print(f"{rng:8s} {statistics.median(ts) / count * 1e3:.3f} ms/job  B {bu[0]}  sha {hashlib.sha256(outs[1].numpy().tobytes()).hexdigest()[:16]}", flush=True)
