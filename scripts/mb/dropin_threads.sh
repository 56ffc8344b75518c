# drop-in host entry (pageable in, fresh/reused pageable out) against the host pool's thread count
for t in 16 8 4 2 16 8 4 2; do
MGP_HOST_TRACE=1 MGP_HOST_THREADS=$t python - <<'PY' >> gpurun_out/dropin_threads.txt 2>/dev/null
import ctypes, os, sys, time, statistics
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2109_13504_b200 as mg
from paper_2109_13504_b200 import _lib
n, b = 1 << 24, 354
L = _lib.lib()
w = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, n), 20240, "single").values
reused = np.empty(n, dtype=np.int64); reused.fill(1)
def host(out):
    bu = ctypes.c_int32(0)
    t0 = time.perf_counter()
    _lib.check(L.mgp_resample_host(_lib.KIND["megopolis"], w.ctypes.data, 0, n, b, 0.0, 7, 32, 0, 1, _lib.RNG["philox"], out.ctypes.data, ctypes.byref(bu), -1))
    return 1e3 * (time.perf_counter() - t0)
host(reused)
for name, mk in (("fresh", lambda: np.empty(n, dtype=np.int64)), ("reused", lambda: reused)):
    ts = [host(mk()) for _ in range(6)]
    print(f"threads {os.environ['MGP_HOST_THREADS']:>2s} {name:6s} median {statistics.median(ts):6.2f} min {min(ts):6.2f} ms", flush=True)
PY
done
