# staged-copy phase times (MGP_HOST_TRACE) for a fresh vs a resident pageable output
MGP_HOST_TRACE=1 python - <<'PY' > gpurun_out/dropin_trace.txt 2>&1
import ctypes, os, sys, time
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
    print(f"total {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
for name, mk in (("fresh", lambda: np.empty(n, dtype=np.int64)), ("reused", lambda: reused), ("fresh", lambda: np.empty(n, dtype=np.int64)), ("reused", lambda: reused)):
    print("==", name, file=sys.stderr, flush=True)
    for _ in range(4):
        host(mk())
PY
