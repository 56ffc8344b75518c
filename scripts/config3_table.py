"""SURVEY config 3: Metropolis-C1/C2 at N=2^20 over partition sizes 128..2048 B, y in {0, 4},
C1 with and without shared-memory staging, both streams; plus Megopolis and Metropolis.

    python scripts/config3_table.py > profiles/rNN_config3.json
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

L = _lib.lib()
n = 1 << 20
out = {"n": n, "rows": []}
anc = torch.empty(n, dtype=torch.int64, device="cuda")
ref_anc = torch.empty(n, dtype=torch.int64, device="cuda")
sp = D.stream_ptr()
stream = torch.cuda.current_stream()


def timeit(fn, reps=5):
    ts = []
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for y in (0.0, 4.0):
    w = mg.gen_gaussian_weights(mg.GaussianWeightParams(y, n), 2024, "single", device="cuda")
    b = mg.iterations_for(w, 0.01).b
    for rng in ("megores", "philox"):
        def run(kind, ps, flags, dst):
            _lib.check(L.mgp_resample_range(_lib.KIND[kind], D.ptr(w.values), 0, n, b, 7, 32, ps, 1, _lib.RNG[rng],
                                            flags, 0, n, D.ptr(dst), sp))
        for kind in ("megopolis", "metropolis"):
            ms = timeit(lambda: run(kind, 0, 1, anc))
            out["rows"].append({"y": y, "B": b, "rng": rng, "kind": kind, "ps": None, "staged": None, "ms": ms})
        for ps in (128, 256, 512, 1024, 2048):
            for kind, flags in (("c1", 1), ("c1", 1 | _lib.FLAG_NO_STAGE), ("c2", 1)):
                ms = timeit(lambda: run(kind, ps, flags, anc))
                if kind == "c1" and flags & _lib.FLAG_NO_STAGE:
                    run(kind, ps, 1, ref_anc)
                    assert torch.equal(anc, ref_anc), "staged and direct C1 differ"
                out["rows"].append({"y": y, "B": b, "rng": rng, "kind": kind, "ps": ps,
                                    "staged": (kind == "c1" and not flags & _lib.FLAG_NO_STAGE), "ms": ms})
for r in out["rows"]:
    print(f"y={r['y']:.0f} B={r['B']:3d} {r['rng']:8s} {r['kind']:10s} ps={str(r['ps']):5s} staged={str(r['staged']):5s} "
          f"{r['ms']:.4f} ms", file=sys.stderr)
print(json.dumps(out, indent=1))
