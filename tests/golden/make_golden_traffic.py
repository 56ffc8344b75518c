"""Golden comparison-index traces and traffic reports from the UNMODIFIED reference
(megores.resample.comparison_indices, M/resample.py:384-428; megores.warpsim, M/warpsim.py).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_traffic.py

Writes tests/golden/golden_traffic.json: per case the sha256 of the int64 (B, N) index matrix
and the TrafficReport fields.  tests/test_warpsim_gpu.py checks the device replay against it.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_traffic.json")

# (kind, n, b, seed, warp_size, partition_bytes)
CASES = [
    ("metropolis", 64, 32, 3, 32, None),
    ("metropolis", 4096, 8, 11, 32, None),
    ("metropolis", 1000, 5, 2, 8, None),
    ("c1", 4096, 8, 7, 32, 128),
    ("c1", 1024, 4, 9, 32, 2048),
    ("c1", 960, 6, 4, 7, 64),
    ("c2", 4096, 8, 5, 32, 256),
    ("c2", 2048, 3, 1, 16, 128),
    ("megopolis", 4096, 6, 5, 32, None),
    ("megopolis", 1000, 7, 12, 8, None),
    ("megopolis", 96, 9, 2**64 - 1, 7, None),
]


def main():
    import megores as m
    from megores.resample import comparison_indices
    from megores.warpsim import AccessTrace, traffic_report

    rows = []
    for kind, n, b, seed, ws, part in CASES:
        warp = m.WarpConfig(ws)
        idx = comparison_indices(kind, n, b, seed, warp, part)
        ent = {"kind": kind, "n": n, "b": b, "seed": seed, "warp": ws, "partition_bytes": part,
               "sha": hashlib.sha256(np.ascontiguousarray(idx, dtype=np.int64).tobytes()).hexdigest()[:32],
               "first": idx[0, :8].tolist()}
        if n % ws == 0:
            rep = traffic_report(AccessTrace(idx, warp))
            ent["report"] = [rep.total_transactions, rep.per_iteration_mean, rep.per_warp_max, rep.unnecessary_words]
        rows.append(ent)
    with open(OUT, "w") as fh:
        json.dump({"cases": rows}, fh, indent=1)
    print("wrote", OUT, len(rows))


if __name__ == "__main__":
    main()
