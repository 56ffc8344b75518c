"""Golden CLI outputs from the UNMODIFIED reference (``megores`` console script, M/bench.py).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_cli.py

Runs the reference CLI on the argument lists in CASES and stores each output file under
tests/golden/cli/<name>.  tests/test_cli_gpu.py runs ``python -m paper_2109_13504_b200`` with
the same arguments and compares the files (byte for byte, except the particle-filter RMSE).
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")

# name -> (argv with {out}/{dir} placeholders, produced files)
CASES = {
    "quality_single": (["quality", "--algorithms", "megopolis,metropolis,c1:128,c2:256,multinomial,systematic",
                        "--n-grid", "256,2048", "--params", "0,1,4", "--k-runs", "4", "--sequences", "2",
                        "--seed", "11", "--out", "{out}"], ["{out}"]),
    "quality_double_gamma": (["quality", "--algorithms", "megopolis,c1:128", "--n-grid", "1024", "--family", "gamma",
                              "--params", "0.5,3", "--k-runs", "3", "--sequences", "2", "--precision", "double",
                              "--seed", "12", "--out", "{out}"], ["{out}"]),
    "gen_weights_gamma.bin": (["gen-weights", "--family", "gamma", "--param", "3", "--n", "3000", "--precision",
                               "double", "--seed", "9", "--out", "{out}"], ["{out}"]),
    "pf_small": (["pf", "--algorithms", "megopolis,c1:128,systematic", "--n", "1024", "--b-grid", "4,8",
                  "--trajectories", "2", "--runs", "2", "--t-steps", "20", "--seed", "5", "--out", "{out}"],
                 ["{out}", "{out}.timings.csv"]),
}
CASES.update({
    "traffic_desk": (["traffic", "--algorithms", "megopolis,metropolis,c1:128,c2:128,c1:2048,systematic",
                      "--n-grid", "1024,4096,65536", "--b", "8", "--seed", "13", "--out", "{out}"], ["{out}"]),
    "traffic_small": (["traffic", "--algorithms", "metropolis,c2:256,megopolis", "--n-grid", "64,256",
                       "--b", "32", "--seed", "3", "--out", "{out}"], ["{out}"]),
})
PLOT = ("plot_mse", ["plotdata", "--results", "{dir}/quality_single", "--figure", "mse-vs-N", "--out", "{out}"])


def main(only=None):
    """Regenerate every case, or only the named ones (``python make_golden_cli.py traffic_desk``)."""
    from megores import bench

    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        for name, (argv, files) in list(CASES.items()) + [(PLOT[0], (PLOT[1], ["{out}"]))]:
            if only and name not in only:
                continue
            out = os.path.join(tmp, name)
            rc = bench.main([a.format(out=out, dir=OUT) for a in argv])
            assert rc == 0, (name, rc)
            for f in files:
                src = f.format(out=out)
                shutil.copy(src, os.path.join(OUT, os.path.basename(src)))
            print("wrote", name, flush=True)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
