"""The C ABI from a plain-C host (examples/resample_host.c): compiled with gcc against
include/megopolis_b200.h and libmgp.so, no Python on its compute path.

* CPU: the header and the example compile as strict C99 with every warning an error;
* GPU: the program's int64 ancestors (raw file and the reference's `<Q`-header weight file,
  M/storage.py:29-91) equal the Python API's and the oracle's, and invalid input exits 2 with
  the reference's message.
"""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

SRC = os.path.join(ROOT, "examples", "resample_host.c")
LIBDIR = os.path.join(ROOT, "paper_2109_13504_b200")


def _compile(tmp_path, link=True):
    exe = str(tmp_path / "resample_host")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), SRC]
    if link:
        cmd += ["-L", LIBDIR, "-lmgp", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    else:
        cmd += ["-c", "-o", exe + ".o"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_header_compiles_as_c99(tmp_path):
    _compile(tmp_path, link=False)


@pytest.mark.gpu
def test_c_host_matches_python_api(tmp_path, oracle):
    import paper_2109_13504_b200 as mg
    from paper_2109_13504_b200 import storage

    exe = _compile(tmp_path)
    n = 1 << 16
    w = oracle.gen_gaussian_weights(3.0, n, 99, "single")
    raw = tmp_path / "w.raw"
    w.tofile(raw)
    hdr = tmp_path / "w.bin"
    storage.save_weights(str(hdr), mg.WeightVector(w, "single"))
    b = mg.iterations_for(mg.WeightVector(w, "single"), 0.01).b
    for path, kind, rng in ((raw, 3, 0), (hdr, 3, 1), (raw, 0, 0)):
        out = subprocess.run([exe, str(path), "7", str(kind), str(rng)], capture_output=True, check=True)
        anc = np.frombuffer(out.stdout, dtype=np.int64)
        name = {3: "megopolis", 0: "metropolis"}[kind]
        rname = {0: "megores", 1: "philox"}[rng]
        assert np.array_equal(anc, mg.make_resampler(name, rng=rname)(w, b, 7))
        assert np.array_equal(anc, oracle.resample(name, w, b, 7, 32, None, True, rname))
    zero = tmp_path / "z.raw"
    np.zeros(64, np.float32).tofile(zero)
    bad = subprocess.run([exe, str(zero), "1"], capture_output=True, text=True)
    assert bad.returncode == 2 and "megores: error: all weights are zero" in bad.stderr
