"""CPU-side checks of the C ABI and the host logic (no GPU needed).

libmgp.so loads without a device; its host-only entry points (B rule, offsets,
argument validation) are exercised here against the golden vectors.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2109_13504_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2109_13504_b200 import build

    build.build()
    return _lib.lib()


def header_symbols():
    with open(os.path.join(ROOT, "include", "megopolis_b200.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(mgp_\w+)\(", txt, re.M)))


def test_every_header_symbol_exported(L):
    syms = header_symbols()
    assert set(syms) == set(_lib.SIGNATURES)
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} not bound in _lib.SIGNATURES"
    assert L.mgp_abi_version() == 1


def test_nm_exports_are_c_linkage(L):
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for s in header_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_compute_iterations_kats(L, golden):
    meta, _ = golden
    b = ctypes.c_int32()
    for r in meta["b_rule"]:
        assert L.mgp_compute_iterations(r["eps"], r["mean"], r["max"], ctypes.byref(b)) == 0
        assert b.value == r["b"], r
    # closed-form budgets T/test_weights.py:74-79
    import math

    for y, expect in {0: 4, 1: 6, 2: 16, 3: 60, 4: 354}.items():
        ratio = math.exp(-(y**2) / 4.0) / math.sqrt(2.0)
        assert L.mgp_compute_iterations(0.01, ratio, 1.0, ctypes.byref(b)) == 0 and b.value == expect
    assert L.mgp_compute_iterations(0.0, 0.5, 1.0, ctypes.byref(b)) == _lib.MGP_EINVAL
    assert L.mgp_compute_iterations(0.01, 2.0, 1.0, ctypes.byref(b)) == _lib.MGP_EINVAL
    assert b"exceeds" in L.mgp_last_error()


def test_python_compute_iterations_matches(golden):
    import paper_2109_13504_b200 as mg

    meta, _ = golden
    for r in meta["b_rule"]:
        assert mg.compute_iterations(r["eps"], r["mean"], r["max"]).b == r["b"]
    with pytest.raises(ValueError):
        mg.compute_iterations(0.0, 0.5, 1.0)


def test_offsets_host_golden(L, golden):
    import paper_2109_13504_b200 as mg

    meta, z = golden
    for o in meta["offsets"]:
        got = mg.megopolis_offsets(o["n"], o["b"], o["seed"])
        assert np.array_equal(got, z[o["name"]]), o


def test_offsets_host_philox_matches_oracle(oracle):
    import paper_2109_13504_b200 as mg

    for n, b, s in [(64, 9, 3), (2**24, 354, 7), (1000, 33, 2**64 - 1)]:
        assert np.array_equal(mg.megopolis_offsets(n, b, s, rng="philox"),
                              oracle.megopolis_offsets(n, b, s, rng="philox"))


def test_argument_validation_before_device(L):
    # invalid arguments are rejected on the host, before any device work
    null = ctypes.c_void_p(0)
    rc = L.mgp_megopolis(null, 0, 33, 4, 0, 32, 1, 0, 0, null, null)
    assert rc == _lib.MGP_EINVAL
    assert L.mgp_last_error() == b"megopolis requires N (33) to be a multiple of the warp size (32) in strict mode"
    assert L.mgp_metropolis(null, 0, 16, 0, 0, 0, 0, null, null) == _lib.MGP_EINVAL
    assert L.mgp_last_error() == b"B must be >= 1, got 0"
    assert L.mgp_metropolis_c1(null, 0, 64, 4, 0, 32, 130, 1, 0, 0, null, null) == _lib.MGP_EINVAL
    assert L.mgp_last_error() == b"partition_bytes must be a positive multiple of word_bytes"
    assert L.mgp_metropolis_c2(null, 0, 64, 4, 0, 32, 384, 1, 0, 0, null, null) == _lib.MGP_EINVAL
    assert L.mgp_last_error() == b"N=64 is not divisible by the partition width 96"
    assert L.mgp_megopolis(null, 7, 64, 4, 0, 32, 1, 0, 0, null, null) == _lib.MGP_EINVAL
    assert L.mgp_megopolis(null, 0, 2**31, 4, 0, 32, 1, 0, 0, null, null) == _lib.MGP_EUNSUPPORTED


def test_python_api_validation_cpu():
    import paper_2109_13504_b200 as mg

    with pytest.raises(ValueError):
        mg.WarpConfig(warp_size=0)
    with pytest.raises(ValueError):
        mg.PartitionConfig(0).n_weights(mg.WarpConfig())
    with pytest.raises(ValueError):
        mg.PartitionConfig(130).n_weights(mg.WarpConfig())
    with pytest.raises(ValueError):
        mg.PartitionConfig(3 * 128).n_partitions(64, mg.WarpConfig())
    assert mg.PartitionConfig(128).n_partitions(2**14, mg.WarpConfig()) == 512
    with pytest.raises(ValueError):
        mg.WeightVector(np.array([1.0, -0.5]))
    with pytest.raises(ValueError):
        mg.WeightVector(np.array([1.0, np.inf]))
    with pytest.raises(ValueError):
        mg.WeightVector(np.array([]))
    with pytest.raises(ValueError):
        mg.WeightVector(np.array([1.0]), precision="half")
    with pytest.raises(ValueError):
        mg.make_resampler("nope")
    with pytest.raises(ValueError):
        mg.make_resampler("c1")
    # megopolis_index hand traces (T/test_resample.py:126-151)
    W = mg.WarpConfig()
    assert mg.megopolis_index(5, 70, W, 128) == 75
    for i in (0, 5, 31, 127):
        assert mg.megopolis_index(i, 0, W, 128) == i
    for o in (0, 3, 70, 255):
        outs = {mg.megopolis_index(i, o, W, 256) for i in range(32, 64)}
        base = min(outs)
        assert base % 32 == 0 and outs == set(range(base, base + 32))


def test_derive_seed_matches_golden(golden):
    import paper_2109_13504_b200 as mg

    meta, _ = golden
    for parts, expect in meta["rng"]["derive_seed"]:
        assert mg.derive_seed(parts[0], *parts[1:]) == expect


def test_cpu_only_compute_fails_loudly():
    """No CPU fallback: compute entry points raise without a device."""
    import torch

    import paper_2109_13504_b200 as mg

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        mg.megopolis(mg.WeightVector(np.ones(64)), 4, seed=0)
    with pytest.raises(RuntimeError, match="CUDA device"):
        mg.ancestors_to_offspring(np.zeros(4, dtype=np.int64))


def test_shim_patches_both_namespaces(tmp_path, monkeypatch):
    """shim.install patches megores.<fn> and megores.resample.<fn> (M/__init__.py:12-28 binds at
    import; make_resampler resolves resample globals at call time, M/resample.py:441-454).
    Uses a stand-in package with the reference's layout; the GPU run of the real reference
    through the shim is tests/test_parity_gpu.py::test_shim_routes_reference_api."""
    import importlib
    import sys

    from paper_2109_13504_b200 import resample as R
    from paper_2109_13504_b200 import shim

    pkg = tmp_path / "fake_megores"
    pkg.mkdir()
    (pkg / "resample.py").write_text(
        "def metropolis(*a, **k): return 'cpu'\n"
        "def metropolis_c1(*a, **k): return 'cpu'\n"
        "def metropolis_c2(*a, **k): return 'cpu'\n"
        "def megopolis(*a, **k): return 'cpu'\n"
        "def ancestors_to_offspring(*a, **k): return 'cpu'\n"
        "def apply_ancestors(*a, **k): return 'cpu'\n"
        "def make_resampler(kind):\n"
        "    if kind == 'megopolis':\n"
        "        return lambda w, b, seed: megopolis(w, b, seed)\n"
        "    return lambda w, b, seed: metropolis(w, b, seed)\n")
    (pkg / "__init__.py").write_text("from .resample import (metropolis, metropolis_c1, metropolis_c2, megopolis,\n"
                                     "    ancestors_to_offspring, apply_ancestors, make_resampler)\n"
                                     "from .warpsim import traffic_report, count_transactions\n")
    (pkg / "warpsim.py").write_text("def trace_algorithm(*a, **k): return 'cpu'\n"
                                    "def traffic_report(*a, **k): return 'cpu'\n"
                                    "def count_transactions(*a, **k): return 'cpu'\n")
    (pkg / "bench.py").write_text("from .warpsim import trace_algorithm, traffic_report\n")
    monkeypatch.syspath_prepend(str(tmp_path))
    fm = importlib.import_module("fake_megores")
    saved = shim.install(fm, offspring=True, traffic=True)
    try:
        assert fm.megopolis is R.megopolis and fm.resample.megopolis is R.megopolis
        assert fm.metropolis_c2 is R.metropolis_c2 and fm.resample.apply_ancestors is R.apply_ancestors
        # make_resampler (resolved at call time) now reaches the B200 function
        fn = fm.make_resampler("megopolis")
        assert fn.__code__.co_names[0] == "megopolis" and fm.resample.megopolis is R.megopolis
        from paper_2109_13504_b200 import warpsim as W

        bench = sys.modules["fake_megores.bench"]
        assert fm.traffic_report is W.traffic_report and fm.warpsim.trace_algorithm is W.trace_algorithm
        assert bench.trace_algorithm is W.trace_algorithm and bench.traffic_report is W.traffic_report
    finally:
        shim.uninstall(fm, saved)
    assert fm.megopolis(1) == "cpu" and fm.resample.megopolis(1) == "cpu"
    assert fm.traffic_report() == "cpu" and sys.modules["fake_megores.bench"].trace_algorithm() == "cpu"
    for name in ("fake_megores", "fake_megores.resample", "fake_megores.warpsim", "fake_megores.bench"):
        sys.modules.pop(name, None)
