"""The bench contract's CPU side: ``bench.py --impl reference`` (the reference arm: the CPU port of
the path, timed on the host's cores) prints one JSON line with the contract's keys, on a machine
without a GPU."""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                        "--n", "65536"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "particles/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"] and d["config"]["N"] == 65536
    assert d["config"]["rng"] == "philox" and d["scaling"] == "strong"
    assert d["cpu_baseline"]["cpu_model"] and d["cpu_baseline"]["median_s"] > 0


def test_reference_arm_loads_no_product_library():
    """The reference arm's process maps liboracle.so and never libmgp.so (its inputs are the
    reference's weight bytes from the oracle, not the product's generator)."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '1', "
            "'--n', '8192']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "sys.stderr.write('MAPS ' + str('libmgp' in maps) + ' ' + str('liboracle.so' in maps) + '\\n')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "MAPS False True" in r.stderr


def test_both_arms_print_the_same_config():
    sys.path.insert(0, ROOT)
    import bench

    a = bench.workload_config(1 << 24, 354, "philox", 1)
    assert a == bench.workload_config(1 << 24, 354, "philox", 1)
    assert a["N"] == 1 << 24 and a["B"] == 354 and "strong" in a["parallelism"]
