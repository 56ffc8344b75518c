"""The reference's own test files, UNMODIFIED, with the B200 shim installed.

The unmodified reference package and its tests are staged under ``baseline/_ref/``
(``megores/`` and ``tests/``, copied from /root/reference/pkg by
``scripts/stage_reference.sh``; git-ignored, shipped to the GPU box with the snapshot).
A child pytest runs T/test_resample.py, T/test_acceptance.py and T/test_pfilter.py there
with ``-p mgp_ref_shim`` (tests/mgp_ref_shim.py), which patches megores' resamplers,
``ancestors_to_offspring`` and ``apply_ancestors`` (M/__init__.py:12-28,
M/resample.py:431-455) before collection.  The reference's exact pins then compare the
B200 kernels against the reference's own numba code on the same process:
``test_trace_fidelity_all_kernels`` (T/test_resample.py:353-376) checks every kernel's
comparison indices against ``comparison_indices``; the acceptance criteria
(T/test_acceptance.py) run their quality grid through the GPU.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
FILES = ("test_resample.py", "test_acceptance.py", "test_pfilter.py")


def _staged():
    return os.path.isfile(os.path.join(REF, "megores", "resample.py")) and all(
        os.path.isfile(os.path.join(REF, "tests", f)) for f in FILES)


@pytest.mark.parametrize("fname", FILES)
def test_reference_file_with_shim(fname, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pytest.importorskip("numba")
    assert _staged(), "unmodified reference not staged under baseline/_ref (scripts/stage_reference.sh)"
    report = tmp_path / "report.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests"), ROOT, env.get("PYTHONPATH", "")])
    env["MGP_REF_SHIM_REPORT"] = str(report)
    env.setdefault("NUMBA_CACHE_DIR", str(tmp_path / "numba"))
    ini = tmp_path / "pytest.ini"  # keep the repo's pytest.ini out of the child run
    ini.write_text("[pytest]\n")
    cmd = [sys.executable, "-m", "pytest", "-q", "-c", str(ini), "-p", "mgp_ref_shim", "-p", "no:cacheprovider",
           "--rootdir", os.path.join(REF, "tests"), os.path.join(REF, "tests", fname)]
    r = subprocess.run(cmd, cwd=os.path.join(REF, "tests"), env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    rep = json.loads(report.read_text())
    assert os.path.realpath(rep["megores"]) == os.path.realpath(os.path.join(REF, "megores"))
    assert rep["libmgp_mapped"], "libmgp.so was not loaded by the reference suite"
    routed = sum(v for k, v in rep["calls"].items())
    assert routed > 0, f"no resampler call went through the shim: {rep}"
    print(fname, rep["calls"])
