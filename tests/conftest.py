import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libmgp.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()
    return o


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="session")
def ref_megores():
    """The UNMODIFIED reference package staged under baseline/_ref (scripts/stage_reference.sh);
    a missing stage is a failure, not a skip."""
    if not os.path.isfile(os.path.join(REF_DIR, "megores", "resample.py")) and os.path.isdir("/root/reference/pkg"):
        import subprocess  # build container only: the GPU box has no /root/reference (it gets the staged copy)

        subprocess.run(["sh", os.path.join(ROOT, "scripts", "stage_reference.sh")], check=True)
    if not os.path.isfile(os.path.join(REF_DIR, "megores", "resample.py")):
        pytest.fail("unmodified reference not staged under baseline/_ref (run scripts/stage_reference.sh)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import megores

    assert os.path.realpath(os.path.dirname(megores.__file__)) == os.path.realpath(os.path.join(REF_DIR, "megores"))
    return megores
