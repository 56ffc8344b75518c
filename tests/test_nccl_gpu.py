"""The NCCL data plane, executed: torchrun with one process on the box's GPU (world size 1),
``ShardedResampler(force_collectives=True)`` so every exchange of the sharded path -- weight
all-gathers, the stats all-gather behind the bit-exact global B, the owner-bucketed
all-to-alls of offspring counts and of apply_ancestors -- is a real NCCL collective, each
result checked bit for bit against one device's public API (tests/nccl_worker.py).  The
bench's sharded step runs the same way (``bench.py --sharded``), its timed ancestors checked
against the oracle.  NCCL_DEBUG=INFO must report the communicator (nRanks 1)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun(args, timeout=900):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, NCCL_DEBUG="INFO", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:]
    return json.loads(lines[-1]), r.stdout + r.stderr


def test_sharded_path_over_nccl_bit_exact():
    d, log = torchrun([os.path.join("tests", "nccl_worker.py")])
    assert d["backend"] == "nccl" and d["world"] == 1
    assert "nRanks 1" in log, "NCCL_DEBUG=INFO did not report the communicator"
    for c in d["checks"]:
        assert c["ancestors"] and c["offspring"], c
    assert d["quality"] and d["exchange"]


def test_bench_sharded_step_over_nccl():
    d, log = torchrun(["bench.py", "--sharded", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-config5",
                       "--no-probe", "--quality-runs", "2", "--no-e2e"])
    assert "nRanks 1" in log
    assert d["n_gpus"] == 1 and d["config"]["N"] == 1 << 24 and d["config"]["B"] == 354
    assert "sharded" in d["step_breakdown_ms"]["what"]
    assert d["parity"]["mismatches"] == 0 and d["parity"]["checked"] >= 1 << 20
    assert d["parity"]["other_stream"]["mismatches"] == 0
    assert d["quality"]["megopolis"]["mse_per_particle"] > 0
