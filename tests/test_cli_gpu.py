"""The B200 CLI (``python -m paper_2109_13504_b200``) against the reference CLI's own output
files (tests/golden/cli/, made by tests/golden/make_golden_cli.py from the unmodified
``megores`` console script, M/bench.py).

* quality and traffic grids: byte-identical CSVs (bit-exact weights, B rule, resamplers, offspring and
  quality statistics, and the same float formatting);
* gen-weights and plotdata: byte-identical files (CPU only);
* pf: identical rows up to the filter's libm-rounded stages (rtol 1e-6);
* the reference's CLI contract: exit 2 + "megores: error:" on bad input, unknown config keys.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, ROOT)

from make_golden_cli import CASES, OUT, PLOT  # noqa: E402

from paper_2109_13504_b200 import cli  # noqa: E402


def run_cli(argv, tmp_path, name):
    out = str(tmp_path / name)
    rc = cli.main([a.format(out=out, dir=OUT) for a in argv])
    return rc, out


def gold(name):
    with open(os.path.join(OUT, name), "rb") as fh:
        return fh.read()


def test_gen_weights_byte_identical(tmp_path):
    argv, _ = CASES["gen_weights_gamma.bin"]
    rc, out = run_cli(argv, tmp_path, "gen_weights_gamma.bin")
    assert rc == 0
    assert open(out, "rb").read() == gold("gen_weights_gamma.bin")


def test_plotdata_byte_identical(tmp_path):
    rc, out = run_cli(PLOT[1], tmp_path, PLOT[0])
    assert rc == 0
    assert open(out, "rb").read() == gold(PLOT[0])


def test_cli_errors(tmp_path, capsys):
    assert cli.main(["traffic", "--algorithms", "c7", "--out", str(tmp_path / "t.csv")]) == 2
    assert "megores: error: unknown algorithm 'c7'" in capsys.readouterr().err
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"k_runs": 4, "bogus": 1}))
    assert cli.main(["quality", "--config", str(cfg), "--out", str(tmp_path / "q.csv")]) == 2
    assert "unknown config keys: ['bogus']" in capsys.readouterr().err
    assert cli.main(["quality", "--algorithms", "c1", "--out", str(tmp_path / "q.csv")]) == 2
    assert "c1 needs a partition size" in capsys.readouterr().err
    assert cli.main(["quality", "--k-runs", "1", "--out", str(tmp_path / "q.csv")]) == 2


def test_module_entry_point(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_2109_13504_b200", "gen-weights", "--family", "gaussian",
                        "--param", "1", "--n", "64", "--out", str(tmp_path / "w.bin")], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0 and "wrote" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["quality_single", "quality_double_gamma", "traffic_desk", "traffic_small"])
def test_quality_byte_identical(tmp_path, name):
    argv, _ = CASES[name]
    rc, out = run_cli(argv, tmp_path, name)
    assert rc == 0
    assert open(out, "rb").read() == gold(name)


@pytest.mark.gpu
def test_pf_matches_reference(tmp_path):
    argv, _ = CASES["pf_small"]
    rc, out = run_cli(argv, tmp_path, "pf_small")
    assert rc == 0
    ours = cli.read_csv(out)
    ref = cli.read_csv(os.path.join(OUT, "pf_small"))
    assert [r["algorithm"] for r in ours] == [r["algorithm"] for r in ref]
    for a, b in zip(ours, ref):
        assert {k: v for k, v in a.items() if k != "rmse"} == {k: v for k, v in b.items() if k != "rmse"}
        assert abs(float(a["rmse"]) - float(b["rmse"])) <= 1e-6 * float(b["rmse"])
    timings = cli.read_csv(out + ".timings.csv")
    assert len(timings) == len(ref) and all(0.0 < float(r["resample_ratio"]) < 1.0 for r in timings)
