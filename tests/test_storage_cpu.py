"""Flat-file formats (M/storage.py) -- byte-compatible with the reference (T/test_storage.py)."""

import numpy as np
import pytest

import paper_2109_13504_b200 as mg
from paper_2109_13504_b200 import storage


def test_weight_roundtrip_both_precisions(tmp_path, oracle):
    for prec, n, width in (("single", 100, 4), ("double", 33, 8)):
        w = mg.WeightVector(oracle.gen_gaussian_weights(1.0, n, 3, prec), prec)
        p = tmp_path / f"w_{prec}.bin"
        storage.save_weights(p, w)
        assert p.stat().st_size == 8 + width * n
        back = storage.load_weights(p)
        assert back.precision == prec and np.array_equal(back.values, w.values)


def test_layout_is_reference_layout(tmp_path):
    p = tmp_path / "w.bin"
    storage.save_weights(p, mg.WeightVector(np.array([1.0, 2.0], dtype=np.float32), "single"))
    raw = p.read_bytes()
    assert raw[:8] == (2).to_bytes(8, "little") and np.frombuffer(raw[8:], "<f4").tolist() == [1.0, 2.0]


def test_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"\x01\x02")
    with pytest.raises(ValueError):
        storage.load_weights(p)
    p.write_bytes((3).to_bytes(8, "little") + b"\x00" * 10)
    with pytest.raises(ValueError):
        storage.load_weights(p)
    with pytest.raises(ValueError):
        storage.load_indices(p)


def test_indices_and_csv(tmp_path):
    idx = np.array([5, 0, 2**40, 7], dtype=np.int64)
    storage.save_indices(tmp_path / "i.bin", idx)
    assert np.array_equal(storage.load_indices(tmp_path / "i.bin"), idx)
    storage.save_weights_csv(tmp_path / "w.csv", mg.WeightVector(np.array([0.5, 1.25]), "double"))
    assert (tmp_path / "w.csv").read_text().strip().splitlines() == ["index,weight", "0,0.5", "1,1.25"]
    storage.save_indices_csv(tmp_path / "i.csv", [3, 1], column="ancestor")
    assert (tmp_path / "i.csv").read_text().strip().splitlines() == ["ancestor", "3", "1"]
    storage.save_trajectory_csv(tmp_path / "t.csv", [1.5, -2.0], [0.1, 0.2])
    lines = (tmp_path / "t.csv").read_text().strip().splitlines()
    assert lines[0] == "t,truth,observation" and lines[1].startswith("1,1.5,")
    with pytest.raises(ValueError):
        storage.save_trajectory_csv(tmp_path / "t.csv", [1.0], [1.0, 2.0])


def test_reads_files_written_by_the_reference(tmp_path, ref_megores):
    """Byte compatibility with the unmodified reference's storage module (staged under
    baseline/_ref by scripts/stage_reference.sh)."""
    megores = ref_megores
    from megores import storage as ref_storage

    w = megores.WeightVector(np.arange(1, 9, dtype=np.float32), "single")
    ref_storage.save_weights(tmp_path / "r.bin", w)
    back = storage.load_weights(tmp_path / "r.bin")
    assert back.precision == "single" and np.array_equal(back.values, w.values)
    storage.save_indices(tmp_path / "o.bin", np.array([3, 2, 1]))
    assert ref_storage.load_indices(tmp_path / "o.bin").tolist() == [3, 2, 1]
