"""Device weight generators: gen_gamma_weights / gen_gaussian_weights with
``device=`` against the reference's host formulas (M/weights.py:100-111).

Tolerances (the device path is not bit-exact; the default host path is):
* gamma, float64: |x_dev - x_scipy| <= 1e-12 * x_scipy for alpha in the reference CLI's grid
  (0.5, 2, 3, 10, 50) and alpha = 1 (M/bench.py:50), measured ~1e-14;
* gamma, float32: at most 1e-5 of the draws differ from scipy's float32 bytes, each by one ulp;
* the default (host) path is scipy's own bytes.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def mg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_13504_b200 as m

    return m


def scipy_gamma(alpha, beta, n, seed):
    from scipy import stats

    from paper_2109_13504_b200.rng import uniform_open01_at

    u = uniform_open01_at(seed, np.arange(n), 0)
    return stats.gamma.ppf(u, a=alpha, scale=1.0 / beta)


@pytest.mark.parametrize("alpha", [0.5, 1.0, 2.0, 3.0, 10.0, 50.0])
def test_device_gamma_vs_scipy(mg, alpha):
    n = 1 << 17
    ref = scipy_gamma(alpha, 1.0, n, 4242)
    w64 = mg.gen_gamma_weights(mg.GammaWeightParams(alpha, 1.0, n), 4242, "double", device="cuda")
    assert w64.on_device and w64.values.dtype == torch.float64
    got = w64.values.cpu().numpy()
    rel = np.abs(got - ref) / ref
    assert rel.max() <= 1e-12, rel.max()
    w32 = mg.gen_gamma_weights(mg.GammaWeightParams(alpha, 1.0, n), 4242, "single", device=0).values.cpu().numpy()
    r32 = ref.astype(np.float32)
    bad = w32 != r32
    assert bad.mean() <= 1e-5
    ulps = np.abs(w32.view(np.int32).astype(np.int64) - r32.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1


def test_device_gamma_rate_and_extremes(mg):
    n = 4096
    for alpha, beta in ((2.0, 0.25), (0.5, 8.0)):
        ref = scipy_gamma(alpha, beta, n, 9)
        got = mg.gen_gamma_weights(mg.GammaWeightParams(alpha, beta, n), 9, "double", device="cuda").values.cpu().numpy()
        assert np.allclose(got, ref, rtol=1e-12, atol=0)
    # extreme uniforms through the kernel's own draws: every value finite and positive
    big = mg.gen_gamma_weights(mg.GammaWeightParams(3.0, 1.0, 1 << 20), 1, "double", device="cuda").values
    assert bool(torch.isfinite(big).all()) and float(big.min()) > 0


def test_default_gamma_is_reference_bytes(mg):
    n = 2048
    w = mg.gen_gamma_weights(mg.GammaWeightParams(2.0, 1.0, n), 77, "single")
    assert isinstance(w.values, np.ndarray)
    assert np.array_equal(w.values, scipy_gamma(2.0, 1.0, n, 77).astype(np.float32))


def test_gamma_moments_2p24(mg):
    """T/test_weights.py:32-42 at 2^24 on the device: exponential mean 1; alpha = 50 mean/var."""
    n = 1 << 24
    w = mg.gen_gamma_weights(mg.GammaWeightParams(1.0, 1.0, n), 8, "double", device="cuda").values
    assert abs(float(w.mean()) - 1.0) < 5 * (1.0 / np.sqrt(n))
    w = mg.gen_gamma_weights(mg.GammaWeightParams(50.0, 1.0, n), 9, "double", device="cuda").values
    assert abs(float(w.mean()) - 50.0) < 5 * np.sqrt(50.0 / n)
    assert abs(float(w.var()) - 50.0) < 0.5


def test_gamma_rejects_bad_shape(mg):
    from paper_2109_13504_b200 import _lib

    out = torch.empty(4, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError, match="alpha and beta must be > 0"):
        _lib.check(_lib.lib().mgp_gen_gamma(0.0, 1.0, 4, 1, 0, out.data_ptr(), None))


def test_cli_device_weights_route(mg, tmp_path):
    """cli gen-weights/quality with --device-weights-from: the HBM generators feed the same
    pipeline; below the threshold the bytes stay the reference's."""
    from paper_2109_13504_b200 import cli, storage

    out = str(tmp_path / "g.bin")
    assert cli.main(["gen-weights", "--family", "gamma", "--param", "3", "--n", "8192", "--seed", "5", "--out", out,
                     "--device-weights-from", "4096"]) == 0
    dev = storage.load_weights(out)
    out2 = str(tmp_path / "h.bin")
    assert cli.main(["gen-weights", "--family", "gamma", "--param", "3", "--n", "8192", "--seed", "5", "--out", out2]) == 0
    host = storage.load_weights(out2)
    dv, hv = np.asarray(dev.values), np.asarray(host.values)
    assert np.allclose(dv, hv, rtol=1e-6, atol=0) and (dv != hv).mean() <= 1e-3
    q = str(tmp_path / "q.csv")
    assert cli.main(["quality", "--algorithms", "megopolis", "--n-grid", "4096", "--family", "gamma", "--params", "2",
                     "--k-runs", "4", "--sequences", "1", "--out", q, "--device-weights-from", "1"]) == 0
    assert sum(1 for ln in open(q) if ln.strip() and not ln.startswith("#")) == 2  # header + one row
