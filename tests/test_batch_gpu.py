"""mgp_resample_host_batch / resample_batch: independent host-buffer resamples pipelined over two
device slots give the same ancestors (and B) as one mgp_resample_host call per job, for every
resampler kind and both streams, with page-locked and pageable buffers, outputs repeating every
other job, and per-job validation errors."""

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


def jobs(n, count, seed):
    rs = np.random.default_rng(seed)
    ws = [(rs.random(n) ** (1 + k)).astype(np.float32) for k in range(count)]
    ws[1][rs.random(n) < 0.05] = 0  # zero weights in one job (no NONZERO fast path there)
    return ws


CASES = [(k, p, r) for k, p in (("megopolis", None), ("c1", 128), ("c2", 256), ("metropolis", None))
         for r in ("megores", "philox")] + [("multinomial", None, "megores"), ("systematic", None, "megores")]


@pytest.mark.parametrize("kind,part,rng", CASES)
def test_batch_matches_single_calls(mg, kind, part, rng):
    n, count = 1 << 14, 5
    ws = jobs(n, count, 3)
    seeds = [11 * k + 1 for k in range(count)]
    pc = mg.PartitionConfig(part) if part else None
    outs, bs = mg.resample_batch(kind, ws, 0, seeds, part=pc, rng=rng)
    # against the one-call host entry for every job: same B, same ancestors
    import ctypes

    from paper_2109_13504_b200 import _lib
    from paper_2109_13504_b200.resample import abi_partition_bytes

    pb = abi_partition_bytes(part, mg.WarpConfig()) if part else 0
    for k in range(count):
        one = np.empty(n, dtype=np.int64)
        bu = ctypes.c_int32(0)
        _lib.check(_lib.lib().mgp_resample_host(_lib.KIND[kind], ws[k].ctypes.data, 0, n, 0, 0.01, seeds[k], 32, pb, 1,
                                                _lib.RNG[rng], one.ctypes.data, ctypes.byref(bu), -1))
        assert bs[k] == bu.value, k
        assert np.array_equal(outs[k], one), (kind, rng, k)


def test_batch_pinned_aliased_outputs_and_errors(mg):
    n, count = 1 << 20, 6
    ws = [torch.from_numpy(w).pin_memory().numpy() for w in jobs(n, count, 5)]
    seeds = list(range(100, 100 + count))
    ref = [mg.megopolis(ws[k], 40, seed=seeds[k], rng="philox") for k in range(count)]
    pinned = [torch.empty(n, dtype=torch.int64).pin_memory().numpy() for _ in range(2)]
    got, bs = mg.resample_batch("megopolis", ws, 40, seeds, rng="philox", out=[pinned[k & 1] for k in range(count)])
    assert bs == [40] * count
    # outputs repeat every other job: the last two jobs' ancestors remain
    assert np.array_equal(pinned[(count - 1) & 1], ref[count - 1])
    assert np.array_equal(pinned[(count - 2) & 1], ref[count - 2])
    bad = [w.copy() for w in ws[:3]]
    bad[2][7] = np.nan
    with pytest.raises(ValueError, match="finite"):
        mg.resample_batch("megopolis", bad, 0, [1, 2, 3])
    with pytest.raises(ValueError):
        mg.resample_batch("megopolis", ws[:2], 0, [1])


@pytest.mark.parametrize("kind,part,rng,n", [("megopolis", None, "philox", 1 << 22), ("megopolis", None, "megores", 1 << 21),
                                             ("megopolis", None, "megores", (1 << 21) + 4096),
                                             ("c2", 128, "philox", 3 << 20), ("systematic", None, "megores", 1 << 21)])
def test_batch_last_job_chunked(mg, kind, part, rng, n):
    """n >= 2^21: the batch's last job runs in particle chunks (last chunk split) with per-chunk
    downloads (MGP_BATCH_LAST_CHUNKED); every job, the chunked last one included, equals one
    mgp_resample_host call, into page-locked outputs."""
    import ctypes

    from paper_2109_13504_b200 import _lib
    from paper_2109_13504_b200.resample import abi_partition_bytes

    count = 3
    ws = [torch.from_numpy(w).pin_memory().numpy() for w in jobs(n, count, 9)]
    outs = [torch.empty(n, dtype=torch.int64).pin_memory().numpy() for _ in range(count)]
    seeds = [5 * k + 2 for k in range(count)]
    pc = mg.PartitionConfig(part) if part else None
    got, bs = mg.resample_batch(kind, ws, 0, seeds, part=pc, rng=rng, out=outs)
    pb = abi_partition_bytes(part, mg.WarpConfig()) if part else 0
    for k in range(count):
        one = np.empty(n, dtype=np.int64)
        bu = ctypes.c_int32(0)
        _lib.check(_lib.lib().mgp_resample_host(_lib.KIND[kind], ws[k].ctypes.data, 0, n, 0, 0.01, seeds[k], 32, pb, 1,
                                                _lib.RNG[rng], one.ctypes.data, ctypes.byref(bu), -1))
        assert bs[k] == bu.value, k
        assert np.array_equal(got[k], one), (kind, rng, n, k)
