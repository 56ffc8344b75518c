"""Library contract details (ADVICE round 1 and VERDICT "library hygiene"):

* C1/C2 over a particle range whose end is not warp-aligned (the straddling warp stays whole);
* WarpConfig.word_bytes reaches the partition geometry (n_w = partition_bytes // word_bytes,
  M/resample.py:84-87), checked against the unmodified reference;
* QualityAccumulator rejects length mismatches before any launch (M/metrics.py:86-93);
* a WeightVector over a caller's CUDA tensor sees in-place updates (no stale statistics);
* the weight-texture LRU evicts safely past its capacity;
* scratch comes from the library's private pool: the device default pool is untouched;
* pageable and pinned host buffers give the same ancestors.
"""

import ctypes

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


def lib():
    from paper_2109_13504_b200 import _lib

    return _lib


@pytest.mark.parametrize("kind,part", [("c1", 256), ("c2", 128), ("c1", 2048), ("megopolis", 0), ("metropolis", 0)])
def test_unaligned_range_end(mg, oracle, kind, part):
    L = lib()
    n, b = 1 << 14, 23
    w = oracle.gen_gaussian_weights(3.0, n, 5, "single")
    wd = torch.from_numpy(w).cuda()
    full = oracle.resample(kind, w, b, 17, 32, part or None, True, "megores")
    for p0, p1 in ((0, 7), (32, 61), (4096, 4096 + 1000), (n - 64, n - 1), (96, 97)):
        out = torch.full((p1 - p0,), -1, dtype=torch.int64, device="cuda")
        L.check(L.lib().mgp_resample_range(L.KIND[kind], wd.data_ptr(), 0, n, b, 17, 32, part, 1, L.RNG["megores"], 0,
                                           p0, p1, out.data_ptr(), None))
        assert np.array_equal(out.cpu().numpy(), full[p0:p1]), (kind, p0, p1)


def test_word_bytes_geometry(mg, ref_megores):
    m = ref_megores
    rs = np.random.default_rng(4)
    w = rs.random(4096).astype(np.float32) ** 3
    for kind in ("c1", "c2"):
        for wb, pb in ((8, 256), (8, 1024), (4, 256), (16, 512)):
            warp_ref = m.WarpConfig(word_bytes=wb, segment_bytes=max(32, wb))
            fn_ref = m.metropolis_c1 if kind == "c1" else m.metropolis_c2
            want = fn_ref(m.WeightVector(w, "single"), 9, m.PartitionConfig(pb), warp_ref, 21)
            warp = mg.WarpConfig(word_bytes=wb, segment_bytes=max(32, wb))
            fn = mg.metropolis_c1 if kind == "c1" else mg.metropolis_c2
            got = fn(mg.WeightVector(w, "single"), 9, mg.PartitionConfig(pb), warp, 21)
            assert np.array_equal(got, want), (kind, wb, pb)
            gd = fn(mg.WeightVector(torch.from_numpy(w).cuda(), "single"), 9, mg.PartitionConfig(pb), warp, 21)
            assert np.array_equal(gd.cpu().numpy(), want), (kind, wb, pb)


def test_quality_length_checks(mg):
    acc = mg.QualityAccumulator(64)
    w = mg.WeightVector(np.ones(64), "double")
    with pytest.raises(ValueError, match="length mismatch"):
        acc.add(np.ones(32, dtype=np.int64), w)
    with pytest.raises(ValueError, match="length mismatch"):
        acc.add(np.ones(64, dtype=np.int64), mg.WeightVector(np.ones(32), "double"))
    with pytest.raises(ValueError, match="length mismatch"):
        acc.add_runs("megopolis", mg.WeightVector(np.ones(128), "double"), 3, [1, 2])
    assert acc.k == 0
    acc.add(np.ones(64, dtype=np.int64), w)
    acc.add(np.ones(64, dtype=np.int64), w)
    assert acc.finalize().mse == 0.0


def test_device_weights_follow_inplace_updates(mg, oracle):
    n = 4096
    w = oracle.gen_gaussian_weights(1.0, n, 3, "single")
    t = torch.from_numpy(w).cuda()
    wv = mg.WeightVector(t, "single")
    a0 = mg.megopolis(wv, 7, seed=1).cpu().numpy()
    assert np.array_equal(a0, oracle.megopolis(w, 7, seed=1))
    t[: n // 2] = 0.0  # zeros now present: the non-zero fast path must not be taken
    w2 = t.cpu().numpy()
    a1 = mg.megopolis(wv, 7, seed=1).cpu().numpy()
    assert np.array_equal(a1, oracle.megopolis(w2, 7, seed=1))
    assert wv.stats().n_zero == n // 2
    t[0] = float("nan")
    with pytest.raises(ValueError, match="finite"):
        mg.megopolis(wv, 7, seed=1)


def test_texture_cache_eviction(mg, oracle):
    """More distinct float32 weight arrays than the texture LRU holds (64), interleaved with
    re-use of the first ones: every result stays bit-exact."""
    n = 2048
    ws = [oracle.gen_gaussian_weights(2.0, n, 100 + k, "single") for k in range(80)]
    dev = [torch.from_numpy(w).cuda() for w in ws]
    refs = [oracle.megopolis(w, 5, seed=9) for w in ws]
    s = torch.cuda.Stream()
    for k in list(range(80)) + [0, 1, 2, 79, 40]:
        with torch.cuda.stream(s if k % 3 == 0 else torch.cuda.current_stream()):
            got = mg.megopolis(mg.WeightVector(dev[k], "single"), 5, seed=9)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), refs[k]), k


def test_private_pool_leaves_default_pool(mg, oracle):
    rt = pytest.importorskip("cuda.bindings.runtime")
    dev = torch.cuda.current_device()
    err, pool = rt.cudaDeviceGetDefaultMemPool(dev)
    assert int(err) == 0
    attr = rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold
    err, before = rt.cudaMemPoolGetAttribute(pool, attr)
    w = oracle.gen_gaussian_weights(2.0, 1 << 16, 1, "single")
    mg.megopolis(mg.WeightVector(w, "single"), 6, seed=2)  # host path: scratch + buffers
    mg.multinomial(mg.WeightVector(torch.from_numpy(w).cuda(), "single"), 3)  # prefix-sum scratch
    torch.cuda.synchronize()
    err, after = rt.cudaMemPoolGetAttribute(pool, attr)
    assert int(after) == int(before)
    assert int(after) != 2**64 - 1
    L = lib()
    L.check(L.lib().mgp_release_cached_memory(-1))
    L.check(L.lib().mgp_release_cached_memory(dev))


def test_pageable_and_pinned_host_buffers(mg, oracle):
    L = lib()
    n = 1 << 22
    w = oracle.gen_gaussian_weights(4.0, n, 11, "single")
    outs = []
    for pinned in (False, True):
        hw = torch.from_numpy(w)
        ha = torch.empty(n, dtype=torch.int64)
        if pinned:
            hw, ha = hw.pin_memory(), ha.pin_memory()
        bu = ctypes.c_int32(0)
        for rng in ("philox", "megores"):
            L.check(L.lib().mgp_resample_host(L.KIND["megopolis"], hw.data_ptr(), 0, n, 0, 0.01, 3, 32, 0, 1,
                                              L.RNG[rng], ha.data_ptr(), ctypes.byref(bu), -1))
            outs.append((rng, ha.numpy().copy()))
    assert np.array_equal(outs[0][1], outs[2][1]) and np.array_equal(outs[1][1], outs[3][1])
    b = int(bu.value)
    for rng, a in outs[:2]:
        for p0 in (0, n // 2 - 64, n - 128):
            ref = oracle.megopolis(w, b, seed=3, rng=rng, p0=p0, p1=p0 + 128)
            assert np.array_equal(a[p0:p0 + 128], ref[p0:p0 + 128]), (rng, p0)
