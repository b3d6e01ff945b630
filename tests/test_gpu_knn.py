"""Stage 1 parity on the GPU: carma_knn_* vs the oracle restatement of
LearnedEstimator::predict_scalar (estimators.cpp:438-475). Bit-exact: buckets,
bytes, and the k nearest (d2, training index) pairs."""
import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi
from oracle_bind import oracle_predict

pytestmark = pytest.mark.gpu

FAMILIES = [(0, 11, 12345), (1, 112, 2024), (2, 213, 2025)]


def _device_predict(knn, rows, family=None, default_family=0, k=5, fmt=abi.ROWS_FEATURES):
    import torch

    q = len(rows)
    raw = torch.from_numpy(np.ascontiguousarray(rows).view(np.uint8).reshape(-1)).cuda()
    fam = None if family is None else torch.from_numpy(np.ascontiguousarray(family, np.int8)).cuda()
    b = torch.empty(q, dtype=torch.int32, device="cuda")
    by = torch.empty(q, dtype=torch.int64, device="cuda")
    d2 = torch.empty(q * k, dtype=torch.float64, device="cuda")
    idx = torch.empty(q * k, dtype=torch.int64, device="cuda")
    abi.check(abi.lib.carma_knn_predict_device(knn.handle, raw.data_ptr(), fmt,
                                               None if fam is None else fam.data_ptr(), default_family, q,
                                               b.data_ptr(), by.data_ptr(), d2.data_ptr(), idx.data_ptr(), None))
    torch.cuda.synchronize()
    return (b.cpu().numpy(), by.cpu().numpy().view(np.uint64), d2.cpu().numpy().reshape(q, k),
            idx.cpu().numpy().reshape(q, k))


@pytest.fixture(scope="module")
def models():
    return {f: cb.fit_knn(f, 4000, s, 5) for f, s, _ in FAMILIES}


@pytest.mark.parametrize("path", [1, 2], ids=["exact-fp64", "fp32-prefilter"])
@pytest.mark.parametrize("fam,seed,qseed", FAMILIES)
def test_knn_matches_oracle_bit_exact(gpu, olib, models, fam, seed, qseed, path):
    m = models[fam]
    knn = cb.GpuKnn(gpu)
    knn.set_model(m)
    abi.check(abi.lib.carma_knn_set_path(knn.handle, path))
    ds = cb.generate_synthetic_dataset(fam, 4096, qseed)
    raw = cb.scalar_features(ds.rows)
    ob, oby, od2, oidx = oracle_predict(olib, m, raw)
    b, by = knn.predict(ds.rows, default_family=fam)
    assert np.array_equal(b, ob)
    assert np.array_equal(by, oby)
    gb, gby, gd2, gidx = _device_predict(knn, ds.rows, default_family=fam)
    assert np.array_equal(gb, ob)
    assert np.array_equal(gd2.view(np.uint64), od2.view(np.uint64))  # same IEEE bits
    assert np.array_equal(gidx, oidx)
    # raw 19-feature rows (predict_scalar) give the same answer
    sb, sby = knn.predict(raw, default_family=fam)
    assert np.array_equal(sb, ob)
    launches, evals = knn.last_stats()
    assert launches >= 4 and 0 < evals < 4096 * len(m.labels)


def test_bank_routes_by_family_and_flags_mismatch(gpu, olib, models):
    knn = cb.GpuKnn(gpu)
    knn.set_model(models[1])
    knn.set_model(models[2])  # no MLP model: family 0 rows -> no estimate
    rows, fams, want_b = [], [], []
    for f, _, qs in FAMILIES:
        ds = cb.generate_synthetic_dataset(f, 700, qs + 1)
        rows.append(ds.rows)
        fams.append(np.full(700, f, np.int8))
        if f == 0:
            want_b.append(np.full(700, -1, np.int32))
        else:
            want_b.append(oracle_predict(olib, models[f], cb.scalar_features(ds.rows))[0])
    rows = np.concatenate(rows)
    fams = np.concatenate(fams)
    want_b = np.concatenate(want_b)
    perm = np.random.default_rng(5).permutation(len(rows))
    b, by = knn.predict(rows[perm], family=fams[perm])
    assert np.array_equal(b, want_b[perm])
    assert np.all(by[fams[perm] == 0] == np.uint64(0xFFFFFFFFFFFFFFFF))


@pytest.mark.parametrize("path", [1, 2], ids=["exact-fp64", "fp32-prefilter"])
@pytest.mark.parametrize("k", [1, 2, 4, 8, 16, 17, 40, 101])
def test_knn_k_variants_and_vote_ties(gpu, olib, k, path):
    """k <= 16: the register top-k search kernels; k > 16: the exact brute-force
    kernel (any k, estimators.cpp:460 kk = min(k, n))."""
    m = cb.fit_knn(1, 1500, 77, k)
    knn = cb.GpuKnn(gpu)
    knn.set_model(m)
    abi.check(abi.lib.carma_knn_set_path(knn.handle, path))
    ds = cb.generate_synthetic_dataset(1, 2000, 99)
    raw = cb.scalar_features(ds.rows)
    ob, oby, od2, oidx = oracle_predict(olib, m, raw)
    gb, gby, gd2, gidx = _device_predict(knn, ds.rows, default_family=1, k=k)
    assert np.array_equal(gb, ob)
    assert np.array_equal(gd2.view(np.uint64), od2.view(np.uint64))
    assert np.array_equal(gidx, oidx)


def test_knn_degenerate_models_ties_and_outliers(gpu, olib):
    rng = np.random.default_rng(3)
    # Duplicated points -> exact d2 ties broken by training index; k > n.
    n = 7
    pts = np.repeat(rng.random((3, 19)), [3, 2, 2], axis=0)[:n]
    pts[:, 5] = 0.0
    lo = np.zeros(19)
    hi = np.ones(19)
    hi[5] = 0.0  # a constant feature (hi == lo -> normalised to 0)
    labels = np.array([4, 4, 1, 2, 2, 3, 0], np.int32)
    for k in (3, 5, 9, 16, 25):
        m = cb.KnnModel(1, k, 8 * abi.GiB, lo, hi, pts.copy(), labels, np.zeros(0, np.int64))
        knn = cb.GpuKnn(gpu)
        knn.set_model(m)
        q = np.concatenate([pts, rng.random((200, 19)) * 3 - 1, np.full((1, 19), 1e12), np.zeros((1, 19))])
        ob, oby, od2, oidx = oracle_predict(olib, m, q, k=k)
        gb, gby, gd2, gidx = _device_predict(knn, q, default_family=1, k=k, fmt=abi.ROWS_SCALAR)
        assert np.array_equal(gb, ob)
        kk = min(k, n)
        assert np.array_equal(gd2[:, :kk].view(np.uint64), od2[:, :kk].view(np.uint64))
        assert np.array_equal(gidx[:, :kk], oidx[:, :kk])


def test_knn_empty_and_single(gpu, models):
    knn = cb.GpuKnn(gpu)
    knn.set_model(models[0])
    b, by = knn.predict(np.zeros(0, abi.feature_row_dtype), default_family=0)
    assert len(b) == 0
    ds = cb.generate_synthetic_dataset(0, 1, 5)
    b, _ = knn.predict(ds.rows, default_family=0)
    assert b.shape == (1,)


def test_knn_large_batch_subsample_parity(gpu, olib, models):
    """1M rows through the chunked host pipeline; a 3000-row sample vs the oracle,
    and determinism of the whole output."""
    ds = cb.generate_synthetic_dataset(2, 50_000, 31)
    rows = np.tile(ds.rows, 20)
    knn = cb.GpuKnn(gpu)
    knn.set_model(models[2])
    b1, by1 = knn.predict(rows, default_family=2)
    b2, _ = knn.predict(rows, default_family=2)
    assert np.array_equal(b1, b2)
    assert np.array_equal(b1.reshape(20, -1), np.broadcast_to(b1[:50_000], (20, 50_000)))
    sel = np.random.default_rng(0).choice(50_000, 3000, replace=False)
    ob, _, _, _ = oracle_predict(olib, models[2], cb.scalar_features(ds.rows[sel]))
    assert np.array_equal(b1[sel], ob)


def test_packed_rows_match_oracle(gpu, olib, models):
    """The 64-byte packed format (host + device paths) gives identical results."""
    rows, fams, want = [], [], []
    for f, _, qs in FAMILIES:
        ds = cb.generate_synthetic_dataset(f, 1500, qs + 7)
        rows.append(ds.rows)
        fams.append(np.full(1500, f, np.int8))
        want.append(oracle_predict(olib, models[f], cb.scalar_features(ds.rows))[0])
    rows, fams, want = np.concatenate(rows), np.concatenate(fams), np.concatenate(want)
    knn = cb.GpuKnn(gpu)
    for f in models:
        knn.set_model(models[f])
    packed, table = cb.pack_features(rows, fams)
    b, by = knn.predict_packed(packed, table)
    assert np.array_equal(b, want)
    abi.check(abi.lib.carma_knn_set_act_table(knn.handle, table.ctypes.data))
    gb, _, _, _ = _device_predict(knn, packed, k=5, fmt=abi.ROWS_PACKED)
    assert np.array_equal(gb, want)


@pytest.mark.parametrize("family", [0, 1, 2])
def test_gpu_knn_matches_reference_golden(gpu, family):
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "knn.npz"))
    fam, mseed, qseed, n = (int(x) for x in g["cases"][family])
    knn = cb.GpuKnn(gpu)
    knn.set_model(cb.fit_knn(fam, 4000, mseed, 5))
    ds = cb.generate_synthetic_dataset(fam, n, qseed)
    b, by = knn.predict(ds.rows, default_family=fam)
    assert np.array_equal(b, g[f"bucket_{family}"]) and np.array_equal(by, g[f"bytes_{family}"])


@pytest.mark.parametrize("path", [1, 2], ids=["exact-fp64", "fp32-prefilter"])
def test_knn_outlier_queries_and_near_ties(gpu, olib, models, path):
    """Queries far outside the training range (fp32 filter loses precision or
    would overflow -> exact fallback), duplicated training points (exact d2
    ties) and queries sitting exactly on training points."""
    m = models[1]
    pts = m.points.copy()
    pts[100:140] = pts[60:100]  # exact duplicates -> ties broken by index
    mm = cb.KnnModel(1, 5, m.bucket_range, m.lo, m.hi, pts, m.labels, m.holdout_rows)
    knn = cb.GpuKnn(gpu)
    knn.set_model(mm)
    abi.check(abi.lib.carma_knn_set_path(knn.handle, path))
    rng = np.random.default_rng(11)
    raw = cb.scalar_features(cb.generate_synthetic_dataset(1, 600, 4).rows)
    span = np.where(m.hi > m.lo, m.hi - m.lo, 1.0)
    on_pts = pts[55:105] * span + m.lo  # de-normalised training points
    huge = raw[:40].copy()
    huge[:, 5] *= 1e9
    huge[:10, 18] = 1e40
    q = np.concatenate([raw, on_pts, huge, raw[:20] * (1 + 1e-12)])
    ob, oby, od2, oidx = oracle_predict(olib, mm, q)
    gb, gby, gd2, gidx = _device_predict(knn, q, default_family=1, k=5, fmt=abi.ROWS_SCALAR)
    assert np.array_equal(gb, ob)
    assert np.array_equal(gd2.view(np.uint64), od2.view(np.uint64))
    assert np.array_equal(gidx, oidx)


def test_fp32_prefilter_cuts_fp64_work(gpu, models):
    knn = cb.GpuKnn(gpu)
    knn.set_model(models[2])
    ds = cb.generate_synthetic_dataset(2, 20000, 77)
    import ctypes
    la, e64, e32 = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    abi.check(abi.lib.carma_knn_set_path(knn.handle, 1))
    b1, _ = knn.predict(ds.rows, default_family=2)
    abi.check(abi.lib.carma_knn_last_work(knn.handle, ctypes.byref(la), ctypes.byref(e64), ctypes.byref(e32)))
    exact_only = e64.value
    abi.check(abi.lib.carma_knn_set_path(knn.handle, 2))
    b2, _ = knn.predict(ds.rows, default_family=2)
    abi.check(abi.lib.carma_knn_last_work(knn.handle, ctypes.byref(la), ctypes.byref(e64), ctypes.byref(e32)))
    assert np.array_equal(b1, b2)
    assert e32.value > 0 and e64.value * 4 < exact_only, (e64.value, e32.value, exact_only)


def test_bitpacked_rows_match_oracle(gpu, olib, models):
    rows, fams, want = [], [], []
    for f, _, qs in FAMILIES:
        ds = cb.generate_synthetic_dataset(f, 1200, qs + 9)
        rows.append(ds.rows)
        fams.append(np.full(1200, f, np.int8))
        want.append(oracle_predict(olib, models[f], cb.scalar_features(ds.rows))[0])
    rows, fams, want = np.concatenate(rows), np.concatenate(fams), np.concatenate(want)
    knn = cb.GpuKnn(gpu)
    for f in models:
        knn.set_model(models[f])
    words, schema = cb.pack_features_bits(rows, fams)
    b, by = knn.predict_bitpacked(words, schema, len(rows))
    assert np.array_equal(b, want)


@pytest.mark.parametrize("family", [0, 1, 2])
def test_train_learned_estimator_holdout_matches_reference(gpu, family):
    """train_learned_estimator's 30% holdout report, scored with the GPU
    predict: accuracy, macro-F1 and underestimate rate equal the reference's
    doubles bit for bit (estimators.cpp:396-434)."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "knn.npz"))
    fam, mseed, _, _ = (int(x) for x in g["cases"][family])
    est = cb.train_learned_estimator(fam, 4000, mseed, 5, device=gpu)
    want = g[f"holdout_{family}"]
    got = np.array([est.holdout.accuracy, est.holdout.macro_f1, est.holdout.underestimate_rate])
    assert got.tobytes() == want.tobytes(), (got, want)
    assert est.holdout.train_size == 2800 and est.holdout.holdout_size == 1200


@pytest.mark.parametrize("family,samples,seed", [(0, 4000, 11), (1, 4000, 112), (2, 4000, 213), (1, 777, 5),
                                                 (2, 5000, 3)])
def test_train_on_device_equals_host_fit(gpu, family, samples, seed):
    """carma_knn_train (bounds, normalised points and holdout on the GPU) fits
    exactly the model of the host restatement of estimators.cpp:344-395."""
    est = cb.train_learned_estimator(family, samples, seed, 5, device=gpu)
    m = cb.fit_knn(family, samples, seed, 5)
    assert np.array_equal(est.model.lo.view(np.uint64), m.lo.view(np.uint64))
    assert np.array_equal(est.model.hi.view(np.uint64), m.hi.view(np.uint64))
    assert np.array_equal(est.model.points.view(np.uint64), m.points.view(np.uint64))
    assert np.array_equal(est.model.labels, m.labels)
    assert np.array_equal(est.model.holdout_rows, m.holdout_rows)
    assert est.holdout.train_size == len(m.labels) and est.holdout.holdout_size == len(m.holdout_rows)
    ds = cb.generate_synthetic_dataset(family, 3000, seed + 1)
    k2 = cb.GpuKnn(gpu)
    k2.set_model(m)
    assert np.array_equal(est.predict(ds.rows), k2.predict(ds.rows, default_family=family)[0])


def _mixed_rows():
    """~700k rows over 3+ host-pipeline chunks: the three families, rows whose
    family is negative or has no model, and in one chunk a row whose
    activation is not a registry activation (that chunk cannot travel packed
    and goes as raw 136-byte rows)."""
    parts, fams = [], []
    for f, s in ((0, 3), (1, 4), (2, 5)):
        ds = cb.generate_synthetic_dataset(f, 230_000, s)
        parts.append(ds.rows)
        fams.append(np.full(230_000, f, np.int8))
    rows, fam = np.concatenate(parts), np.concatenate(fams)
    perm = np.random.default_rng(1).permutation(len(rows))
    rows, fam = rows[perm].copy(), fam[perm].copy()
    fam[::997] = -1
    fam[5::1009] = 7
    rows["act_cos"][400_123] = 0.3
    rows["act_sin"][400_123] = 0.25
    return rows, fam


def test_host_api_packed_staging_and_raw_fallback(gpu, models):
    """carma_knn_predict re-encodes host feature rows per chunk
    (csrc/host/stage.cpp): 40-byte compact rows (bit-packed, fixed schema)
    when every row fits, else 64-byte packed rows, else the raw rows.
    Chunks here: [0, 2^18) compact, [2^18, 2^19) raw (a non-registry
    activation), the rest 64-byte packed (a total_params >= 2^32). Results
    equal the device-resident raw-row path bit for bit."""
    import ctypes
    rows, fam = _mixed_rows()
    rows["total_params"][600_000] = 2**33 + 5
    knn = cb.GpuKnn(gpu)
    for f in models:
        knn.set_model(models[f])
    hb, hby = knn.predict(rows, family=fam, default_family=0)
    n = ctypes.c_uint64()
    abi.check(abi.lib.carma_knn_last_h2d_bytes(knn.handle, ctypes.byref(n)))
    c = 1 << 18
    assert n.value == 40 * c + 137 * c + 64 * (len(rows) - 2 * c)
    db, dby, _, _ = _device_predict(knn, rows, family=fam, default_family=0)
    assert np.array_equal(hb, db) and np.array_equal(hby, dby)
    assert (hb[fam == -1] == -1).all() and (hby[fam == 7] == np.uint64(2**64 - 1)).all()
    # no family array: default_family for every row, also out of range
    hb2, _ = knn.predict(rows[:300_000], default_family=2)
    db2, _, _, _ = _device_predict(knn, rows[:300_000], default_family=2)
    assert np.array_equal(hb2, db2)
    hb3, _ = knn.predict(rows[:1000], default_family=9)
    assert (hb3 == -1).all()


def test_host_api_pinned_rows_mix_raw_and_packed_chunks(gpu, models):
    """Pinned inputs: every other chunk ships raw (the copy engine reads the
    rows while the host pool packs the next chunk); results are identical."""
    import torch
    rows, fam = _mixed_rows()
    h_rows = torch.from_numpy(rows.view(np.uint8).reshape(-1)).pin_memory().numpy().view(abi.feature_row_dtype)
    h_fam = torch.from_numpy(fam).pin_memory().numpy()
    knn = cb.GpuKnn(gpu)
    for f in models:
        knn.set_model(models[f])
    hb, hby = knn.predict(h_rows, family=h_fam, default_family=0)
    import ctypes
    n = ctypes.c_uint64()
    abi.check(abi.lib.carma_knn_last_h2d_bytes(knn.handle, ctypes.byref(n)))
    assert 40 * len(rows) < n.value < 137 * len(rows)  # a mix of compact and raw chunks
    db, dby, _, _ = _device_predict(knn, rows, family=fam, default_family=0)
    assert np.array_equal(hb, db) and np.array_equal(hby, dby)
