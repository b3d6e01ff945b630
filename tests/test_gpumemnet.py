"""Neural GPUMemNet ensemble (carma_nn_*): the oracle pinned
to the torch model that defines the weights (CPU), and the tcgen05 kernel
against the oracle (GPU).

Tolerances (BASELINE.json north_star): logits within 1e-3 relative —
written here as |gpu - oracle| <= 1e-3 * max(1, |oracle|) — and identical
bins wherever the oracle's top-2 ensemble-probability margin exceeds 1e-3.
"""
import os

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi
from paper_2508_19073_b200 import gpumemnet as gm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "gpumemnet.npz")
TOL = 1e-3


def _oracle():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import gpumemnet_oracle
    return gpumemnet_oracle


@pytest.fixture(scope="module")
def models():
    m = gm.load_default_models()
    assert set(m) == {0, 1, 2}
    return m


def _golden(name):
    z = np.load(GOLDEN)
    rows = z[f"{name}_rows"].reshape(-1).view(abi.feature_row_dtype)
    return rows, z[f"{name}_raw"], z[f"{name}_logits"], z[f"{name}_labels"]


def _margin(probs):
    s = np.sort(probs, axis=1)
    return s[:, -1] - s[:, -2]


def _close(a, b, tol=TOL):
    return np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b))


# ------------------------------------------------------------------ CPU

@pytest.mark.parametrize("fam", [0, 1, 2])
def test_oracle_matches_torch_golden(models, fam):
    orc = _oracle()
    m = models[fam]
    rows, raw, logits, labels = _golden(gm.FAMILY_NAMES[fam])
    assert np.array_equal(cb.scalar_features(rows), raw)
    ol, op, ob, oby = orc.forward(m.spec()[0], m.params, raw)
    # golden logits are the torch fp64 forward stored as fp32
    assert np.all(np.abs(ol - logits) <= 1e-6 * np.maximum(1.0, np.abs(logits)))
    assert np.all((ob >= 0) & (ob < m.classes))
    assert np.array_equal(oby, (ob.astype(np.uint64) + 1) * np.uint64(m.bucket_range))
    assert np.allclose(op.sum(axis=1), 1.0)
    # the trained ensembles are useful estimators on fresh rows
    assert (ob == np.minimum(labels, m.classes - 1)).mean() > 0.9


@pytest.mark.parametrize("fam", [0, 1, 2])
def test_param_layout(models, fam):
    m = models[fam]
    assert gm.param_count(m) == len(m.params)
    assert 1 <= m.members <= abi.NN_MAX_MEMBERS
    assert all(1 <= d <= abi.NN_MAX_DEPTH for d in m.depth)
    assert m.classes == (41 if fam == 0 else 6)
    assert m.holdout_accuracy > 0.95
    orc = _oracle()
    assert len(orc.unpack_params(m.spec()[0], m.params)) == m.members


def test_bf16_rounding_is_nearest_even():
    orc = _oracle()
    x = np.array([1.0, 1.00390625, 1.01171875, -3.3, 0.0, 1e-30], np.float32)
    import torch
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(orc.bf16_round(x), ref)


# ------------------------------------------------------------------ GPU

def _predict_device(net, rows, fmt, q, family=None, default_family=0):
    import torch
    raw = torch.from_numpy(np.ascontiguousarray(rows).view(np.uint8).reshape(-1)).cuda()
    fam = None if family is None else torch.from_numpy(np.ascontiguousarray(family, np.int8)).cuda()
    b = torch.empty(q, dtype=torch.int32, device="cuda")
    by = torch.empty(q, dtype=torch.int64, device="cuda")
    pr = torch.full((q, abi.NN_MAX_CLASSES), float("nan"), dtype=torch.float32, device="cuda")
    lg = torch.full((q, abi.NN_MAX_MEMBERS, abi.NN_MAX_CLASSES), float("nan"), dtype=torch.float32, device="cuda")
    net.predict_device(raw, fmt, q, b, by, family=fam, default_family=default_family, probs=pr, logits=lg)
    torch.cuda.synchronize()
    return b.cpu().numpy(), by.cpu().numpy().view(np.uint64), pr.cpu().numpy(), lg.cpu().numpy()


def _check(m, raw, b, by, pr, lg):
    orc = _oracle()
    ol, op, ob, oby = orc.forward(m.spec()[0], m.params, raw)
    E, C = m.members, m.classes
    assert np.all(_close(lg[:, :E, :C], ol)), np.max(np.abs(lg[:, :E, :C] - ol))
    assert np.all(_close(pr[:, :C], op))
    sure = _margin(op) > TOL
    assert np.array_equal(b[sure], ob[sure])
    assert np.array_equal(by[sure], oby[sure])
    assert np.array_equal(by, (b.astype(np.uint64) + 1) * np.uint64(m.bucket_range))
    return float(np.max(np.abs(lg[:, :E, :C] - ol) / np.maximum(1.0, np.abs(ol))))


@pytest.mark.gpu
@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("path", [1, 2], ids=["tcgen05", "cuda-cores"])
def test_kernel_matches_oracle(gpu, models, fam, path):
    m = models[fam]
    net = gm.GpuMemNet(gpu)
    net.set_path(path)
    net.set_model(m)
    ds = cb.generate_synthetic_dataset(fam, 3000, 777 + fam)
    raw = cb.scalar_features(ds.rows)
    for fmt, rows in ((abi.ROWS_FEATURES, ds.rows), (abi.ROWS_SCALAR, raw)):
        b, by, pr, lg = _predict_device(net, rows, fmt, len(ds.rows), default_family=fam)
        err = _check(m, raw, b, by, pr, lg)
        assert err < 1e-4  # fp32 FMAs / three bf16 activation parts keep ~24 bits per layer
    t = net.last_timing()
    assert t["launches"] >= 1 and (t["mmas"] > 0) == (path == 1)
    # host-buffer API: same bins
    hb, hby = net.predict(ds.rows, default_family=fam)
    assert np.array_equal(hb, b) and np.array_equal(hby, by)
    net.close()


@pytest.mark.gpu
@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("path", [1, 2], ids=["tcgen05", "cuda-cores"])
def test_kernel_matches_golden(gpu, models, fam, path):
    m = models[fam]
    rows, raw, logits, _ = _golden(gm.FAMILY_NAMES[fam])
    net = gm.GpuMemNet(gpu)
    net.set_path(path)
    net.set_model(m)
    b, by, pr, lg = _predict_device(net, rows, abi.ROWS_FEATURES, len(rows), default_family=fam)
    assert np.all(_close(lg[:, : m.members, : m.classes], logits))
    net.close()


@pytest.mark.gpu
@pytest.mark.parametrize("q", [1, 2, 127, 128, 129, 1000, 100_003])
@pytest.mark.parametrize("path", [1, 2], ids=["tcgen05", "cuda-cores"])
def test_ragged_batches(gpu, models, q, path):
    m = models[1]
    net = gm.GpuMemNet(gpu)
    net.set_path(path)
    net.set_model(m)
    ds = cb.generate_synthetic_dataset(1, q, 99 + q)
    raw = cb.scalar_features(ds.rows)
    b, by, pr, lg = _predict_device(net, ds.rows, abi.ROWS_FEATURES, q, default_family=1)
    _check(m, raw, b, by, pr, lg)
    net.close()


@pytest.mark.gpu
@pytest.mark.parametrize("path", [1, 2], ids=["tcgen05", "cuda-cores"])
def test_mixed_families_route_by_row(gpu, models, path):
    """Packed / bit-packed rows carry their family: one call routes CNN, TF and
    MLP rows to their own ensembles; a family without a model -> no estimate."""
    net = gm.GpuMemNet(gpu)
    net.set_path(path)
    for f in (0, 1):
        net.set_model(models[f])  # no Transformer model installed
    parts = [cb.generate_synthetic_dataset(f, n, 50 + f) for f, n in ((0, 700), (1, 1300), (2, 500))]
    rows = np.concatenate([p.rows for p in parts])
    fams = np.concatenate([np.full(len(p.rows), p.family, np.int8) for p in parts])
    order = np.random.default_rng(3).permutation(len(rows))
    rows, fams = rows[order], fams[order]
    raw = cb.scalar_features(rows)
    q = len(rows)
    outs = []
    packed, table = cb.pack_features(rows, fams)
    net.set_act_table(table)
    outs.append(_predict_device(net, packed, abi.ROWS_PACKED, q))
    words, schema = cb.pack_features_bits(rows, fams)
    net.set_bit_schema(schema)
    outs.append(_predict_device(net, words, abi.ROWS_BITPACKED, q))
    outs.append(_predict_device(net, rows, abi.ROWS_FEATURES, q, family=fams))
    for b, by, pr, lg in outs:
        assert np.array_equal(b, outs[0][0]) and np.array_equal(by, outs[0][1])
        miss = fams == 2
        assert np.all(b[miss] == -1) and np.all(by[miss] == np.uint64(0xFFFFFFFFFFFFFFFF))
        for f in (0, 1):
            sel = fams == f
            _check(models[f], raw[sel], b[sel], by[sel], pr[sel], lg[sel])
    hb, hby = net.predict_bitpacked(words, schema, q)
    assert np.array_equal(hb, outs[0][0]) and np.array_equal(hby, outs[0][1])
    net.close()


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(8, 8, 48), (1, 1, 2), (3, 5, 17), (8, 1, 8)],
                         ids=["E8-L8-C48", "E1-L1-C2", "E3-L5-C17", "E8-L1-C8"])
@pytest.mark.parametrize("path", [1, 2], ids=["tcgen05", "cuda-cores"])
def test_extreme_shapes_random_weights(gpu, shape, path):
    """Random models at the limits of the spec: 8 members x 8 layers x 48
    bins (4 head passes), a single 1-layer member, odd widths."""
    E, L, C = shape
    rng = np.random.default_rng(E * 100 + L * 10 + C)
    depth = [int(rng.integers(1, L + 1)) if e else L for e in range(E)]
    width = [[int(rng.integers(1, 9)) for _ in range(d)] for d in depth]
    m = gm.NnModel(0, abi.GiB, C, depth, width, rng.normal(0, 1, 19).astype(np.float32) * 0.1,
                   np.full(19, 0.5, np.float32), np.zeros(1, np.float32))
    n = gm.param_count(m)
    m.params = (rng.normal(0, 0.6, n)).astype(np.float32)
    net = gm.GpuMemNet(gpu)
    net.set_path(path)
    net.set_model(m)
    ds = cb.generate_synthetic_dataset(0, 2000, 5)
    raw = cb.scalar_features(ds.rows)
    b, by, pr, lg = _predict_device(net, raw, abi.ROWS_SCALAR, len(raw), default_family=0)
    _check(m, raw, b, by, pr, lg)
    net.close()


@pytest.mark.gpu
def test_large_batch_host_api(gpu, models):
    """1M rows through the chunked host API equal the device call."""
    import torch
    m = models[2]
    net = gm.GpuMemNet(gpu)
    net.set_model(m)
    base = cb.generate_synthetic_dataset(2, 1 << 16, 11)
    rows = np.tile(base.rows, 16)
    hb, hby = net.predict(rows, default_family=2)
    db, dby, _, _ = _predict_device(net, base.rows, abi.ROWS_FEATURES, len(base.rows), default_family=2)
    assert np.array_equal(hb, np.tile(db, 16)) and np.array_equal(hby, np.tile(dby, 16))
    torch.cuda.synchronize()
    net.close()


@pytest.mark.gpu
def test_invalid_models_rejected(gpu, models):
    net = gm.GpuMemNet(gpu)
    m = models[1]
    bad = gm.NnModel(1, m.bucket_range, 49, m.depth, m.width, m.shift, m.scale, m.params)
    with pytest.raises(abi.CarmaError):
        net.set_model(bad)
    short = gm.NnModel(1, m.bucket_range, m.classes, m.depth, m.width, m.shift, m.scale, m.params[:-1])
    with pytest.raises(abi.CarmaError):
        net.set_model(short)
    with pytest.raises(abi.CarmaError):  # no model installed yet
        net.predict(cb.generate_synthetic_dataset(1, 4, 1).rows, default_family=1)
    net.close()


@pytest.mark.gpu
def test_neural_estimates_drive_the_replay(gpu, models):
    """The neural estimator in the loop: run_simulation with estimator
    'neural' places with the ensemble's bytes, and the fused device path
    (estimates written on the GPU, read by the replay) gives the same run."""
    rc = cb.RunConfig(mix="t90", trace_seed=3, policy=cb.PolicyConfig(policy="magm", estimator="neural"))
    m = cb.materialize_trace(cb.generate_trace("t90", 3))
    cb.provision_estimates(rc, m, gpu)
    net = gm.GpuMemNet(gpu)
    for mdl in models.values():
        net.set_model(mdl)
    _, nby = net.predict(m.features, family=m.family)
    assert np.array_equal(m.tasks["estimate"], nby)
    cfg = cb.make_config(rc.policy, rc.constants)
    host = cb.replay(cfg, [m.tasks], device=gpu)
    fr = cb.FusedReplay(cb.materialize_trace(cb.generate_trace("t90", 3)), cfg, net, gpu)
    fr.run()
    dev = fr.results()
    fr.close()
    assert dev.traces.tobytes() == host.traces.tobytes()
    assert dev.tasks.tobytes() == host.tasks.tobytes()
    tr, _, _ = cb.run_simulation(rc, device=gpu)
    assert tr.tobytes() == host.traces[0].tobytes()
    net.close()


# ------------------------------------------------- the Transformer ensemble

GOLDEN_TF = os.path.join(ROOT, "tests", "golden", "gpumemnet_tf.npz")


@pytest.fixture(scope="module")
def tf_models():
    m = gm.load_default_models(gm.ARCH_TRANSFORMER)
    assert set(m) == {0, 1, 2}
    return m


@pytest.mark.parametrize("fam", [0, 1, 2])
def test_tf_oracle_matches_torch_golden(tf_models, fam):
    orc = _oracle()
    m = tf_models[fam]
    z = np.load(GOLDEN_TF)
    name = gm.FAMILY_NAMES[fam]
    raw, logits = z[f"{name}_raw"], z[f"{name}_logits"]
    ol, op, ob, oby = orc.forward(m.spec()[0], m.params, raw)
    assert np.all(np.abs(ol - logits) <= 1e-5 * np.maximum(1.0, np.abs(logits)))
    assert gm.param_count(m) == len(m.params)
    assert m.holdout_accuracy > 0.9
    assert (ob == np.minimum(z[f"{name}_labels"], m.classes - 1)).mean() > 0.85


@pytest.mark.gpu
@pytest.mark.parametrize("fam", [0, 1, 2])
def test_tf_kernel_matches_oracle(gpu, tf_models, fam):
    m = tf_models[fam]
    net = gm.GpuMemNet(gpu)
    net.set_model(m)
    ds = cb.generate_synthetic_dataset(fam, 3000, 555 + fam)
    raw = cb.scalar_features(ds.rows)
    for fmt, rows in ((abi.ROWS_FEATURES, ds.rows), (abi.ROWS_SCALAR, raw)):
        b, by, pr, lg = _predict_device(net, rows, fmt, len(ds.rows), default_family=fam)
        assert _check(m, raw, b, by, pr, lg) < 1e-4
    hb, hby = net.predict(ds.rows, default_family=fam)
    assert np.array_equal(hb, b) and np.array_equal(hby, by)
    net.close()


@pytest.mark.gpu
def test_tf_and_mlp_banks_mix_by_family(gpu, models, tf_models):
    """A bank may hold a Transformer ensemble for one family and an MLP
    ensemble for another; bit-packed rows route per family."""
    net = gm.GpuMemNet(gpu)
    net.set_model(tf_models[1])
    net.set_model(models[2])
    parts = [cb.generate_synthetic_dataset(f, n, 70 + f) for f, n in ((1, 900), (2, 1100))]
    rows = np.concatenate([p.rows for p in parts])
    fams = np.concatenate([np.full(len(p.rows), p.family, np.int8) for p in parts])
    order = np.random.default_rng(4).permutation(len(rows))
    rows, fams = rows[order], fams[order]
    raw = cb.scalar_features(rows)
    words, schema = cb.pack_features_bits(rows, fams)
    net.set_bit_schema(schema)
    b, by, pr, lg = _predict_device(net, words, abi.ROWS_BITPACKED, len(rows))
    for f, mdl in ((1, tf_models[1]), (2, models[2])):
        sel = fams == f
        _check(mdl, raw[sel], b[sel], by[sel], pr[sel], lg[sel])
    net.close()


@pytest.mark.gpu
def test_grouped_rows_read_in_place(gpu, models):
    """Rows already grouped by family (the c2 batch) skip the permutation;
    the answers equal those of the same rows shuffled."""
    net = gm.GpuMemNet(gpu)
    for f in (0, 1):
        net.set_model(models[f])  # family 2 rows (last) have no model
    parts = [cb.generate_synthetic_dataset(f, n, 80 + f) for f, n in ((0, 1000), (1, 2100), (2, 300))]
    rows = np.concatenate([p.rows for p in parts])
    fams = np.concatenate([np.full(len(p.rows), p.family, np.int8) for p in parts])
    words, schema = cb.pack_features_bits(rows, fams)
    net.set_bit_schema(schema)
    gb, gby, _, _ = _predict_device(net, words, abi.ROWS_BITPACKED, len(rows))
    order = np.random.default_rng(5).permutation(len(rows))
    words2, schema2 = cb.pack_features_bits(rows[order], fams[order])
    net.set_bit_schema(schema2)
    sb, sby, _, _ = _predict_device(net, words2, abi.ROWS_BITPACKED, len(rows))
    assert np.array_equal(gb[order], sb) and np.array_equal(gby[order], sby)
    assert np.all(gb[fams == 2] == -1)
    net.close()


@pytest.mark.gpu
@pytest.mark.parametrize("path", [1, 2], ids=["tcgen05", "cuda-cores"])
def test_host_api_packed_staging_and_raw_fallback(gpu, models, path):
    """carma_nn_predict re-encodes host feature rows as 64-byte packed rows per
    chunk and falls back to raw rows for a chunk holding a non-registry
    activation; identical to the device-resident raw-row path."""
    parts = [cb.generate_synthetic_dataset(f, 200_000, 60 + f) for f in (0, 1, 2)]
    rows = np.concatenate([p.rows for p in parts])
    fams = np.concatenate([np.full(len(p.rows), p.family, np.int8) for p in parts])
    order = np.random.default_rng(4).permutation(len(rows))
    rows, fams = rows[order].copy(), fams[order].copy()
    fams[::991] = -1
    rows["act_cos"][350_001] = 0.3
    rows["total_params"][590_000] = 2**33 + 5  # that chunk: 64-byte rows, not the 40-byte compact ones
    net = gm.GpuMemNet(gpu)
    net.set_path(path)
    for f in (0, 1, 2):
        net.set_model(models[f])
    hb, hby = net.predict(rows, family=fams, default_family=0)
    import ctypes
    n = ctypes.c_uint64()
    abi.check(abi.lib.carma_nn_last_h2d_bytes(net.handle, ctypes.byref(n)))
    assert 40 * len(rows) < n.value < 137 * len(rows)  # compact, 64-byte and raw chunks
    db, dby, _, _ = _predict_device(net, rows, abi.ROWS_FEATURES, len(rows), family=fams)
    assert np.array_equal(hb, db) and np.array_equal(hby, dby)
    assert (hb[fams == -1] == -1).all()
    net.close()
