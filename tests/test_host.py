"""CPU tests of the host side: the C-ABI library loads and exports every
declared symbol, compute entry points fail loudly without a GPU, and the
host provisioning (traces, datasets, features, packing) behaves."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = []
    for h in ("carma_gpu.h", "carma_host.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"^(?:carma_status|int|const char\*)\s+(carma_\w+)\(", text, re.M)
    return names


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 30
    lib = ctypes.CDLL(abi.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(abi.SIGNATURES), set(names) - set(abi.SIGNATURES)


def test_no_gpu_fails_loudly():
    if abi.lib.carma_device_count() > 0:
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    st = abi.lib.carma_knn_create(0, ctypes.byref(h))
    assert st == 2  # CARMA_ERR_CUDA: no CPU fallback
    assert b"no CPU fallback" in abi.lib.carma_last_error()


def test_catalog_and_trace_shapes():
    cat = cb.builtin_catalog()
    assert len(cat) == 35
    assert sum(1 for e in cat if e.gpus == 2) == 3
    t90 = cb.generate_trace("t90", 1)
    t60 = cb.generate_trace("t60", 1)
    assert len(t90) == 90 and len(t60) == 60
    assert np.all(np.diff(t90.submit) >= 0) and t90.submit[0] == 0.0
    m = cb.materialize_trace(t90)
    assert sorted(m.tasks["rank"].tolist()) == list(range(90))
    assert np.array_equal(m.tasks["rank"], np.arange(90))  # 3-digit ids sort in index order


def test_rank_is_lexicographic_beyond_999(tmp_path):
    tr = cb.generate_uniform_trace(1200, 3.0, 7)
    m = cb.materialize_trace(tr)
    cat = cb.builtin_catalog()
    ids = ["t%03d-%s" % (i, cat[e].key) for i, e in enumerate(tr.entry)]
    want = np.empty(len(ids), np.uint32)
    want[np.argsort(ids, kind="stable")] = np.arange(len(ids))
    assert np.array_equal(m.tasks["rank"], want)


def test_trace_file_round_trip(tmp_path):
    tr = cb.generate_trace("t60", 3)
    p = str(tmp_path / "t.trace")
    cb.save_trace(tr, p)
    back = cb.load_trace(p)
    assert np.array_equal(back.submit, tr.submit)
    assert np.array_equal(back.entry, tr.entry) and np.array_equal(back.epochs, tr.epochs)
    assert open(p).readline().startswith("#carma-trace v1 seed=3 mix=t60")
    bad = tmp_path / "bad.trace"
    bad.write_text("#carma-trace v1\n5.0,resnet18_cifar100_bs32,20\n1.0,resnet18_cifar100_bs32,20\n")
    with pytest.raises(abi.CarmaError):
        cb.load_trace(str(bad))


def unpack(packed, table):
    w = packed["w"].astype(np.uint64)
    m48 = np.uint64((1 << 48) - 1)
    s = np.zeros((len(w), 19))
    s[:, 0] = (w[:, 0] >> np.uint64(48)) & np.uint64(0xff)
    s[:, 1] = w[:, 0] >> np.uint64(56)
    s[:, 2] = (w[:, 1] >> np.uint64(48)) & np.uint64(0xff)
    s[:, 3] = w[:, 1] >> np.uint64(56)
    batch = (w[:, 2] >> np.uint64(48)) | ((w[:, 5] >> np.uint64(48)) << np.uint64(16))
    s[:, 4] = batch
    s[:, 5] = w[:, 0] & m48
    s[:, 6] = w[:, 1] & m48
    code = (w[:, 3] >> np.uint64(61)).astype(np.int64)
    s[:, 7] = table[2 * code]
    s[:, 8] = table[2 * code + 1]
    for k in range(3):
        s[:, 9 + 3 * k] = (w[:, 3] >> np.uint64(48 + 4 * k)) & np.uint64(0xf)
        s[:, 10 + 3 * k] = w[:, 2 + 2 * k] & m48
        s[:, 11 + 3 * k] = w[:, 3 + 2 * k] & m48
    s[:, 18] = 16.0 * s[:, 5] + (4.0 * s[:, 4]) * s[:, 6]
    fam = ((w[:, 4] >> np.uint64(48)) & np.uint64(0xff)).astype(np.int8)
    return s, fam


@pytest.mark.parametrize("family", [0, 1, 2])
def test_packed_format_is_lossless(family):
    ds = cb.generate_synthetic_dataset(family, 3000, 9)
    packed, table = cb.pack_features(ds.rows, default_family=family)
    s, fam = unpack(packed, table)
    want = cb.scalar_features(ds.rows)
    assert np.array_equal(s.view(np.uint64), want.view(np.uint64))
    assert np.all(fam == family)


def test_packed_format_rejects_out_of_range_rows():
    ds = cb.generate_synthetic_dataset(0, 4, 9)
    rows = ds.rows.copy()
    rows["total_params"][2] = 1 << 50
    with pytest.raises(abi.CarmaError) as e:
        cb.pack_features(rows, default_family=0)
    assert e.value.status == 5


def test_fit_shapes_and_holdout_split():
    m = cb.fit_knn(0, 4000, 11, 5)
    assert len(m.labels) == 2800 and len(m.holdout_rows) == 1200
    assert m.points.shape == (2800, 19)
    lo, hi = m.lo, m.hi
    active = hi > lo
    assert np.all(m.points[:, active] >= 0.0) and np.all(m.points[:, active] <= 1.0)
    assert np.all(m.points[:, ~active] == 0.0)
    assert m.bucket_range == 1 << 30


def unpack_bits(words, schema, n):
    s = schema[0]
    wpr = int(s["words_per_row"])
    base_idx = np.arange(n, dtype=np.int64) * wpr
    w = words.astype(np.uint64)
    out = np.zeros((n, 19), np.uint64)
    for f in range(19):
        width, off, base = int(s["width"][f]), int(s["offset"][f]), np.uint64(s["base"][f])
        if width == 0:
            out[:, f] = base
            continue
        i = base_idx + (off >> 5)
        sh = off & 31
        v = (w[i] | (w[i + 1] << np.uint64(32))) >> np.uint64(sh)
        if sh + width > 64:
            v |= w[i + 2] << np.uint64(64 - sh)
        out[:, f] = base + (v & np.uint64((1 << width) - 1))
    return out


@pytest.mark.parametrize("families", [(0,), (1, 2), (0, 1, 2)])
def test_bitpacked_format_is_lossless(families):
    rows, fams = [], []
    for f in families:
        ds = cb.generate_synthetic_dataset(f, 2000, 21 + f)
        rows.append(ds.rows)
        fams.append(np.full(2000, f, np.int8))
    rows, fams = np.concatenate(rows), np.concatenate(fams)
    words, schema = cb.pack_features_bits(rows, fams)
    n = len(rows)
    assert len(words) == n * int(schema["words_per_row"][0]) + 2
    v = unpack_bits(words, schema, n)
    assert np.array_equal(v[:, 0], rows["n_linear"]) and np.array_equal(v[:, 3], rows["n_conv"])
    assert np.array_equal(v[:, 4], rows["batch_size"]) and np.array_equal(v[:, 5], rows["total_params"])
    assert np.array_equal(v[:, 6], rows["total_activations"])
    table = schema["act_table"][0]
    assert np.array_equal(table[2 * v[:, 7].astype(np.int64)], rows["act_cos"])
    assert np.array_equal(table[2 * v[:, 7].astype(np.int64) + 1], rows["act_sin"])
    for k in range(3):
        assert np.array_equal(v[:, 8 + k].astype(np.int32), rows["kind"][:, k])
        assert np.array_equal(v[:, 12 + 2 * k], rows["tuple_acts"][:, k])
        assert np.array_equal(v[:, 13 + 2 * k], rows["tuple_params"][:, k])
    assert np.array_equal(v[:, 18].astype(np.int8), fams)
    assert int(schema["words_per_row"][0]) * 4 < 64  # denser than the fixed 64-byte packing


def test_compact_format_is_lossless_and_rejects_wide_rows():
    """The fixed-schema 40-byte rows the host-buffer predicts ship (stage.cpp)."""
    rows, fams = [], []
    for f in (0, 1, 2):
        ds = cb.generate_synthetic_dataset(f, 2000, 31 + f)
        rows.append(ds.rows)
        fams.append(np.full(2000, f, np.int8))
    rows, fams = np.concatenate(rows), np.concatenate(fams)
    fams[::7] = -1
    fams[3::11] = 9
    words, schema = cb.pack_features_compact(rows, fams)
    n = len(rows)
    assert int(schema["words_per_row"][0]) == 10 and len(words) == 10 * n + 2
    v = unpack_bits(words, schema, n)
    for f, name in enumerate(("n_linear", "n_batchnorm", "n_dropout", "n_conv", "batch_size", "total_params",
                              "total_activations")):
        assert np.array_equal(v[:, f], rows[name])
    table = schema["act_table"][0]
    assert np.array_equal(table[2 * v[:, 7].astype(np.int64)], rows["act_cos"])
    assert np.array_equal(table[2 * v[:, 7].astype(np.int64) + 1], rows["act_sin"])
    for k in range(3):
        assert np.array_equal(v[:, 8 + k].astype(np.int32), rows["kind"][:, k])
        assert np.array_equal(v[:, 12 + 2 * k], rows["tuple_acts"][:, k])
        assert np.array_equal(v[:, 13 + 2 * k], rows["tuple_params"][:, k])
    assert np.array_equal(v[:, 11], (rows["has_layers"] != 0).astype(np.uint64))
    want_f = np.where((fams >= 0) & (fams < 15), fams, 15).astype(np.uint64)
    assert np.array_equal(v[:, 18], want_f)
    for field, value in (("total_params", 2**32), ("batch_size", 4096), ("tuple_acts", 2**32)):
        bad = rows[:3].copy()
        bad[field][1] = value
        with pytest.raises(abi.CarmaError) as e:
            cb.pack_features_compact(bad, default_family=0)
        assert e.value.status == 5


def test_mig_layout_matches_gpudevice():
    c = cb.make_config(cb.PolicyConfig(collocation_mode="mig"), cb.SimConstants(), None)
    assert c["mig_count"][0] == 2 and list(c["mig_blocks"][0, :2]) == [40, 40]
    c = cb.make_config(cb.PolicyConfig(collocation_mode="mig"), cb.SimConstants(), (0.3, 0.3, 0.4))
    # round_up(trunc(0.3 * 40 GiB)) = 12 GiB = 24 blocks of 512 MiB; the last instance absorbs the rest
    assert list(c["mig_base"][0, :3]) == [0, 24, 48] and list(c["mig_blocks"][0, :3]) == [24, 24, 32]
    c = cb.make_config(cb.PolicyConfig(collocation_mode="mig"), cb.SimConstants(), (0.5, 0.2))
    # sum < 1: nothing absorbs the tail (gpu.cpp:44-46)
    assert list(c["mig_blocks"][0, :2]) == [40, 16] and c["mig_count"][0] == 2
    for bad in ((0.6, 0.6), (0.0, 0.5), (1.5,)):
        with pytest.raises(abi.CarmaError):
            cb.make_config(cb.PolicyConfig(collocation_mode="mig"), cb.SimConstants(), bad)
    with pytest.raises(abi.CarmaError):
        cb.make_config(cb.PolicyConfig(collocation_mode="mig"), cb.SimConstants(), (0.1,) * 9)


def test_reference_bridge_loads_and_fails_loudly_without_gpu():
    """integration/_build/libcarma_bridge.so (built where /root/reference
    exists) links the reference library and libcarma_b200.so; on a box with
    no GPU its GPU side raises the C ABI's error through the reference's
    exception types while the reference side still runs."""
    from bridge_bind import case, load_bridge, run_pair
    lib = load_bridge()
    if lib is None:
        pytest.skip("bridge not built (needs /root/reference)")
    for sym in ("bridge_run_pair", "bridge_sweep_pair", "bridge_estimate_pair", "bridge_manager_estimates"):
        assert hasattr(lib, sym)
    if abi.lib.carma_device_count() > 0:
        pytest.skip("a GPU is present")
    ref, got = run_pair(lib, case(policy="magm", estimator="oracle"))
    assert ref.startswith("OK:{") and '"trace_name": "t90-seed1"' in ref or ref.startswith("OK:")
    assert got.startswith("ERR:") and "no CPU fallback" in got


def test_device_log1p_is_glibc_bit_for_bit():
    """The trace generator's log1p (glibc_log1p.cuh, the code the device runs)
    equals the C library's on 6M inputs: the generator's domain (-u, u in
    [0, 1)), tiny arguments, both sides of every branch boundary."""
    import ctypes
    bad = ctypes.c_uint64()
    abi.check(abi.lib.carma_host_check_log1p(6_000_000, 12345, ctypes.byref(bad)))
    assert bad.value == 0


@pytest.mark.parametrize("b", [0, 1, 2])
def test_mt_jump_ahead_tables(b):
    """The device dataset generator's jump-ahead (csrc/cuda/dataset.cu): the
    characteristic polynomial of mt19937_64 (Berlekamp-Massey) and
    x^(156 * 2^(13+b)) mod P applied by Horner's rule give exactly the window
    that stepping the recurrence reaches."""
    import ctypes
    for seed in (1, 2**63 + 5):
        m = ctypes.c_uint64()
        abi.check(abi.lib.carma_host_check_mt_jump(seed, b, ctypes.byref(m)))
        assert m.value == 0
