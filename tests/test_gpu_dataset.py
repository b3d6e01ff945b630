"""Device-side generate_synthetic_dataset (csrc/cuda/dataset.cu) against the
host generator (itself pinned to the reference, test_oracle_vs_ref.py) and
against the compiled reference directly: every byte of every carma_feature_row,
every bucket label and ground-truth byte count must be identical
(estimators.cpp:221-264)."""
import os

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi

pytestmark = pytest.mark.gpu


def same(a, b):
    return a.rows.tobytes() == b.rows.tobytes() and np.array_equal(a.bucket, b.bucket) and \
        np.array_equal(a.mem, b.mem)


@pytest.mark.parametrize("family", [0, 1, 2])
@pytest.mark.parametrize("n,seed", [(1, 0), (7, 1), (1000, 12345), (100_003, 2**63 + 11)])
def test_device_dataset_equals_host(gpu, family, n, seed):
    assert same(cb.generate_synthetic_dataset(family, n, seed, device=gpu),
                cb.generate_synthetic_dataset(family, n, seed))


@pytest.mark.parametrize("family", [0, 1, 2])
def test_many_rounds_carry_row_boundaries(gpu, family, monkeypatch):
    """Rounds of 4096 words: rows straddling a round's end are carried over."""
    monkeypatch.setenv("CARMA_DATASET_ROUND_WORDS", "4096")
    st = np.zeros(1, abi.dataset_stats_dtype)
    n = 20_000
    rows = np.zeros(n, abi.feature_row_dtype)
    b, m = np.zeros(n, np.int32), np.zeros(n, np.uint64)
    abi.check(abi.lib.carma_dataset_generate(gpu, family, n, 77, rows.ctypes.data, b.ctypes.data, m.ctypes.data,
                                             st.ctypes.data))
    assert st[0]["rounds"] > 20
    h = cb.generate_synthetic_dataset(family, n, 77)
    assert rows.tobytes() == h.rows.tobytes() and np.array_equal(b, h.bucket) and np.array_equal(m, h.mem)


def test_device_dataset_matches_reference(gpu, ref):
    """Straight against the reference's generate_synthetic_dataset (oracle/_ref)."""
    for family, seed in ((0, 5), (1, 2024), (2, 2025)):
        n = 30_000
        f, b, mm = np.zeros((n, 19)), np.zeros(n, np.int32), np.zeros(n, np.uint64)
        assert ref.ref_dataset(family, n, seed, f.ctypes.data, b.ctypes.data, mm.ctypes.data) == 0
        ds = cb.generate_synthetic_dataset(family, n, seed, device=gpu)
        assert np.array_equal(cb.scalar_features(ds.rows).view(np.uint64), f.view(np.uint64))
        assert np.array_equal(ds.bucket, b) and np.array_equal(ds.mem, mm)


def test_c2_batch_full_size(gpu):
    """The bench's c2 inputs (8,388,608 CNN rows seed 2024 + 8,388,608
    Transformer rows seed 2025), generated into device memory, equal the host
    generator's."""
    import torch
    n = 8_388_608
    for family, seed in ((1, 2024), (2, 2025)):
        rows = torch.empty(n * abi.feature_row_dtype.itemsize, dtype=torch.uint8, device=f"cuda:{gpu}")
        b = torch.empty(n, dtype=torch.int32, device=f"cuda:{gpu}")
        m = torch.empty(n, dtype=torch.int64, device=f"cuda:{gpu}")
        st = cb.generate_synthetic_dataset_device(family, n, seed, rows, b, m, device=gpu)
        torch.cuda.synchronize()
        assert st["rows_accepted"] >= n
        h = cb.generate_synthetic_dataset(family, n, seed)
        assert rows.cpu().numpy().tobytes() == h.rows.tobytes()
        assert np.array_equal(b.cpu().numpy(), h.bucket)
        assert np.array_equal(m.cpu().numpy().view(np.uint64), h.mem)


def test_invalid_arguments(gpu):
    rows = np.zeros(1, abi.feature_row_dtype)
    assert abi.lib.carma_dataset_generate(gpu, 0, 0, 1, rows.ctypes.data, None, None, None) == abi.CARMA_ERR_INVALID
    assert abi.lib.carma_dataset_generate(gpu, 3, 1, 1, rows.ctypes.data, None, None, None) == abi.CARMA_ERR_INVALID
