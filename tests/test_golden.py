"""The oracle restatement against the reference's own outputs (committed
golden fixtures, tests/golden/make_golden.py) — runs anywhere, no reference
sources needed."""
import os

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from cases import assert_matches_ref, case_inputs, model
from oracle_bind import oracle_predict, oracle_replay

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def knn_golden():
    return np.load(os.path.join(GOLDEN, "knn.npz"))


@pytest.fixture(scope="module")
def replay_golden():
    return np.load(os.path.join(GOLDEN, "replay.npz"))


@pytest.mark.parametrize("family", [0, 1, 2])
def test_oracle_knn_matches_reference_golden(olib, knn_golden, family):
    fam, mseed, qseed, n = knn_golden["cases"][family]
    ds = cb.generate_synthetic_dataset(int(fam), int(n), int(qseed))
    b, by, _, _ = oracle_predict(olib, model(int(fam), 4000, int(mseed)), cb.scalar_features(ds.rows))
    assert np.array_equal(b, knn_golden[f"bucket_{family}"])
    assert np.array_equal(by, knn_golden[f"bytes_{family}"])


def test_oracle_replay_matches_reference_golden(olib, replay_golden):
    cases = replay_golden["cases"]
    for i, case in enumerate(cases):
        cfg, tasks = case_inputs(olib, str(case))
        rc, ot, otr, og = oracle_replay(olib, cfg, tasks)
        assert rc == 0, case
        assert_matches_ref(replay_golden, i, ot, otr, og)
