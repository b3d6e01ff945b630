"""run_sweep (runner.cpp:192-283) on the GPU against the reference's own
run_sweep: the whole sweep CSV (per-seed report rows + median rows, printf
formatting included) must be identical."""
import ctypes

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from oracle_bind import ref_config

pytestmark = pytest.mark.gpu

CELLS = [dict(policy="exclusive"), dict(policy="rr"), dict(policy="magm", estimator="learned"),
         dict(policy="lug", estimator="oracle"), dict(policy="magm", min_free=3 << 30, window=30.0),
         dict(policy="mug", mode="streams", max_smact=1.0)]


def policy_of(kw):
    return cb.PolicyConfig(policy=kw["policy"], estimator=kw.get("estimator", "none"),
                           collocation_mode=kw.get("mode", "mps"), max_smact=kw.get("max_smact", 0.8),
                           min_free_mem=kw.get("min_free"), monitor_window=kw.get("window", 60.0))


@pytest.mark.parametrize("mix,seeds", [("t90", [1, 2, 3, 4]), ("t60", [5, 6, 7])])
def test_run_sweep_csv_matches_reference(gpu, ref, mix, seeds):
    cfg = cb.SweepConfig(base=cb.RunConfig(mix=mix), cells=[cb.SweepCell(policy_of(kw)) for kw in CELLS],
                         seeds=seeds)
    res = cb.run_sweep(cfg, device=gpu)
    rows = np.concatenate([ref_config(**kw) for kw in CELLS])
    s = np.ascontiguousarray(seeds, np.uint64)
    buf = ctypes.create_string_buffer(1 << 16)
    assert ref.ref_run_sweep(rows.ctypes.data, len(CELLS), cb.abi.MIX[mix], s.ctypes.data, len(seeds), buf,
                             len(buf)) == 0
    assert res.csv == buf.value.decode()
    assert len(res.reports) == len(CELLS) and all(len(r) == len(seeds) for r in res.reports)


def test_run_sweep_rejects_empty(gpu):
    with pytest.raises(cb.abi.CarmaError):
        cb.run_sweep(cb.SweepConfig(base=cb.RunConfig(), cells=[]))
