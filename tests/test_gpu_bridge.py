"""The reference-side bridge (integration/carma_bridge.cpp), compiled against
the reference's headers and linked with the UNMODIFIED reference library:
gpu_run_simulation / gpu_run_sweep / GpuEstimatorBank must give the
reference's own run_simulation / run_sweep / make_estimate results byte for
byte (emit_report JSON of every report, the sweep CSV, every estimate), and
fail with the same messages where the reference fails."""
import ctypes

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from bridge_bind import GiB, MiB, case, load_bridge, run_pair, sweep_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bridge(gpu):
    lib = load_bridge()
    if lib is None:
        pytest.fail("integration/_build/libcarma_bridge.so not built (__graft_entry__.build())")
    return lib


RUNS = [
    dict(policy=p, estimator=e) for p in ("exclusive", "rr", "magm", "lug", "mug")
    for e in ("none", "oracle", "analytical", "static_graph", "learned")
] + [
    dict(mix="t60", policy="magm", estimator="learned", seed=4),
    dict(policy="magm", mode="streams", seed=2),
    dict(policy="rr", rr_pre=True, min_free=4 * GiB, seed=3),
    dict(policy="lug", max_smact=0.5, window=30.0, gpu_count=8, seed=5),
    dict(policy="magm", mode="mig", mig=(0.75, 0.125, 0.125), seed=6),
    dict(policy="mug", mode="mig", mig=(0.8, 0.2), seed=7, estimator="oracle"),
    dict(policy="magm", capacity=80 * GiB, block=256 * MiB, gpu_count=2, seed=8, estimator="learned"),
    dict(policy="lug", capacity=192 * GiB, gpu_count=8, seed=9, estimator="oracle"),
    # byte-granular segment allocator (generic replay instantiations)
    dict(policy="rr", block=0, seed=10),
    dict(policy="magm", capacity=40 * GiB + 100 * MiB, seed=11, estimator="learned"),
    dict(policy="magm", gpu_count=100, seed=12, estimator="oracle"),
    dict(policy="magm", mode="mig", mig=(0.75, 0.25), block=0, seed=13),
]


@pytest.mark.parametrize("kw", RUNS, ids=lambda kw: "-".join(f"{k}={v}" for k, v in kw.items()))
def test_gpu_run_simulation_report_equals_reference(bridge, kw):
    ref, got = run_pair(bridge, case(**kw))
    assert ref.startswith("OK:"), ref[:300]
    assert got == ref


def test_gpu_run_simulation_failure_equals_reference(bridge):
    # one 40 GiB GPU cannot host the heavy two-GPU tasks: IncompleteRun on both sides
    ref, got = run_pair(bridge, case(policy="magm", gpu_count=1))
    assert ref.startswith("ERR:") and got == ref


def test_gpu_run_sweep_csv_and_reports_equal_reference(bridge):
    cells = [case(policy=p) for p in ("exclusive", "rr", "magm", "lug")]
    cells.append(case(policy="magm", estimator="learned"))
    ref, got = sweep_pair(bridge, cells, list(range(1, 26)))
    assert ref.startswith("OK:policy,estimator"), ref[:300]
    assert got == ref


def test_gpu_run_sweep_t60_mig_equals_reference(bridge):
    cells = [case(mix="t60", policy=p, mode="mig", mig=(0.75, 0.25)) for p in ("magm", "mug")]
    ref, got = sweep_pair(bridge, cells, [3, 9, 27])
    assert ref.startswith("OK:") and got == ref


@pytest.mark.parametrize("k", [5, 31])
@pytest.mark.parametrize("how", [0, 1, 2], ids=["add", "train", "load"])
@pytest.mark.parametrize("family", [0, 1, 2])
def test_estimator_bank_equals_estimate_learned(bridge, family, how, k):
    import ctypes
    n = 3000
    rb, gb = np.zeros(n, np.int32), np.full(n, -9, np.int32)
    rby, gby = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    err = ctypes.create_string_buffer(512)
    rc = bridge.bridge_estimate_pair(family, n, 777 + family, 4000, 11 + 101 * family, k, how, 0, rb.ctypes.data,
                                     rby.ctypes.data, gb.ctypes.data, gby.ctypes.data, err, 512)
    assert rc == 0, err.value.decode()
    assert np.array_equal(rb, gb) and np.array_equal(rby, gby)


@pytest.mark.parametrize("mix,seed", [(0, 1), (0, 42), (1, 5)])
def test_estimator_bank_equals_manager_make_estimate(bridge, mix, seed):
    import ctypes
    cap = 128
    r, g = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64)
    n = ctypes.c_uint64()
    err = ctypes.create_string_buffer(512)
    assert bridge.bridge_manager_estimates(mix, seed, 0, r.ctypes.data, g.ctypes.data, cap, ctypes.byref(n), err,
                                           512) == 0, err.value.decode()
    assert n.value in (60, 90)
    assert np.array_equal(r[: n.value], g[: n.value])


@pytest.mark.parametrize("family", [0, 1, 2])
def test_snapshot_saved_here_loads_in_the_reference(bridge, gpu, tmp_path, family):
    """train_learned_estimator on the GPU, LearnedEstimator.save here, then the
    reference's own LearnedEstimator::load + estimate_learned: its buckets equal
    the GPU bank's for the same queries (the snapshot round-trips exactly)."""
    est = cb.train_learned_estimator(family, 4000, 11 + 101 * family, 5, device=gpu)
    path = str(tmp_path / "est.json")
    est.save(path)
    n, qseed = 3000, 4242
    rb = np.zeros(n, np.int32)
    err = ctypes.create_string_buffer(512)
    assert bridge.bridge_snapshot_predict(path.encode(), family, n, qseed, rb.ctypes.data, err, 512) == 0, err.value
    rows = cb.generate_synthetic_dataset(family, n, qseed).rows
    assert np.array_equal(est.predict(rows), rb)
    knn = cb.GpuKnn(gpu)  # and carma_knn_load_snapshot reads it back to the same predictions
    knn.load_snapshot(path)
    assert np.array_equal(knn.predict(rows, default_family=family)[0], rb)
    knn.close()
