"""Pins the oracle restatement and the product's host provisioning to the
compiled reference (oracle/_ref) on fresh seeds. Skips where the reference
library is not built."""
import ctypes

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi
from cases import model
from oracle_bind import GiB, MiB, oracle_predict, oracle_replay, ref_config, ref_run, replay_config_from


@pytest.mark.parametrize("family,seed", [(0, 11), (1, 112), (2, 213), (1, 7)])
def test_fit_matches_reference_train(ref, family, seed):
    lo, hi = np.zeros(19), np.zeros(19)
    pts, lab = np.zeros((4000, 19)), np.zeros(4000, np.int32)
    n, br, h = ctypes.c_uint64(), ctypes.c_uint64(), np.zeros(3)
    assert ref.ref_train(family, 4000, seed, 5, b"/tmp/carma_ref_model.json", lo.ctypes.data, hi.ctypes.data,
                         pts.ctypes.data, lab.ctypes.data, 4000, ctypes.byref(n), ctypes.byref(br),
                         h.ctypes.data) == 0
    m = cb.fit_knn(family, 4000, seed, 5)
    assert np.array_equal(m.lo, lo) and np.array_equal(m.hi, hi)
    assert np.array_equal(m.points, pts[: n.value]) and np.array_equal(m.labels, lab[: n.value])
    assert m.bucket_range == br.value


@pytest.mark.parametrize("family,seed", [(0, 3), (1, 5), (2, 8)])
def test_dataset_and_predict_match_reference(ref, olib, family, seed):
    n = 1500
    f, b, mm = np.zeros((n, 19)), np.zeros(n, np.int32), np.zeros(n, np.uint64)
    assert ref.ref_dataset(family, n, seed, f.ctypes.data, b.ctypes.data, mm.ctypes.data) == 0
    ds = cb.generate_synthetic_dataset(family, n, seed)
    raw = cb.scalar_features(ds.rows)
    assert np.array_equal(raw.view(np.uint64), f.view(np.uint64))
    assert np.array_equal(ds.bucket, b) and np.array_equal(ds.mem, mm)
    pb, pby = np.zeros(n, np.int32), np.zeros(n, np.uint64)
    mseed = 11 + 101 * family
    assert ref.ref_predict_dataset(family, 4000, mseed, 5, n, seed, pb.ctypes.data, pby.ctypes.data) == 0
    ob, oby, _, _ = oracle_predict(olib, model(family, 4000, mseed), raw)
    assert np.array_equal(ob, pb) and np.array_equal(oby, pby)


def test_traces_and_materialize_match_reference(ref, tmp_path):
    for mix in (0, 1):
        for seed in (1, 17, 99):
            sub, ent, ep = np.zeros(128), np.zeros(128, np.int32), np.zeros(128, np.uint64)
            n = ctypes.c_uint64()
            assert ref.ref_gen_trace(mix, seed, sub.ctypes.data, ent.ctypes.data, ep.ctypes.data, 128,
                                     ctypes.byref(n)) == 0
            tr = cb.generate_trace("t90" if mix == 0 else "t60", seed)
            k = n.value
            assert np.array_equal(tr.submit, sub[:k]) and np.array_equal(tr.entry, ent[:k])
            assert np.array_equal(tr.epochs, ep[:k])
    tr = cb.generate_uniform_trace(1500, 3.0, 7)
    path = str(tmp_path / "u.trace")
    cb.save_trace(tr, path)
    cap = 2000
    arrs = dict(submit=np.zeros(cap), true_mem=np.zeros(cap, np.uint64), work=np.zeros(cap),
                demand=np.zeros(cap), gpus=np.zeros(cap, np.uint64), family=np.zeros(cap, np.int32),
                batch=np.zeros(cap, np.uint64), feats=np.zeros((cap, 19)))
    n = ctypes.c_uint64()
    assert ref.ref_materialize(path.encode(), cap, *[a.ctypes.data for a in arrs.values()], None, 0,
                               ctypes.byref(n)) == 0
    m = cb.materialize_trace(tr)
    k = n.value
    assert k == 1500
    for f in ("submit", "true_mem", "work", "demand", "gpus"):
        assert np.array_equal(m.tasks[f], arrs[f][:k].astype(m.tasks[f].dtype)), f
    assert np.array_equal(m.family, arrs["family"][:k].astype(np.int8))
    assert np.array_equal(cb.scalar_features(m.features).view(np.uint64), arrs["feats"][:k].view(np.uint64))


GRID = [dict(policy=p) for p in ("exclusive", "rr", "magm", "lug", "mug")] + [
    dict(policy="rr", rr_pre=True, estimator="oracle"),
    dict(policy="magm", estimator="analytical"),
    dict(policy="magm", estimator="static_graph"),
    dict(policy="magm", mode="streams", max_smact=1.0),
    dict(policy="lug", gpu_count=8, window=5.0),
    dict(policy="magm", gpu_count=2, window=5.0, min_free=3 << 30),
    # MIG: instance 0 must hold the largest catalog task (27.9 GiB) or the
    # reference never terminates (exclusive recovery retries instance 0).
    dict(policy="magm", mode="mig", mig=(0.75, 0.25)),
    dict(policy="rr", mode="mig", mig=(0.7, 0.15, 0.15)),
    dict(policy="exclusive", mode="mig", mig=(0.75, 0.125)),
    dict(policy="lug", mode="mig", mig=(0.8, 0.2), estimator="oracle"),
    dict(policy="mug", mode="mig", mig=(1.0,), gpu_count=8),
    dict(policy="magm", mode="mig", mig=(0.75, 0.125, 0.125), estimator="analytical"),
    dict(policy="rr", mode="mig", mig=(0.8, 0.2), rr_pre=True, estimator="oracle", gpu_count=2),
    # more than 256 allocation blocks per GPU (the wide global tier)
    dict(policy="magm", capacity=192 * GiB, block=512 * MiB, gpu_count=8),
    dict(policy="rr", capacity=40 * GiB, block=16 * MiB),
    dict(policy="lug", capacity=192 * GiB, block=64 * MiB, mode="mig", mig=(0.75, 0.25), estimator="oracle"),
]


@pytest.mark.parametrize("kw", GRID, ids=[str(i) for i in range(len(GRID))])
def test_oracle_replay_matches_reference(ref, olib, kw):
    for mix in ("t90", "t60"):
        for seed in (11, 12):
            cfg = ref_config(**kw)
            tout, rout, ge, gs, gp = ref_run(ref, cfg, mix=mix, seed=seed)
            m = cb.materialize_trace(cb.generate_trace(mix, seed))
            cb.set_persona_estimates(m, kw.get("estimator", "none"))
            rc, ot, otr, og = oracle_replay(olib, replay_config_from(cfg), m.tasks)
            assert rc == 0
            for a, b in (("final_dispatch", "final_dispatch"), ("complete", "complete"), ("ooms", "ooms"),
                         ("executed", "executed"), ("first_attempt", "first_attempt"),
                         ("last_crash", "last_crash"), ("attempts", "n_attempts")):
                assert np.array_equal(ot[a], tout[b]), (kw, mix, seed, a)
            assert np.array_equal(ot["gpu"][:, 0], tout["gpu0"]) and np.array_equal(ot["gpu"][:, 1], tout["gpu1"])
            for f in ("avg_wait", "avg_exec", "avg_jct", "energy_mj", "trace_total_time"):
                assert otr[f] == rout[f], (kw, mix, seed, f)
            assert np.array_equal(og["energy_j"], ge) and np.array_equal(og["mean_smact"], gs)
            assert np.array_equal(og["peak_used"], gp)


def test_oracle_large_trace_matches_reference(ref, olib, tmp_path):
    """2000 uniform-catalog tasks on 64 GPUs, W = 5 s, learned estimates, loaded
    from a #carma-trace v1 file (ids past t999: lexicographic order matters)."""
    tr = cb.generate_uniform_trace(2000, 3.0, 7)
    path = str(tmp_path / "big.trace")
    cb.save_trace(tr, path)
    cfg = ref_config(policy="magm", estimator="learned", gpu_count=64, window=5.0)
    tout, rout, ge, gs, gp = ref_run(ref, cfg, path=path)
    m = cb.materialize_trace(cb.load_trace(path))
    raw = cb.scalar_features(m.features)
    e = np.zeros(len(m.tasks), np.uint64)
    for f in set(m.family.tolist()):
        sel = m.family == f
        e[sel] = oracle_predict(olib, model(f), raw[sel])[1]
    m.tasks["estimate"] = e
    rc, ot, otr, og = oracle_replay(olib, replay_config_from(cfg), m.tasks)
    assert rc == 0
    assert np.array_equal(ot["complete"], tout["complete"]) and np.array_equal(ot["ooms"], tout["ooms"])
    assert np.array_equal(ot["gpu"][:, 0], tout["gpu0"])
    assert otr["energy_mj"] == rout["energy_mj"] and otr["avg_jct"] == rout["avg_jct"]
    assert np.array_equal(og["mean_smact"], gs)


def test_ref_batch_entries_match_single_calls(ref, olib):
    """The full-size parity tests' reference entries (ref_estimate_rows over
    feature rows, ref_run_jobs over a threaded job pool) agree with the
    reference's per-dataset predict and single run_simulation, and the oracle."""
    from oracle_bind import ref_estimate_rows, ref_run_jobs
    rows = np.concatenate([cb.generate_synthetic_dataset(f, 1200, 40 + f).rows for f in (0, 1, 2)])
    fam = np.repeat(np.array([0, 1, 2], np.int8), 1200)
    b, by = ref_estimate_rows(ref, rows, fam, threads=3)
    for f in (0, 1, 2):
        sel = fam == f
        ob, oby, _, _ = oracle_predict(olib, cb.fit_knn(f, 4000, 11 + 101 * f, 5), cb.scalar_features(rows[sel]))
        assert np.array_equal(b[sel], ob) and np.array_equal(by[sel], oby)
    cfgs = np.concatenate([ref_config(policy=p, max_smact=0.8) for p in ("exclusive", "rr", "magm", "lug")])
    tout, rout, ge, gs, gp = ref_run_jobs(ref, cfgs, "t90", 3, 6, 90, threads=3)
    for c, p in enumerate(("exclusive", "rr", "magm", "lug")):
        for s in (0, 5):
            j = c * 6 + s
            one = ref_run(ref, ref_config(policy=p, max_smact=0.8), mix="t90", seed=3 + s)
            assert tout[j * 90:(j + 1) * 90].tobytes() == one[0].tobytes()
            assert rout[j].tobytes() == one[1].tobytes()
            assert ge[j * 4:(j + 1) * 4].tobytes() == one[2].tobytes()
            assert np.array_equal(gp[j * 4:(j + 1) * 4], one[4])


@pytest.mark.parametrize("family,seed", [(0, 11), (1, 112), (2, 213)])
def test_snapshot_written_by_reference_parses_to_its_state(ref, tmp_path, family, seed):
    """carma_host_parse_snapshot reads LearnedEstimator::save's JSON
    (estimators.cpp:481-501) back to the reference's fitted state bit for bit
    (and to the host fit the GPU bank installs)."""
    path = str(tmp_path / f"est{family}.json")
    lo, hi = np.zeros(19), np.zeros(19)
    pts, lab = np.zeros((4000, 19)), np.zeros(4000, np.int32)
    n, br, h = ctypes.c_uint64(), ctypes.c_uint64(), np.zeros(3)
    assert ref.ref_train(family, 4000, seed, 5, path.encode(), lo.ctypes.data, hi.ctypes.data, pts.ctypes.data,
                         lab.ctypes.data, 4000, ctypes.byref(n), ctypes.byref(br), h.ctypes.data) == 0
    m = cb.parse_snapshot(open(path, "rb").read())
    assert m.family == family and m.k == 5 and m.bucket_range == br.value and m.seed == seed
    assert m.lo.tobytes() == lo.tobytes() and m.hi.tobytes() == hi.tobytes()
    assert m.points.tobytes() == pts[: n.value].tobytes() and np.array_equal(m.labels, lab[: n.value])
    assert np.float64(m.holdout["accuracy"]).tobytes() == np.float64(h[0]).tobytes()
    assert np.float64(m.holdout["macro_f1"]).tobytes() == np.float64(h[1]).tobytes()
    assert np.float64(m.holdout["underestimate_rate"]).tobytes() == np.float64(h[2]).tobytes()
    f = cb.fit_knn(family, 4000, seed, 5)
    assert f.points.tobytes() == m.points.tobytes()


def test_snapshot_errors_follow_the_reference():
    from paper_2508_19073_b200 import abi
    with pytest.raises(abi.CarmaError, match="unrecognized estimator snapshot schema"):
        cb.parse_snapshot(b'{"schema": "other"}')
    bad = (b'{"schema": "carma-knn-estimator/v1", "family": "cnn", "bucket_range": 8, "k": 5, "seed": 1, '
           b'"lo": [' + b",".join([b"0.0"] * 19) + b'], "hi": [' + b",".join([b"1.0"] * 19) + b'], '
           b'"labels": [1, 2], "points": [[' + b",".join([b"0.5"] * 19) + b']], "holdout": {}}')
    with pytest.raises(abi.CarmaError, match="labels/points mismatch"):
        cb.parse_snapshot(bad)
    with pytest.raises(abi.CarmaError, match="unsupported model family"):
        cb.parse_snapshot(bad.replace(b'"cnn"', b'"rnn"'))
    with pytest.raises(abi.CarmaError, match="malformed"):
        cb.parse_snapshot(b'{"schema": "carma-knn-estimator/v1", ')


@pytest.mark.parametrize("gpus,policy", [(128, "magm"), (256, "lug"), (100, "rr")])
def test_oracle_many_gpus_matches_reference(ref, olib, tmp_path, gpus, policy):
    """Pins the oracle beyond 64 simulated GPUs (the GPU's many-GPU tier is
    checked against it in tests/test_gpu_replay.py)."""
    tr = cb.generate_uniform_trace(1500, 0.3, 9)
    path = str(tmp_path / "many.trace")
    cb.save_trace(tr, path)
    cfg = ref_config(policy=policy, estimator="oracle", gpu_count=gpus, window=5.0)
    tout, rout, ge, gs, gp = ref_run(ref, cfg, path=path)
    m = cb.materialize_trace(cb.load_trace(path))
    cb.set_persona_estimates(m, "oracle")
    rc, ot, otr, og = oracle_replay(olib, replay_config_from(cfg), m.tasks)
    assert rc == 0
    assert np.array_equal(ot["complete"], tout["complete"]) and np.array_equal(ot["ooms"], tout["ooms"])
    assert np.array_equal(ot["gpu"][:, 0], tout["gpu0"])
    assert otr["energy_mj"] == rout["energy_mj"] and otr["avg_jct"] == rout["avg_jct"]
    assert np.array_equal(og["mean_smact"], gs)


@pytest.mark.parametrize("capacity,block", [(40 * GiB, 0), (40 * GiB + 100 * MiB, 512 * MiB)])
def test_oracle_byte_granular_allocator_matches_reference(ref, olib, capacity, block):
    """The oracle's segment allocator against the reference's GpuDevice with
    alloc_block = 0 and a capacity that is not a block multiple (RR without
    preconditions stacks tasks, so OOM crashes and free/largest reports occur)."""
    for policy, pre in (("rr", False), ("magm", False)):
        cfg = ref_config(policy=policy, rr_pre=pre, gpu_count=4, capacity=capacity, block=block, max_smact=1.0)
        for seed in (1, 2, 3):
            tout, rout, ge, gs, gp = ref_run(ref, cfg, mix="t90", seed=seed)
            m = cb.materialize_trace(cb.generate_trace("t90", seed))
            rc, ot, otr, og = oracle_replay(olib, replay_config_from(cfg), m.tasks)
            assert rc == 0
            assert np.array_equal(ot["complete"], tout["complete"]) and np.array_equal(ot["ooms"], tout["ooms"])
            assert otr["energy_mj"] == rout["energy_mj"] and otr["avg_jct"] == rout["avg_jct"]
            assert np.array_equal(og["peak_used"], gp)


@pytest.mark.parametrize("block,capacity", [(0, 40 * GiB), (512 * MiB, 40 * GiB + 100 * MiB)])
def test_oracle_mig_byte_instances_match_reference(ref, olib, block, capacity):
    """MIG on a byte-granular device (instance tables in bytes, carma_mig_layout)."""
    for mig in ((0.7, 0.3), (0.75, 0.125, 0.125)):  # the largest instance holds every catalog task
        cfg = ref_config(policy="magm", mode="mig", mig=mig, capacity=capacity, block=block)
        for seed in (1, 2):
            tout, rout, ge, gs, gp = ref_run(ref, cfg, mix="t90", seed=seed)
            m = cb.materialize_trace(cb.generate_trace("t90", seed))
            rc, ot, otr, og = oracle_replay(olib, replay_config_from(cfg), m.tasks)
            assert rc == 0
            assert np.array_equal(ot["complete"], tout["complete"]) and np.array_equal(ot["ooms"], tout["ooms"])
            assert otr["energy_mj"] == rout["energy_mj"] and np.array_equal(og["peak_used"], gp)
