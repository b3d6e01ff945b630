"""Parity at the benchmarked sizes (BASELINE configs[1], [3], [4]): every
output of the bench's GPU workloads against the UNMODIFIED reference
(oracle/_ref) on the same inputs.

* c2: all 16,777,216 estimates (bucket and bytes) of the k-NN ensemble batch
  against the reference's estimate_learned (estimators.cpp:540-551) on all
  host threads, through both the device-resident bit-packed path the bench
  times and the 136-B feature-row host API its e2e times.
* c4: all 400,000 replays of the policy sweep (t90 seeds 1..100,000 x
  {exclusive, rr, magm, lug}): every task's (first attempt, final dispatch,
  completion, crash times, executed work, attempts, OOMs, GPU ids), every
  report and every per-GPU result against the reference's run_simulation
  (runner.cpp:40-147) pool, bit for bit.
* c5: the 10^6-task fused estimator-in-the-loop trace on 64 GPUs against the
  committed golden of the reference's full run (tests/golden/c5_ref.json,
  written by tests/golden/make_c5_golden.py): report and per-GPU bits, a
  SHA-256 digest of every per-task field, and a sample of full records.
"""
import json
import os

import numpy as np
import pytest

import bench
import paper_2508_19073_b200 as cb
from fullsize import first_mismatch, gpu_tasks_canonical, ref_tasks_canonical, digest_fields, sample_records
from paper_2508_19073_b200 import abi

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_c2_full_batch_matches_reference(gpu, ref):
    import torch
    from oracle_bind import ref_estimate_rows
    rows, fam = bench.knn_inputs(cb)
    q = len(rows)
    assert q == 16_777_216
    knn = cb.GpuKnn(gpu)
    for f in (1, 2):
        knn.set_model(cb.fit_knn(f, 4000, bench.MODEL_SEEDS[f], 5))
    # the bench's device-resident path: bit-packed rows, explicit stream
    words, schema = cb.pack_features_bits(rows, fam)
    abi.check(abi.lib.carma_knn_set_bit_schema(knn.handle, schema.ctypes.data))
    s = torch.cuda.Stream()
    d_rows = torch.from_numpy(words.view(np.uint8)).to("cuda")
    d_b = torch.full((q,), -7, dtype=torch.int32, device="cuda")
    d_by = torch.zeros(q, dtype=torch.int64, device="cuda")
    abi.check(abi.lib.carma_knn_predict_device(knn.handle, d_rows.data_ptr(), abi.ROWS_BITPACKED, None, 1, q,
                                               d_b.data_ptr(), d_by.data_ptr(), None, None, abi.stream_arg(s)))
    s.synchronize()
    gb, gby = d_b.cpu().numpy(), d_by.cpu().numpy().view(np.uint64)
    del d_rows, d_b, d_by
    # the e2e path: 136-B feature rows from host memory
    hb, hby = knn.predict(rows, family=fam)
    knn.close()
    rb, rby = ref_estimate_rows(ref, rows, fam, samples=4000, est_seed=11, k=5)
    bad = np.nonzero(gb != rb)[0]
    assert len(bad) == 0, f"{len(bad)} buckets differ, first row {bad[0]}: gpu {gb[bad[0]]} ref {rb[bad[0]]}"
    assert np.array_equal(gby, rby)
    assert np.array_equal(hb, rb) and np.array_equal(hby, rby)


def test_c4_full_sweep_matches_reference(gpu, ref):
    from oracle_bind import ref_config, ref_run_jobs
    n_tr = bench.SWEEP_TRACES
    cfgs, tasks, offs, jobs = bench.sweep_inputs(cb, n_tr)
    plan = cb.ReplayPlan(cfgs, tasks, offs, jobs, device=gpu)
    plan.run()
    res = plan.results()
    plan.close()
    assert (res.traces["status"] == 0).all()
    gtask = gpu_tasks_canonical(res.tasks)
    rcfgs = np.concatenate([ref_config(policy=p, max_smact=0.8) for p in bench.SWEEP_POLICIES])
    chunk = 12_500
    for s0 in range(0, n_tr, chunk):
        tout, rout, ge, gs, gp = ref_run_jobs(ref, rcfgs, "t90", 1 + s0, chunk, 90)
        for c in range(len(bench.SWEEP_POLICIES)):
            j0 = c * n_tr + s0                      # GPU job = policy * n_tr + trace
            rsl = slice(c * chunk, (c + 1) * chunk)  # ref job = cfg * chunk + seed offset
            g = res.traces[j0: j0 + chunk]
            r = rout[rsl]
            for f in ("trace_total_time", "avg_wait", "avg_exec", "avg_jct", "energy_mj", "last_complete",
                      "first_submit"):
                assert g[f].tobytes() == r[f].tobytes(), (bench.SWEEP_POLICIES[c], s0, f)
            assert np.array_equal(g["oom_count"], r["oom_count"])
            gt = gtask[res.task_offsets[j0]: res.task_offsets[j0 + chunk]]
            rt = ref_tasks_canonical(tout[c * chunk * 90: (c + 1) * chunk * 90])
            mm = first_mismatch(gt, rt)
            assert mm is None, f"policy {bench.SWEEP_POLICIES[c]} seeds {1 + s0}..: task field {mm[0]} " \
                               f"row {mm[1]} (trace seed {1 + s0 + mm[1] // 90})"
            gg = res.gpus[res.gpu_offsets[j0]: res.gpu_offsets[j0 + chunk]]
            sl = slice(c * chunk * 4, (c + 1) * chunk * 4)
            assert gg["energy_j"].tobytes() == ge[sl].tobytes()
            assert gg["mean_smact"].tobytes() == gs[sl].tobytes()
            assert np.array_equal(gg["peak_used"], gp[sl])


@pytest.mark.parametrize("estimator", ["learned", "none"])
def test_c5_full_trace_matches_reference_golden(gpu, estimator):
    import hashlib
    import tempfile
    path = os.path.join(HERE, "golden", "c5_ref.json")
    if not os.path.exists(path):
        pytest.fail("tests/golden/c5_ref.json missing (python tests/golden/make_c5_golden.py)")
    gold = json.load(open(path))
    want = gold["runs"][estimator]
    n = gold["n_tasks"]
    tr = cb.generate_uniform_trace(n, 3.0, 7)
    tp = os.path.join(tempfile.mkdtemp(), "c5.trace")
    cb.save_trace(tr, tp)
    with open(tp, "rb") as f:
        assert hashlib.sha256(f.read()).hexdigest() == gold["trace_sha256"], "c5 input trace differs"
    m = cb.materialize_trace(tr)
    cfg = cb.make_config(cb.PolicyConfig(policy="magm", max_smact=0.8, monitor_window=5.0),
                         cb.SimConstants(gpu_count=64))
    if estimator == "learned":
        knn = cb.GpuKnn(gpu)
        for f in sorted(set(m.family.tolist())):
            knn.set_model(cb.fit_knn(f, 4000, 11 + 101 * f, 5))
        fused = cb.FusedReplay(m, cfg, knn, gpu)
        fused.run()
        res = fused.results()
        fused.close()
        knn.close()
    else:
        res = cb.replay(cfg, [m.tasks], device=gpu)
    t = res.traces[0]
    assert int(t["status"]) == 0
    assert int(t["oom_count"]) == want["oom_count"]
    for k, v in want["report"].items():
        assert np.float64(t[k]).view(np.uint64).item().to_bytes(8, "big").hex() == v, k
    g = res.job_gpus(0)
    assert [int(x).to_bytes(8, "big").hex() for x in g["energy_j"].view(np.uint64)] == want["gpu_energy_j"]
    assert [int(x).to_bytes(8, "big").hex() for x in g["mean_smact"].view(np.uint64)] == want["gpu_mean_smact"]
    assert [int(x) for x in g["peak_used"]] == want["gpu_peak_used"]
    rec = gpu_tasks_canonical(res.job_tasks(0))
    assert sample_records(rec, want["sample_stride"]) == want["sample"]
    assert digest_fields(rec) == want["task_digest"]
