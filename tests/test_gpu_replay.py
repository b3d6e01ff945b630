"""Stage 2 parity on the GPU: carma_replay_* vs the oracle restatement of
run_simulation (world.cpp / manager.cpp / gpu.cpp / runner.cpp / metrics.cpp).
Every output field is compared bit-for-bit: per task (attempts, dispatch,
completion, crash times, OOMs, GPU ids, executed work), per GPU (energy,
mean SMACT, peak memory, step count) and per trace (report scalars, events)."""
import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi
from oracle_bind import oracle_predict, oracle_replay

pytestmark = pytest.mark.gpu


def cfg_of(policy="magm", mode="mps", gpu_count=4, max_smact=0.8, min_free=None, window=60.0, rr_pre=False,
           capacity=40 * abi.GiB, block=512 * abi.MiB, mig=None):
    return cb.make_config(cb.PolicyConfig(policy=policy, collocation_mode=mode, max_smact=max_smact,
                                          min_free_mem=min_free, monitor_window=window,
                                          rr_apply_preconditions=rr_pre),
                          cb.SimConstants(gpu_count=gpu_count, gpu_capacity=capacity, alloc_block=block), mig)


def learned_estimates(olib, m, models):
    raw = cb.scalar_features(m.features)
    est = np.zeros(len(m.tasks), np.uint64)
    for f in set(m.family.tolist()):
        sel = m.family == f
        est[sel] = oracle_predict(olib, models[f], raw[sel])[1]
    return est


@pytest.fixture(scope="module")
def models():
    return {f: cb.fit_knn(f, 4000, 11 + 101 * f, 5) for f in range(3)}


def check_jobs(olib, res, cfgs, task_lists, jobs):
    for j, (t, c) in enumerate(jobs):
        cfg = cfgs[c: c + 1]
        rc, ot, otr, og = oracle_replay(olib, cfg, task_lists[t])
        assert rc == 0
        gt = res.job_tasks(j)
        assert gt.tobytes() == ot.tobytes(), f"job {j} task results differ"
        assert res.traces[j: j + 1].tobytes() == np.array([otr]).tobytes(), f"job {j} report differs"
        assert res.job_gpus(j).tobytes() == og.tobytes(), f"job {j} gpu results differ"


def test_replay_policies_mixes_estimators(gpu, olib, models):
    """t90/t60 seeds 1..6 x {exclusive, rr, magm, lug, mug} x estimator personas."""
    task_lists = []
    for mix in ("t90", "t60"):
        for seed in range(1, 7):
            for est in ("none", "oracle", "learned", "static_graph"):
                m = cb.materialize_trace(cb.generate_trace(mix, seed))
                if est == "learned":
                    m.tasks["estimate"] = learned_estimates(olib, m, models)
                else:
                    cb.set_persona_estimates(m, est)
                task_lists.append(m.tasks)
    cfgs = np.concatenate([cfg_of(p) for p in ("exclusive", "rr", "magm", "lug", "mug")] +
                          [cfg_of("rr", rr_pre=True), cfg_of("magm", min_free=2 * abi.GiB),
                           cfg_of("magm", max_smact=1.0, mode="streams"), cfg_of("rr", mode="streams")])
    jobs = [(t, c) for c in range(len(cfgs)) for t in range(len(task_lists))]
    res = cb.replay(cfgs, task_lists, jobs)
    check_jobs(olib, res, cfgs, task_lists, jobs)


@pytest.mark.parametrize("gpus,window", [(8, 60.0), (2, 5.0), (16, 5.0), (64, 5.0)])
def test_replay_gpu_counts_and_windows(gpu, olib, models, gpus, window):
    task_lists = []
    for seed in (1, 2, 3):
        m = cb.materialize_trace(cb.generate_trace("t90", seed))
        m.tasks["estimate"] = learned_estimates(olib, m, models)
        task_lists.append(m.tasks)
    cfgs = np.concatenate([cfg_of(p, gpu_count=gpus, window=window) for p in ("magm", "lug", "rr", "exclusive")])
    jobs = [(t, c) for c in range(len(cfgs)) for t in range(len(task_lists))]
    res = cb.replay(cfgs, task_lists, jobs)
    check_jobs(olib, res, cfgs, task_lists, jobs)


def test_replay_large_trace_many_gpus(gpu, olib):
    """A 4000-task uniform-catalog trace on 64 GPUs (ids beyond t999 exercise
    the lexicographic rank order) — runs in the global-memory state tier."""
    tr = cb.generate_uniform_trace(4000, 3.0, 7)
    m = cb.materialize_trace(tr)
    cb.set_persona_estimates(m, "oracle")
    cfgs = np.concatenate([cfg_of("magm", gpu_count=64, window=5.0), cfg_of("rr", gpu_count=64, window=5.0)])
    jobs = [(0, 0), (0, 1)]
    res = cb.replay(cfgs, [m.tasks], jobs)
    check_jobs(olib, res, cfgs, [m.tasks], jobs)
    assert not np.array_equal(m.tasks["rank"], np.arange(4000))


@pytest.mark.parametrize("gpus", [65, 100, 128, 256])
def test_replay_more_than_64_gpus(gpu, olib, gpus):
    """65..256 simulated GPUs run in the many-GPU global tier (8 GPUs per
    lane, multi-word eligibility sets): every policy, 1- and 2-GPU tasks,
    bit-exact against the oracle (pinned to the reference beyond 64 GPUs in
    test_oracle_vs_ref.py)."""
    tr = cb.generate_uniform_trace(3000, 0.2, 13)
    m = cb.materialize_trace(tr)
    cb.set_persona_estimates(m, "oracle")
    assert (m.tasks["gpus"] == 2).any()
    cfgs = np.concatenate([cfg_of(p, gpu_count=gpus, window=5.0, rr_pre=pre)
                           for p, pre in (("magm", False), ("lug", False), ("mug", False), ("rr", False),
                                          ("rr", True), ("exclusive", False))])
    jobs = [(0, c) for c in range(len(cfgs))]
    res = cb.replay(cfgs, [m.tasks], jobs)
    check_jobs(olib, res, cfgs, [m.tasks], jobs)
    used = set(res.job_tasks(0)["gpu"][:, 0].tolist())
    assert max(used) >= 64, "the trace must reach GPUs past 63"


def test_replay_overflow_tier_escalation(gpu, olib):
    """RR without preconditions on 80 GiB GPUs stacks > 24 residents per GPU:
    the shared-memory tier overflows and the job re-runs in the global tier."""
    tr = cb.generate_uniform_trace(600, 1.0, 11)
    m = cb.materialize_trace(tr)
    cfg = cfg_of("rr", gpu_count=2, capacity=80 * abi.GiB, window=1.0)
    offs = np.array([0, len(m.tasks)], np.uint64)
    jobs = np.zeros(1, abi.job_dtype)
    plan = cb.ReplayPlan(cfg, m.tasks, offs, jobs)
    plan.run()
    res = plan.results()
    launches, retried = plan.stats()
    check_jobs(olib, res, cfg, [m.tasks], [(0, 0)])
    assert res.traces["status"][0] == 0


def test_replay_deterministic_and_resident(gpu, olib):
    task_lists = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in range(1, 65)]
    cfgs = np.concatenate([cfg_of(p) for p in ("exclusive", "rr", "magm", "lug")])
    offs = np.concatenate([[0], np.cumsum([len(t) for t in task_lists])]).astype(np.uint64)
    jobs = np.zeros(len(task_lists) * 4, abi.job_dtype)
    jobs["trace"] = np.tile(np.arange(len(task_lists)), 4)
    jobs["config"] = np.repeat(np.arange(4), len(task_lists))
    plan = cb.ReplayPlan(cfgs, np.concatenate(task_lists), offs, jobs)
    plan.run()
    r1 = plan.results()
    plan.run()
    r2 = plan.results()
    assert r1.tasks.tobytes() == r2.tasks.tobytes()
    assert r1.traces.tobytes() == r2.traces.tobytes()
    for j in range(0, len(jobs), 37):
        t, c = int(jobs["trace"][j]), int(jobs["config"][j])
        rc, ot, otr, og = oracle_replay(olib, cfgs[c: c + 1], task_lists[t])
        assert r1.job_tasks(j).tobytes() == ot.tobytes()


def test_pick_batch_matches_oracle(gpu, olib):
    rng = np.random.default_rng(1)
    for g in (1, 3, 4, 8, 17, 32, 64):
        n = 3000
        views = np.zeros((n, g), abi.gpu_view_dtype)
        views["total_free"] = rng.integers(0, 81, (n, g)).astype(np.uint64) * (512 * abi.MiB)
        views["total_free"][:, ::3] = 20 * abi.GiB  # ties
        views["windowed_smact"] = np.round(rng.random((n, g)), 1)
        views["idle"] = rng.random((n, g)) < 0.3
        reqs = np.zeros(n, abi.pick_request_dtype)
        reqs["estimate"] = np.where(rng.random(n) < 0.3, abi.NO_ESTIMATE,
                                    rng.integers(0, 45, n).astype(np.uint64) * abi.GiB)
        reqs["want"] = np.where(rng.random(n) < 0.2, 2, 1).astype(np.uint32)
        if g == 1:
            reqs["want"] = 1
        reqs["from_recovery"] = rng.random(n) < 0.1
        cursor = rng.integers(0, g, n).astype(np.int32)
        for policy in ("exclusive", "rr", "magm", "lug", "mug"):
            for rr_pre in (False, True):
                cfg = cfg_of(policy, gpu_count=g, min_free=abi.GiB, rr_pre=rr_pre)
                out, cur = cb.pick_batch(cfg, views, reqs, cursor)
                for i in range(0, n, 7):
                    oc = np.array([cursor[i]], np.int32)
                    oo = np.zeros(2, np.int32)
                    olib.oracle_pick(cfg.ctypes.data, views[i].ctypes.data, g, reqs[i: i + 1].ctypes.data,
                                     oc.ctypes.data, oo.ctypes.data)
                    assert out[i].tolist() == oo.tolist(), (g, policy, i)
                    assert cur[i] == oc[0]


def test_gpu_replay_matches_reference_golden(gpu, olib):
    """All 72 golden reference runs (12 of them MIG) (tests/golden/replay.npz) in one batch; learned
    estimates come from the GPU k-NN (GPUMemNet stage feeding stage 2)."""
    import os

    from cases import assert_matches_ref, case_inputs
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "replay.npz"))
    knn = cb.GpuKnn(gpu)
    cfgs, lists = [], []
    for case in g["cases"]:
        cfg, tasks = case_inputs(olib, str(case), knn=knn)
        cfgs.append(cfg)
        lists.append(tasks)
    jobs = [(i, i) for i in range(len(lists))]
    res = cb.replay(np.concatenate(cfgs), lists, jobs)
    for i in range(len(lists)):
        assert_matches_ref(g, i, res.job_tasks(i), res.traces[i], res.job_gpus(i))


def test_plan_upload_and_outcomes(gpu, olib):
    """Re-uploading a different task set into a plan and the compact outcome path."""
    a = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in (1, 2)]
    b = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in (3, 4)]
    cfg = cfg_of("magm")
    offs = np.array([0, 90, 180], np.uint64)
    jobs = np.zeros(2, abi.job_dtype)
    jobs["trace"] = [0, 1]
    plan = cb.ReplayPlan(cfg, np.concatenate(a), offs, jobs)
    plan.run()
    plan.upload_tasks(np.concatenate(b))
    plan.run()
    to, jr, gr = plan.outcomes()
    for j in range(2):
        rc, ot, otr, og = oracle_replay(olib, cfg, b[j])
        sl = slice(90 * j, 90 * (j + 1))
        assert np.array_equal(to["complete"][sl], ot["complete"])
        assert np.array_equal(to["final_dispatch"][sl], ot["final_dispatch"])
        assert np.array_equal(to["ooms"][sl], ot["ooms"]) and np.array_equal(to["attempts"][sl], ot["attempts"])
        assert jr[j].tobytes() == np.array([otr]).tobytes()


@pytest.mark.parametrize("estimator", ["learned", "none"])
def test_fused_c5_prefix_matches_oracle(gpu, olib, estimator):
    """BASELINE c5 shape on a 20k-task prefix: uniform catalog, 3 s mean gaps,
    64 GPUs, MAGM u=0.8, W=5 s; learned estimates from the on-device k-NN
    pre-pass feed the replay without leaving the GPU."""
    from cases import model
    m = cb.materialize_trace(cb.generate_uniform_trace(20000, 3.0, 7))
    cfg = cfg_of("magm", gpu_count=64, window=5.0)
    knn = cb.GpuKnn(gpu)
    for f in (1, 2):
        knn.set_model(model(f))
    want_tasks = m.tasks.copy()
    if estimator == "learned":
        raw = cb.scalar_features(m.features)
        e = np.zeros(len(m.tasks), np.uint64)
        for f in set(m.family.tolist()):
            sel = m.family == f
            e[sel] = oracle_predict(olib, model(f), raw[sel])[1]
        want_tasks["estimate"] = e
        fused = cb.FusedReplay(m, cfg, knn, gpu)
        fused.run()
        res = fused.results()
        fused.close()
    else:
        res = cb.replay(cfg, [m.tasks])
    rc, ot, otr, og = oracle_replay(olib, cfg, want_tasks)
    assert rc == 0
    assert res.job_tasks(0).tobytes() == ot.tobytes()
    assert res.traces[0:1].tobytes() == np.array([otr]).tobytes()
    assert res.job_gpus(0).tobytes() == og.tobytes()


def test_fused_orders_prepass_before_replay(gpu, olib):
    """FusedReplay regression (round-1 race): the k-NN pre-pass and the replay
    that reads its bytes run on one stream, after the caller's queued work.
    The caller's stream is kept busy (a device sleep) and then overwrites the
    estimates with a sentinel (0 bytes: every task fits anywhere); if the
    replay read them before the pre-pass rewrote them, placements would
    differ from the oracle's learned run."""
    import torch
    from cases import model
    m = cb.materialize_trace(cb.generate_uniform_trace(4000, 3.0, 7))
    cfg = cfg_of("magm", gpu_count=8, window=5.0)
    knn = cb.GpuKnn(gpu)
    for f in (1, 2):
        knn.set_model(model(f))
    want = m.tasks.copy()
    raw = cb.scalar_features(m.features)
    e = np.zeros(len(m.tasks), np.uint64)
    for f in set(m.family.tolist()):
        sel = m.family == f
        e[sel] = oracle_predict(olib, model(f), raw[sel])[1]
    want["estimate"] = e
    rc, ot, otr, og = oracle_replay(olib, cfg, want)
    assert rc == 0 and int(otr["oom_count"]) >= 0
    fused = cb.FusedReplay(m, cfg, knn, gpu)
    side = torch.cuda.Stream()
    for caller in (torch.cuda.current_stream(), side):
        for _ in range(3):
            with torch.cuda.stream(caller):
                torch.cuda._sleep(20_000_000)       # ~10 ms of queued caller work
                fused.d_bytes.fill_(0)               # sentinel, ordered before the pre-pass
                fused.run(stream=caller)
                after = fused.d_bytes.clone()        # caller work after run() sees the pre-pass output
            res = fused.results()
            assert res.job_tasks(0).tobytes() == ot.tobytes()
            assert res.traces[0:1].tobytes() == np.array([otr]).tobytes()
            torch.cuda.synchronize()
            assert np.array_equal(after.cpu().numpy().view(np.uint64), e)
    fused.close()
    knn.close()


# MIG (gpu.cpp:29-51, :151-195; manager.cpp:125-134, :176-187, :236-243).
# Instance 0 holds the largest catalog task, so every run terminates (the
# reference retries crashed tasks exclusively on instance 0).
MIG_CASES = [("magm", (0.75, 0.25), "none", 4), ("rr", (0.7, 0.15, 0.15), "none", 4),
             ("exclusive", (0.75, 0.125), "none", 4), ("lug", (0.8, 0.2), "oracle", 4),
             ("mug", (1.0,), "none", 8), ("magm", (0.75, 0.125, 0.125), "analytical", 4),
             ("magm", (0.9, 0.05, 0.05), "learned", 8), ("rr", (0.8, 0.2), "oracle", 2)]


def test_replay_mig_matches_oracle(gpu, olib, models):
    task_lists, cfgs, jobs = [], [], []
    for c, (pol, fr, est, g) in enumerate(MIG_CASES):
        cfgs.append(cb.make_config(cb.PolicyConfig(policy=pol, collocation_mode="mig",
                                                   rr_apply_preconditions=pol == "rr" and est != "none"),
                                   cb.SimConstants(gpu_count=g), fr))
        for mix in ("t90", "t60"):
            for seed in (11, 12, 13):
                m = cb.materialize_trace(cb.generate_trace(mix, seed))
                if est == "learned":
                    m.tasks["estimate"] = learned_estimates(olib, m, models)
                else:
                    cb.set_persona_estimates(m, est)
                task_lists.append(m.tasks)
                jobs.append((len(task_lists) - 1, c))
    cfgs = np.concatenate(cfgs)
    res = cb.replay(cfgs, task_lists, jobs)
    assert (res.traces["oom_count"] > 0).any()  # the instance limits bite
    check_jobs(olib, res, cfgs, task_lists, jobs)



def test_pick_batch_device_matches_host_path(gpu, olib):
    """carma_pick_batch_device on device-resident arrays (the bench's scoring
    workload shape) equals the host-buffer path decision for decision."""
    import torch
    rng = np.random.default_rng(7)
    for g in (4, 8, 64):
        n = 50000
        views = np.zeros((n, g), abi.gpu_view_dtype)
        views["total_free"] = rng.integers(0, 81, (n, g)).astype(np.uint64) * (512 * abi.MiB)
        views["windowed_smact"] = rng.random((n, g))
        views["idle"] = rng.random((n, g)) < 0.3
        reqs = np.zeros(n, abi.pick_request_dtype)
        reqs["estimate"] = rng.integers(0, 45, n).astype(np.uint64) * abi.GiB
        reqs["want"] = np.where(rng.random(n) < 0.2, 2, 1).astype(np.uint32)
        cursor = rng.integers(0, g, n).astype(np.int32)
        for policy in ("rr", "magm", "lug"):
            cfg = cfg_of(policy, gpu_count=g, rr_pre=True)
            out, cur = cb.pick_batch(cfg, views, reqs, cursor)
            dv = torch.from_numpy(views.view(np.uint8).reshape(-1)).cuda()
            dr = torch.from_numpy(reqs.view(np.uint8).reshape(-1)).cuda()
            dc = torch.from_numpy(cursor.copy()).cuda()
            do = torch.empty(2 * n, dtype=torch.int32, device="cuda")
            abi.check(abi.lib.carma_pick_batch_device(gpu, cfg.ctypes.data, dv.data_ptr(), g, dr.data_ptr(), n,
                                                      dc.data_ptr(), do.data_ptr(), None))
            torch.cuda.synchronize()
            assert np.array_equal(do.cpu().numpy().reshape(n, 2), out), (g, policy)
            assert np.array_equal(dc.cpu().numpy(), cur), (g, policy)


@pytest.mark.parametrize("capacity,block", [(192 * abi.GiB, 512 * abi.MiB), (40 * abi.GiB, 16 * abi.MiB),
                                            (192 * abi.GiB, 48 * abi.MiB)])
def test_replay_more_than_256_blocks(gpu, olib, models, capacity, block):
    """Devices with 384 / 2560 / 4096 allocation blocks (a 192 GiB B200-class
    GPU at 512 MiB blocks, fine 16 MiB blocks): the wide global tier's 64-word
    bitmaps, every policy, MPS / streams / MIG, against the oracle."""
    task_lists = []
    for mix, seed in (("t90", 1), ("t90", 2), ("t60", 3)):
        m = cb.materialize_trace(cb.generate_trace(mix, seed))
        m.tasks["estimate"] = learned_estimates(olib, m, models)
        task_lists.append(m.tasks)
    cfgs = np.concatenate([cfg_of(p, gpu_count=g, capacity=capacity, block=block)
                           for p in ("exclusive", "rr", "magm", "lug", "mug") for g in (4, 8)] +
                          [cfg_of("magm", mode="streams", max_smact=1.0, capacity=capacity, block=block)] +
                          ([cfg_of("lug", mode="mig", mig=[0.75, 0.25], capacity=capacity, block=block)]
                           if capacity > 64 * abi.GiB else []))
    jobs = [(t, c) for c in range(len(cfgs)) for t in range(len(task_lists))]
    res = cb.replay(cfgs, task_lists, jobs)
    check_jobs(olib, res, cfgs, task_lists, jobs)


@pytest.mark.parametrize("gpus,mode", [(8, "mps"), (64, "mps"), (130, "mps"), (16, "mig"), (12, "streams")])
def test_replay_tasks_requesting_up_to_8_gpus(gpu, olib, gpus, mode):
    """Tasks asking for 1..8 GPUs (TaskSpec::gpus_requested; the catalog only
    has 1 and 2) run in the multi-GPU instantiations (F bit 4): allocation on
    every device with roll-back, the task rate as the min over its devices,
    affected-task de-duplication over all touched devices; bit-exact against
    the oracle for every policy."""
    m = cb.materialize_trace(cb.generate_uniform_trace(1500, 0.5, 21))
    cb.set_persona_estimates(m, "oracle")
    rng = np.random.default_rng(gpus)
    m.tasks["gpus"] = rng.integers(1, 9, len(m.tasks)).astype(np.uint32)
    mig = [0.75, 0.25] if mode == "mig" else None
    cfgs = np.concatenate([cfg_of(p, mode=mode, gpu_count=gpus, window=5.0, rr_pre=pre, mig=mig)
                           for p, pre in (("magm", False), ("lug", False), ("mug", False), ("rr", False),
                                          ("rr", True), ("exclusive", False))])
    jobs = [(0, c) for c in range(len(cfgs))]
    res = cb.replay(cfgs, [m.tasks], jobs)
    check_jobs(olib, res, cfgs, [m.tasks], jobs)
    placed = res.job_tasks(0)
    assert (placed["final_dispatch"][m.tasks["gpus"] > 2] >= 0).any(), "some wide tasks must be placed"


def test_replay_rejects_wide_tasks_uploaded_into_a_narrow_plan(gpu):
    """A plan classified with 1-2 GPU tasks reports UNSUPPORTED per job when
    re-uploaded tasks ask for more (device-side check; no silent misplacement)."""
    m = cb.materialize_trace(cb.generate_uniform_trace(200, 1.0, 3))
    cfg = cfg_of("magm", gpu_count=8, window=5.0)
    offs = np.array([0, len(m.tasks)], np.uint64)
    jobs = np.zeros(1, abi.job_dtype)
    plan = cb.ReplayPlan(cfg, m.tasks, offs, jobs)
    t2 = m.tasks.copy()
    t2["gpus"][5] = 4
    abi.check(abi.lib.carma_replay_plan_upload_tasks(plan._h, t2.ctypes.data))
    plan.run()
    assert plan.results().traces["status"][0] == abi.CARMA_ERR_UNSUPPORTED
    plan.close()


@pytest.mark.parametrize("capacity,block", [(40 * abi.GiB, 0), (40 * abi.GiB + 100 * abi.MiB, 512 * abi.MiB),
                                            (192 * abi.GiB, 8 * abi.MiB), (32 * abi.GiB + 7, 0)])
def test_replay_byte_granular_allocator(gpu, olib, capacity, block):
    """alloc_block = 0 (round_up is the identity), capacities that are not a
    block multiple (tail carving leaves unaligned offsets) and > 4096 blocks
    run on the segment allocator (gpu.cpp:58-130) of the generic
    instantiations; bit-exact against the oracle, whose allocator is the same
    segment list and is pinned to the reference (test_oracle_vs_ref.py)."""
    m = cb.materialize_trace(cb.generate_uniform_trace(1200, 0.5, 17))
    cb.set_persona_estimates(m, "oracle")
    cfgs = np.concatenate([cfg_of(p, gpu_count=g, window=5.0, rr_pre=pre, capacity=capacity, block=block)
                           for p, pre, g in (("magm", False, 8), ("lug", False, 8), ("rr", False, 4),
                                             ("exclusive", False, 8), ("magm", False, 100))])
    jobs = [(0, c) for c in range(len(cfgs))]
    res = cb.replay(cfgs, [m.tasks], jobs)
    check_jobs(olib, res, cfgs, [m.tasks], jobs)
    assert res.traces["oom_count"][2] > 0  # RR stacking: OOM crashes and their free / largest reports


def test_outcome_sink_streams_the_same_outcomes(gpu):
    """carma_replay_plan_set_outcome_sink: the per-task outcomes written to
    pinned host memory by the kernel as jobs finish equal the compacted
    read-back (incl. jobs that overflow a tier and re-run)."""
    import torch
    lists = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in range(1, 201)]
    tasks = np.concatenate(lists)
    offs = np.concatenate([[0], np.cumsum([len(t) for t in lists])]).astype(np.uint64)
    cfgs = np.concatenate([cfg_of(p, gpu_count=4) for p in ("exclusive", "rr", "magm", "lug")] +
                          [cfg_of("rr", gpu_count=2, capacity=80 * abi.GiB, window=1.0)])
    jobs = np.zeros(len(lists) * len(cfgs), abi.job_dtype)
    jobs["trace"] = np.tile(np.arange(len(lists), dtype=np.uint32), len(cfgs))
    jobs["config"] = np.repeat(np.arange(len(cfgs), dtype=np.uint32), len(lists))
    plan = cb.ReplayPlan(cfgs, tasks, offs, jobs)
    n_out = int(np.diff(offs.astype(np.int64))[jobs["trace"]].sum())
    sink = torch.empty(n_out * 24, dtype=torch.uint8).pin_memory().numpy().view(abi.task_outcome_dtype)
    sink[:] = np.frombuffer(b"\xff" * sink.nbytes, dtype=abi.task_outcome_dtype)
    abi.check(abi.lib.carma_replay_plan_set_outcome_sink(plan._h, sink.ctypes.data))
    plan.run()
    ref_o = np.zeros(n_out, abi.task_outcome_dtype)
    abi.check(abi.lib.carma_replay_plan_outcomes(plan._h, ref_o.ctypes.data, None, None))
    assert sink.tobytes() == ref_o.tobytes()
    pageable = np.zeros(4, abi.task_outcome_dtype)
    assert abi.lib.carma_replay_plan_set_outcome_sink(plan._h, pageable.ctypes.data) == abi.CARMA_ERR_INVALID
    abi.check(abi.lib.carma_replay_plan_set_outcome_sink(plan._h, None))
    plan.close()


def test_pick_batch_wide_matches_oracle(gpu, olib):
    """carma_pick_batch_wide: up to 256 GPUs per snapshot, up to 8 GPUs per
    decision, every policy, against the oracle's map_task (oracle_pick_wide)."""
    rng = np.random.default_rng(2)
    for g in (1, 5, 40, 64, 100, 256):
        n = 800
        views = np.zeros((n, g), abi.gpu_view_dtype)
        views["total_free"] = rng.integers(0, 81, (n, g)).astype(np.uint64) * (512 * abi.MiB)
        views["total_free"][:, ::3] = 20 * abi.GiB  # ties
        views["windowed_smact"] = np.round(rng.random((n, g)), 1)
        views["idle"] = rng.random((n, g)) < 0.4
        reqs = np.zeros(n, abi.pick_request_dtype)
        reqs["estimate"] = np.where(rng.random(n) < 0.3, abi.NO_ESTIMATE,
                                    rng.integers(0, 45, n).astype(np.uint64) * abi.GiB)
        reqs["want"] = rng.integers(1, min(8, g) + 1, n).astype(np.uint32)
        reqs["from_recovery"] = rng.random(n) < 0.1
        cursor0 = rng.integers(0, g, n).astype(np.int32)
        for policy in ("exclusive", "rr", "magm", "lug", "mug"):
            for rr_pre in (False, True):
                cfg = cfg_of(policy, gpu_count=g, min_free=abi.GiB, rr_pre=rr_pre)
                cur = cursor0.copy()
                out = np.zeros((n, 8), np.int32)
                abi.check(abi.lib.carma_pick_batch_wide(gpu, cfg.ctypes.data, views.ctypes.data, g,
                                                        reqs.ctypes.data, n, cur.ctypes.data, out.ctypes.data))
                for i in range(0, n, 3):
                    oc = np.array([cursor0[i]], np.int32)
                    oo = np.zeros(8, np.int32)
                    olib.oracle_pick_wide(cfg.ctypes.data, views[i].ctypes.data, g, reqs[i: i + 1].ctypes.data,
                                          oc.ctypes.data, oo.ctypes.data)
                    assert out[i].tolist() == oo.tolist(), (g, policy, rr_pre, i)
                    assert cur[i] == oc[0]
