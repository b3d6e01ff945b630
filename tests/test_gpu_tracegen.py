"""Device-side sweep inputs (carma_replay_plan_create_generated): every task of
generate_trace(mix, seed) + materialisation (traces.cpp:238-306), generated on
the GPU, must equal the host generator's bit for bit — submit times, work,
demand, memory, GPUs, rank, estimates and catalog entries — and replaying the
generated plan must equal replaying the host-built one."""
import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi

pytestmark = pytest.mark.gpu


def host_tasks(mix, seeds):
    ts, es = [], []
    for s in seeds:
        m = cb.materialize_trace(cb.generate_trace(mix, int(s)))
        ts.append(m.tasks)
        es.append(m.entry)
    return np.concatenate(ts), np.concatenate(es)


def one_config():
    return cb.make_config(cb.PolicyConfig(policy="magm", max_smact=0.8), cb.SimConstants())


@pytest.mark.parametrize("mix,n,first", [("t90", 100_000, 1), ("t60", 20_000, 1),
                                         ("t90", 50_000, 0), ("t60", 50_000, 0)])
def test_generated_tasks_equal_host_generator(gpu, mix, n, first):
    """first = 0: random 64-bit seeds (the device log1p is glibc's algorithm,
    so no seed range is special)."""
    seeds = np.arange(first, first + n, dtype=np.uint64) if first else \
        np.random.default_rng(2026).integers(1, 2**63, n, dtype=np.uint64)
    jobs = np.zeros(n, abi.job_dtype)
    jobs["trace"] = np.arange(n, dtype=np.uint32)
    plan = cb.ReplayPlan.generated(one_config(), mix, seeds, jobs, device=gpu)
    dt, de = plan.device_tasks()
    plan.close()
    ht, he = host_tasks(mix, seeds)
    assert np.array_equal(de, he)
    for f in ("submit", "work", "demand"):
        bad = np.nonzero(dt[f].view(np.uint64) != ht[f].view(np.uint64))[0]
        assert len(bad) == 0, (f, bad[:5], dt[f][bad[:5]], ht[f][bad[:5]])
    for f in ("true_mem", "estimate", "gpus", "rank"):
        assert np.array_equal(dt[f], ht[f]), f


@pytest.mark.parametrize("estimator", ["oracle", "analytical", "learned"])
def test_generated_estimates_match_provisioning(gpu, estimator):
    seeds = np.arange(40, 60, dtype=np.uint64)
    rc = cb.RunConfig(mix="t90", policy=cb.PolicyConfig(policy="magm", estimator=estimator))
    knn = cb.GpuKnn(gpu)
    table = cb.entry_estimates(rc, gpu, knn)
    jobs = np.zeros(len(seeds), abi.job_dtype)
    jobs["trace"] = np.arange(len(seeds), dtype=np.uint32)
    plan = cb.ReplayPlan.generated(one_config(), "t90", seeds, jobs, table[None, :], device=gpu)
    dt, _ = plan.device_tasks()
    plan.close()
    for i, s in enumerate(seeds):
        m = cb.materialize_trace(cb.generate_trace("t90", int(s)))
        cb.provision_estimates(rc, m, gpu, knn)
        assert np.array_equal(dt["estimate"][90 * i: 90 * (i + 1)], m.tasks["estimate"])
    knn.close()


def test_generated_plan_replays_like_host_plan(gpu):
    seeds = np.arange(1, 2001, dtype=np.uint64)
    pols = ("exclusive", "rr", "magm", "lug")
    cfgs = np.concatenate([cb.make_config(cb.PolicyConfig(policy=p, max_smact=0.8), cb.SimConstants())
                           for p in pols])
    n = len(seeds)
    jobs = np.zeros(n * len(pols), abi.job_dtype)
    jobs["trace"] = np.tile(np.arange(n, dtype=np.uint32), len(pols))
    jobs["config"] = np.repeat(np.arange(len(pols), dtype=np.uint32), n)
    g = cb.ReplayPlan.generated(cfgs, "t90", seeds, jobs, device=gpu)
    g.run()
    rg = g.results()
    g.close()
    ht, _ = host_tasks("t90", seeds)
    offs = np.arange(n + 1, dtype=np.uint64) * np.uint64(90)
    h = cb.ReplayPlan(cfgs, ht, offs, jobs, device=gpu)
    h.run()
    rh = h.results()
    h.close()
    assert rg.traces.tobytes() == rh.traces.tobytes()
    assert rg.tasks.tobytes() == rh.tasks.tobytes()
    assert rg.gpus.tobytes() == rh.gpus.tobytes()


def test_generated_rejects_bad_input(gpu):
    jobs = np.zeros(1, abi.job_dtype)
    with pytest.raises(abi.CarmaError):
        cb.ReplayPlan.generated(one_config(), "t90", np.zeros(0, np.uint64), jobs, device=gpu)
    bad = np.zeros(1, abi.job_dtype)
    bad["trace"] = 5
    with pytest.raises(abi.CarmaError):
        cb.ReplayPlan.generated(one_config(), "t90", np.ones(2, np.uint64), bad, device=gpu)
