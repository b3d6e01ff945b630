"""RunConfig::enable_timeline on the GPU replay against the reference itself
(oracle/_ref): the sample ticks are events, so every output (energy bits,
completions, reports) must match the reference run WITH the timeline, and the
timeline text (runner.cpp:80-93, world.cpp:210-219) must be identical."""
import ctypes
import dataclasses

import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from oracle_bind import ref_config, ref_run

pytestmark = pytest.mark.gpu

CASES = [dict(policy="magm", interval=10.0), dict(policy="rr", interval=7.3),
         dict(policy="lug", interval=60.0, gpu_count=8, window=5.0),
         dict(policy="exclusive", interval=10.0, estimator="oracle"),
         dict(policy="magm", interval=10.0, mode="mig", mig=(0.75, 0.25)),
         # byte-granular allocator (generic instantiations): alloc_block 0, non-multiple capacity
         dict(policy="rr", interval=7.3, block=0),
         dict(policy="magm", interval=10.0, capacity=40 * 2**30 + 100 * 2**20),
         # MIG on a byte-granular device: instance boundaries in bytes
         dict(policy="magm", interval=10.0, mode="mig", mig=(0.7, 0.3), block=0),
         dict(policy="lug", interval=7.3, mode="mig", mig=(0.75, 0.25), capacity=40 * 2**30 + 100 * 2**20)]


@pytest.mark.parametrize("case", CASES, ids=[str(i) for i in range(len(CASES))])
@pytest.mark.parametrize("mix,seed", [("t90", 1), ("t60", 4)])
def test_timeline_matches_reference(gpu, ref, case, mix, seed):
    kw = dict(case)
    interval = kw.pop("interval")
    est = kw.get("estimator", "none")
    rc = cb.RunConfig(mix=mix, trace_seed=seed, enable_timeline=True, sample_interval=interval,
                      policy=cb.PolicyConfig(policy=kw["policy"], estimator=est,
                                             collocation_mode=kw.get("mode", "mps"),
                                             monitor_window=kw.get("window", 60.0)),
                      constants=cb.SimConstants(gpu_count=kw.get("gpu_count", 4),
                                                **({"gpu_capacity": kw["capacity"]} if "capacity" in kw else {}),
                                                **({"alloc_block": kw["block"]} if "block" in kw else {})),
                      mig_instances=list(kw.get("mig", ())))
    art = cb.run_simulation_artifacts(rc, device=gpu)
    cfg = ref_config(**kw, sample_interval=interval)
    tout, rout, ge, gs, gp = ref_run(ref, cfg, mix=mix, seed=seed)
    buf = ctypes.create_string_buffer(1 << 22)
    assert ref.ref_timeline(cfg.ctypes.data, cb.abi.MIX[mix], seed, buf, len(buf)) == 0
    assert "\n".join(art.timeline) + "\n" == buf.value.decode()
    assert np.array_equal(art.tasks["complete"], tout["complete"])
    assert np.array_equal(art.tasks["executed"], tout["executed"])
    assert art.report["energy_mj"] == rout["energy_mj"] and art.report["avg_jct"] == rout["avg_jct"]
    assert np.array_equal(art.gpus["energy_j"], ge) and np.array_equal(art.gpus["mean_smact"], gs)


def test_timeline_off_is_unchanged(gpu):
    rc = cb.RunConfig(mix="t90", trace_seed=2)
    a = cb.run_simulation_artifacts(rc, device=gpu)
    r, t, g = cb.run_simulation(rc, device=gpu)
    assert a.timeline == [] and a.report.tobytes() == r.tobytes() and a.tasks.tobytes() == t.tobytes()


LOG_CASES = [dict(policy="magm"), dict(policy="rr"), dict(policy="lug", estimator="oracle"),
             dict(policy="magm", mode="mig", mig=(0.75, 0.25)), dict(policy="exclusive", gpu_count=8),
             dict(policy="rr", block=0), dict(policy="rr", capacity=40 * 2**30 + 100 * 2**20),
             dict(policy="magm", mode="mig", mig=(0.75, 0.25), block=0)]


@pytest.mark.parametrize("case", LOG_CASES, ids=[str(i) for i in range(len(LOG_CASES))])
@pytest.mark.parametrize("mix,seed", [("t90", 2), ("t60", 5)])
def test_event_and_decision_logs_match_reference(gpu, ref, case, mix, seed):
    """RunConfig::enable_event_log + verbose_decisions: place / complete /
    alloc_oom lines (world.cpp:94-153) and decide lines (manager.cpp:298-318)
    identical to the reference's, and the run itself unchanged."""
    kw = dict(case)
    est = kw.get("estimator", "none")
    rc = cb.RunConfig(mix=mix, trace_seed=seed, enable_event_log=True, verbose_decisions=True,
                      policy=cb.PolicyConfig(policy=kw["policy"], estimator=est,
                                             collocation_mode=kw.get("mode", "mps")),
                      constants=cb.SimConstants(gpu_count=kw.get("gpu_count", 4),
                                                **({"gpu_capacity": kw["capacity"]} if "capacity" in kw else {}),
                                                **({"alloc_block": kw["block"]} if "block" in kw else {})),
                      mig_instances=list(kw.get("mig", ())))
    art = cb.run_simulation_artifacts(rc, device=gpu)
    cfg = ref_config(**kw, log_flags=3)
    ev = ctypes.create_string_buffer(1 << 22)
    de = ctypes.create_string_buffer(1 << 22)
    assert ref.ref_logs(cfg.ctypes.data, cb.abi.MIX[mix], seed, ev, len(ev), de, len(de)) == 0
    assert "".join(l + "\n" for l in art.event_log) == ev.value.decode()
    assert "".join(l + "\n" for l in art.decision_log) == de.value.decode()
    if kw["policy"] == "rr":  # stacking without preconditions: OOM lines are exercised
        assert any("alloc_oom" in l for l in art.event_log)
    r, t, g = cb.run_simulation(dataclasses.replace(rc, enable_event_log=False, verbose_decisions=False), device=gpu)
    assert r.tobytes() == art.report.tobytes() and t.tobytes() == art.tasks.tobytes()
