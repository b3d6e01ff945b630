"""Shared builders: reference-style case dicts -> replay inputs."""
import ast

import numpy as np

import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi
from oracle_bind import oracle_predict, ref_config, replay_config_from

_MODELS = {}


def model(family, samples=4000, seed=None, k=5):
    seed = 11 + 101 * family if seed is None else seed
    key = (family, samples, seed, k)
    if key not in _MODELS:
        _MODELS[key] = cb.fit_knn(family, samples, seed, k)
    return _MODELS[key]


def case_inputs(olib, case, knn=None):
    """(replay config row, task array) for a golden case; learned estimates come
    from the oracle k-NN, or from `knn` (a GpuKnn) when given."""
    if isinstance(case, str):
        case = ast.literal_eval(case)
    kw = {k: v for k, v in case.items() if k not in ("mix", "seed")}
    cfg = replay_config_from(ref_config(**kw))
    m = cb.materialize_trace(cb.generate_trace(case["mix"], case["seed"]))
    est = case.get("estimator", "none")
    if est == "learned":
        if knn is not None:
            for f in set(m.family.tolist()):
                if f not in knn.models:
                    knn.set_model(model(f))
            m.tasks["estimate"] = knn.predict(m.features, family=m.family)[1]
        else:
            raw = cb.scalar_features(m.features)
            e = np.zeros(len(m.tasks), np.uint64)
            for f in set(m.family.tolist()):
                sel = m.family == f
                e[sel] = oracle_predict(olib, model(f), raw[sel])[1]
            m.tasks["estimate"] = e
    else:
        cb.set_persona_estimates(m, est)
    return cfg, m.tasks


def assert_matches_ref(golden, i, tasks_out, trace_out, gpus_out):
    """Compare replay outputs (carma_* layouts) to golden reference case i."""
    rt = golden[f"tasks_{i}"]
    for ours, theirs in (("first_attempt", "first_attempt"), ("final_dispatch", "final_dispatch"),
                         ("complete", "complete"), ("first_crash", "first_crash"), ("last_crash", "last_crash"),
                         ("executed", "executed"), ("attempts", "n_attempts"), ("ooms", "ooms")):
        a, b = tasks_out[ours], rt[theirs]
        assert np.array_equal(np.asarray(a).view(np.uint64) if a.dtype == np.float64 else a,
                              np.asarray(b).view(np.uint64) if b.dtype == np.float64 else b), (i, ours)
    assert np.array_equal(tasks_out["gpu"][:, 0], rt["gpu0"]) and np.array_equal(tasks_out["gpu"][:, 1], rt["gpu1"])
    rr = golden[f"report_{i}"][0]
    for f in ("trace_total_time", "avg_wait", "avg_exec", "avg_jct", "energy_mj", "last_complete", "first_submit"):
        assert np.float64(trace_out[f]).tobytes() == np.float64(rr[f]).tobytes(), (i, f)
    assert int(trace_out["oom_count"]) == int(rr["oom_count"])
    assert np.array_equal(gpus_out["energy_j"].view(np.uint64), golden[f"gpu_energy_{i}"].view(np.uint64))
    assert np.array_equal(gpus_out["mean_smact"].view(np.uint64), golden[f"gpu_smact_{i}"].view(np.uint64))
    assert np.array_equal(gpus_out["peak_used"], golden[f"gpu_peak_{i}"])
