"""ctypes bindings of the test oracles (test infrastructure only).

* ``oracle``  — oracle/build/liboracle.so: the CPU restatement (always buildable).
* ``ref``     — oracle/_ref/libcarma_ref.so: the UNMODIFIED reference library +
                marshalling shim; present when built here (needs /root/reference)
                or shipped prebuilt to the GPU box.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_uint32, c_uint64, c_void_p

import numpy as np

# Enum values of the reference's public types (manager.hpp:15-19, gpu.hpp:14,
# traces.hpp). Kept here, not imported from the product package, so a process
# that only drives the reference (bench.py --impl reference) never maps
# libcarma_b200.so.
POLICY = {"exclusive": 0, "rr": 1, "magm": 2, "lug": 3, "mug": 4}
MODE = {"streams": 0, "mps": 1, "mig": 2}
ESTIMATOR = {"none": 0, "oracle": 1, "analytical": 2, "static_graph": 3, "learned": 4}
MIX = {"t90": 0, "t60": 1}
GiB = 1 << 30
MiB = 1 << 20

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcarma_ref.so")
P = c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data


def load_oracle() -> ctypes.CDLL:
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       stdout=subprocess.DEVNULL)
    lib = ctypes.CDLL(ORACLE_SO)
    lib.oracle_knn_predict.restype = c_int
    lib.oracle_knn_predict.argtypes = [P, P, P, P, c_uint64, c_uint32, c_uint64, P, c_uint64, P, P, P, P]
    lib.oracle_replay.restype = c_int
    lib.oracle_replay.argtypes = [P, P, c_uint32, P, P, P]
    lib.oracle_pick.restype = c_int
    lib.oracle_pick.argtypes = [P, P, c_uint32, P, P, P]
    lib.oracle_pick_wide.restype = c_int
    lib.oracle_pick_wide.argtypes = [P, P, c_uint32, P, P, P]
    return lib


def load_ref():
    if not os.path.exists(REF_SO):
        return None
    lib = ctypes.CDLL(REF_SO)
    lib.ref_last_error.restype = c_char_p
    lib.ref_train.argtypes = [c_int, c_uint64, c_uint64, c_uint64, c_char_p, P, P, P, P, c_uint64,
                              POINTER(c_uint64), POINTER(c_uint64), P]
    lib.ref_dataset.argtypes = [c_int, c_uint64, c_uint64, P, P, P]
    lib.ref_dataset_fv.argtypes = [c_int, c_uint64, c_uint64, P, P, P, P, P]
    lib.ref_predict_dataset.argtypes = [c_int, c_uint64, c_uint64, c_uint64, c_uint64, c_uint64, P, P]
    lib.ref_bench_predict.restype = c_double
    lib.ref_bench_predict.argtypes = [c_int, c_uint64, c_uint64, c_uint64, c_uint64, c_uint64, c_int, c_int,
                                      POINTER(c_uint64)]
    lib.ref_gen_trace.argtypes = [c_int, c_uint64, P, P, P, c_uint64, POINTER(c_uint64)]
    lib.ref_save_trace.argtypes = [c_char_p, c_uint64, c_char_p, P, P, P, c_uint64]
    lib.ref_materialize.argtypes = [c_char_p, c_uint64, P, P, P, P, P, P, P, P, P, c_int, POINTER(c_uint64)]
    lib.ref_run.argtypes = [P, c_int, c_uint64, c_char_p, P, c_uint64, P, P, P, P]
    lib.ref_bench_sweep.restype = c_double
    lib.ref_bench_sweep.argtypes = [P, c_int, c_uint64, c_uint64, P, c_int, c_int, POINTER(c_uint64),
                                    POINTER(c_double)]
    lib.ref_estimate_rows.argtypes = [P, P, c_uint64, c_uint64, c_uint64, c_uint64, c_int, P, P]
    lib.ref_run_jobs.argtypes = [P, c_int, c_int, c_uint64, c_uint64, c_int, c_uint64, P, P, P, P, P]
    lib.ref_run_sweep.argtypes = [P, c_int, c_int, P, c_int, c_char_p, c_uint64]
    lib.ref_timeline.argtypes = [P, c_int, c_uint64, c_char_p, c_uint64]
    lib.ref_logs.argtypes = [P, c_int, c_uint64, c_char_p, c_uint64, c_char_p, c_uint64]
    return lib


ref_config_dtype = np.dtype([
    ("policy", "<i4"), ("estimator", "<i4"), ("mode", "<i4"), ("rr_apply_preconditions", "<i4"),
    ("max_smact", "<f8"), ("has_min_free", "<i4"), ("min_free", "<u8"), ("safety_margin", "<u8"),
    ("monitor_window", "<f8"), ("gpu_count", "<i4"), ("gpu_capacity", "<u8"), ("alloc_block", "<u8"),
    ("estimator_seed", "<u8"), ("estimator_k", "<u8"), ("estimator_samples", "<u8"),
    ("mig_count", "<i4"), ("mig_reserved", "<i4"), ("mig_fractions", "<f8", (8,)), ("sample_interval", "<f8"),
    ("log_flags", "<i4"), ("log_reserved", "<i4"),
], align=True)

ref_task_out_dtype = np.dtype([
    ("submit", "<f8"), ("first_attempt", "<f8"), ("final_dispatch", "<f8"), ("complete", "<f8"),
    ("first_crash", "<f8"), ("last_crash", "<f8"), ("executed", "<f8"), ("n_attempts", "<u4"),
    ("ooms", "<u4"), ("gpu0", "<i4"), ("gpu1", "<i4"),
], align=True)

ref_trace_out_dtype = np.dtype([
    ("trace_total_time", "<f8"), ("avg_wait", "<f8"), ("avg_exec", "<f8"), ("avg_jct", "<f8"),
    ("energy_mj", "<f8"), ("last_complete", "<f8"), ("first_submit", "<f8"), ("oom_count", "<i4"),
    ("n_tasks", "<i4"),
], align=True)


def ref_config(policy="magm", estimator="none", mode="mps", rr_pre=False, max_smact=0.8, min_free=None,
               margin=2 * GiB, window=60.0, gpu_count=4, capacity=40 * GiB, block=512 * MiB,
               est_seed=11, est_k=5, est_samples=4000, mig=(), sample_interval=0.0, log_flags=0):
    c = np.zeros(1, ref_config_dtype)
    c["log_flags"] = log_flags
    c["sample_interval"] = sample_interval
    c["mig_count"] = len(mig)
    c["mig_fractions"][0, : len(mig)] = mig
    c["policy"] = POLICY[policy]
    c["estimator"] = ESTIMATOR[estimator]
    c["mode"] = MODE[mode]
    c["rr_apply_preconditions"] = int(rr_pre)
    c["max_smact"] = max_smact
    c["has_min_free"] = int(min_free is not None)
    c["min_free"] = min_free or 0
    c["safety_margin"] = margin
    c["monitor_window"] = window
    c["gpu_count"] = gpu_count
    c["gpu_capacity"] = capacity
    c["alloc_block"] = block
    c["estimator_seed"] = est_seed
    c["estimator_k"] = est_k
    c["estimator_samples"] = est_samples
    return c


def replay_config_from(c):
    """The carma_replay_config equivalent of a ref config row."""
    from paper_2508_19073_b200 import abi
    r = np.zeros(1, abi.replay_config_dtype)
    for f in ("policy", "mode", "gpu_count", "rr_apply_preconditions", "max_smact", "monitor_window",
              "gpu_capacity", "alloc_block"):
        r[f] = c[f]
    r["min_free"] = c["min_free"] if c["has_min_free"][0] else 0
    r["p_idle_w"], r["p_max_w"], r["p_boost_w"], r["boost_threshold"] = 55.0, 400.0, 30.0, 0.9
    r["oom_startup_delay"] = 5.0
    r["sample_interval"] = c["sample_interval"]
    r["log_flags"] = c["log_flags"]
    if int(c["mode"][0]) == abi.MODE["mig"]:
        n = int(c["mig_count"][0])
        fr = np.ascontiguousarray(c["mig_fractions"][0, :n], np.float64)
        abi.check(abi.lib.carma_mig_layout(fr.ctypes.data if n else None, n, r.ctypes.data))
    return r


def ref_run(ref, cfg, mix=None, seed=1, path=None, cap=1 << 20):
    tout = np.zeros(cap, ref_task_out_dtype)
    rout = np.zeros(1, ref_trace_out_dtype)
    g = int(cfg["gpu_count"][0])
    ge = np.zeros(g)
    gs = np.zeros(g)
    gp = np.zeros(g, np.uint64)
    rc = ref.ref_run(_ptr(cfg), MIX[mix] if mix else -1, seed, path.encode() if path else None,
                     _ptr(tout), cap, _ptr(rout), _ptr(ge), _ptr(gs), _ptr(gp))
    if rc != 0:
        raise RuntimeError(ref.ref_last_error().decode())
    n = int(rout["n_tasks"][0])
    return tout[:n], rout[0], ge, gs, gp


def oracle_replay(olib, cfg, tasks):
    from paper_2508_19073_b200 import abi
    n = len(tasks)
    tout = np.zeros(n, abi.task_result_dtype)
    tr = np.zeros(1, abi.trace_result_dtype)
    g = np.zeros(int(cfg["gpu_count"][0]), abi.gpu_result_dtype)
    tasks = np.ascontiguousarray(tasks)
    rc = olib.oracle_replay(_ptr(cfg), _ptr(tasks), n, _ptr(tout), _ptr(tr), _ptr(g))
    return rc, tout, tr[0], g


def oracle_predict(olib, m, raw, k=None):
    raw = np.ascontiguousarray(raw, np.float64)
    q = len(raw)
    k = k or m.k
    b = np.zeros(q, np.int32)
    by = np.zeros(q, np.uint64)
    d2 = np.zeros((q, k))
    idx = np.zeros((q, k), np.int64)
    pts = np.ascontiguousarray(m.points)
    rc = olib.oracle_knn_predict(_ptr(m.lo), _ptr(m.hi), _ptr(pts), _ptr(m.labels), len(m.labels), k,
                                 m.bucket_range, _ptr(raw), q, _ptr(b), _ptr(by), _ptr(d2), _ptr(idx))
    assert rc == 0
    return b, by, d2, idx


def ref_estimate_rows(ref, rows, family, samples=4000, est_seed=11, k=5, threads=None):
    """The reference's estimate_learned over feature rows (abi.feature_row_dtype),
    per-row family, models as provision_estimators trains them; host threads."""
    rows = np.ascontiguousarray(rows)
    family = np.ascontiguousarray(family, np.int8)
    n = len(rows)
    b = np.zeros(n, np.int32)
    by = np.zeros(n, np.uint64)
    rc = ref.ref_estimate_rows(_ptr(rows), _ptr(family), n, samples, est_seed, k, threads or os.cpu_count() or 1,
                               _ptr(b), _ptr(by))
    if rc != 0:
        raise RuntimeError(ref.ref_last_error().decode())
    return b, by


def ref_run_jobs(ref, cfgs, mix, seed0, n_seeds, tasks_per_trace, threads=None):
    """run_simulation of every (config, seed) job (job = c * n_seeds + s)."""
    cfgs = np.ascontiguousarray(cfgs, ref_config_dtype)
    nj = len(cfgs) * n_seeds
    g = int(cfgs["gpu_count"].max())
    assert (cfgs["gpu_count"] == g).all()
    tout = np.zeros(nj * tasks_per_trace, ref_task_out_dtype)
    rout = np.zeros(nj, ref_trace_out_dtype)
    ge, gs = np.zeros(nj * g), np.zeros(nj * g)
    gp = np.zeros(nj * g, np.uint64)
    rc = ref.ref_run_jobs(_ptr(cfgs), len(cfgs), MIX[mix], seed0, n_seeds, threads or os.cpu_count() or 1,
                          tasks_per_trace, _ptr(tout), _ptr(rout), _ptr(ge), _ptr(gs), _ptr(gp))
    if rc != 0:
        raise RuntimeError(ref.ref_last_error().decode())
    return tout, rout, ge, gs, gp
