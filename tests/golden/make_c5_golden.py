"""Writes tests/golden/c5_ref.json: the UNMODIFIED reference (oracle/_ref) run
on the FULL c5 workload (BASELINE configs[4]): 10^6 arrivals, uniform catalog,
exponential gaps of mean 3 s, seed 7, 64 simulated GPUs, MAGM u=0.8, W=5 s,
estimator learned (and the estimator-none twin, which exercises OOM recovery).

Each run is one single-threaded run_simulation (runner.cpp:40-147) over the
#carma-trace v1 file; ~20-25 min of CPU each, so the two runs go
in parallel processes. The golden holds the report scalars and per-GPU results
as IEEE bit patterns, a SHA-256 digest per task field (trace row order) and a
sparse sample of full task records, so tests/test_gpu_fullsize.py can assert
bit-equality of every task of the GPU run without shipping 10^6 records.

TEST INFRASTRUCTURE ONLY. Needs oracle/_ref/libcarma_ref.so (built from
/root/reference by oracle/Makefile).

  python tests/golden/make_c5_golden.py [n_tasks]
"""
from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

N_DEFAULT = 1_000_000
SAMPLE_STRIDE = 4999


def trace_path(n: int) -> str:
    import paper_2508_19073_b200 as cb
    path = os.path.join(tempfile.gettempdir(), f"c5_{n}.trace")
    if not os.path.exists(path):
        cb.save_trace(cb.generate_uniform_trace(n, 3.0, 7), path)
    return path


def _run(args):
    est, n, path = args
    from oracle_bind import load_ref, ref_config, ref_run
    import fullsize
    ref = load_ref()
    cfg = ref_config(policy="magm", estimator=est, gpu_count=64, window=5.0)
    t = time.perf_counter()
    tout, rout, ge, gs, gp = ref_run(ref, cfg, path=path, cap=n)
    dt = time.perf_counter() - t
    rec = fullsize.ref_tasks_canonical(tout)
    return est, {
        "seconds": dt,
        "report": fullsize.bits_of({k: float(rout[k]) for k in ("trace_total_time", "avg_wait", "avg_exec",
                                                                 "avg_jct", "energy_mj", "last_complete",
                                                                 "first_submit")}),
        "oom_count": int(rout["oom_count"]),
        "n_tasks": int(rout["n_tasks"]),
        "gpu_energy_j": fullsize.hex_f64(ge), "gpu_mean_smact": fullsize.hex_f64(gs),
        "gpu_peak_used": [int(x) for x in gp],
        "task_digest": fullsize.digest_fields(rec),
        "sample_stride": SAMPLE_STRIDE,
        "sample": fullsize.sample_records(rec, SAMPLE_STRIDE),
    }


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else N_DEFAULT
    path = trace_path(n)
    with open(path, "rb") as f:
        tsha = hashlib.sha256(f.read()).hexdigest()
    with mp.get_context("spawn").Pool(2) as pool:
        runs = dict(pool.map(_run, [("learned", n, path), ("none", n, path)]))
    out = {"workload": f"c5: {n} arrivals, uniform catalog, exp gaps mean 3 s, seed 7; 64 GPUs, MAGM u=0.8, "
                       "W=5 s, MPS; estimator learned (provision_estimators: 4000 samples, k=5, seed 11) and none",
           "n_tasks": n, "trace_sha256": tsha, "generator": "tests/golden/make_c5_golden.py",
           "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t"),
           "runs": runs}
    dst = os.path.join(HERE, "c5_ref.json" if n == N_DEFAULT else f"c5_ref_{n}.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(dst, {k: (v["seconds"], v["oom_count"]) for k, v in runs.items()})


if __name__ == "__main__":
    main()
