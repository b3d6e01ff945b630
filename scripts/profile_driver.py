"""Small single-purpose drivers for ncu captures (one GPU).

  python scripts/profile_driver.py replay --traces 20000 --policies magm,rr
  python scripts/profile_driver.py knn --rows 4194304 [--format rows|bitpacked]

Each runs the workload `--reps` times (default 2) so `ncu -k regex:<kernel> -s <n> -c 1`
can skip the first launch.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_19073_b200 as cb  # noqa: E402
from paper_2508_19073_b200 import abi  # noqa: E402


def replay(args):
    pols = args.policies.split(",")
    lists = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in range(1, args.traces + 1)]
    tasks = np.concatenate(lists)
    offs = np.concatenate([[0], np.cumsum([len(t) for t in lists])]).astype(np.uint64)
    cfgs = np.concatenate([cb.make_config(cb.PolicyConfig(policy=p, max_smact=0.8), cb.SimConstants()) for p in pols])
    jobs = np.zeros(args.traces * len(pols), abi.job_dtype)
    jobs["trace"] = np.tile(np.arange(args.traces, dtype=np.uint32), len(pols))
    jobs["config"] = np.repeat(np.arange(len(pols), dtype=np.uint32), args.traces)
    plan = cb.ReplayPlan(cfgs, tasks, offs, jobs)
    import ctypes
    km, rm = ctypes.c_double(), ctypes.c_double()
    for _ in range(args.reps):
        plan.run()
        abi.check(abi.lib.carma_replay_plan_timing(plan._h, ctypes.byref(km), ctypes.byref(rm)))
        print(f"replay {len(jobs)} jobs: tier0 {km.value:.2f} ms, run {rm.value:.2f} ms, "
              f"stats {plan.stats()}", flush=True)
    res = plan.results(tasks=False)
    print("events", int(res.traces["events"].sum()), "status!=0", int((res.traces["status"] != 0).sum()))


def knn(args):
    import torch
    ds = [cb.generate_synthetic_dataset(f, args.rows // 2, s) for f, s in ((1, 2024), (2, 2025))]
    rows = np.concatenate([d.rows for d in ds])
    fam = np.concatenate([np.full(args.rows // 2, 1, np.int8), np.full(args.rows // 2, 2, np.int8)])
    k = cb.GpuKnn(0)
    k.set_model(cb.fit_knn(1, 4000, 112, 5))
    k.set_model(cb.fit_knn(2, 4000, 213, 5))
    fmt, fam_ptr = 0, None
    if args.format == "bitpacked":  # the bench's device path (36 B rows, family inside)
        words, schema = cb.pack_features_bits(rows, fam)
        abi.check(abi.lib.carma_knn_set_bit_schema(k.handle, schema.ctypes.data))
        d_rows = torch.from_numpy(words.view(np.uint8)).cuda()
        fmt = abi.ROWS_BITPACKED
    else:
        d_rows = torch.from_numpy(rows.view(np.uint8)).cuda()
        d_fam = torch.from_numpy(fam).cuda()
        fam_ptr = d_fam.data_ptr()
    b = torch.empty(len(rows), dtype=torch.int32, device="cuda")
    by = torch.empty(len(rows), dtype=torch.int64, device="cuda")
    import ctypes
    sm, pm = ctypes.c_double(), ctypes.c_double()
    for _ in range(args.reps):
        abi.check(abi.lib.carma_knn_predict_device(k.handle, d_rows.data_ptr(), fmt, fam_ptr, 1, len(rows),
                                                   b.data_ptr(), by.data_ptr(), None, None, None))
        abi.check(abi.lib.carma_knn_last_timing(k.handle, ctypes.byref(sm), ctypes.byref(pm)))
        print(f"knn {len(rows)} rows: search {sm.value:.2f} ms pipeline {pm.value:.2f} ms stats {k.last_stats()}",
              flush=True)
    fn = getattr(abi.lib, "carma_debug_knn_chunk_times", None)
    if fn is not None:
        fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
        out = np.zeros(16, np.float32)
        n = ctypes.c_int32()
        abi.check(fn(k.handle, out.ctypes.data, 16, ctypes.byref(n)))
        print("chunk search windows (ms from pipeline start):",
              [(round(float(out[2 * c]), 3), round(float(out[2 * c + 1]), 3)) for c in range(min(n.value, 8))])


def nn(args):
    """The neural GPUMemNet ensemble (carma_nn_*) over the bench's bit-packed
    CNN + Transformer rows."""
    import torch
    from paper_2508_19073_b200 import gpumemnet as gm
    ds = [cb.generate_synthetic_dataset(f, args.rows // 2, s) for f, s in ((1, 2024), (2, 2025))]
    rows = np.concatenate([d.rows for d in ds])
    fam = np.concatenate([np.full(args.rows // 2, 1, np.int8), np.full(args.rows // 2, 2, np.int8)])
    net = gm.GpuMemNet(0)
    models = gm.load_default_models(gm.ARCH_TRANSFORMER if args.arch == "transformer" else gm.ARCH_MLP)
    for f in (1, 2):
        net.set_model(models[f])
    net.set_path(args.path)
    words, schema = cb.pack_features_bits(rows, fam)
    net.set_bit_schema(schema)
    d_rows = torch.from_numpy(words.view(np.uint8)).cuda()
    b = torch.empty(len(rows), dtype=torch.int32, device="cuda")
    by = torch.empty(len(rows), dtype=torch.int64, device="cuda")
    for _ in range(args.reps):
        net.predict_device(d_rows, abi.ROWS_BITPACKED, len(rows), b, by)
        print(f"nn {len(rows)} rows: {net.last_timing()}", flush=True)


def fused(args):
    import ctypes
    m = cb.materialize_trace(cb.generate_uniform_trace(args.tasks, 3.0, 7))
    cfg = cb.make_config(cb.PolicyConfig(policy="magm", max_smact=0.8, monitor_window=5.0),
                         cb.SimConstants(gpu_count=64))
    knn = cb.GpuKnn(0)
    for f in (1, 2):
        knn.set_model(cb.fit_knn(f, 4000, 11 + 101 * f, 5))
    fr = cb.FusedReplay(m, cfg, knn, 0)
    import torch
    for _ in range(args.reps):
        t = time.perf_counter()
        fr.run()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        km, rm = ctypes.c_double(), ctypes.c_double()
        abi.check(abi.lib.carma_replay_plan_timing(fr.plan._h, ctypes.byref(km), ctypes.byref(rm)))
        print(f"fused {args.tasks} tasks: wall {dt * 1e3:.1f} ms, replay run {rm.value:.1f} ms "
              f"(tier0 {km.value:.1f}), stats {fr.plan.stats()}", flush=True)
    r = fr.results().traces[0]
    print("oom", r["oom_count"], "events", r["events"], "makespan", r["trace_total_time"], "status", r["status"])
    if hasattr(abi.lib, "carma_debug_replay_prof"):  # REPLAY_PROF builds: cycles per event-loop region
        v = (ctypes.c_ulonglong * 16)()
        abi.lib.carma_debug_replay_prof(v)
        names = ["next_event", "integrate", "handle", "refresh", "decide", "place", "push", "events"]
        tot = sum(v[:7])
        for n, x in zip(names, v):
            print(f"  {n:10s} {x:16d}" + (f"  {100 * x / tot:5.1f}%  {x / max(v[7], 1):8.1f} cyc/event" if n != "events" else ""))
        print(f"  heap pops {v[9]}, mean heap size {v[8] / max(v[9], 1):.1f}; decides {v[11]}, with a head {v[10]}; "
              f"refreshes {v[13]}, mean residents on touched GPUs {v[12] / max(v[13], 1):.2f}, "
              f"mean ring entries {v[14] / max(v[13], 1):.2f}; pushes {v[15]}")
        u = (ctypes.c_ulonglong * 8)()
        abi.lib.carma_debug_replay_sub(u)
        for n, x in zip(["refresh_gpu", "affected+sort", "re-push loop", "decide gate/head", "decide inputs",
                         "decide pick"], u):
            print(f"    {n:16s} {x / max(v[7], 1):8.1f} cyc/event")


def scoring(args):
    """The bench's scoring workload (bench.scoring_bench) once per rep."""
    import torch
    sys.path.insert(0, ROOT)
    import bench

    class One:
        n = 1

        def barrier(self):
            pass

        def max(self, x):
            return x

    r = bench.scoring_bench(abi, cb, 0, torch.cuda.current_stream(), 1, args.reps, One())
    print(f"scoring: {r['ms_per_step']:.3f} ms, {r['roofline']['achieved']:.0f} GB/s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=("replay", "knn", "fused", "scoring", "nn"))
    ap.add_argument("--tasks", type=int, default=1_000_000)
    ap.add_argument("--traces", type=int, default=20000)
    ap.add_argument("--policies", default="exclusive,rr,magm,lug")
    ap.add_argument("--rows", type=int, default=1 << 22)
    ap.add_argument("--format", choices=("rows", "bitpacked"), default="bitpacked")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--arch", choices=("mlp", "transformer"), default="mlp")
    ap.add_argument("--path", type=int, default=0, help="neural MLP: 0 auto, 1 tcgen05, 2 CUDA cores")
    a = ap.parse_args()
    {"replay": replay, "knn": knn, "fused": fused, "scoring": scoring, "nn": nn}[a.what](a)
