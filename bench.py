#!/usr/bin/env python
"""Benchmark of the CARMA hot path on B200.

Headline (BASELINE.json configs[1]): GPUMemNet estimates/s — the reference's
k-NN memory-bin classifier over the 16,777,216-row CNN + Transformer batch
(generate_synthetic_dataset(CNN, 8388608, 2024) + (Transformer, 8388608, 2025)),
routed per family to the models provision_estimators trains (seeds 112, 213).
The paper's neural GPUMemNet ensembles (MLP on tcgen05, Transformer on CUDA
cores) run over the same rows (line key "neural").
Second half of the metric (configs[3], line key "replay", printed last so the
driver's stdout tail keeps it): trace-replay placed tasks/s for the policy
sweep t90 seeds 1..100000 x {exclusive, rr, magm, lug}.

Scaling is STRONG: the 16.7M rows and the 400k replay jobs are the whole
job; rank r of N takes the contiguous shard dist.balanced_shards gives it
(rows by count, jobs by task count) with no data-path collective, and
value = all units / max-over-ranks time. configs[4] (one 10^6-task trace),
the scoring kernel and the small configs run at N = 1 only (a single trace
does not shard; replicas would add nothing).

The full measurement record goes to gpurun_out/bench_detail.json; stdout
carries one compact JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl carma|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KNN_ROWS_PER_FAMILY = 8_388_608
KNN_SEEDS = {1: 2024, 2: 2025}          # query datasets (family -> seed)
MODEL_SEEDS = {1: 11 + 101, 2: 11 + 202}  # provision_estimators: estimator_seed + 101*family
SWEEP_TRACES = 100_000
SWEEP_POLICIES = ("exclusive", "rr", "magm", "lug")
ALG_BYTES_PER_ESTIMATE = 164       # 19 f64 in + i32 bucket + u64 bytes
ALG_BYTES_PER_TASK = 80            # 45 B in + 35 B out per placed task
FLOPS_PER_EVAL = 58                # 19 x (sub, mul, add) + 1 weight mul, FMA-free
FLOPS_PER_F32_EVAL = 48            # fp32 pre-filter: 16 dims x (sub + fma)
FEATURE_ROW_BYTES = 136
# host-buffer calls re-encode every other chunk of 136-B rows (+ 1-B family)
# into 40-B compact rows on host threads while the copy engine ships the
# other chunks raw, so PCIe and host memory bandwidth overlap
# (csrc/host/stage.cpp); h2d_bytes_per_step is the call's own count
E2E_API = ("{fn} (pinned 136-B carma_feature_row + family in, bucket + bytes out; half the chunks re-encoded to "
           "40-B compact rows by the host thread pool inside the call, overlapped with the raw chunks' H2D)")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def host_cpus() -> dict:
    import psutil
    return {"logical_cpus": psutil.cpu_count(logical=True), "physical_cores": psutil.cpu_count(logical=False)}


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None

    def __enter__(self):
        self.t_busy = time.time()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(1.0)  # nvidia-smi needs ~0.5 s before its first sample
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def mark(self, name: str) -> None:
        setattr(self, name, time.time())

    def summary(self):
        """Median SM clock over samples inside [t_begin, t_end] (the timed
        region); if the region is shorter than the sampling period, the
        samples of the surrounding busy window (warm-up + timed) are used."""
        import datetime
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except OSError:
            rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        parsed = []
        for r in rows:
            try:
                ts = datetime.datetime.strptime(r[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
                parsed.append((ts, float(r[2]), float(r[3]), [n for n, v in zip(names, r[6:10])
                                                              if v.strip().lower() == "active"]))
            except (ValueError, IndexError):
                continue
        t0, t1 = getattr(self, "t_begin", 0.0), getattr(self, "t_end", 1e30)
        inside = [p for p in parsed if t0 - 0.05 <= p[0] <= t1 + 0.05]
        window = "timed region"
        if not inside:
            w0 = getattr(self, "t_busy", t0)
            inside = [p for p in parsed if w0 <= p[0] <= t1 + 0.2]
            window = "warm-up + timed (timed region shorter than the 100 ms sampling period)"
        sm = [p[1] for p in inside]
        reasons = sorted({n for p in inside for n in p[3]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max((p[2] for p in parsed), default=None),
                "reasons": reasons, "samples": len(sm), "window": window}


# ------------------------------------------------------------------ dist
class Dist:
    """One process per GPU (torchrun); NCCL only for the barrier and the
    max-over-ranks of the timings (no data-path collective)."""

    def __init__(self, gpus: int, backend: str = "nccl"):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.n = max(self.world, 1)
        self.backend = backend
        if gpus and self.world > 1 and gpus != self.world:
            log(f"warning: --gpus {gpus} but WORLD_SIZE {self.world}")
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            if backend == "nccl":
                import torch
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ------------------------------------------------------------------ data
def knn_inputs(cb, dev: int = 0):
    """The c2 batch: 8,388,608 CNN rows (seed 2024) + 8,388,608 Transformer rows
    (seed 2025), from the device generator (carma_dataset_generate_device,
    bit-identical to the host / reference generator: tests/test_gpu_dataset.py)
    and copied to host memory once (the e2e arms start from host rows)."""
    import torch
    from paper_2508_19073_b200 import abi
    n = KNN_ROWS_PER_FAMILY
    rb = abi.feature_row_dtype.itemsize
    d_rows = torch.empty(2 * n * rb, dtype=torch.uint8, device=f"cuda:{dev}")
    for k, f in enumerate(KNN_SEEDS):
        cb.generate_synthetic_dataset_device(f, n, KNN_SEEDS[f], d_rows[k * n * rb:(k + 1) * n * rb], device=dev)
    torch.cuda.synchronize(dev)
    rows = d_rows.cpu().numpy().view(abi.feature_row_dtype)
    del d_rows
    fam = np.concatenate([np.full(KNN_ROWS_PER_FAMILY, 1, np.int8), np.full(KNN_ROWS_PER_FAMILY, 2, np.int8)])
    return rows, fam


def sweep_inputs(cb, n_traces: int):
    """t90 seeds 1..n_traces, materialised once; jobs = traces x 4 policies
    (job = policy * n_traces + trace)."""
    lists = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in range(1, n_traces + 1)]
    tasks = np.concatenate(lists)
    offs = np.concatenate([[0], np.cumsum([len(t) for t in lists])]).astype(np.uint64)
    cfgs = np.concatenate([cb.make_config(cb.PolicyConfig(policy=p, max_smact=0.8), cb.SimConstants())
                           for p in SWEEP_POLICIES])
    from paper_2508_19073_b200 import abi
    jobs = np.zeros(n_traces * len(SWEEP_POLICIES), abi.job_dtype)
    jobs["trace"] = np.tile(np.arange(n_traces, dtype=np.uint32), len(SWEEP_POLICIES))
    jobs["config"] = np.repeat(np.arange(len(SWEEP_POLICIES), dtype=np.uint32), n_traces)
    return cfgs, tasks, offs, jobs


def shard_jobs(tasks, offs, jobs, b: int, e: int):
    """The replay inputs of jobs [b, e): only the traces they reference,
    renumbered (what a rank uploads)."""
    sub = jobs[b:e].copy()
    used = np.unique(sub["trace"])
    remap = np.zeros(len(offs) - 1, np.uint32)
    remap[used] = np.arange(len(used), dtype=np.uint32)
    sub["trace"] = remap[sub["trace"]]
    o = offs.astype(np.int64)
    lens = o[used + 1] - o[used]
    idx = np.concatenate([np.arange(o[t], o[t + 1]) for t in used]) if len(used) else np.zeros(0, np.int64)
    return tasks[idx], np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64), sub


def profile_traffic(*names):
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(path))
    except (OSError, ValueError):
        return None
    for n in names:
        if n in t:
            return t[n]
    return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def knn_config(n: int, rows_shard: int) -> dict:
    return {"workload": "c2: GPUMemNet k-NN ensemble over 8,388,608 CNN (seed 2024) + 8,388,608 Transformer "
                        "(seed 2025) feature vectors in total; models = provision_estimators (4000 samples, k=5, "
                        "seeds 112/213)",
            "rows_total": 2 * KNN_ROWS_PER_FAMILY, "rows_per_gpu": rows_shard, "row_format": "carma_feature_row (136 B)",
            "parallelism": f"dp{n}: contiguous row shards, no collective",
            "l2": "inputs 2.28 GB > 126 MB L2 (no flush needed)"}


def nn_tile_flops(m) -> tuple:
    """(executed tensor-pipe flops per 128-row tile, useful dense flops per row)
    of a GPUMemNet ensemble on the kernel's layout (csrc/cuda/gpumemnet.cu):
    members sorted by depth, layer l over the running prefix (N = 8 alive_l,
    K = 8 alive_{l-1}, padded to 16; layer 0 K = 32), the head passes (K = 64),
    3 bf16 activation parts, 2*M*N*K flops per MMA (M = 128)."""
    L = max(m.depth)
    alive = [sum(1 for d in m.depth if d > l) for l in range(L)]
    pad = lambda x: (x + 15) // 16 * 16  # noqa: E731
    cp = (m.classes + 7) // 8 * 8
    mpp = min(m.members, 128 // cp)
    passes = [min(mpp, m.members - p * mpp) for p in range((m.members + mpp - 1) // mpp)]
    head_n = sum(pad(k * cp) for k in passes)
    mnk = pad(8 * alive[0]) * 32 + sum(pad(8 * alive[l]) * pad(8 * alive[l - 1]) for l in range(1, L))
    executed = 3 * 2 * 128 * (mnk + head_n * 64)
    useful = 0
    for d, w in zip(m.depth, m.width):
        fan = 19
        for x in w:
            useful += 2 * fan * x
            fan = x
        useful += 2 * fan * m.classes
    return executed, useful


def timed_device_steps(step, stream, warmup: int, steps: int, d, clk=None):
    """W warm-up steps, barrier + sync, K steps bracketed by CUDA events on
    `stream`, sync + barrier; returns max-over-ranks ms per step."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    if clk:
        clk.mark("t_begin")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.mark("t_end")
    d.barrier()
    return d.max(e0.elapsed_time(e1) / steps)


def timed_host_steps(step, warmup: int, steps: int, d):
    """Host API calls (synchronous, host buffers in and out): wall clock per
    step, max over ranks."""
    for _ in range(warmup):
        step()
    d.barrier()
    t = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t) / steps
    d.barrier()
    return d.max(dt)


# ------------------------------------------------------------ reference arm
def ref_lib():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import load_ref
    return load_ref()


def cpu_knn_baseline(ref, threads: int, target_s: float = 10.0):
    """The reference predict (estimate_learned, oracle/_ref) on `threads` host
    threads over CNN (seed 2024) and Transformer (seed 2025) rows, sized for
    ~target_s of wall time. Returns (estimates/s, sample description)."""
    import ctypes
    n = 50_000
    ck = ctypes.c_uint64()
    # warm the model cache + calibrate
    t = ref.ref_bench_predict(1, 4000, MODEL_SEEDS[1], 5, 4000, KNN_SEEDS[1], threads, 1, ctypes.byref(ck))
    rate = 4000 / max(t, 1e-6)
    reps = max(1, int(rate * target_s / 2 / n))
    tot, rows = 0.0, 0
    for f in (1, 2):
        s = ref.ref_bench_predict(f, 4000, MODEL_SEEDS[f], 5, n, KNN_SEEDS[f], threads, reps, ctypes.byref(ck))
        if s < 0:
            raise RuntimeError(ref.ref_last_error().decode())
        tot += s
        rows += n * reps
    return rows / tot, f"{reps} x {n} CNN (seed 2024) + {reps} x {n} Transformer (seed 2025) rows; " \
                       f"models trained as provision_estimators (seeds 112, 213)"


def cpu_sweep_baseline(ref, threads: int, target_s: float = 10.0):
    """The reference run_simulation pool (run_sweep shape) over t90 seeds x 4 policies."""
    import ctypes
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import POLICY, ref_config
    cfg = ref_config(policy="magm", max_smact=0.8)
    pols = np.array([POLICY[p] for p in SWEEP_POLICIES], np.int32)
    placed, esum = ctypes.c_uint64(), ctypes.c_double()
    n0 = max(8, threads)
    t = ref.ref_bench_sweep(cfg.ctypes.data, 0, 1, n0, pols.ctypes.data, len(pols), threads,
                            ctypes.byref(placed), ctypes.byref(esum))
    rate = n0 * len(pols) / max(t, 1e-6)
    n = max(n0, int(rate * target_s / len(pols)))
    t = ref.ref_bench_sweep(cfg.ctypes.data, 0, 1, n, pols.ctypes.data, len(pols), threads,
                            ctypes.byref(placed), ctypes.byref(esum))
    if t < 0:
        raise RuntimeError(ref.ref_last_error().decode())
    return placed.value / t, f"t90 seeds 1..{n} x {{exclusive, rr, magm, lug}} ({n * len(pols)} runs)", n


def cpu_fused_baseline(ref, n_tasks: int):
    """One reference run_simulation (single-threaded by design, runner.cpp:40)
    on the first n_tasks rows of the c5 trace, loaded from a #carma-trace v1
    file, learned estimator provisioned in-process as the reference does."""
    import paper_2508_19073_b200 as cb
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import ref_config, ref_run
    path = os.path.join(tempfile.mkdtemp(), "c5_prefix.trace")
    cb.save_trace(cb.generate_uniform_trace(n_tasks, 3.0, 7), path)
    cfg = ref_config(policy="magm", estimator="learned", gpu_count=64, window=5.0)
    t = time.perf_counter()
    ref_run(ref, cfg, path=path, cap=n_tasks)
    dt = time.perf_counter() - t
    return n_tasks / dt, (f"first {n_tasks} rows of the c5 trace, one run_simulation on 1 core "
                          f"(reference cost grows superlinearly with trace length, SURVEY F7)")


def c5_golden():
    try:
        return json.load(open(os.path.join(ROOT, "tests", "golden", "c5_ref.json")))
    except (OSError, ValueError):
        return None


def run_reference(args, d: Dist):
    """The reference's own CPU implementation of the path (oracle/_ref, the
    unmodified library) on all host threads; rank 0 only."""
    if d.rank != 0:
        return
    ref = ref_lib()
    threads = os.cpu_count() or 1
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcarma_ref.so not built"}))
        return
    steps = []
    for _ in range(args.warmup + args.steps):
        rate, sample = cpu_knn_baseline(ref, threads, target_s=4.0)
        steps.append(rate)
    vals = steps[args.warmup:]
    value = statistics.median(vals)
    srate, ssample, _ = cpu_sweep_baseline(ref, threads, target_s=4.0)
    cpus = host_cpus()
    line = {
        "impl": "reference", "metric": "GPUMemNet estimates/sec (k-NN, CNN+Transformer ensemble)",
        "value": value, "unit": "estimates/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * 2 * KNN_ROWS_PER_FAMILY / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": knn_config(1, 2 * KNN_ROWS_PER_FAMILY),
        "cpu_baseline": {"value": value, "unit": "estimates/s", "cores": threads, "kind": "reference",
                         "sample": sample, **cpus},
        "e2e": {"value": value, "unit": "estimates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "replay": {"value": srate, "unit": "placed tasks/s", "cores": threads, "sample": ssample},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ stage 1
def knn_stage(abi, cb, dev, stream, args, d, rows, fam, b, e):
    """The k-NN GPUMemNet over this rank's contiguous shard [b, e) of the c2
    batch: device-resident 136-B feature rows (value) and the host API from
    pinned 136-B rows (e2e)."""
    import ctypes

    import torch
    Q = e - b
    knn = cb.GpuKnn(dev)
    for f in (1, 2):
        knn.set_model(cb.fit_knn(f, 4000, MODEL_SEEDS[f], 5))
    h_rows = torch.from_numpy(rows[b:e].view(np.uint8).reshape(-1)).pin_memory()
    h_fam = torch.from_numpy(fam[b:e]).pin_memory()
    d_rows = h_rows.to("cuda")
    d_fam = h_fam.to("cuda")
    d_b = torch.empty(Q, dtype=torch.int32, device="cuda")
    d_by = torch.empty(Q, dtype=torch.int64, device="cuda")
    search_ms, pipe_ms = [], []
    sm, pm = ctypes.c_double(), ctypes.c_double()

    def step():
        abi.check(abi.lib.carma_knn_predict_device(knn.handle, d_rows.data_ptr(), abi.ROWS_FEATURES,
                                                   d_fam.data_ptr(), 1, Q, d_b.data_ptr(), d_by.data_ptr(),
                                                   None, None, abi.stream_arg(stream)))
        abi.check(abi.lib.carma_knn_last_timing(knn.handle, ctypes.byref(sm), ctypes.byref(pm)))
        search_ms.append(sm.value)
        pipe_ms.append(pm.value)

    with Clocks(dev) as clk:
        ms = timed_device_steps(step, stream, args.warmup, args.steps, d, clk)
    clocks = clk.summary()
    search_ms, pipe_ms = search_ms[args.warmup:], pipe_ms[args.warmup:]
    b_dev = d_b.cpu().numpy()
    by_dev = d_by.cpu().numpy().view(np.uint64)
    launches, evals = knn.last_stats()
    la_, e64_, e32_ = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    abi.check(abi.lib.carma_knn_last_work(knn.handle, ctypes.byref(la_), ctypes.byref(e64_), ctypes.byref(e32_)))
    visits = e32_.value
    del d_rows, d_fam, d_b, d_by

    # e2e: the drop-in call (carma_knn_predict: pinned 136-B rows + families in,
    # buckets + bytes out; chunked H2D / compute / D2H inside)
    h_rows_np = h_rows.numpy().view(abi.feature_row_dtype)
    h_fam_np = h_fam.numpy()
    h_b = torch.empty(Q, dtype=torch.int32).pin_memory().numpy()
    h_by = torch.empty(Q, dtype=torch.int64).pin_memory().numpy().view(np.uint64)

    def e2e_step():
        abi.check(abi.lib.carma_knn_predict(knn.handle, h_rows_np.ctypes.data, h_fam_np.ctypes.data, 1, Q,
                                            h_b.ctypes.data, h_by.ctypes.data))

    e2e_s = timed_host_steps(e2e_step, max(1, args.warmup - 1), args.steps, d)
    h2d = ctypes.c_uint64()
    abi.check(abi.lib.carma_knn_last_h2d_bytes(knn.handle, ctypes.byref(h2d)))
    assert np.array_equal(h_b, b_dev) and np.array_equal(h_by, by_dev), "host-API and device predictions differ"
    knn_handle = knn  # kept for the fused c5 run
    search_avg = statistics.mean(search_ms)
    f32_flops = visits * FLOPS_PER_F32_EVAL
    achieved = f32_flops / (search_avg * 1e-3)
    fp32, fp64 = ctypes.c_double(), ctypes.c_double()
    abi.check(abi.lib.carma_probe_fp32(dev, ctypes.byref(fp32)))
    abi.check(abi.lib.carma_probe_fp64(dev, ctypes.byref(fp64)))
    N = d.n
    QT = 2 * KNN_ROWS_PER_FAMILY
    out = {
        "value": QT / (ms * 1e-3), "ms_per_step": ms, "clocks": clocks,
        "e2e": {"value": QT / e2e_s, "unit": "estimates/s",
                "h2d_bytes_per_step": int(h2d.value),
                "d2h_bytes_per_step": int(Q * 12),
                "api": E2E_API.format(fn="carma_knn_predict"),
                "host_row_bytes_read": int(Q * (FEATURE_ROW_BYTES + 1)),
                "ms_per_step": e2e_s * 1e3,
                "pcie_gbs": (h2d.value + Q * 12) / e2e_s / 1e9},
        "gpu_launches": int(launches) * args.steps,
        "roofline": {"bound": "fp32", "achieved": achieved / 1e12, "peak": fp32.value / 1e12, "unit": "TFLOP/s",
                     "frac": achieved / fp32.value,
                     "traffic": profile_traffic("knn_search_f32", "knn_search"),
                     "kernel": "knn_search_f32", "kernel_ms": search_avg,
                     "kernel_share_of_step": search_avg / statistics.mean(pipe_ms),
                     "peak_source": "measured: carma_probe_fp32 (FFMA2 issue rate; MEASURED_PEAKS.json has no fp32 "
                                    "figure)",
                     "work": f"{visits} fp32 pre-filter evaluations x {FLOPS_PER_F32_EVAL} flops + {evals} exact "
                             f"fp64 evaluations x {FLOPS_PER_EVAL} flops per launch on this rank",
                     "fp64": {"achieved": evals * FLOPS_PER_EVAL / (search_avg * 1e-3) / 1e12,
                              "peak": fp64.value / 1e12, "unit": "TFLOP/s"},
                     "hbm_gbs": ALG_BYTES_PER_ESTIMATE * Q / (search_avg * 1e-3) / 1e9,
                     "hbm_peak_gbs": peaks().get("hbm_gbs")},
    }
    return out, knn_handle, (h_rows_np, h_fam_np, b_dev)


def neural_stage(abi, cb, dev, stream, args, d, h_rows, h_fam, rows_all, fam_all, b):
    """The paper's neural GPUMemNet ensembles (MLP on tcgen05, Transformer on
    CUDA cores) over the same shard of 136-B rows."""
    import ctypes

    import torch

    from paper_2508_19073_b200 import gpumemnet as gm
    Q = len(h_rows)
    QT = 2 * KNN_ROWS_PER_FAMILY
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import gpumemnet_oracle
    d_rows = torch.from_numpy(h_rows.view(np.uint8).reshape(-1)).to("cuda")
    d_fam = torch.from_numpy(h_fam).to("cuda")
    d_b = torch.empty(Q, dtype=torch.int32, device="cuda")
    d_by = torch.empty(Q, dtype=torch.int64, device="cuda")
    h_b = torch.empty(Q, dtype=torch.int32).pin_memory().numpy()
    h_by = torch.empty(Q, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(Q, min(Q, 4096), replace=False))
    raw = cb.scalar_features(h_rows[idx])
    res = {}
    for arch, key in ((gm.ARCH_MLP, "mlp"), (gm.ARCH_TRANSFORMER, "transformer")):
        models = gm.load_default_models(arch)
        net = gm.GpuMemNet(dev)
        for f in (1, 2):
            net.set_model(models[f])
        kernel_ms, call_ms = [], []

        def step():
            net.predict_device(d_rows, abi.ROWS_FEATURES, Q, d_b, d_by, family=d_fam, default_family=1,
                               stream=stream)
            t = net.last_timing()
            kernel_ms.append(t["kernel_ms"])
            call_ms.append(t["call_ms"])

        ms = timed_device_steps(step, stream, args.warmup, args.steps, d)
        t = net.last_timing()
        kernel_ms, call_ms = kernel_ms[args.warmup:], call_ms[args.warmup:]
        b_dev = d_b.cpu().numpy()

        def e2e_step():
            abi.check(abi.lib.carma_nn_predict(net.handle, h_rows.ctypes.data, h_fam.ctypes.data, 1, Q,
                                               h_b.ctypes.data, h_by.ctypes.data))

        e2e_s = timed_host_steps(e2e_step, 1, args.steps, d)
        h2d = ctypes.c_uint64()
        abi.check(abi.lib.carma_nn_last_h2d_bytes(net.handle, ctypes.byref(h2d)))
        assert np.array_equal(h_b, b_dev), f"{key}: host-API and device-resident neural predictions differ"
        agree = 0
        for f in (1, 2):
            sel = h_fam[idx] == f
            if not sel.any():
                continue
            _, op, ob, _ = gpumemnet_oracle.forward(models[f].spec()[0], models[f].params, raw[sel])
            srt = np.sort(op, axis=1)
            sure = srt[:, -1] - srt[:, -2] > 1e-3
            assert np.array_equal(b_dev[idx][sel][sure], ob[sure]), f"{key}: bins differ from the oracle"
            agree += int(sure.sum())
        k_avg = statistics.mean(kernel_ms)
        r = {"value": QT / (ms * 1e-3), "ms_per_step": ms,
             "e2e": {"value": QT / e2e_s, "unit": "estimates/s", "h2d_bytes_per_step": int(h2d.value),
                     "d2h_bytes_per_step": int(Q * 12), "api": E2E_API.format(fn="carma_nn_predict")},
             "gpu_launches": int(t["launches"]) * args.steps, "kernel_ms": k_avg,
             "kernel_share_of_step": k_avg / statistics.mean(call_ms), "oracle_agreement_rows": agree,
             "holdout_accuracy": {gm.FAMILY_NAMES[f]: models[f].holdout_accuracy for f in (1, 2)}}
        rows_f = {f: int((h_fam == f).sum()) for f in (1, 2)}
        useful = sum(rows_f[f] * nn_tile_flops(models[f])[1] for f in (1, 2))
        if key == "mlp":
            # default path: mlp_ffma (fp32 FFMA on the CUDA cores); the tcgen05
            # path (nn_ensemble) is timed beside it for the record
            import ctypes as _ct
            fp32 = _ct.c_double()
            abi.check(abi.lib.carma_probe_fp32(dev, _ct.byref(fp32)))
            ach = useful / (k_avg * 1e-3) / 1e12
            r["dtype"] = "f32"
            r["roofline"] = {"bound": "fp32", "achieved": ach, "peak": fp32.value / 1e12, "unit": "TFLOP/s",
                             "frac": ach / (fp32.value / 1e12), "traffic": profile_traffic("mlp_ffma"),
                             "kernel": "mlp_ffma",
                             "work": f"algorithmic {useful / 1e9:.1f} GFLOP (dense ensemble math, 2 flops per "
                                     "multiply-add) per launch",
                             "peak_source": "measured: carma_probe_fp32 (FFMA2 issue rate)"}
            net.set_path(1)
            tc_ms = []

            def tc_step():
                net.predict_device(d_rows, abi.ROWS_FEATURES, Q, d_b, d_by, family=d_fam, default_family=1,
                                   stream=stream)
                tc_ms.append(net.last_timing()["kernel_ms"])

            timed_device_steps(tc_step, stream, args.warmup, args.steps, d)
            executed = sum((rows_f[f] + 127) // 128 * nn_tile_flops(models[f])[0] for f in (1, 2))
            tc_k = statistics.mean(tc_ms[args.warmup:])
            peak = peaks().get("bf16_tflops", 2250.0)
            r["tcgen05_path"] = {"kernel": "nn_ensemble", "kernel_ms": tc_k, "value": QT / (tc_k * 1e-3),
                                 "useful_tflops": useful / (tc_k * 1e-3) / 1e12,
                                 "executed_tflops": executed / (tc_k * 1e-3) / 1e12,
                                 "executed_frac_of_bf16_peak": executed / (tc_k * 1e-3) / 1e12 / peak,
                                 "traffic": profile_traffic("nn_ensemble"),
                                 "note": "block-diagonal bf16 x3 on tcgen05 (M=128, K=16); slower than the "
                                         "CUDA-core path, kept selectable (carma_nn_set_path)"}
        else:
            r["dtype"] = "f32"
            r["kernel"] = "tf_ensemble (CUDA cores)"
            r["useful_tflops"] = useful / (k_avg * 1e-3) / 1e12
        res[key] = r
        net.close()
    cpu = None
    if d.rank == 0 and d.n == 1 and not args.skip_cpu:
        from threadpoolctl import threadpool_info
        threads = max([p.get("num_threads", 1) for p in threadpool_info()] or [1])
        ns = 1 << 18
        sidx = np.concatenate([np.arange(ns // 2), KNN_ROWS_PER_FAMILY + np.arange(ns // 2)])
        sraw = cb.scalar_features(rows_all[sidx])
        models = gm.load_default_models()
        t0 = time.perf_counter()
        for f in (1, 2):
            sel = fam_all[sidx] == f
            gpumemnet_oracle.forward(models[f].spec()[0], models[f].params, sraw[sel])
        cpu_s = time.perf_counter() - t0
        cpu = {"value": ns / cpu_s, "unit": "estimates/s", "cores": threads, "kind": "port",
               "sample": f"MLP ensemble, first {ns // 2} CNN + first {ns // 2} Transformer rows through "
                         "oracle/gpumemnet_oracle.py (numpy; no reference implementation exists)"}
    res["mlp"]["cpu_baseline"] = cpu
    return res


# ------------------------------------------------------------------ stage 2
def replay_stage(abi, cb, dev, stream, args, d):
    """The c4 policy sweep, jobs sharded by task count across ranks."""
    import ctypes

    import torch

    from paper_2508_19073_b200 import dist as cdist
    t0 = time.time()
    n_tr = args.sweep_traces
    cfgs, tasks_all, offs_all, jobs_all = sweep_inputs(cb, n_tr)
    counts = np.diff(offs_all.astype(np.int64))[jobs_all["trace"]]
    b, e = cdist.balanced_shards(counts, d.n)[d.rank]
    tasks, offs, jobs = shard_jobs(tasks_all, offs_all, jobs_all, b, e)
    n_placed = int(np.diff(offs.astype(np.int64))[jobs["trace"]].sum())
    total_placed = int(counts.sum())
    log(f"[rank {d.rank}] sweep inputs {n_tr} traces x {len(SWEEP_POLICIES)}, jobs [{b}, {e}) in "
        f"{time.time() - t0:.1f}s")
    plan = cb.ReplayPlan(cfgs, tasks, offs, jobs, device=dev)
    km, rm = ctypes.c_double(), ctypes.c_double()
    kernel_ms = []

    def step():
        plan.run(stream)
        abi.check(abi.lib.carma_replay_plan_timing(plan._h, ctypes.byref(km), ctypes.byref(rm)))
        kernel_ms.append(km.value)

    ms = timed_device_steps(step, stream, args.warmup, args.steps, d)
    kernel_ms = kernel_ms[args.warmup:]
    res = plan.results(tasks=False)
    assert (res.traces["status"] == 0).all()
    launches_r, retried = plan.stats()
    events = int(res.traces["events"].sum())
    plan.close()
    # e2e through the plan's host API: every step uploads the shard's tasks
    # from pinned memory, replays, and reads back per-task outcomes, reports
    # and per-GPU results into pinned memory
    plan = cb.ReplayPlan(cfgs, tasks, offs, jobs, device=dev)
    h_tasks = torch.from_numpy(tasks.view(np.uint8)).pin_memory().numpy().view(tasks.dtype)
    o_t = torch.empty(n_placed * 24, dtype=torch.uint8).pin_memory().numpy().view(abi.task_outcome_dtype)
    o_j = torch.empty(len(jobs) * 80, dtype=torch.uint8).pin_memory().numpy().view(abi.trace_result_dtype)
    o_g = torch.empty(len(jobs) * 4 * 32, dtype=torch.uint8).pin_memory().numpy().view(abi.gpu_result_dtype)

    # per-task outcomes stream into the pinned buffer as each job finishes
    # (carma_replay_plan_set_outcome_sink); reports and per-GPU results follow
    abi.check(abi.lib.carma_replay_plan_set_outcome_sink(plan._h, o_t.ctypes.data))

    def e2e_step():
        abi.check(abi.lib.carma_replay_plan_upload_tasks(plan._h, h_tasks.ctypes.data))
        abi.check(abi.lib.carma_replay_plan_run(plan._h, None))
        abi.check(abi.lib.carma_replay_plan_outcomes(plan._h, None, o_j.ctypes.data, o_g.ctypes.data))

    r_e2e = timed_host_steps(e2e_step, 1, args.steps, d)
    plan.close()
    assert o_j.tobytes() == res.traces.tobytes(), "replay e2e reports differ from the device-timed run"
    k_avg = statistics.mean(kernel_ms)
    hbm = peaks().get("hbm_gbs", 6650.0)
    ach = ALG_BYTES_PER_TASK * n_placed / (k_avg * 1e-3) / 1e9
    return {
        "metric": "trace-replay placed tasks/sec", "unit": "placed tasks/s",
        "value": total_placed / (ms * 1e-3), "ms_per_step": ms,
        "config": {"workload": f"c4 policy sweep: t90 seeds 1..{n_tr} x {{exclusive, rr, magm, lug}} "
                               f"({len(jobs_all)} jobs, {total_placed} placed tasks in total), MPS, u=0.8, "
                               "no estimator, 4 GPUs x 40 GiB, W=60 s",
                   "parallelism": f"dp{d.n}: contiguous job shards balanced by task count",
                   "jobs_this_rank": int(e - b), "placed_tasks_this_rank": n_placed},
        "events_per_s": d.sum(events) / (ms * 1e-3),
        "e2e": {"value": total_placed / r_e2e, "unit": "placed tasks/s", "ms_per_step": r_e2e * 1e3,
                "h2d_bytes_per_step": int(h_tasks.nbytes),
                "d2h_bytes_per_step": int(o_t.nbytes + o_j.nbytes + o_g.nbytes),
                "api": "carma_replay_plan_upload_tasks + run (per-task outcomes streamed into a pinned sink as jobs "
                       "finish) + outcomes (reports, per-GPU results)"},
        "gpu_launches": int(launches_r) * args.steps, "retried_jobs": int(retried),
        "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                     "traffic": profile_traffic("replay_kernel"), "kernel": "replay_kernel", "kernel_ms": k_avg,
                     "note": "latency/issue-bound event loop; algorithmic bytes = 80 B per placed task"},
    }


SCORING_DECISIONS = 1 << 24  # per GPU
SCORING_GPUS = 8


def scoring_bench(abi, cb, dev, stream, warmup, steps, d):
    """Batched eligible_gpus + map_task (manager.cpp:109-245): one decision per
    (task, server view) over device-resident views (24 B per simulated GPU) and
    requests (16 B), writing 2 GPU ids + the RR cursor. A pure HBM stream:
    algorithmic bytes per decision = G*24 + 16 + 4 (cursor in) + 4 (out) + 8."""
    import torch
    n, g = SCORING_DECISIONS, SCORING_GPUS
    rng = np.random.default_rng(5)
    views = np.zeros((n, g), abi.gpu_view_dtype)
    views["total_free"] = rng.integers(0, 81, (n, g), dtype=np.uint64) * np.uint64(512 << 20)
    views["windowed_smact"] = rng.random((n, g))
    views["idle"] = rng.random((n, g)) < 0.25
    reqs = np.zeros(n, abi.pick_request_dtype)
    reqs["estimate"] = rng.integers(0, 45, n, dtype=np.uint64) * np.uint64(1 << 30)
    reqs["want"] = np.where(rng.random(n) < 0.15, 2, 1).astype(np.uint32)
    cfg = cb.make_config(cb.PolicyConfig(policy="magm", max_smact=0.8), cb.SimConstants(gpu_count=g))
    dv = torch.from_numpy(views.view(np.uint8).reshape(-1)).to("cuda")
    dr = torch.from_numpy(reqs.view(np.uint8).reshape(-1)).to("cuda")
    dc = torch.zeros(n, dtype=torch.int32, device="cuda")
    do = torch.empty(2 * n, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2: every step starts cold

    def step():
        abi.check(abi.lib.carma_pick_batch_device(dev, cfg.ctypes.data, dv.data_ptr(), g, dr.data_ptr(), n,
                                                  dc.data_ptr(), do.data_ptr(), abi.stream_arg(stream)))

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            flush.zero_()
            step()
        torch.cuda.synchronize()
        times = []
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    per = g * 24 + 16 + 4 + 4 + 8
    gbs = per * n / (ms * 1e-3) / 1e9
    hbm = peaks().get("hbm_gbs", 6650.0)
    return {"metric": "placement decisions/sec (feasibility + MAGM score matrix)", "unit": "decisions/s",
            "value": n / (ms * 1e-3), "ms_per_step": ms,
            "config": {"workload": f"{n} decisions x {g} simulated GPUs, MAGM u=0.8, random views "
                                   f"(free in 512 MiB blocks, SMACT, idle), 15% two-GPU requests",
                       "l2": "256 MiB buffer written between steps"},
            "gpu_launches": 1,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                         "traffic": profile_traffic("pick_kernel"),
                         "algorithmic_bytes_per_decision": per, "kernel": "pick_kernel"}}


def fused_stage(abi, cb, dev, stream, args, knn):
    """configs[4] (c5): one 10^6-task trace, k-NN pre-pass over every arrival
    feeding the replay on 64 simulated GPUs; checked against the committed
    golden of the reference's full run (tests/golden/c5_ref.json)."""
    import torch
    t0 = time.time()
    mf = cb.materialize_trace(cb.generate_uniform_trace(args.fused_tasks, 3.0, 7))
    cfg5 = cb.make_config(cb.PolicyConfig(policy="magm", max_smact=0.8, monitor_window=5.0),
                          cb.SimConstants(gpu_count=64))
    for f in sorted(set(mf.family.tolist())):
        if f not in knn.models:
            knn.set_model(cb.fit_knn(f, 4000, 11 + 101 * f, 5))
    fr = cb.FusedReplay(mf, cfg5, knn, dev)
    log(f"fused inputs {args.fused_tasks} tasks in {time.time() - t0:.1f}s")
    fr.run(stream)  # warm-up (one: a step is ~11 s at 10^6 tasks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fr.run(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    f_ms = e0.elapsed_time(e1)
    res = fr.results()
    fr.close()
    t = res.traces[0]
    assert t["status"] == 0
    parity = "not checked (golden missing or different size)"
    gold = c5_golden()
    if gold and gold["n_tasks"] == args.fused_tasks:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import fullsize
        want = gold["runs"]["learned"]
        rec = fullsize.gpu_tasks_canonical(res.job_tasks(0))
        ok = (int(t["oom_count"]) == want["oom_count"] and fullsize.digest_fields(rec) == want["task_digest"]
              and all(np.float64(t[k]).view(np.uint64).item().to_bytes(8, "big").hex() == v
                      for k, v in want["report"].items()))
        assert ok, "c5 run differs from the reference golden"
        parity = "bit-exact vs tests/golden/c5_ref.json (report, per-task digests of every field)"
    full = gold["runs"]["learned"]["seconds"] if gold else None
    # Like-for-like with the CPU sample: the same prefix replayed on the GPU
    # (the per-event cost grows with the queue on both sides).
    ns = min(args.fused_cpu_tasks, args.fused_tasks)
    fs = cb.FusedReplay(cb.materialize_trace(cb.generate_uniform_trace(ns, 3.0, 7)), cfg5, knn, dev)
    fs.run(stream)
    torch.cuda.synchronize()
    e0.record(stream)
    fs.run(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    s_ms = e0.elapsed_time(e1)
    assert fs.results().traces[0]["status"] == 0
    fs.close()
    return {"metric": "fused estimator-in-the-loop placed tasks/sec", "unit": "placed tasks/s",
            "value": args.fused_tasks / (f_ms * 1e-3), "ms_per_step": f_ms, "steps": 1, "warmup": 1,
            "config": {"workload": f"c5: {args.fused_tasks} arrivals, uniform catalog, exp gaps mean 3 s, seed 7; "
                                   "k-NN pre-pass over every arrival feeding the replay; MAGM + learned, u=0.8, "
                                   "W=5 s, 64 simulated GPUs"},
            "events": int(t["events"]), "oom_count": int(t["oom_count"]), "parity": parity,
            "cpu_reference_full_trace": None if full is None else
            {"value": args.fused_tasks / full, "unit": "placed tasks/s", "cores": 1, "kind": "reference",
             "seconds": full, "source": "tests/golden/c5_ref.json (make_c5_golden.py, the full reference run)"},
            "gpu_same_sample": {"value": ns / (s_ms * 1e-3), "unit": "placed tasks/s", "ms": s_ms,
                                "sample": f"first {ns} rows of the c5 trace (the CPU sample's input)"},
            "note": "one trace: a single warp replays it (sequential event loop); not sharded"}


def small_configs(cb, abi, dev, stream, ref):
    """configs[0] (c1: 4096 MLP vectors, the reference's CPU batch) and
    configs[2] (c3: one paper-style t90 trace on an 8-GPU server, MAGM u=0.8
    with OOM recovery, estimator none and learned): latency-style lines."""
    import ctypes

    import torch
    out = {}
    m = cb.fit_knn(0, 4000, 11, 5)
    knn = cb.GpuKnn(dev)
    knn.set_model(m)
    ds = cb.generate_synthetic_dataset(0, 4096, 12345)
    d_rows = torch.from_numpy(ds.rows.view(np.uint8).reshape(-1)).to("cuda")
    d_b = torch.empty(4096, dtype=torch.int32, device="cuda")
    d_by = torch.empty(4096, dtype=torch.int64, device="cuda")

    def step():
        abi.check(abi.lib.carma_knn_predict_device(knn.handle, d_rows.data_ptr(), abi.ROWS_FEATURES, None, 0, 4096,
                                                   d_b.data_ptr(), d_by.data_ptr(), None, None,
                                                   abi.stream_arg(stream)))
    for _ in range(5):
        step()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / reps
    for _ in range(3):
        knn.predict(ds.rows, default_family=0)
    t = time.perf_counter()
    for _ in range(reps):
        h_b, _ = knn.predict(ds.rows, default_family=0)
    e2e_ms = (time.perf_counter() - t) / reps * 1e3
    assert np.array_equal(h_b, d_b.cpu().numpy())
    c1 = {"workload": "c1: GPUMemNet MLP k-NN over 4096 MLP feature vectors (seed 12345), model seed 11",
          "unit": "ms per 4096-row batch", "device_ms": dev_ms, "e2e_ms": e2e_ms,
          "estimates_per_s": 4096 / (dev_ms * 1e-3), "e2e_estimates_per_s": 4096 / (e2e_ms * 1e-3)}
    if ref is not None:
        ck = ctypes.c_uint64()
        ref.ref_bench_predict(0, 4000, 11, 5, 4096, 12345, 1, 1, ctypes.byref(ck))  # model cache
        cpu_s = ref.ref_bench_predict(0, 4000, 11, 5, 4096, 12345, 1, 3, ctypes.byref(ck)) / 3
        c1["cpu_baseline"] = {"value": cpu_s * 1e3, "unit": "ms per 4096-row batch", "cores": 1,
                              "kind": "reference", "sample": "the same 4096 rows, estimate_learned, 1 thread"}
    out["c1"] = c1
    knn.close()
    c3 = {"workload": "c3: one t90 trace (seed 1) on an 8-GPU server, MAGM u=0.8, MPS, W=60 s; "
                      "estimator none and learned", "unit": "ms per trace replay"}
    for est in ("none", "learned"):
        rc = cb.RunConfig(mix="t90", trace_seed=1,
                          policy=cb.PolicyConfig(policy="magm", max_smact=0.8, estimator=est),
                          constants=cb.SimConstants(gpu_count=8))
        mt = cb.materialize_trace(cb.generate_trace("t90", 1))
        cb.provision_estimates(rc, mt, dev)
        cfg = cb.make_config(rc.policy, rc.constants)
        plan = cb.ReplayPlan(cfg, mt.tasks, np.array([0, len(mt.tasks)], np.uint64), np.zeros(1, abi.job_dtype), dev)
        for _ in range(3):
            plan.run()
        km, rm = ctypes.c_double(), ctypes.c_double()
        runs = []
        for _ in range(10):
            plan.run()
            abi.check(abi.lib.carma_replay_plan_timing(plan._h, ctypes.byref(km), ctypes.byref(rm)))
            runs.append(rm.value)
        r = plan.results().traces[0]
        plan.close()
        t = time.perf_counter()
        for _ in range(10):
            cb.run_simulation(rc, device=dev)
        e2e_ms = (time.perf_counter() - t) / 10 * 1e3
        c3[est] = {"device_ms": statistics.median(runs), "e2e_ms": e2e_ms, "oom_count": int(r["oom_count"]),
                   "events": int(r["events"])}
        if ref is not None:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from oracle_bind import ref_config, ref_run
            rcfg = ref_config(policy="magm", estimator=est, gpu_count=8)
            ref_run(ref, rcfg, mix="t90", seed=1)
            t = time.perf_counter()
            for _ in range(5):
                ref_run(ref, rcfg, mix="t90", seed=1)
            c3[est]["cpu_baseline_ms"] = (time.perf_counter() - t) / 5 * 1e3
    c3["note"] = ("a single 90-task trace is one warp of sequential events (~2 us per event); e2e and the CPU "
                  "line both time run_simulation, learned estimators trained in-process on both sides")
    out["c3"] = c3
    return out


# ------------------------------------------------------------------ ours
def compact(x, keep):
    return None if x is None else {k: x[k] for k in keep if k in x}


def run_carma(args, d: Dist):
    import torch

    import paper_2508_19073_b200 as cb
    from paper_2508_19073_b200 import abi
    from paper_2508_19073_b200 import dist as cdist

    dev = int(os.environ.get("BENCH_DEVICE", d.local))
    if dev != d.local:
        log(f"[rank {d.rank}] dry run: device {dev} (BENCH_DEVICE), backend {d.backend}")
    torch.cuda.set_device(dev)
    if abi.lib.carma_device_count() < 1:
        raise SystemExit("no sm_100 device visible")
    N = d.n
    stream = torch.cuda.Stream(dev)  # every timed call runs on this explicit stream
    t0 = time.time()
    rows, fam = knn_inputs(cb, dev)
    QT = len(rows)
    b, e = cdist.balanced_shards_count(QT, N)[d.rank]
    gen_s = time.time() - t0
    log(f"[rank {d.rank}] knn inputs {QT} rows generated on the device in {gen_s:.2f}s; shard [{b}, {e})")
    knn_res, knn, (h_rows, h_fam, _) = knn_stage(abi, cb, dev, stream, args, d, rows, fam, b, e)
    neural = None
    if not args.skip_neural:
        neural = neural_stage(abi, cb, dev, stream, args, d, h_rows, h_fam, rows, fam, b)
    replay = None if args.skip_replay else replay_stage(abi, cb, dev, stream, args, d)
    scoring = fused = small = None
    if N == 1:
        if not args.skip_scoring:
            scoring = scoring_bench(abi, cb, dev, stream, args.warmup, args.steps, d)
        if not args.skip_fused:
            fused = fused_stage(abi, cb, dev, stream, args, knn)
    knn.close()

    cpu = None
    cpus = host_cpus()
    if d.rank == 0 and N == 1 and not args.skip_cpu:
        ref = ref_lib()
        threads = os.cpu_count() or 1
        if ref is not None:
            rate, sample = cpu_knn_baseline(ref, threads)
            cpu = {"value": rate, "unit": "estimates/s", "cores": threads, "kind": "reference", "sample": sample,
                   **cpus}
            if replay is not None:
                srate, ssample, _ = cpu_sweep_baseline(ref, threads)
                replay["cpu_baseline"] = {"value": srate, "unit": "placed tasks/s", "cores": threads,
                                          "kind": "reference", "sample": ssample, **cpus}
            if fused is not None:
                frate, fsample = cpu_fused_baseline(ref, args.fused_cpu_tasks)
                fused["cpu_baseline"] = {"value": frate, "unit": "placed tasks/s", "cores": 1, "kind": "reference",
                                         "sample": fsample}
    if d.rank == 0 and N == 1 and not args.skip_small:
        small = small_configs(cb, abi, dev, stream, None if args.skip_cpu else ref_lib())
    if d.rank != 0:
        return
    line = {
        "metric": "GPUMemNet estimates/sec (k-NN, CNN+Transformer ensemble)",
        "value": knn_res["value"], "unit": "estimates/s", "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": knn_res["ms_per_step"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generators, seeded)",
        "config": {**knn_config(N, e - b), "input_generation_s": gen_s},
        "e2e": knn_res["e2e"], "gpu_launches": knn_res["gpu_launches"], "roofline": knn_res["roofline"],
        "cpu_baseline": cpu, "clocks": knn_res["clocks"],
        "neural": neural, "scoring": scoring, "fused": fused, "small_configs": small, "replay": replay,
    }
    detail_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(detail_dir, exist_ok=True)
    with open(os.path.join(detail_dir, f"bench_detail_n{N}.json"), "w") as f:
        json.dump(line, f, indent=1)
    # the stdout line: the contract keys, then short sub-objects, the replay half last
    short = dict(line)
    short["roofline"] = compact(line["roofline"], ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel",
                                                   "kernel_ms", "kernel_share_of_step", "peak_source"))
    short["e2e"] = compact(line["e2e"], ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step", "api"))
    short["cpu_baseline"] = compact(cpu, ("value", "unit", "cores", "kind", "logical_cpus", "physical_cores"))
    short["clocks"] = compact(line["clocks"], ("sm_mhz", "sm_max_mhz", "reasons"))
    short["neural"] = None if neural is None else {
        "mlp": {"value": neural["mlp"]["value"], "ms_per_step": neural["mlp"]["ms_per_step"],
                "e2e": neural["mlp"]["e2e"]["value"], "roofline_frac": neural["mlp"]["roofline"]["frac"]},
        "transformer": {"value": neural["transformer"]["value"],
                        "ms_per_step": neural["transformer"]["ms_per_step"],
                        "e2e": neural["transformer"]["e2e"]["value"]}}
    short["scoring"] = None if scoring is None else {"value": scoring["value"], "unit": scoring["unit"],
                                                     "roofline_frac": scoring["roofline"]["frac"]}
    short["fused"] = None if fused is None else {"value": fused["value"], "unit": fused["unit"],
                                                 "ms_per_step": fused["ms_per_step"], "parity": fused["parity"][:12],
                                                 "cpu_sample": (fused.get("cpu_baseline") or {}).get("value"),
                                                 "gpu_same_sample": fused["gpu_same_sample"]["value"],
                                                 "cpu_full": (fused.get("cpu_reference_full_trace") or {}).get("value")}
    short["small_configs"] = None if small is None else "gpurun_out/bench_detail_n1.json"
    short["detail"] = f"gpurun_out/bench_detail_n{N}.json"
    if replay is not None:
        short["replay"] = {"metric": replay["metric"], "value": replay["value"], "unit": replay["unit"],
                           "ms_per_step": replay["ms_per_step"], "e2e": replay["e2e"]["value"],
                           "cpu_baseline": compact(replay.get("cpu_baseline"), ("value", "cores", "kind")),
                           "roofline_frac": replay["roofline"]["frac"], "scaling": "strong"}
    print(json.dumps(short))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("carma", "reference"), default="carma")
    ap.add_argument("--sweep-traces", type=int, default=SWEEP_TRACES)
    ap.add_argument("--skip-replay", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-fused", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    ap.add_argument("--skip-scoring", action="store_true")
    ap.add_argument("--skip-neural", action="store_true")
    ap.add_argument("--fused-tasks", type=int, default=1_000_000)
    ap.add_argument("--fused-cpu-tasks", type=int, default=100_000)
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        # the reference arm never touches the GPU or libcarma_b200.so: no NCCL
        d = Dist(args.gpus, backend="gloo")
    else:
        # BENCH_DIST_BACKEND=gloo + BENCH_DEVICE=0: a dry run of the N > 1
        # orchestration (sharding, barrier, max-over-ranks) on one GPU
        d = Dist(args.gpus, backend=os.environ.get("BENCH_DIST_BACKEND", "nccl"))
    try:
        if args.impl == "reference":
            run_reference(args, d)
        else:
            run_carma(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
