#!/usr/bin/env python
"""Benchmark of the CARMA hot path on B200.

Headline (BASELINE.json configs[1]): GPUMemNet estimates/s — the reference's
k-NN memory-bin classifier over the 16,777,216-row CNN + Transformer batch
(generate_synthetic_dataset(CNN, 8388608, 2024) + (Transformer, 8388608, 2025)),
routed per family to the models provision_estimators trains (seeds 112, 213).
Secondary (configs[3], same JSON line under "replay"): trace-replay placed
tasks/s for the policy sweep t90 seeds 1..100000 x {exclusive, rr, magm, lug}.

Scaling is weak: every rank runs the full per-GPU workload on its own GPU
with no data-path collective; value = all ranks' units / max-over-ranks time.

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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


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
    def __init__(self, gpus: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.n = max(self.world, 1)
        if gpus and self.world > 1 and gpus != self.world:
            log(f"warning: --gpus {gpus} but WORLD_SIZE {self.world}")
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ------------------------------------------------------------------ data
def knn_inputs(cb):
    """The c2 batch: 8,388,608 CNN rows (seed 2024) + 8,388,608 Transformer rows (seed 2025)."""
    out = {}

    def gen(f):
        out[f] = cb.generate_synthetic_dataset(f, KNN_ROWS_PER_FAMILY, KNN_SEEDS[f])

    th = [threading.Thread(target=gen, args=(f,)) for f in KNN_SEEDS]
    for t in th:
        t.start()
    for t in th:
        t.join()
    rows = np.concatenate([out[1].rows, out[2].rows])
    fam = np.concatenate([np.full(KNN_ROWS_PER_FAMILY, 1, np.int8), np.full(KNN_ROWS_PER_FAMILY, 2, np.int8)])
    return rows, fam


def sweep_inputs(cb, n_traces: int):
    """t90 seeds 1..n_traces, materialised once; jobs = traces x 4 policies."""
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


def profile_traffic(name: str):
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(path)).get(name)
    except (OSError, ValueError):
        return None


def recorded(name: str):
    """A measurement too long for the bounded bench run (e.g. the reference on the
    full 10^6-task c5 trace, scripts/c5_cpu_full.py, ~21 min), recorded once per
    round under profiles/."""
    try:
        r = json.load(open(os.path.join(ROOT, "profiles", name)))
        r["source"] = f"profiles/{name} (scripts/c5_cpu_full.py on the GPU box host, not re-run here)"
        return r
    except (OSError, ValueError):
        return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def knn_config(n: int) -> dict:
    return {"workload": "c2: GPUMemNet k-NN ensemble over 8,388,608 CNN (seed 2024) + 8,388,608 "
                        "Transformer (seed 2025) feature vectors per GPU; models = provision_estimators "
                        "(4000 samples, k=5, seeds 112/213)",
            "rows_per_gpu": 2 * KNN_ROWS_PER_FAMILY, "parallelism": f"dp{n} (independent shards, no collective)",
            "l2": "inputs 2.28 GB per GPU > 126 MB L2 (no flush needed)"}


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


def neural_bench(abi, cb, dev, stream, args, d, words, schema, rows, fam):
    """The paper's neural GPUMemNet (MLP ensemble, 8 members)
    over the same c2 batch as the k-NN headline: 16,777,216 bit-packed CNN +
    Transformer rows, routed per family, on the tcgen05 kernel."""
    import ctypes

    import torch

    from paper_2508_19073_b200 import gpumemnet as gm
    Q = len(rows)
    models = gm.load_default_models()
    net = gm.GpuMemNet(dev)
    for f in (1, 2):
        net.set_model(models[f])
    net.set_bit_schema(schema)
    d_rows = torch.from_numpy(words.view(np.uint8)).to("cuda")
    d_b = torch.empty(Q, dtype=torch.int32, device="cuda")
    d_by = torch.empty(Q, dtype=torch.int64, device="cuda")

    def step():
        net.predict_device(d_rows, abi.ROWS_BITPACKED, Q, d_b, d_by, stream=stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    d.barrier()
    kernel_ms, call_ms = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
        t = net.last_timing()
        kernel_ms.append(t["kernel_ms"])
        call_ms.append(t["call_ms"])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = d.max(e0.elapsed_time(e1) / args.steps)
    t = net.last_timing()
    b_dev = d_b.cpu().numpy()
    # e2e: pinned host bit-packed rows -> carma_nn_predict_bitpacked -> pinned host outputs
    h_rows = torch.from_numpy(words.view(np.uint8)).pin_memory().numpy().view(np.uint32)
    h_b = torch.empty(Q, dtype=torch.int32).pin_memory().numpy()
    h_by = torch.empty(Q, dtype=torch.int64).pin_memory().numpy().view(np.uint64)

    def e2e_step():
        abi.check(abi.lib.carma_nn_predict_bitpacked(net.handle, h_rows.ctypes.data, schema.ctypes.data, Q,
                                                     h_b.ctypes.data, h_by.ctypes.data))

    e2e_step()
    d.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = d.max((time.perf_counter() - t0) / args.steps)
    assert np.array_equal(h_b, b_dev), "host-API and device-resident neural predictions differ"
    # parity spot check against the oracle on a sample of the batch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import gpumemnet_oracle
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(Q, 4096, replace=False))
    agree = 0
    raw = cb.scalar_features(rows[idx])
    for f in (1, 2):
        sel = fam[idx] == f
        _, op, ob, _ = gpumemnet_oracle.forward(models[f].spec()[0], models[f].params, raw[sel])
        srt = np.sort(op, axis=1)
        sure = srt[:, -1] - srt[:, -2] > 1e-3
        assert np.array_equal(b_dev[idx][sel][sure], ob[sure]), "neural bins differ from the oracle"
        agree += int(sure.sum())
    cpu = None
    if d.rank == 0 and d.n == 1 and not args.skip_cpu:
        # The reference has no neural estimator: the CPU baseline is the numpy
        # oracle ("port", fp64 layers, BLAS threads) on a bounded sample.
        from threadpoolctl import threadpool_info
        threads = max([p.get("num_threads", 1) for p in threadpool_info()] or [1])
        ns = 1 << 18
        sidx = np.concatenate([np.arange(ns // 2), KNN_ROWS_PER_FAMILY + np.arange(ns // 2)])
        sraw = cb.scalar_features(rows[sidx])
        t0 = time.perf_counter()
        for f in (1, 2):
            sel = fam[sidx] == f
            gpumemnet_oracle.forward(models[f].spec()[0], models[f].params, sraw[sel])
        cpu_s = time.perf_counter() - t0
        cpu = {"value": ns / cpu_s, "unit": "estimates/s", "cores": threads, "kind": "port",
               "sample": f"first {ns // 2} CNN + first {ns // 2} Transformer rows of the batch through "
                         "oracle/gpumemnet_oracle.py (numpy; no reference implementation exists)"}
    # the paper's Transformer ensemble on the same batch (CUDA cores)
    tfm = gm.load_default_models(gm.ARCH_TRANSFORMER)
    tnet = gm.GpuMemNet(dev)
    for f in (1, 2):
        tnet.set_model(tfm[f])
    tnet.set_bit_schema(schema)

    def tf_step():
        tnet.predict_device(d_rows, abi.ROWS_BITPACKED, Q, d_b, d_by, stream=stream.cuda_stream)

    for _ in range(args.warmup):
        tf_step()
    torch.cuda.synchronize()
    d.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        tf_step()
    f1.record(stream)
    torch.cuda.synchronize()
    tf_ms = d.max(f0.elapsed_time(f1) / args.steps)
    tb = d_b.cpu().numpy()
    tf_agree = 0
    for f in (1, 2):
        sel = fam[idx] == f
        _, op, ob, _ = gpumemnet_oracle.forward(tfm[f].spec()[0], tfm[f].params, raw[sel])
        srt = np.sort(op, axis=1)
        sure = srt[:, -1] - srt[:, -2] > 1e-3
        assert np.array_equal(tb[idx][sel][sure], ob[sure]), "transformer bins differ from the oracle"
        tf_agree += int(sure.sum())
    tnet.close()
    transformer = {"metric": "GPUMemNet estimates/sec (Transformer ensemble, 8 members)", "unit": "estimates/s",
                   "value": d.n * Q / (tf_ms * 1e-3), "ms_per_step": tf_ms, "dtype": "f32",
                   "kernel": "tf_ensemble (thread per row, three-token attention in registers, CUDA cores)",
                   "oracle_agreement_rows": tf_agree,
                   "holdout_accuracy": {gm.FAMILY_NAMES[f]: tfm[f].holdout_accuracy for f in (1, 2)}}
    k_avg = statistics.mean(kernel_ms)
    rows_f = {f: int((fam == f).sum()) for f in (1, 2)}
    executed = sum((rows_f[f] + 127) // 128 * nn_tile_flops(models[f])[0] for f in (1, 2))
    useful = sum(rows_f[f] * nn_tile_flops(models[f])[1] for f in (1, 2))
    peak = peaks().get("bf16_tflops", 2250.0)
    ach = useful / (k_avg * 1e-3) / 1e12          # algorithmic (the ensemble's dense math)
    ach_exec = executed / (k_avg * 1e-3) / 1e12   # what the tensor pipe executed
    wpr = int(schema["words_per_row"][0])
    hbm_bytes = Q * (4 * wpr + 12)
    net.close()
    return {
        "metric": "GPUMemNet estimates/sec (neural MLP ensemble, 8 members, CNN+Transformer)",
        "unit": "estimates/s", "value": d.n * Q / (ms * 1e-3), "ms_per_step": ms, "dtype": "bf16 x3 -> fp32",
        "config": {"workload": f"c2 batch ({Q} bit-packed rows, {4 * wpr} B each) through the neural GPUMemNet "
                               "ensembles of paper_2508_19073_b200/weights (scripts/train_gpumemnet.py)",
                   "l2": "inputs larger than L2 (no flush needed)"},
        "e2e": {"value": d.n * Q / e2e_s, "unit": "estimates/s", "h2d_bytes_per_step": int(h_rows.nbytes),
                "d2h_bytes_per_step": int(h_b.nbytes + h_by.nbytes),
                "api": "carma_nn_predict_bitpacked (pinned host buffers)"},
        "gpu_launches": int(t["launches"]) * args.steps,
        "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                     "traffic": profile_traffic("nn_ensemble"), "kernel": "nn_ensemble", "kernel_ms": k_avg,
                     "kernel_share_of_step": k_avg / statistics.mean(call_ms),
                     "work": f"algorithmic: {useful / 1e9:.1f} GFLOP of dense ensemble math per step (DESIGN §3); "
                             f"executed: {t['mmas']} tcgen05.mma (M=128, K=16) = {executed / 1e9:.1f} GFLOP "
                             "(block-diagonal padding, 3 bf16 activation parts)",
                     "executed_tflops": ach_exec, "executed_frac": ach_exec / peak,
                     "note": "latency-bound: a 9-stage dependent MMA -> epilogue chain per 128-row tile, "
                             "3 tiles in flight per SM (shared memory); tiny layers (<= 8 neurons per member)",
                     "hbm_gbs": hbm_bytes / (k_avg * 1e-3) / 1e9, "hbm_peak_gbs": peaks().get("hbm_gbs"),
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)"},
        "cpu_baseline": cpu,
        "transformer": transformer,
        "oracle_agreement_rows": agree,
        "holdout_accuracy": {gm.FAMILY_NAMES[f]: models[f].holdout_accuracy for f in (1, 2)},
    }



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
    from oracle_bind import ref_config
    from paper_2508_19073_b200 import abi
    cfg = ref_config(policy="magm", max_smact=0.8)
    pols = np.array([abi.POLICY[p] for p in SWEEP_POLICIES], np.int32)
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
                                                  dc.data_ptr(), do.data_ptr(), stream.cuda_stream))

    for _ in range(warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    d.barrier()
    times = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = d.max(statistics.mean(times))
    per = g * 24 + 16 + 4 + 4 + 8
    gbs = per * n / (ms * 1e-3) / 1e9
    hbm = peaks().get("hbm_gbs", 6650.0)
    return {"metric": "placement decisions/sec (feasibility + MAGM score matrix)", "unit": "decisions/s",
            "value": d.n * n / (ms * 1e-3), "ms_per_step": ms,
            "config": {"workload": f"{n} decisions x {g} simulated GPUs per rank, MAGM u=0.8, random views "
                                   f"(free in 512 MiB blocks, SMACT, idle), 15% two-GPU requests",
                       "l2": "256 MiB buffer written between steps"},
            "gpu_launches": 1,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                         "traffic": profile_traffic("pick_kernel"),
                         "algorithmic_bytes_per_decision": per, "kernel": "pick_kernel"}}


def small_configs(cb, abi, dev, ref):
    """configs[0] (c1: 4096 MLP vectors, the reference's CPU batch) and
    configs[2] (c3: one paper-style t90 trace on an 8-GPU server, MAGM u=0.8
    with OOM recovery, estimator none and learned): latency-style lines."""
    import ctypes

    import torch
    out = {}
    # ---- c1
    m = cb.fit_knn(0, 4000, 11, 5)
    knn = cb.GpuKnn(dev)
    knn.set_model(m)
    ds = cb.generate_synthetic_dataset(0, 4096, 12345)
    words, schema = cb.pack_features_bits(ds.rows, np.zeros(4096, np.int8))
    abi.check(abi.lib.carma_knn_set_bit_schema(knn.handle, schema.ctypes.data))
    d_rows = torch.from_numpy(words.view(np.uint8)).to("cuda")
    d_b = torch.empty(4096, dtype=torch.int32, device="cuda")
    d_by = torch.empty(4096, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()

    def step():
        abi.check(abi.lib.carma_knn_predict_device(knn.handle, d_rows.data_ptr(), abi.ROWS_BITPACKED, None, 0, 4096,
                                                   d_b.data_ptr(), d_by.data_ptr(), None, None, s.cuda_stream))
    for _ in range(5):
        step()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / reps
    h_b = np.zeros(4096, np.int32)
    h_by = np.zeros(4096, np.uint64)
    for _ in range(3):
        knn.predict_bitpacked(words, schema, 4096)
    t = time.perf_counter()
    for _ in range(reps):
        h_b, h_by = knn.predict_bitpacked(words, schema, 4096)
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
    # ---- c3
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
        # e2e: the user's call, run_simulation (trace generation, estimator
        # provisioning incl. training for "learned", the replay, read-back),
        # like the reference's run_simulation the CPU line times
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


def run_reference(args, d: Dist):
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
    line = {
        "impl": "reference", "metric": "GPUMemNet estimates/sec (k-NN, CNN+Transformer ensemble)",
        "value": value, "unit": "estimates/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": knn_config(1),
        "cpu_baseline": {"value": value, "unit": "estimates/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "estimates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "replay": {"value": srate, "unit": "placed tasks/s", "cores": threads, "sample": ssample},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ ours
def run_carma(args, d: Dist):
    import torch

    import paper_2508_19073_b200 as cb
    from paper_2508_19073_b200 import abi

    dev = d.local
    torch.cuda.set_device(dev)
    if abi.lib.carma_device_count() < 1:
        raise SystemExit("no sm_100 device visible")
    N = d.n
    import ctypes
    fp64 = ctypes.c_double()
    abi.check(abi.lib.carma_probe_fp64(dev, ctypes.byref(fp64)))
    fp32 = ctypes.c_double()
    abi.check(abi.lib.carma_probe_fp32(dev, ctypes.byref(fp32)))

    # ---------------- stage 1 inputs
    t0 = time.time()
    rows, fam = knn_inputs(cb)
    Q = len(rows)
    knn = cb.GpuKnn(dev)
    for f in (1, 2):
        knn.set_model(cb.fit_knn(f, 4000, MODEL_SEEDS[f], 5))
    log(f"[rank {d.rank}] knn inputs {Q} rows in {time.time() - t0:.1f}s; fp64 probe {fp64.value / 1e12:.2f} TF/s")
    # Bit-packed rows (lossless frame-of-reference packing, family inside;
    # include/carma_gpu.h): 36 B/row on this batch instead of 136 B.
    words, schema = cb.pack_features_bits(rows, fam)
    abi.check(abi.lib.carma_knn_set_bit_schema(knn.handle, schema.ctypes.data))
    wpr = int(schema["words_per_row"][0])
    stream = torch.cuda.current_stream()
    d_rows = torch.from_numpy(words.view(np.uint8)).to("cuda")
    d_b = torch.empty(Q, dtype=torch.int32, device="cuda")
    d_by = torch.empty(Q, dtype=torch.int64, device="cuda")

    def knn_step():
        abi.check(abi.lib.carma_knn_predict_device(knn.handle, d_rows.data_ptr(), abi.ROWS_BITPACKED, None, 1, Q,
                                                   d_b.data_ptr(), d_by.data_ptr(), None, None, stream.cuda_stream))

    search_ms, pipe_ms = [], []
    sm, pm = ctypes.c_double(), ctypes.c_double()
    with Clocks(dev) as clk:
        clk.mark("t_busy")
        for _ in range(args.warmup):
            knn_step()
        torch.cuda.synchronize()
        d.barrier()
        torch.cuda.synchronize()
        clk.mark("t_begin")
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            knn_step()
            abi.check(abi.lib.carma_knn_last_timing(knn.handle, ctypes.byref(sm), ctypes.byref(pm)))
            search_ms.append(sm.value)
            pipe_ms.append(pm.value)
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark("t_end")
        d.barrier()
    knn_ms = d.max(e0.elapsed_time(e1) / args.steps)
    clocks = clk.summary()
    b_dev = d_b.cpu().numpy()
    launches, evals = knn.last_stats()
    la_, e64_, e32_ = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    abi.check(abi.lib.carma_knn_last_work(knn.handle, ctypes.byref(la_), ctypes.byref(e64_), ctypes.byref(e32_)))
    visits = e32_.value
    value = N * Q / (knn_ms * 1e-3)

    # e2e: pinned host bit-packed rows -> carma_knn_predict_bitpacked (chunked
    # H2D / compute / D2H on two streams) -> pinned host buckets + bytes
    h_rows = torch.from_numpy(words.view(np.uint8)).pin_memory().numpy().view(np.uint32)
    h_b = torch.empty(Q, dtype=torch.int32).pin_memory().numpy()
    h_by = torch.empty(Q, dtype=torch.int64).pin_memory().numpy().view(np.uint64)

    def e2e_step():
        abi.check(abi.lib.carma_knn_predict_bitpacked(knn.handle, h_rows.ctypes.data, schema.ctypes.data, Q,
                                                      h_b.ctypes.data, h_by.ctypes.data))

    for _ in range(max(1, args.warmup - 1)):
        e2e_step()
    d.barrier()
    t = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = d.max((time.perf_counter() - t) / args.steps)
    d.barrier()
    assert np.array_equal(h_b, b_dev), "host-API and device-resident predictions differ"
    # the other host formats, warm, once each: 64-B packed rows and the
    # 136-B FeatureVector rows
    packed, table = cb.pack_features(rows, fam)
    h_pk = torch.from_numpy(packed.view(np.uint8).reshape(-1)).pin_memory().numpy().view(packed.dtype)
    for _ in range(2):
        t = time.perf_counter()
        abi.check(abi.lib.carma_knn_predict_packed(knn.handle, h_pk.ctypes.data, table.ctypes.data, Q,
                                                   h_b.ctypes.data, h_by.ctypes.data))
        e2e_pk_s = time.perf_counter() - t
    assert np.array_equal(h_b, b_dev)
    h_full = torch.from_numpy(rows.view(np.uint8).reshape(-1)).pin_memory().numpy().view(rows.dtype)
    h_fam = torch.from_numpy(fam).pin_memory().numpy()
    for _ in range(2):  # warm-up: scratch sized for 136-B rows
        t = time.perf_counter()
        abi.check(abi.lib.carma_knn_predict(knn.handle, h_full.ctypes.data, h_fam.ctypes.data, 1, Q,
                                            h_b.ctypes.data, h_by.ctypes.data))
        e2e_full_s = time.perf_counter() - t
    assert np.array_equal(h_b, b_dev)
    del d_rows, d_b, d_by, h_full, h_fam, h_pk
    abi.check(abi.lib.carma_knn_set_act_table(knn.handle, table.ctypes.data))

    search_avg = statistics.mean(search_ms)
    # executed work of the exact pruned search: fp32 pre-filter evaluations
    # (16 dims x (sub + fma) = 48 flops) dominate; exact fp64 evaluations are
    # reported beside them
    f32_flops = visits * FLOPS_PER_F32_EVAL
    achieved = f32_flops / (search_avg * 1e-3)
    traffic = profile_traffic("knn_search_f32")

    # ---------------- stage 1, neural GPUMemNet (tcgen05 MLP ensemble)
    neural = None
    if not args.skip_neural:
        neural = neural_bench(abi, cb, dev, stream, args, d, words, schema, rows, fam)

    # ---------------- stage 2: policy sweep
    replay = None
    if not args.skip_replay:
        t0 = time.time()
        n_tr = args.sweep_traces
        cfgs, tasks, offs, jobs = sweep_inputs(cb, n_tr)
        sweep_gen_s = time.time() - t0
        n_placed = int(np.diff(offs.astype(np.int64))[jobs["trace"]].sum())
        plan = cb.ReplayPlan(cfgs, tasks, offs, jobs, device=dev)
        log(f"[rank {d.rank}] sweep inputs {n_tr} traces x {len(SWEEP_POLICIES)} in {time.time() - t0:.1f}s")
        for _ in range(args.warmup):
            plan.run()
        km, rm = ctypes.c_double(), ctypes.c_double()
        kernel_ms, run_ms = [], []
        d.barrier()
        for _ in range(args.steps):
            plan.run()
            abi.check(abi.lib.carma_replay_plan_timing(plan._h, ctypes.byref(km), ctypes.byref(rm)))
            kernel_ms.append(km.value)
            run_ms.append(rm.value)
        d.barrier()
        res = plan.results(tasks=False)
        assert (res.traces["status"] == 0).all()
        launches_r, retried = plan.stats()
        events = int(res.traces["events"].sum())
        plan.close()
        run_avg = d.max(statistics.mean(run_ms))
        k_avg = statistics.mean(kernel_ms)
        # e2e through the plan's host API: every step uploads the tasks from
        # pinned memory, replays, and reads back per-task outcomes + reports
        plan = cb.ReplayPlan(cfgs, tasks, offs, jobs, device=dev)
        h_tasks = torch.from_numpy(tasks.view(np.uint8)).pin_memory().numpy().view(tasks.dtype)
        o_t = torch.empty(n_placed * 24, dtype=torch.uint8).pin_memory().numpy().view(abi.task_outcome_dtype)
        o_j = torch.empty(len(jobs) * 80, dtype=torch.uint8).pin_memory().numpy().view(abi.trace_result_dtype)
        o_g = torch.empty(len(jobs) * 4 * 32, dtype=torch.uint8).pin_memory().numpy().view(abi.gpu_result_dtype)

        def e2e_step():
            abi.check(abi.lib.carma_replay_plan_upload_tasks(plan._h, h_tasks.ctypes.data))
            abi.check(abi.lib.carma_replay_plan_run(plan._h, None))
            abi.check(abi.lib.carma_replay_plan_outcomes(plan._h, o_t.ctypes.data, o_j.ctypes.data,
                                                         o_g.ctypes.data))

        e2e_step()
        d.barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        r_e2e = d.max((time.perf_counter() - t) / args.steps)
        plan.close()
        assert np.array_equal(o_j["energy_mj"], res.traces["energy_mj"])
        # e2e from seeds: the sweep's traces generated and materialised on the
        # device (carma_replay_plan_create_generated), replayed, outcomes read
        # back — run_sweep's inputs without the host trace loop
        seeds = np.arange(1, n_tr + 1, dtype=np.uint64)

        def gen_step():
            p = cb.ReplayPlan.generated(cfgs, "t90", seeds, jobs, device=dev)
            abi.check(abi.lib.carma_replay_plan_run(p._h, None))
            abi.check(abi.lib.carma_replay_plan_outcomes(p._h, o_t.ctypes.data, o_j.ctypes.data, o_g.ctypes.data))
            p.close()

        gen_step()
        d.barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            gen_step()
        r_gen = d.max((time.perf_counter() - t) / args.steps)
        assert np.array_equal(o_j["energy_mj"], res.traces["energy_mj"]), "generated sweep differs"
        replay = {
            "metric": "trace-replay placed tasks/sec", "unit": "placed tasks/s",
            "value": N * n_placed / (run_avg * 1e-3), "ms_per_step": run_avg,
            "config": {"workload": f"c4 policy sweep: t90 seeds 1..{n_tr} x {{exclusive, rr, magm, lug}}, "
                                   "MPS, u=0.8, no estimator, 4 GPUs x 40 GiB, W=60 s",
                       "jobs_per_gpu": len(jobs), "placed_tasks_per_gpu": n_placed},
            "events_per_s": N * events / (run_avg * 1e-3),
            "e2e": {"value": N * n_placed / r_e2e, "unit": "placed tasks/s",
                    "h2d_bytes_per_step": int(h_tasks.nbytes),
                    "d2h_bytes_per_step": int(o_t.nbytes + o_j.nbytes + o_g.nbytes),
                    "api": "carma_replay_plan_upload_tasks + run + outcomes (per-task outcomes, reports, per-GPU)",
                    "from_seeds": {"value": N * n_placed / r_gen, "unit": "placed tasks/s",
                                   "h2d_bytes_per_step": int(seeds.nbytes),
                                   "d2h_bytes_per_step": int(o_t.nbytes + o_j.nbytes + o_g.nbytes),
                                   "api": "carma_replay_plan_create_generated (traces generated on the device) "
                                          "+ run + outcomes"},
                    "host_trace_generation_s": sweep_gen_s},
            "gpu_launches": int(launches_r) * args.steps,
            "retried_jobs": int(retried),
            "roofline": {"bound": "hbm", "achieved": ALG_BYTES_PER_TASK * n_placed / (k_avg * 1e-3) / 1e9,
                         "peak": peaks().get("hbm_gbs", 6650.0), "unit": "GB/s",
                         "frac": ALG_BYTES_PER_TASK * n_placed / (k_avg * 1e-3) / 1e9 / peaks().get("hbm_gbs", 6650.0),
                         "traffic": profile_traffic("replay_kernel"),
                         "note": "latency/issue bound event loop; algorithmic bytes = 80 B per placed task"},
        }

    # ---------------- placement scoring (feasibility / score matrix, B9)
    scoring = None
    if not args.skip_scoring:
        scoring = scoring_bench(abi, cb, dev, stream, args.warmup, args.steps, d)

    # ---------------- stage 1 -> 2 fused (configs[4], c5)
    fused = None
    if not args.skip_fused:
        t0 = time.time()
        mf = cb.materialize_trace(cb.generate_uniform_trace(args.fused_tasks, 3.0, 7))
        cfg5 = cb.make_config(cb.PolicyConfig(policy="magm", max_smact=0.8, monitor_window=5.0),
                              cb.SimConstants(gpu_count=64))
        fr = cb.FusedReplay(mf, cfg5, knn, dev)
        log(f"[rank {d.rank}] fused inputs {args.fused_tasks} tasks in {time.time() - t0:.1f}s")
        fr.run()  # warm-up (one: a step is ~13 s at 10^6 tasks)
        torch.cuda.synchronize()
        d.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fr.run()
        e1.record(stream)
        torch.cuda.synchronize()
        f_ms = d.max(e0.elapsed_time(e1))
        fres = fr.results().traces[0]
        assert fres["status"] == 0
        fr.close()
        fused = {"metric": "fused estimator-in-the-loop placed tasks/sec", "unit": "placed tasks/s",
                 "value": N * args.fused_tasks / (f_ms * 1e-3), "ms_per_step": f_ms, "steps": 1, "warmup": 1,
                 "config": {"workload": f"c5: {args.fused_tasks} arrivals, uniform catalog, exp gaps mean 3 s, "
                                        "seed 7; k-NN pre-pass over every arrival on device feeding the replay; "
                                        "MAGM + learned, u=0.8, W=5 s, 64 simulated GPUs"},
                 "events": int(fres["events"]), "oom_count": int(fres["oom_count"]),
                 "note": "one trace: a single warp replays it (sequential event loop); replicas only across GPUs",
                 "cpu_reference_full_trace": recorded("c5_cpu_full_r01.json")}

    # ---------------- CPU baselines (rank 0, N = 1)
    cpu = None
    if d.rank == 0 and N == 1 and not args.skip_cpu:
        ref = ref_lib()
        threads = os.cpu_count() or 1
        if ref is not None:
            rate, sample = cpu_knn_baseline(ref, threads)
            cpu = {"value": rate, "unit": "estimates/s", "cores": threads, "kind": "reference", "sample": sample}
            if replay is not None:
                srate, ssample, _ = cpu_sweep_baseline(ref, threads)
                replay["cpu_baseline"] = {"value": srate, "unit": "placed tasks/s", "cores": threads,
                                          "kind": "reference", "sample": ssample}
            if fused is not None:
                frate, fsample = cpu_fused_baseline(ref, args.fused_cpu_tasks)
                fused["cpu_baseline"] = {"value": frate, "unit": "placed tasks/s", "cores": 1, "kind": "reference",
                                         "sample": fsample}

    small = None
    if d.rank == 0 and N == 1 and not args.skip_small:
        small = small_configs(cb, abi, dev, None if args.skip_cpu else ref_lib())

    if d.rank != 0:
        return
    hbm = peaks().get("hbm_gbs")
    line = {
        "metric": "GPUMemNet estimates/sec (k-NN, CNN+Transformer ensemble)",
        "value": value, "unit": "estimates/s", "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": knn_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generators, seeded)",
        "config": knn_config(N),
        "e2e": {"value": N * Q / e2e_s, "unit": "estimates/s",
                "h2d_bytes_per_step": int(h_rows.nbytes),
                "d2h_bytes_per_step": int(h_b.nbytes + h_by.nbytes),
                "api": f"carma_knn_predict_bitpacked ({4 * wpr} B bit-packed rows, pinned host buffers)",
                "packed64_api_estimates_per_s": N * Q / e2e_pk_s,
                "feature_row_api_estimates_per_s": N * Q / e2e_full_s},
        "gpu_launches": int(launches) * args.steps,
        "roofline": {"bound": "fp32", "achieved": achieved / 1e12, "peak": fp32.value / 1e12, "unit": "TFLOP/s",
                     "frac": achieved / fp32.value, "traffic": traffic,
                     "kernel": "knn_search_f32", "kernel_ms": search_avg,
                     "kernel_share_of_step": search_avg / statistics.mean(pipe_ms),
                     "peak_source": "measured: carma_probe_fp32 (FFMA2 issue rate; the contract's MEASURED_PEAKS "
                                    "file has no fp32/fp64 figures)",
                     "work": f"{visits} fp32 pre-filter evaluations x {FLOPS_PER_F32_EVAL} flops + {evals} exact "
                             f"fp64 evaluations x {FLOPS_PER_EVAL} flops",
                     "fp64": {"achieved": evals * FLOPS_PER_EVAL / (search_avg * 1e-3) / 1e12,
                              "peak": fp64.value / 1e12, "unit": "TFLOP/s"},
                     "brute_force_equivalent_tflops": Q * 162_400 / (search_avg * 1e-3) / 1e12,
                     "hbm_gbs": ALG_BYTES_PER_ESTIMATE * Q / (search_avg * 1e-3) / 1e9, "hbm_peak_gbs": hbm,
                     "note": "exact pruned search: the bound is instruction issue over the fp32 pass; the brute-force "
                             "figure (162,400 flops/estimate) is what the pruning avoids"},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "replay": replay,
        "neural": neural,
        "scoring": scoring,
        "fused": fused,
        "small_configs": small,
    }
    print(json.dumps(line))


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
    d = Dist(args.gpus)
    try:
        if args.impl == "reference":
            run_reference(args, d)
        else:
            run_carma(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
