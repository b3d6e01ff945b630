"""Reference-shaped host API over the C ABI.

Mirrors the parts of the reference's public C++ API that sit on the hot path
(names follow proj/include/carma/*.hpp):

* ``generate_synthetic_dataset`` / ``train_learned_estimator`` /
  ``LearnedEstimator.predict`` / ``estimate_learned``  (estimators.hpp:98-142)
* ``generate_trace`` / ``materialize_trace`` / ``save_trace`` / ``load_trace``
  (traces.hpp:42-62)
* ``PolicyConfig`` / ``SimConstants`` / ``RunConfig`` / ``run_simulation`` /
  ``run_sweep`` (manager.hpp:29-37, memory_model.hpp:11-29, runner.hpp:18-72)
* ``pick_batch``: batched ``Manager::eligible_gpus`` + ``map_task``
  (manager.hpp:82-86)

Everything numeric runs in libcarma_b200.so: the k-NN and the replay on the
GPU, trace/dataset provisioning in its host C++ half. Errors surface as
:class:`abi.CarmaError` (the reference's CarmaError family).
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import Dict, Iterable, List, Optional, Sequence

import numpy as np

from . import abi
from .abi import check, lib, ptr

# ----------------------------------------------------------------- catalog


@dataclasses.dataclass(frozen=True)
class CatalogEntry:
    key: str
    family: int
    gpus: int
    batch: int
    mem_gib: float


def builtin_catalog() -> List[CatalogEntry]:
    out = []
    for i in range(lib.carma_host_catalog_size()):
        key = ctypes.create_string_buffer(96)
        fam, gpus, batch, mem = ctypes.c_int32(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_double()
        check(lib.carma_host_catalog_entry(i, key, 96, ctypes.addressof(fam), ctypes.addressof(gpus),
                                           ctypes.addressof(batch), ctypes.addressof(mem)))
        out.append(CatalogEntry(key.value.decode(), fam.value, gpus.value, batch.value, mem.value))
    return out


# ------------------------------------------------------------------ traces


@dataclasses.dataclass
class Trace:
    """TraceFile (traces.hpp:43-52): rows of (submit_s, catalog index, epochs)."""

    submit: np.ndarray
    entry: np.ndarray
    epochs: np.ndarray
    seed: int = 0
    mix: str = ""

    def __len__(self) -> int:
        return len(self.submit)


def generate_trace(mix: str, seed: int) -> Trace:
    cap = 128
    sub = np.zeros(cap, np.float64)
    ent = np.zeros(cap, np.int32)
    ep = np.zeros(cap, np.uint64)
    n = ctypes.c_uint64()
    check(lib.carma_host_generate_trace(abi.MIX[mix], seed, ptr(sub), ptr(ent), ptr(ep), cap, ctypes.byref(n)))
    k = n.value
    return Trace(sub[:k].copy(), ent[:k].copy(), ep[:k].copy(), seed, mix)


def generate_uniform_trace(n: int, mean_gap: float, seed: int) -> Trace:
    sub = np.zeros(n, np.float64)
    ent = np.zeros(n, np.int32)
    ep = np.zeros(n, np.uint64)
    check(lib.carma_host_generate_uniform_trace(n, mean_gap, seed, ptr(sub), ptr(ent), ptr(ep)))
    return Trace(sub, ent, ep, seed, "uniform")


def save_trace(trace: Trace, path: str) -> None:
    check(lib.carma_host_save_trace(path.encode(), trace.seed, trace.mix.encode(), ptr(trace.submit),
                                    ptr(trace.entry), ptr(trace.epochs), len(trace)))


def load_trace(path: str) -> Trace:
    n = ctypes.c_uint64()
    check(lib.carma_host_load_trace(path.encode(), None, None, None, 0, ctypes.byref(n)))
    sub = np.zeros(n.value, np.float64)
    ent = np.zeros(n.value, np.int32)
    ep = np.zeros(n.value, np.uint64)
    check(lib.carma_host_load_trace(path.encode(), ptr(sub), ptr(ent), ptr(ep), n.value, ctypes.byref(n)))
    return Trace(sub, ent, ep)


@dataclasses.dataclass
class Materialized:
    tasks: np.ndarray      # task_dtype
    features: np.ndarray   # feature_row_dtype
    family: np.ndarray     # int8
    entry: np.ndarray      # int32 catalog index


def materialize_trace(trace: Trace) -> Materialized:
    n = len(trace)
    tasks = np.zeros(n, abi.task_dtype)
    feats = np.zeros(n, abi.feature_row_dtype)
    fam = np.zeros(n, np.int8)
    check(lib.carma_host_materialize(ptr(trace.submit), ptr(trace.entry), ptr(trace.epochs), n, ptr(tasks),
                                     ptr(feats), ptr(fam)))
    return Materialized(tasks, feats, fam, trace.entry.copy())


def set_persona_estimates(m: Materialized, estimator: str, safety_margin: int = 2 * abi.GiB) -> None:
    """oracle / analytical / static_graph / none into m.tasks['estimate'] (manager.cpp:80-107)."""
    check(lib.carma_host_estimates(abi.ESTIMATOR[estimator], safety_margin, ptr(m.entry), len(m.tasks),
                                   ptr(m.tasks)))


# ---------------------------------------------------------------- datasets


@dataclasses.dataclass
class EstimatorDataset:
    rows: np.ndarray     # feature_row_dtype
    bucket: np.ndarray   # int32
    mem: np.ndarray      # uint64
    family: int
    seed: int

    @property
    def bucket_range(self) -> int:
        return abi.GiB if self.family == 0 else 8 * abi.GiB


def generate_synthetic_dataset(family: int, n: int, seed: int, device: Optional[int] = None) -> EstimatorDataset:
    """generate_synthetic_dataset (estimators.cpp:221-264). device=None: the
    host generator (csrc/host/model.cpp); device=d: the GPU generator
    (csrc/cuda/dataset.cu, carma_dataset_generate), bit-identical."""
    rows = np.zeros(n, abi.feature_row_dtype)
    b = np.zeros(n, np.int32)
    m = np.zeros(n, np.uint64)
    if device is None:
        check(lib.carma_host_dataset(family, n, seed, ptr(rows), ptr(b), ptr(m)))
    else:
        check(lib.carma_dataset_generate(device, family, n, seed, ptr(rows), ptr(b), ptr(m), None))
    return EstimatorDataset(rows, b, m, family, seed)


def generate_synthetic_dataset_device(family: int, n: int, seed: int, rows=None, bucket=None, mem=None,
                                      device: int = 0, stream=None) -> np.ndarray:
    """The GPU generator into device tensors (torch, any nullable): rows as
    n x 136 bytes (carma_feature_row), bucket int32[n], mem int64[n] (u64
    bits). Returns the carma_dataset_stats record."""
    st = np.zeros(1, abi.dataset_stats_dtype)
    check(lib.carma_dataset_generate_device(device, family, n, seed, ptr(rows), ptr(bucket), ptr(mem),
                                            abi.stream_arg(stream, device), ptr(st)))
    return st[0]


def pack_features(rows: np.ndarray, family=None, default_family: int = 0):
    """64-byte packed rows (family inside) + the 16-double activation table."""
    rows = np.ascontiguousarray(rows, abi.feature_row_dtype)
    fam = None if family is None else np.ascontiguousarray(family, np.int8)
    out = np.zeros(len(rows), abi.feature_packed_dtype)
    table = np.zeros(16, np.float64)
    check(lib.carma_pack_features(ptr(rows), ptr(fam), default_family, len(rows), ptr(table), ptr(out)))
    return out, table


def pack_features_bits(rows: np.ndarray, family=None, default_family: int = 0):
    """Frame-of-reference bit-packed rows: (u32 words incl. 2 padding words, schema)."""
    rows = np.ascontiguousarray(rows, abi.feature_row_dtype)
    fam = None if family is None else np.ascontiguousarray(family, np.int8)
    schema = np.zeros(1, abi.bit_schema_dtype)
    nw = ctypes.c_uint64()
    check(lib.carma_pack_features_bits(ptr(rows), ptr(fam), default_family, len(rows), ptr(schema), None,
                                       ctypes.byref(nw)))
    words = np.zeros(nw.value, np.uint32)
    check(lib.carma_pack_features_bits(ptr(rows), ptr(fam), default_family, len(rows), ptr(schema), ptr(words),
                                       ctypes.byref(nw)))
    return words, schema


def pack_features_compact(rows: np.ndarray, family=None, default_family: int = 0):
    """The fixed-schema 40-byte rows the host-buffer predicts ship: (u32 words
    incl. 2 padding words, schema); CarmaError(UNSUPPORTED) if a row does not fit."""
    rows = np.ascontiguousarray(rows, abi.feature_row_dtype)
    fam = None if family is None else np.ascontiguousarray(family, np.int8)
    schema = np.zeros(1, abi.bit_schema_dtype)
    words = np.zeros(len(rows) * 10 + 2, np.uint32)
    check(lib.carma_pack_features_compact(ptr(rows), ptr(fam), default_family, len(rows), ptr(schema), ptr(words)))
    return words, schema


def scalar_features(rows: np.ndarray) -> np.ndarray:
    out = np.zeros((len(rows), 19), np.float64)
    rows = np.ascontiguousarray(rows)
    check(lib.carma_host_scalar_features(ptr(rows), len(rows), ptr(out)))
    return out


@dataclasses.dataclass
class HoldoutReport:
    accuracy: float = 0.0
    macro_f1: float = 0.0
    train_size: int = 0
    holdout_size: int = 0
    underestimate_rate: float = 0.0


@dataclasses.dataclass
class KnnModel:
    family: int
    k: int
    bucket_range: int
    lo: np.ndarray
    hi: np.ndarray
    points: np.ndarray   # n x 19 normalised
    labels: np.ndarray   # int32
    holdout_rows: np.ndarray
    seed: int = 0


def fit_knn(family: int, samples: int, seed: int, k: int = 5) -> KnnModel:
    lo = np.zeros(19)
    hi = np.zeros(19)
    pts = np.zeros((samples, 19))
    lab = np.zeros(samples, np.int32)
    hold = np.zeros(samples, np.uint64)
    n, br, nh = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    check(lib.carma_host_fit(family, samples, seed, k, ptr(lo), ptr(hi), ptr(pts), ptr(lab), samples,
                             ctypes.byref(n), ctypes.byref(br), ptr(hold), ctypes.byref(nh)))
    m = KnnModel(family, k, br.value, lo, hi, pts[: n.value].copy(), lab[: n.value].copy(),
                 hold[: nh.value].astype(np.int64), seed)
    m.samples = samples
    return m


def parse_snapshot(text) -> KnnModel:
    """A LearnedEstimator snapshot ("carma-knn-estimator/v1" JSON, the file
    LearnedEstimator::save writes, estimators.cpp:481-538) as a KnnModel."""
    raw = text.encode() if isinstance(text, str) else bytes(text)
    n, k, br, seed = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    fam = ctypes.c_int32()
    check(lib.carma_host_parse_snapshot(raw, len(raw), ctypes.byref(fam), ctypes.byref(k), ctypes.byref(br),
                                        ctypes.byref(seed), None, None, None, None, 0, ctypes.byref(n), None))
    lo, hi = np.zeros(19), np.zeros(19)
    pts = np.zeros((n.value, 19))
    lab = np.zeros(n.value, np.int32)
    hold = np.zeros(1, abi.holdout_report_dtype)
    check(lib.carma_host_parse_snapshot(raw, len(raw), None, None, None, None, ptr(lo), ptr(hi), ptr(pts), ptr(lab),
                                        n.value, ctypes.byref(n), ptr(hold)))
    m = KnnModel(fam.value, k.value, br.value, lo, hi, pts, lab, np.zeros(0, np.int64), seed.value)
    m.holdout = hold[0]
    return m


class GpuKnn:
    """A device-resident bank of k-NN models, one per family (the drop-in for
    Manager::set_learned_estimators + estimate_learned, manager.cpp:91-97)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        check(lib.carma_knn_create(device, ctypes.byref(h)))
        self._h = h
        self.models: Dict[int, KnnModel] = {}

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def set_model(self, m: KnnModel) -> None:
        pts = np.ascontiguousarray(m.points, np.float64)
        check(lib.carma_knn_set_model(self._h, m.family, ptr(m.lo), ptr(m.hi), ptr(pts), ptr(m.labels), len(m.labels),
                                      m.k, m.bucket_range))
        self.models[m.family] = m

    def load_snapshot(self, path: str) -> int:
        """LearnedEstimator::load straight into the bank (carma_knn_load_snapshot_file);
        returns the snapshot's family."""
        fam = ctypes.c_int32()
        check(lib.carma_knn_load_snapshot_file(self._h, path.encode(), ctypes.byref(fam), None))
        with open(path, "rb") as f:
            self.models[fam.value] = parse_snapshot(f.read())
        return fam.value

    def predict(self, rows: np.ndarray, family=None, default_family: Optional[int] = None):
        """Buckets and upper-edge bytes for feature rows (or raw n x 19 scalar rows)."""
        q = len(rows)
        bucket = np.zeros(q, np.int32)
        nbytes = np.zeros(q, np.uint64)
        fam = None if family is None else np.ascontiguousarray(family, np.int8)
        dflt = default_family if default_family is not None else next(iter(self.models))
        rows = np.ascontiguousarray(rows)
        if rows.dtype == abi.feature_row_dtype:
            check(lib.carma_knn_predict(self._h, ptr(rows), ptr(fam), dflt, q, ptr(bucket), ptr(nbytes)))
        else:
            rows = np.ascontiguousarray(rows, np.float64)
            check(lib.carma_knn_predict_scalar(self._h, ptr(rows), ptr(fam), dflt, q, ptr(bucket), ptr(nbytes)))
        return bucket, nbytes

    def predict_packed(self, packed: np.ndarray, table: np.ndarray):
        q = len(packed)
        bucket = np.zeros(q, np.int32)
        nbytes = np.zeros(q, np.uint64)
        check(lib.carma_knn_predict_packed(self._h, ptr(np.ascontiguousarray(packed)), ptr(table), q, ptr(bucket),
                                           ptr(nbytes)))
        return bucket, nbytes

    def predict_bitpacked(self, words: np.ndarray, schema: np.ndarray, q: int):
        bucket = np.zeros(q, np.int32)
        nbytes = np.zeros(q, np.uint64)
        check(lib.carma_knn_predict_bitpacked(self._h, ptr(np.ascontiguousarray(words, np.uint32)), ptr(schema), q,
                                              ptr(bucket), ptr(nbytes)))
        return bucket, nbytes

    def last_stats(self):
        la, ev = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.carma_knn_last_stats(self._h, ctypes.byref(la), ctypes.byref(ev)))
        return la.value, ev.value

    def close(self) -> None:
        if self._h:
            lib.carma_knn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LearnedEstimator:
    """train_learned_estimator's product (estimators.hpp:108-133) on the GPU."""

    def __init__(self, model: KnnModel, knn: GpuKnn, holdout: HoldoutReport):
        self.model = model
        self.knn = knn
        self.holdout = holdout

    @property
    def family(self) -> int:
        return self.model.family

    @property
    def bucket_range(self) -> int:
        return self.model.bucket_range

    def predict(self, rows: np.ndarray) -> np.ndarray:
        return self.knn.predict(rows, default_family=self.model.family)[0]

    def save(self, path: str) -> None:
        """LearnedEstimator::save (estimators.cpp:481-501): the
        "carma-knn-estimator/v1" JSON snapshot, same keys and order; doubles
        in shortest round-trip form, so LearnedEstimator::load (and
        carma_knn_load_snapshot) read back the identical state."""
        m, h = self.model, self.holdout
        names = {0: "mlp", 1: "cnn", 2: "transformer"}
        doc = {"schema": "carma-knn-estimator/v1", "family": names[m.family], "bucket_range": int(m.bucket_range),
               "k": int(m.k), "seed": int(m.seed), "lo": [float(x) for x in m.lo], "hi": [float(x) for x in m.hi],
               "labels": [int(x) for x in m.labels], "points": [[float(x) for x in p] for p in m.points],
               "holdout": {"accuracy": float(h.accuracy), "macro_f1": float(h.macro_f1),
                           "train_size": int(h.train_size), "holdout_size": int(h.holdout_size),
                           "underestimate_rate": float(h.underestimate_rate)}}
        import json
        with open(path, "w") as f:
            f.write(json.dumps(doc, indent=2) + "\n")


def train_learned_estimator(family: int, samples: int, seed: int, k: int = 5, device: int = 0,
                            knn: Optional[GpuKnn] = None) -> LearnedEstimator:
    """train_learned_estimator (estimators.cpp:344-436) on the GPU for
    generate_synthetic_dataset(family, samples, seed): the bounds, normalised
    points, holdout predictions and holdout counts on the device
    (carma_knn_train); the model is installed in `knn`'s bank."""
    ds = generate_synthetic_dataset(family, samples, seed)
    knn = knn or GpuKnn(device)
    order = np.zeros(samples, np.uint64)
    tn = ctypes.c_uint64()
    check(lib.carma_host_split_order(samples, seed, ptr(order), ctypes.byref(tn)))
    n_train = tn.value
    lo, hi = np.zeros(19), np.zeros(19)
    pts, lab = np.zeros((n_train, 19)), np.zeros(n_train, np.int32)
    rep = np.zeros(1, abi.holdout_report_dtype)
    check(lib.carma_knn_train(knn.handle, family, ptr(ds.rows), ptr(ds.bucket), ptr(ds.mem), samples, seed, k,
                              ds.bucket_range, ptr(rep), ptr(lo), ptr(hi), ptr(pts), ptr(lab)))
    m = KnnModel(family, k, ds.bucket_range, lo, hi, pts, lab, order[n_train:].astype(np.int64), seed)
    knn.models[family] = m
    r = rep[0]
    return LearnedEstimator(m, knn, HoldoutReport(float(r["accuracy"]), float(r["macro_f1"]), int(r["train_size"]),
                                                  int(r["holdout_size"]), float(r["underestimate_rate"])))


# ---------------------------------------------------------------- replay


@dataclasses.dataclass
class SimConstants:
    gpu_capacity: int = 40 * abi.GiB
    gpu_count: int = 4
    alloc_block: int = 512 * abi.MiB
    p_idle_w: float = 55.0
    p_max_w: float = 400.0
    p_boost_w: float = 30.0
    boost_threshold: float = 0.9
    oom_startup_delay: float = 5.0


@dataclasses.dataclass
class PolicyConfig:
    policy: str = "magm"
    max_smact: float = 0.80
    min_free_mem: Optional[int] = None
    safety_margin: int = 2 * abi.GiB
    estimator: str = "none"
    collocation_mode: str = "mps"
    monitor_window: float = 60.0
    rr_apply_preconditions: bool = False


def make_config(policy: PolicyConfig, consts: SimConstants, mig_instances: Optional[Sequence[float]] = None,
                sample_interval: float = 0.0, log_flags: int = 0) -> np.ndarray:
    """carma_replay_config of a PolicyConfig + SimConstants (+ RunConfig::mig_instances and, when > 0,
    the timeline's sample_interval, runner.hpp:23-33)."""
    c = np.zeros(1, abi.replay_config_dtype)
    c["policy"] = abi.POLICY[policy.policy]
    c["mode"] = abi.MODE[policy.collocation_mode]
    c["gpu_count"] = consts.gpu_count
    c["rr_apply_preconditions"] = int(policy.rr_apply_preconditions)
    c["max_smact"] = policy.max_smact
    c["min_free"] = policy.min_free_mem or 0
    c["monitor_window"] = policy.monitor_window
    c["gpu_capacity"] = consts.gpu_capacity
    c["alloc_block"] = consts.alloc_block
    c["p_idle_w"] = consts.p_idle_w
    c["p_max_w"] = consts.p_max_w
    c["p_boost_w"] = consts.p_boost_w
    c["boost_threshold"] = consts.boost_threshold
    c["oom_startup_delay"] = consts.oom_startup_delay
    c["sample_interval"] = sample_interval
    c["log_flags"] = log_flags
    if policy.collocation_mode == "mig":
        fr = np.ascontiguousarray([] if mig_instances is None else mig_instances, np.float64)
        check(lib.carma_mig_layout(ptr(fr) if len(fr) else None, len(fr), ptr(c)))
    return c


@dataclasses.dataclass
class ReplayResult:
    tasks: np.ndarray     # task_result_dtype, per job concatenated
    traces: np.ndarray    # trace_result_dtype, per job
    gpus: np.ndarray      # gpu_result_dtype, per job concatenated
    task_offsets: np.ndarray
    gpu_offsets: np.ndarray

    def job_tasks(self, j: int) -> np.ndarray:
        return self.tasks[self.task_offsets[j]: self.task_offsets[j + 1]]

    def job_gpus(self, j: int) -> np.ndarray:
        return self.gpus[self.gpu_offsets[j]: self.gpu_offsets[j + 1]]


class ReplayPlan:
    """Device-resident replay jobs (carma_replay_plan_*)."""

    def __init__(self, configs: np.ndarray, tasks: np.ndarray, trace_offsets: np.ndarray, jobs: np.ndarray,
                 device: int = 0, want_task_results: bool = True):
        self.configs = np.ascontiguousarray(configs, abi.replay_config_dtype)
        self.tasks = np.ascontiguousarray(tasks, abi.task_dtype)
        self.trace_offsets = np.ascontiguousarray(trace_offsets, np.uint64)
        self.jobs = np.ascontiguousarray(jobs, abi.job_dtype)
        h = ctypes.c_void_p()
        check(lib.carma_replay_plan_create(device, ptr(self.configs), len(self.configs), ptr(self.tasks),
                                           ptr(self.trace_offsets), len(self.trace_offsets) - 1, ptr(self.jobs),
                                           len(self.jobs), int(want_task_results), ctypes.byref(h)))
        self._h = h
        n_t = np.diff(self.trace_offsets.astype(np.int64))[self.jobs["trace"]]
        n_g = self.configs["gpu_count"][self.jobs["config"]].astype(np.int64)
        self.task_offsets = np.concatenate([[0], np.cumsum(n_t)])
        self.gpu_offsets = np.concatenate([[0], np.cumsum(n_g)])

    @classmethod
    def generated(cls, configs: np.ndarray, mix: str, seeds, jobs: np.ndarray, tables: Optional[np.ndarray] = None,
                  device: int = 0) -> "ReplayPlan":
        """A plan whose traces are generated on the device
        (carma_replay_plan_create_generated): trace k * len(seeds) + i is
        generate_trace(mix, seeds[i]) materialised with estimate table k (one
        u64 per catalog entry; None = no estimate)."""
        self = cls.__new__(cls)
        self.configs = np.ascontiguousarray(configs, abi.replay_config_dtype)
        self.jobs = np.ascontiguousarray(jobs, abi.job_dtype)
        seeds = np.ascontiguousarray(seeds, np.uint64)
        n_tables = 1 if tables is None else len(tables)
        tab = None if tables is None else np.ascontiguousarray(tables, np.uint64)
        rows = 90 if mix == "t90" else 60
        self.trace_offsets = (np.arange(n_tables * len(seeds) + 1, dtype=np.uint64) * np.uint64(rows))
        self.tasks = None
        h = ctypes.c_void_p()
        check(lib.carma_replay_plan_create_generated(device, ptr(self.configs), len(self.configs), abi.MIX[mix],
                                                     ptr(seeds), len(seeds), ptr(tab), n_tables, ptr(self.jobs),
                                                     len(self.jobs), ctypes.byref(h)))
        self._h = h
        n_t = np.diff(self.trace_offsets.astype(np.int64))[self.jobs["trace"]]
        n_g = self.configs["gpu_count"][self.jobs["config"]].astype(np.int64)
        self.task_offsets = np.concatenate([[0], np.cumsum(n_t)])
        self.gpu_offsets = np.concatenate([[0], np.cumsum(n_g)])
        return self

    def device_tasks(self):
        """(tasks, catalog entries) of a generated plan, read back from the device."""
        n = int(self.trace_offsets[-1])
        t = np.zeros(n, abi.task_dtype)
        e = np.zeros(n, np.int32)
        check(lib.carma_replay_plan_tasks(self._h, ptr(t)))
        check(lib.carma_replay_plan_entries(self._h, ptr(e)))
        return t, e

    def set_estimates_device(self, dev_ptr: int) -> None:
        check(lib.carma_replay_plan_set_estimates_device(self._h, dev_ptr))

    def run(self, stream=None) -> None:
        """Runs every job. stream None: on the plan's own stream (results()
        waits for it); a torch stream / cudaStream_t: ordered after the work
        already queued there, and that stream's later work after the replay."""
        check(lib.carma_replay_plan_run(self._h, None if stream is None else abi.stream_arg(stream)))

    def upload_tasks(self, tasks: np.ndarray) -> None:
        check(lib.carma_replay_plan_upload_tasks(self._h, ptr(np.ascontiguousarray(tasks, abi.task_dtype))))

    def outcomes(self):
        """Compact per-task outcomes + trace reports + per-GPU results."""
        to = np.zeros(int(self.task_offsets[-1]), abi.task_outcome_dtype)
        jr = np.zeros(len(self.jobs), abi.trace_result_dtype)
        gr = np.zeros(int(self.gpu_offsets[-1]), abi.gpu_result_dtype)
        check(lib.carma_replay_plan_outcomes(self._h, ptr(to), ptr(jr), ptr(gr)))
        return to, jr, gr

    def results(self, tasks: bool = True) -> ReplayResult:
        tr = np.zeros(int(self.task_offsets[-1]) if tasks else 0, abi.task_result_dtype)
        jr = np.zeros(len(self.jobs), abi.trace_result_dtype)
        gr = np.zeros(int(self.gpu_offsets[-1]), abi.gpu_result_dtype)
        check(lib.carma_replay_plan_results(self._h, ptr(tr) if tasks else None, ptr(jr), ptr(gr)))
        return ReplayResult(tr, jr, gr, self.task_offsets, self.gpu_offsets)

    def set_timeline_capacity(self, rows_per_job: int) -> None:
        check(lib.carma_replay_plan_set_timeline_capacity(self._h, rows_per_job))

    def timeline(self, job: int) -> np.ndarray:
        """Timeline rows of `job` (timeline_row_dtype); raises if rows were dropped."""
        n = ctypes.c_uint64()
        check(lib.carma_replay_plan_timeline(self._h, job, None, 0, ctypes.byref(n)))
        rows = np.zeros(n.value, abi.timeline_row_dtype)
        check(lib.carma_replay_plan_timeline(self._h, job, ptr(rows), n.value, ctypes.byref(n)))
        if n.value > len(rows):
            raise abi.CarmaError(abi.CARMA_ERR_OVERFLOW, f"timeline capacity too small ({n.value} rows)")
        return rows

    def set_log_capacity(self, records_per_job: int) -> None:
        check(lib.carma_replay_plan_set_log_capacity(self._h, records_per_job))

    def log(self, job: int) -> np.ndarray:
        """Event / decision log records of `job` (log_record_dtype) in run order."""
        n = ctypes.c_uint64()
        check(lib.carma_replay_plan_log(self._h, job, None, 0, ctypes.byref(n)))
        recs = np.zeros(n.value, abi.log_record_dtype)
        check(lib.carma_replay_plan_log(self._h, job, ptr(recs), n.value, ctypes.byref(n)))
        if n.value > len(recs):
            raise abi.CarmaError(abi.CARMA_ERR_OVERFLOW, f"log capacity too small ({n.value} records)")
        return recs

    def stats(self):
        la, rt = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.carma_replay_plan_stats(self._h, ctypes.byref(la), ctypes.byref(rt)))
        return la.value, rt.value

    def close(self) -> None:
        if self._h:
            lib.carma_replay_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def replay(configs: np.ndarray, task_lists: Sequence[np.ndarray], jobs: Iterable = None,
           device: int = 0) -> ReplayResult:
    """One-shot batch replay: traces = task_lists, jobs = [(trace, config)] (default: all x all)."""
    offs = np.concatenate([[0], np.cumsum([len(t) for t in task_lists])]).astype(np.uint64)
    tasks = np.concatenate(task_lists) if len(task_lists) > 1 else np.ascontiguousarray(task_lists[0])
    if jobs is None:
        jobs = [(t, c) for c in range(len(configs)) for t in range(len(task_lists))]
    jarr = np.array(list(jobs), dtype=np.uint32).reshape(-1, 2)
    j = np.zeros(len(jarr), abi.job_dtype)
    j["trace"] = jarr[:, 0]
    j["config"] = jarr[:, 1]
    plan = ReplayPlan(configs, tasks, offs, j, device)
    try:
        plan.run()
        res = plan.results()
    finally:
        plan.close()
    bad = res.traces["status"] != 0
    if bad.any():
        st = int(res.traces["status"][bad][0])
        raise abi.CarmaError(abi.CARMA_OK + (3 if st < 0 else st),
                             f"{int(bad.sum())} job(s) failed (first status {st})")
    return res


def predict_multi(knns: Sequence["GpuKnn"], rows: np.ndarray, family=None, default_family: int = 0):
    """carma_knn_predict_multi: rows sharded over the handles (one per device,
    models installed on each), one host thread per device, results gathered
    into one host buffer at the shard offsets."""
    q = len(rows)
    rows = np.ascontiguousarray(rows, abi.feature_row_dtype)
    fam = None if family is None else np.ascontiguousarray(family, np.int8)
    hs = (ctypes.c_void_p * len(knns))(*[k.handle.value for k in knns])
    bucket = np.zeros(q, np.int32)
    nbytes = np.zeros(q, np.uint64)
    check(lib.carma_knn_predict_multi(ctypes.cast(hs, ctypes.c_void_p), len(knns), ptr(rows), ptr(fam),
                                      default_family, q, ptr(bucket), ptr(nbytes)))
    return bucket, nbytes


def replay_multi(devices: Sequence[int], configs: np.ndarray, tasks: np.ndarray, trace_offsets: np.ndarray,
                 jobs: np.ndarray, task_results: bool = True) -> ReplayResult:
    """carma_replay_batch_multi: jobs sharded by task count over `devices`,
    one host thread + plan + stream per device, outputs in job order."""
    configs = np.ascontiguousarray(configs, abi.replay_config_dtype)
    tasks = np.ascontiguousarray(tasks, abi.task_dtype)
    offs = np.ascontiguousarray(trace_offsets, np.uint64)
    jobs = np.ascontiguousarray(jobs, abi.job_dtype)
    n_t = np.diff(offs.astype(np.int64))[jobs["trace"]]
    n_g = configs["gpu_count"][jobs["config"]].astype(np.int64)
    t_off = np.concatenate([[0], np.cumsum(n_t)])
    g_off = np.concatenate([[0], np.cumsum(n_g)])
    tr = np.zeros(int(t_off[-1]) if task_results else 0, abi.task_result_dtype)
    jr = np.zeros(len(jobs), abi.trace_result_dtype)
    gr = np.zeros(int(g_off[-1]), abi.gpu_result_dtype)
    dv = np.ascontiguousarray(devices, np.int32)
    check(lib.carma_replay_batch_multi(ptr(dv), len(dv), ptr(configs), len(configs), ptr(tasks), ptr(offs),
                                       len(offs) - 1, ptr(jobs), len(jobs), ptr(tr) if task_results else None,
                                       ptr(jr), ptr(gr)))
    return ReplayResult(tr, jr, gr, t_off, g_off)


# ----------------------------------------------------------------- runner


@dataclasses.dataclass
class RunConfig:
    """runner.hpp:18-40 (trace source, policy, constants, estimator provisioning)."""

    mix: Optional[str] = None  # runner.hpp:20: unset by default; trace_path is used when mix is not set
    trace_seed: int = 1
    trace_path: Optional[str] = None
    policy: PolicyConfig = dataclasses.field(default_factory=PolicyConfig)
    constants: SimConstants = dataclasses.field(default_factory=SimConstants)
    estimator_seed: int = 11
    estimator_k: int = 5
    estimator_samples: int = 4000
    mig_instances: List[float] = dataclasses.field(default_factory=list)  # fractions, mig mode only
    enable_timeline: bool = False
    sample_interval: float = 10.0
    enable_event_log: bool = False
    verbose_decisions: bool = False


def provision_estimates(rc: RunConfig, m: Materialized, device: int = 0,
                        knn: Optional[GpuKnn] = None) -> None:
    """make_estimate for every task (manager.cpp:80-107); learned via the GPU k-NN bank
    trained like provision_estimators (runner.cpp:17-38)."""
    est = rc.policy.estimator
    if est == "neural":
        # The paper's neural GPUMemNet (gpumemnet.py), an estimator kind the
        # reference does not ship; families without a model get no estimate.
        from .gpumemnet import GpuMemNet, load_default_models
        net = GpuMemNet(device)
        try:
            for mdl in load_default_models().values():
                net.set_model(mdl)
            _, nbytes = net.predict(m.features, family=m.family)
        finally:
            net.close()
        m.tasks["estimate"] = nbytes
        return
    if est != "learned":
        set_persona_estimates(m, est, rc.policy.safety_margin)
        return
    knn = knn or GpuKnn(device)
    for fam in sorted(set(m.family.tolist())):
        seed = rc.estimator_seed + fam * 101
        have = knn.models.get(fam)
        # provision_estimators (runner.cpp:17-38) trains per config: a bank
        # model trained with other settings is replaced, not reused
        if have is None or (have.seed, have.k, getattr(have, "samples", None)) != \
                (seed, rc.estimator_k, rc.estimator_samples):
            knn.set_model(fit_knn(fam, rc.estimator_samples, seed, rc.estimator_k))
    _, nbytes = knn.predict(m.features, family=m.family)
    m.tasks["estimate"] = nbytes


def entry_estimates(rc: RunConfig, device: int = 0, knn: Optional[GpuKnn] = None) -> np.ndarray:
    """make_estimate of every catalog entry (one u64 each) under rc's estimator:
    estimates are functions of the catalog entry, so a generated trace takes
    its tasks' estimates from this table."""
    n = lib.carma_host_catalog_size()
    tr = Trace(np.zeros(n), np.arange(n, dtype=np.int32), np.ones(n, np.uint64))
    m = materialize_trace(tr)
    provision_estimates(rc, m, device, knn)
    return m.tasks["estimate"].copy()


def _run_trace(rc: "RunConfig"):
    """run_simulation's trace source (runner.cpp:42-55): the mix when set,
    else the trace file, else ConfigError."""
    if rc.mix:
        return generate_trace(rc.mix, rc.trace_seed)
    if not rc.trace_path:
        raise abi.CarmaError(abi.CARMA_ERR_INVALID, "ConfigError: run needs either a trace path or a mix+seed")
    return load_trace(rc.trace_path)


def run_simulation(rc: RunConfig, device: int = 0, knn: Optional[GpuKnn] = None):
    """Replays one trace on the GPU; returns (trace result, task results, gpu results)."""
    trace = _run_trace(rc)
    m = materialize_trace(trace)
    provision_estimates(rc, m, device, knn)
    res = replay(make_config(rc.policy, rc.constants, rc.mig_instances), [m.tasks], device=device)
    return res.traces[0], res.job_tasks(0), res.job_gpus(0)


TIMELINE_HEADER = "t,gpu,smact,mem_used_bytes,power_w"  # runner.cpp:81


def format_timeline(rows: np.ndarray) -> List[str]:
    """World::emit_timeline_row's text (world.cpp:210-219), header first."""
    return [TIMELINE_HEADER] + ["%.3f,%d,%.4f,%d,%.2f" % (r["t"], r["gpu"], r["smact"], r["used"], r["power_w"])
                                for r in rows]


_POLICY_NAMES = {v: k for k, v in abi.POLICY.items()}


def task_ids(m: "Materialized") -> List[str]:
    """TaskSpec ids of materialize_trace (traces.cpp:374): t%03zu-<catalog key>."""
    keys = [e.key for e in builtin_catalog()]
    return ["t%03d-%s" % (i, keys[e]) for i, e in enumerate(m.entry.tolist())]


def format_logs(recs: np.ndarray, ids: Sequence[str]):
    """(event_log, decision_log) lines exactly as World::log_event
    (world.cpp:94-153) and the decision log (manager.cpp:298-318) print them."""
    events, decisions = [], []
    for r in recs:
        t, task, kind = float(r["t"]), ids[int(r["task"])], int(r["kind"])
        if kind == abi.REC_PLACE:
            events.append("t=%.3f ev=place task=%s gpus=%d" % (t, task, int(r["gpu"])))
        elif kind == abi.REC_COMPLETE:
            events.append("t=%.3f ev=complete task=%s" % (t, task))
        elif kind == abi.REC_OOM:
            events.append("t=%.3f ev=alloc_oom gpu=%d task=%s req=%d free=%d largest=%d"
                          % (t, int(r["gpu"]), task, int(r["a"]), int(r["b"]), int(r["c"])))
        else:
            gpu = "defer" if int(r["gpu"]) < 0 else "%d" % int(r["gpu"])
            decisions.append("t=%.3f decide task=%s policy=%s gpu=%s est_bytes=%d"
                             % (t, task, _POLICY_NAMES[int(r["policy"])], gpu, int(r["a"])))
    return events, decisions


@dataclasses.dataclass
class RunArtifacts:
    """run_simulation's artifacts (runner.hpp:38-47): report scalars, per-task and per-GPU results,
    and the timeline / event log / decision log text when the RunConfig switches are set."""

    report: np.ndarray
    tasks: np.ndarray
    gpus: np.ndarray
    timeline: List[str]
    event_log: List[str] = dataclasses.field(default_factory=list)
    decision_log: List[str] = dataclasses.field(default_factory=list)


def run_simulation_artifacts(rc: RunConfig, device: int = 0, knn: Optional[GpuKnn] = None,
                             timeline_rows: int = 1 << 20, log_records: int = 1 << 20) -> RunArtifacts:
    """run_simulation with the reference's output switches: the sample ticks of
    enable_timeline are events of the replay (they split the energy integration
    exactly as in the reference), their rows come back formatted."""
    trace = _run_trace(rc)
    m = materialize_trace(trace)
    provision_estimates(rc, m, device, knn)
    flags = (abi.LOG_EVENTS if rc.enable_event_log else 0) | (abi.LOG_DECISIONS if rc.verbose_decisions else 0)
    cfg = make_config(rc.policy, rc.constants, rc.mig_instances, rc.sample_interval if rc.enable_timeline else 0.0,
                      flags)
    jobs = np.zeros(1, abi.job_dtype)
    plan = ReplayPlan(cfg, m.tasks, np.array([0, len(m.tasks)], np.uint64), jobs, device)
    try:
        if rc.enable_timeline:
            plan.set_timeline_capacity(timeline_rows)
        if flags:
            plan.set_log_capacity(log_records)
        plan.run()
        res = plan.results()
        tl = format_timeline(plan.timeline(0)) if rc.enable_timeline else []
        ev, dec = format_logs(plan.log(0), task_ids(m)) if flags else ([], [])
    finally:
        plan.close()
    st = int(res.traces["status"][0])
    if st != 0:
        raise abi.CarmaError(3 if st < 0 else st, f"run failed (status {st})")
    return RunArtifacts(res.traces[0], res.job_tasks(0), res.job_gpus(0), tl, ev, dec)


class FusedReplay:
    """Estimator-in-the-loop replay (BASELINE c5): the GPUMemNet k-NN pre-pass
    over every arrival writes each task's estimate on the device, and the
    replay reads it there (carma_replay_plan_set_estimates_device) — the
    estimate is a pure function of the task, so a pre-pass gives the bins
    make_estimate computes on every dispatch attempt (manager.cpp:292-294)."""

    def __init__(self, m: "Materialized", cfg: np.ndarray, knn, device: int = 0):
        """knn: a GpuKnn (the reference's learned estimator) or a
        gpumemnet.GpuMemNet (the paper's neural one)."""
        import torch
        self.m, self.cfg, self.knn, self.device = m, cfg, knn, device
        self.neural = not isinstance(knn, GpuKnn)
        self.packed, self.table = pack_features(m.features, m.family)
        if self.neural:
            knn.set_act_table(self.table)
        else:
            abi.check(lib.carma_knn_set_act_table(knn.handle, ptr(self.table)))
        self.d_rows = torch.from_numpy(self.packed.view(np.uint8).reshape(-1)).to(f"cuda:{device}")
        self.d_bucket = torch.empty(len(m.tasks), dtype=torch.int32, device=f"cuda:{device}")
        self.d_bytes = torch.empty(len(m.tasks), dtype=torch.int64, device=f"cuda:{device}")
        # one stream orders the estimator pre-pass before the replay that reads its bytes
        self.stream = torch.cuda.Stream(device)
        jobs = np.zeros(1, abi.job_dtype)
        self.plan = ReplayPlan(cfg, m.tasks, np.array([0, len(m.tasks)], np.uint64), jobs, device)
        self.plan.set_estimates_device(self.d_bytes.data_ptr())

    def run(self, stream=None) -> None:
        """Pre-pass then replay, both on the replay's own stream; `stream`
        (default: torch's current stream) waits for both."""
        import torch
        caller = torch.cuda.current_stream(self.device) if stream is None else stream
        s = self.stream
        s.wait_stream(caller)  # inputs the caller wrote before this call
        if self.neural:
            self.knn.predict_device(self.d_rows, abi.ROWS_PACKED, len(self.m.tasks), self.d_bucket, self.d_bytes,
                                    stream=s)
        else:
            check(lib.carma_knn_predict_device(self.knn.handle, self.d_rows.data_ptr(), abi.ROWS_PACKED, None, 0,
                                               len(self.m.tasks), self.d_bucket.data_ptr(), self.d_bytes.data_ptr(),
                                               None, None, abi.stream_arg(s)))
        self.plan.run(s)
        if hasattr(caller, "wait_stream"):
            caller.wait_stream(s)

    def results(self) -> ReplayResult:
        return self.plan.results()

    def close(self) -> None:
        self.plan.close()


# ------------------------------------------------------------------ sweep


@dataclasses.dataclass
class RunReport:
    """RunReport scalars (metrics.hpp:44-57) of one replay."""

    trace_name: str
    config: PolicyConfig
    trace_total_time: float
    avg_wait: float
    avg_exec: float
    avg_jct: float
    oom_count: int
    energy_mj: float


@dataclasses.dataclass
class SweepCell:
    """runner.hpp:54-57"""

    policy: PolicyConfig
    label: str = ""


@dataclasses.dataclass
class SweepConfig:
    """runner.hpp:59-64 (max_threads is accepted for parity; the GPU runs every cell x seed at once)."""

    base: RunConfig
    cells: List[SweepCell]
    seeds: List[int] = dataclasses.field(default_factory=lambda: [1])
    max_threads: int = 0


@dataclasses.dataclass
class SweepResult:
    """runner.hpp:66-69: reports[cell][seed] and the sweep CSV (per-seed rows + a median row per cell)."""

    reports: List[List[RunReport]]
    csv: str


_CSV_HEADER = ("policy,estimator,mode,max_smact,min_free_gib,window_s,seed,trace,"
               "total_time_s,avg_wait_s,avg_exec_s,avg_jct_s,oom_count,energy_mj")  # metrics.cpp:106-109


def _csv_row(rep: RunReport, seed_field: str) -> str:
    """runner.cpp:169-185 (printf formats reproduced with Python's % operator)."""
    c = rep.config
    min_free = "%.2f" % (c.min_free_mem / float(abi.GiB)) if c.min_free_mem is not None else "none"
    return "%s,%s,%s,%.2f,%s,%.0f,%s,%s,%.3f,%.3f,%.3f,%.3f,%d,%.2f" % (
        c.policy, c.estimator, c.collocation_mode, c.max_smact, min_free, c.monitor_window, seed_field,
        rep.trace_name, rep.trace_total_time, rep.avg_wait, rep.avg_exec, rep.avg_jct, rep.oom_count,
        rep.energy_mj)


def run_sweep(config: SweepConfig, device: int = 0, knn: Optional[GpuKnn] = None) -> SweepResult:
    """run_sweep (runner.cpp:192-283) on the GPU: every (cell, seed) run is one
    replay job of a single plan; any failed run aborts the sweep with the
    reference's message. Traces come from config.base (mix or trace file)."""
    if not config.cells:
        raise abi.CarmaError(abi.CARMA_ERR_INVALID, "ConfigError: sweep has no cells")
    if not config.seeds:
        raise abi.CarmaError(abi.CARMA_ERR_INVALID, "ConfigError: sweep has no seeds")
    base = config.base
    own_knn = knn is None and any(c.policy.estimator == "learned" for c in config.cells)
    if own_knn:
        knn = GpuKnn(device)
    task_lists, trace_of, names = [], {}, {}
    if not base.mix and not base.trace_path:
        raise abi.CarmaError(abi.CARMA_ERR_INVALID, "ConfigError: run needs either a trace path or a mix+seed")
    if base.mix in ("t90", "t60"):
        # Traces generated and materialised on the device, straight into the
        # plan; estimates by catalog entry, one table per (estimator, margin).
        try:
            keys = []
            for c in config.cells:
                k = (c.policy.estimator, c.policy.safety_margin)
                if k not in keys:
                    keys.append(k)
            tables = np.stack([entry_estimates(dataclasses.replace(base, policy=PolicyConfig(
                estimator=e, safety_margin=mg)), device, knn) for e, mg in keys])
            ns = len(config.seeds)
            j = np.zeros(len(config.cells) * ns, abi.job_dtype)
            for ci, c in enumerate(config.cells):
                k = keys.index((c.policy.estimator, c.policy.safety_margin))
                j["trace"][ci * ns:(ci + 1) * ns] = k * ns + np.arange(ns, dtype=np.uint32)
                j["config"][ci * ns:(ci + 1) * ns] = ci
            cfgs = np.concatenate([make_config(c.policy, base.constants, base.mig_instances) for c in config.cells])
            plan = ReplayPlan.generated(cfgs, base.mix, config.seeds, j, tables, device)
            try:
                plan.run()
                res = plan.results(tasks=False)
            finally:
                plan.close()
        finally:
            if own_knn:
                knn.close()
        names = {seed: f"{base.mix}-seed{seed}" for seed in config.seeds}
        return _sweep_result(config, res, names)
    try:
        for seed in config.seeds:
            if base.mix:
                trace, name = generate_trace(base.mix, seed), f"{base.mix}-seed{seed}"
            else:
                trace, name = load_trace(base.trace_path), base.trace_path
            names[seed] = name
            m = None
            for cell in config.cells:
                key = (seed, cell.policy.estimator, cell.policy.safety_margin)
                if key in trace_of:
                    continue
                m = materialize_trace(trace) if m is None else m
                mm = dataclasses.replace(m, tasks=m.tasks.copy())
                rc = dataclasses.replace(base, policy=cell.policy, trace_seed=seed)
                provision_estimates(rc, mm, device, knn)
                trace_of[key] = len(task_lists)
                task_lists.append(mm.tasks)
        cfgs = np.concatenate([make_config(c.policy, base.constants, base.mig_instances) for c in config.cells])
        jobs = [(trace_of[(seed, c.policy.estimator, c.policy.safety_margin)], ci)
                for ci, c in enumerate(config.cells) for seed in config.seeds]
        offs = np.concatenate([[0], np.cumsum([len(t) for t in task_lists])]).astype(np.uint64)
        jarr = np.array(jobs, dtype=np.uint32).reshape(-1, 2)
        j = np.zeros(len(jarr), abi.job_dtype)
        j["trace"], j["config"] = jarr[:, 0], jarr[:, 1]
        plan = ReplayPlan(cfgs, np.concatenate(task_lists), offs, j, device)
        try:
            plan.run()
            res = plan.results(tasks=False)
        finally:
            plan.close()
    finally:
        if own_knn:
            knn.close()
    return _sweep_result(config, res, names)


def _sweep_result(config: SweepConfig, res: ReplayResult, names) -> SweepResult:
    reports, k = [], 0
    for ci, cell in enumerate(config.cells):
        row = []
        for seed in config.seeds:
            t = res.traces[k]
            if int(t["status"]) != 0:
                label = cell.label or cell.policy.policy
                raise abi.CarmaError(abi.CARMA_ERR_INCOMPLETE if int(t["status"]) == abi.CARMA_ERR_INCOMPLETE
                                     else abi.CARMA_ERR_INVALID,
                                     f"sweep cell '{label}' seed {seed} failed: status {int(t['status'])}")
            row.append(RunReport(names[seed], cell.policy, float(t["trace_total_time"]), float(t["avg_wait"]),
                                 float(t["avg_exec"]), float(t["avg_jct"]), int(t["oom_count"]),
                                 float(t["energy_mj"])))
            k += 1
        reports.append(row)
    lines = [_CSV_HEADER]
    for row in reports:
        lines += [_csv_row(r, str(seed)) for r, seed in zip(row, config.seeds)]
        if len(config.seeds) > 1:  # metric-wise medians (runner.cpp:258-276)
            med = dataclasses.replace(
                row[0], trace_total_time=median([r.trace_total_time for r in row]),
                avg_wait=median([r.avg_wait for r in row]), avg_exec=median([r.avg_exec for r in row]),
                avg_jct=median([r.avg_jct for r in row]),
                oom_count=int(math.floor(median([float(r.oom_count) for r in row]) + 0.5)),  # llround, >= 0
                energy_mj=median([r.energy_mj for r in row]))
            lines.append(_csv_row(med, "median"))
    return SweepResult(reports, "\n".join(lines) + "\n")


def median(values) -> float:
    """runner.cpp:149-155"""
    v = sorted(values)
    n = len(v)
    if n == 0:
        return 0.0
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


# ------------------------------------------------------------------ pick


def pick_batch(cfg: np.ndarray, views: np.ndarray, reqs: np.ndarray, rr_cursor: np.ndarray, device: int = 0):
    """Batched eligible_gpus + map_task: views (n x G gpu_view), reqs (n pick_request)."""
    n, g = views.shape
    views = np.ascontiguousarray(views, abi.gpu_view_dtype)
    reqs = np.ascontiguousarray(reqs, abi.pick_request_dtype)
    cur = np.ascontiguousarray(rr_cursor, np.int32).copy()
    out = np.zeros((n, 2), np.int32)
    check(lib.carma_pick_batch(device, ptr(cfg), ptr(views), g, ptr(reqs), n, ptr(cur), ptr(out)))
    return out, cur
