"""ctypes binding of include/carma_gpu.h and include/carma_host.h.

Loads the in-tree ``libcarma_b200.so`` (built by ``__graft_entry__.build()``
or ``make -C paper_2508_19073_b200/csrc``). There is no fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_uint32, c_uint64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CARMA_B200_LIB") or os.path.join(_HERE, "libcarma_b200.so")  # override: A/B builds

CARMA_OK = 0
CARMA_ERR_INVALID, CARMA_ERR_CUDA, CARMA_ERR_OVERFLOW, CARMA_ERR_FAMILY = 1, 2, 3, 4
CARMA_ERR_UNSUPPORTED, CARMA_ERR_INCOMPLETE = 5, 6
STATUS_NAMES = {
    0: "OK", 1: "INVALID", 2: "CUDA", 3: "OVERFLOW", 4: "FAMILY", 5: "UNSUPPORTED", 6: "INCOMPLETE",
}

POLICY = {"exclusive": 0, "rr": 1, "magm": 2, "lug": 3, "mug": 4}
MODE = {"streams": 0, "mps": 1, "mig": 2}
FAMILY = {"mlp": 0, "cnn": 1, "transformer": 2}
ESTIMATOR = {"none": 0, "oracle": 1, "analytical": 2, "static_graph": 3, "learned": 4}
MIX = {"t90": 0, "t60": 1}
NO_ESTIMATE = np.uint64(0xFFFFFFFFFFFFFFFF)
ROWS_FEATURES, ROWS_SCALAR, ROWS_PACKED, ROWS_BITPACKED = 0, 1, 2, 3
GiB = 1 << 30
MiB = 1 << 20

feature_row_dtype = np.dtype([
    ("n_linear", "<u8"), ("n_batchnorm", "<u8"), ("n_dropout", "<u8"), ("n_conv", "<u8"),
    ("batch_size", "<u8"), ("total_params", "<u8"), ("total_activations", "<u8"),
    ("act_cos", "<f8"), ("act_sin", "<f8"), ("kind", "<i4", (3,)), ("has_layers", "<i4"),
    ("tuple_acts", "<u8", (3,)), ("tuple_params", "<u8", (3,)),
], align=True)

feature_packed_dtype = np.dtype([("w", "<u8", (8,))])

bit_schema_dtype = np.dtype([
    ("words_per_row", "<u4"), ("reserved", "<u4"), ("width", "u1", (20,)), ("offset", "<u2", (20,)),
    ("base", "<u8", (20,)), ("act_table", "<f8", (16,)),
], align=True)

task_outcome_dtype = np.dtype([
    ("final_dispatch", "<f8"), ("complete", "<f8"), ("ooms", "<u4"), ("attempts", "<u4"),
], align=True)

replay_config_dtype = np.dtype([
    ("policy", "<i4"), ("mode", "<i4"), ("gpu_count", "<i4"), ("rr_apply_preconditions", "<i4"),
    ("max_smact", "<f8"), ("min_free", "<u8"), ("monitor_window", "<f8"),
    ("gpu_capacity", "<u8"), ("alloc_block", "<u8"),
    ("p_idle_w", "<f8"), ("p_max_w", "<f8"), ("p_boost_w", "<f8"), ("boost_threshold", "<f8"),
    ("oom_startup_delay", "<f8"),
    ("mig_count", "<i4"), ("mig_reserved", "<i4"), ("mig_fraction", "<f8", (8,)),
    ("mig_base", "<u2", (8,)), ("mig_blocks", "<u2", (8,)), ("sample_interval", "<f8"),
    ("log_flags", "<i4"), ("log_reserved", "<i4"),
    ("mig_base_bytes", "<u8", (8,)), ("mig_cap_bytes", "<u8", (8,)),
], align=True)

dataset_stats_dtype = np.dtype([
    ("words_generated", "<u8"), ("rows_parsed", "<u8"), ("rows_accepted", "<u8"), ("rounds", "<u4"),
    ("reserved", "<u4"),
], align=True)

holdout_report_dtype = np.dtype([
    ("accuracy", "<f8"), ("macro_f1", "<f8"), ("underestimate_rate", "<f8"), ("train_size", "<u8"),
    ("holdout_size", "<u8"),
], align=True)

log_record_dtype = np.dtype([
    ("t", "<f8"), ("a", "<u8"), ("b", "<u8"), ("c", "<u8"), ("task", "<u4"), ("gpu", "<i2"), ("kind", "u1"),
    ("policy", "u1"),
], align=True)
LOG_EVENTS, LOG_DECISIONS = 1, 2
REC_PLACE, REC_COMPLETE, REC_OOM, REC_DECIDE = 0, 1, 2, 3

timeline_row_dtype = np.dtype([
    ("t", "<f8"), ("smact", "<f8"), ("power_w", "<f8"), ("used", "<u8"), ("gpu", "<i4"), ("reserved", "<i4"),
], align=True)

task_dtype = np.dtype([
    ("submit", "<f8"), ("work", "<f8"), ("demand", "<f8"), ("true_mem", "<u8"),
    ("estimate", "<u8"), ("gpus", "<u4"), ("rank", "<u4"),
], align=True)

task_result_dtype = np.dtype([
    ("first_attempt", "<f8"), ("final_dispatch", "<f8"), ("complete", "<f8"),
    ("first_crash", "<f8"), ("last_crash", "<f8"), ("executed", "<f8"),
    ("attempts", "<u4"), ("ooms", "<u4"), ("gpu", "<i2", (2,)), ("reserved", "<u4"),
], align=True)

trace_result_dtype = np.dtype([
    ("trace_total_time", "<f8"), ("avg_wait", "<f8"), ("avg_exec", "<f8"), ("avg_jct", "<f8"),
    ("energy_mj", "<f8"), ("first_submit", "<f8"), ("last_complete", "<f8"), ("end_time", "<f8"),
    ("oom_count", "<i4"), ("status", "<i4"), ("events", "<u8"),
], align=True)

gpu_result_dtype = np.dtype([
    ("energy_j", "<f8"), ("mean_smact", "<f8"), ("peak_used", "<u8"), ("smact_steps", "<u8"),
], align=True)

job_dtype = np.dtype([("trace", "<u4"), ("config", "<u4")], align=True)

gpu_view_dtype = np.dtype([
    ("total_free", "<u8"), ("windowed_smact", "<f8"), ("idle", "<i4"), ("reserved", "<i4"),
], align=True)

pick_request_dtype = np.dtype([
    ("estimate", "<u8"), ("want", "<u4"), ("from_recovery", "<i4"),
], align=True)

nn_spec_dtype = np.dtype([
    ("members", "<u4"), ("classes", "<u4"), ("bucket_range", "<u8"), ("depth", "<u4", (8,)),
    ("width", "<u4", (8, 8)), ("log_mask", "<u4"), ("arch", "<u4"), ("shift", "<f4", (19,)),
    ("scale", "<f4", (19,)),
], align=True)
NN_MAX_MEMBERS, NN_MAX_DEPTH, NN_MAX_WIDTH, NN_MAX_CLASSES = 8, 8, 8, 48

assert nn_spec_dtype.itemsize == 464
assert feature_row_dtype.itemsize == 136
assert feature_packed_dtype.itemsize == 64
assert task_outcome_dtype.itemsize == 24
assert replay_config_dtype.itemsize == 344
assert task_dtype.itemsize == 48
assert task_result_dtype.itemsize == 64
assert trace_result_dtype.itemsize == 80
assert gpu_result_dtype.itemsize == 32
assert gpu_view_dtype.itemsize == 24
assert pick_request_dtype.itemsize == 16

P = c_void_p  # every array crosses as a raw pointer

# name -> (restype, argtypes); mirrors the two headers exactly.
SIGNATURES = {
    # carma_gpu.h
    "carma_last_error": (c_char_p, []),
    "carma_version": (c_int, []),
    "carma_device_count": (c_int, []),
    "carma_knn_create": (c_int, [c_int, POINTER(c_void_p)]),
    "carma_knn_destroy": (c_int, [c_void_p]),
    "carma_knn_set_model": (c_int, [c_void_p, c_int32, P, P, P, P, c_uint64, c_uint32, c_uint64]),
    "carma_knn_predict": (c_int, [c_void_p, P, P, c_int32, c_uint64, P, P]),
    "carma_knn_predict_scalar": (c_int, [c_void_p, P, P, c_int32, c_uint64, P, P]),
    "carma_knn_predict_packed": (c_int, [c_void_p, P, P, c_uint64, P, P]),
    "carma_knn_set_act_table": (c_int, [c_void_p, P]),
    "carma_pack_features": (c_int, [P, P, c_int32, c_uint64, P, P]),
    "carma_pack_features_bits": (c_int, [P, P, c_int32, c_uint64, P, P, POINTER(c_uint64)]),
    "carma_pack_features_compact": (c_int, [P, P, c_int32, c_uint64, P, P]),
    "carma_knn_predict_bitpacked": (c_int, [c_void_p, P, P, c_uint64, P, P]),
    "carma_knn_set_bit_schema": (c_int, [c_void_p, P]),
    "carma_replay_plan_upload_tasks": (c_int, [c_void_p, P]),
    "carma_replay_plan_outcomes": (c_int, [c_void_p, P, P, P]),
    "carma_knn_predict_device": (c_int, [c_void_p, P, c_int32, P, c_int32, c_uint64, P, P, P, P, c_void_p]),
    "carma_knn_last_stats": (c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64)]),
    "carma_knn_last_work": (c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64)]),
    "carma_knn_set_path": (c_int, [c_void_p, c_int32]),
    "carma_knn_last_timing": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double)]),
    "carma_replay_plan_timing": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double)]),
    "carma_probe_fp64": (c_int, [c_int, POINTER(c_double)]),
    "carma_probe_fp32": (c_int, [c_int, POINTER(c_double)]),
    "carma_replay_plan_create": (c_int, [c_int, P, c_uint32, P, P, c_uint32, P, c_uint32, c_int32,
                                         POINTER(c_void_p)]),
    "carma_replay_plan_set_estimates_device": (c_int, [c_void_p, P]),
    "carma_replay_plan_run": (c_int, [c_void_p, c_void_p]),
    "carma_replay_plan_results": (c_int, [c_void_p, P, P, P]),
    "carma_replay_plan_stats": (c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64)]),
    "carma_replay_plan_destroy": (c_int, [c_void_p]),
    "carma_replay_batch": (c_int, [c_int, P, c_uint32, P, P, c_uint32, P, c_uint32, P, P, P]),
    "carma_pick_batch": (c_int, [c_int, P, P, c_uint32, P, c_uint64, P, P]),
    "carma_pick_batch_device": (c_int, [c_int, P, P, c_uint32, P, c_uint64, P, P, c_void_p]),
    "carma_replay_plan_set_timeline_capacity": (c_int, [c_void_p, c_uint64]),
    "carma_replay_plan_timeline": (c_int, [c_void_p, c_uint32, P, c_uint64, POINTER(c_uint64)]),
    "carma_replay_plan_set_log_capacity": (c_int, [c_void_p, c_uint64]),
    "carma_nn_param_count": (c_uint64, [P]),
    "carma_nn_create": (c_int, [c_int, POINTER(c_void_p)]),
    "carma_nn_destroy": (c_int, [c_void_p]),
    "carma_nn_set_model": (c_int, [c_void_p, c_int32, P, P, c_uint64]),
    "carma_nn_set_act_table": (c_int, [c_void_p, P]),
    "carma_nn_set_path": (c_int, [c_void_p, c_int32]),
    "carma_nn_set_bit_schema": (c_int, [c_void_p, P]),
    "carma_nn_predict_device": (c_int, [c_void_p, P, c_int32, P, c_int32, c_uint64, P, P, P, P, c_void_p]),
    "carma_nn_predict": (c_int, [c_void_p, P, P, c_int32, c_uint64, P, P]),
    "carma_nn_predict_bitpacked": (c_int, [c_void_p, P, P, c_uint64, P, P]),
    "carma_nn_last_timing": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_uint64),
                                     POINTER(c_uint64)]),
    "carma_replay_plan_create_generated": (c_int, [c_int, P, c_uint32, c_int32, P, c_uint32, P, c_uint32, P, c_uint32,
                                                   POINTER(c_void_p)]),
    "carma_replay_plan_entries": (c_int, [c_void_p, P]),
    "carma_replay_plan_tasks": (c_int, [c_void_p, P]),
    "carma_pick_batch_wide": (c_int, [c_int, P, P, c_uint32, P, c_uint64, P, P]),
    "carma_replay_plan_set_outcome_sink": (c_int, [c_void_p, P]),
    "carma_knn_last_h2d_bytes": (c_int, [c_void_p, POINTER(c_uint64)]),
    "carma_nn_last_h2d_bytes": (c_int, [c_void_p, POINTER(c_uint64)]),
    "carma_dataset_generate_device": (c_int, [c_int32, c_int32, c_uint64, c_uint64, P, P, P, c_void_p, P]),
    "carma_dataset_generate": (c_int, [c_int32, c_int32, c_uint64, c_uint64, P, P, P, P]),
    "carma_knn_train": (c_int, [c_void_p, c_int32, P, P, P, c_uint64, c_uint64, c_uint32, c_uint64, P, P, P, P, P]),
    "carma_host_split_order": (c_int, [c_uint64, c_uint64, P, POINTER(c_uint64)]),
    "carma_replay_plan_log": (c_int, [c_void_p, c_uint32, P, c_uint64, POINTER(c_uint64)]),
    "carma_shard_ranges": (c_int, [P, c_uint64, c_uint32, P]),
    "carma_knn_predict_multi": (c_int, [P, c_uint32, P, P, c_int32, c_uint64, P, P]),
    "carma_nn_predict_multi": (c_int, [P, c_uint32, P, P, c_int32, c_uint64, P, P]),
    "carma_replay_batch_multi": (c_int, [P, c_uint32, P, c_uint32, P, P, c_uint32, P, c_uint32, P, P, P]),
    "carma_knn_load_snapshot": (c_int, [c_void_p, c_char_p, c_uint64, POINTER(c_int32), P]),
    "carma_knn_load_snapshot_file": (c_int, [c_void_p, c_char_p, POINTER(c_int32), P]),
    # carma_host.h
    "carma_host_check_log1p": (c_int, [c_uint64, c_uint64, POINTER(c_uint64)]),
    "carma_host_check_mt_jump": (c_int, [c_uint64, c_int32, POINTER(c_uint64)]),
    "carma_host_parse_snapshot": (c_int, [c_char_p, c_uint64, POINTER(c_int32), POINTER(c_uint64),
                                          POINTER(c_uint64), POINTER(c_uint64), P, P, P, P, c_uint64,
                                          POINTER(c_uint64), P]),
    "carma_host_catalog_size": (c_int, []),
    "carma_host_catalog_entry": (c_int, [c_int, c_char_p, c_int, P, P, P, P]),
    "carma_host_generate_trace": (c_int, [c_int32, c_uint64, P, P, P, c_uint64, POINTER(c_uint64)]),
    "carma_host_generate_uniform_trace": (c_int, [c_uint64, c_double, c_uint64, P, P, P]),
    "carma_host_save_trace": (c_int, [c_char_p, c_uint64, c_char_p, P, P, P, c_uint64]),
    "carma_host_load_trace": (c_int, [c_char_p, P, P, P, c_uint64, POINTER(c_uint64)]),
    "carma_host_materialize": (c_int, [P, P, P, c_uint64, P, P, P]),
    "carma_host_estimates": (c_int, [c_int32, c_uint64, P, c_uint64, P]),
    "carma_host_dataset": (c_int, [c_int32, c_uint64, c_uint64, P, P, P]),
    "carma_host_fit": (c_int, [c_int32, c_uint64, c_uint64, c_uint32, P, P, P, P, c_uint64,
                               POINTER(c_uint64), POINTER(c_uint64), P, POINTER(c_uint64)]),
    "carma_host_scalar_features": (c_int, [P, c_uint64, P]),
    "carma_mig_layout": (c_int, [P, c_uint32, P]),
}


class CarmaError(RuntimeError):
    """A non-OK carma_status; .status holds the code (reference: CarmaError, errors.hpp:12)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status != CARMA_OK:
        raise CarmaError(status, lib.carma_last_error().decode(errors="replace"))


def ptr(a) -> int | None:
    """Raw data pointer of a numpy array / torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays crossing the C ABI must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(f"cannot pass {type(a)} across the C ABI")


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


def stream_arg(stream=None, device: int | None = None) -> int:
    """The caller stream handed to a device-resident C ABI call.

    ``stream``: a torch.cuda.Stream, a raw cudaStream_t (int), or None for
    torch's current stream on ``device``. NULL would select the handle's own
    stream, which the caller's later work is not ordered after; the legacy
    default stream (handle 0) is therefore passed as cudaStreamLegacy."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(device)
    if hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    return int(stream) or CUDA_STREAM_LEGACY
