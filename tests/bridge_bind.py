"""ctypes binding of integration/_build/libcarma_bridge.so (the reference-side
bridge + its test entry points, integration/bridge_capi.cpp). Test
infrastructure only."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_uint64, c_void_p

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BRIDGE_SO = os.path.join(ROOT, "integration", "_build", "libcarma_bridge.so")

case_dtype = np.dtype([
    ("mix", "<i4"), ("policy", "<i4"), ("estimator", "<i4"), ("mode", "<i4"), ("seed", "<u8"),
    ("gpu_count", "<i4"), ("rr_pre", "<i4"), ("has_min_free", "<i4"), ("n_mig", "<i4"),
    ("max_smact", "<f8"), ("window", "<f8"), ("min_free", "<u8"), ("capacity", "<u8"), ("block", "<u8"),
    ("mig", "<f8", (8,)),
])
assert case_dtype.itemsize == 144

POLICY = {"exclusive": 0, "rr": 1, "magm": 2, "lug": 3, "mug": 4}
ESTIMATOR = {"none": 0, "oracle": 1, "analytical": 2, "static_graph": 3, "learned": 4}
MODE = {"streams": 0, "mps": 1, "mig": 2}
GiB, MiB = 1 << 30, 1 << 20


def load_bridge():
    if not os.path.exists(BRIDGE_SO):
        return None
    lib = ctypes.CDLL(BRIDGE_SO)
    P = c_void_p
    lib.bridge_run_pair.argtypes = [P, c_char_p, c_int, c_char_p, c_uint64, c_char_p, c_uint64]
    lib.bridge_sweep_pair.argtypes = [P, c_int, P, c_int, c_int, c_char_p, c_uint64, c_char_p, c_uint64]
    lib.bridge_estimate_pair.argtypes = [c_int, c_uint64, c_uint64, c_uint64, c_uint64, c_uint64, c_int, c_int,
                                         P, P, P, P, c_char_p, c_uint64]
    lib.bridge_manager_estimates.argtypes = [c_int, c_uint64, c_int, P, P, c_uint64, POINTER(c_uint64), c_char_p,
                                             c_uint64]
    lib.bridge_snapshot_predict.argtypes = [c_char_p, c_int, c_uint64, c_uint64, P, c_char_p, c_uint64]
    return lib


def case(mix="t90", seed=1, policy="magm", estimator="none", mode="mps", gpu_count=4, rr_pre=False, min_free=None,
         max_smact=0.8, window=60.0, capacity=40 * GiB, block=512 * MiB, mig=()):
    c = np.zeros(1, case_dtype)
    c["mix"] = {"t90": 0, "t60": 1, None: -1}[mix]
    c["seed"], c["policy"], c["estimator"], c["mode"] = seed, POLICY[policy], ESTIMATOR[estimator], MODE[mode]
    c["gpu_count"], c["rr_pre"], c["max_smact"], c["window"] = gpu_count, int(rr_pre), max_smact, window
    c["has_min_free"], c["min_free"] = int(min_free is not None), min_free or 0
    c["capacity"], c["block"], c["n_mig"] = capacity, block, len(mig)
    c["mig"][0, : len(mig)] = mig
    return c


def run_pair(lib, c, trace_path=None, device=0, cap=1 << 22):
    r, g = ctypes.create_string_buffer(cap), ctypes.create_string_buffer(cap)
    lib.bridge_run_pair(c.ctypes.data, trace_path.encode() if trace_path else None, device, r, cap, g, cap)
    return r.value.decode(), g.value.decode()


def sweep_pair(lib, cells, seeds, device=0, cap=1 << 25):
    cells = np.concatenate(cells)
    seeds = np.ascontiguousarray(seeds, np.uint64)
    r, g = ctypes.create_string_buffer(cap), ctypes.create_string_buffer(cap)
    lib.bridge_sweep_pair(cells.ctypes.data, len(cells), seeds.ctypes.data, len(seeds), device, r, cap, g, cap)
    return r.value.decode(), g.value.decode()
