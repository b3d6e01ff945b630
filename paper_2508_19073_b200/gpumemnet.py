"""Neural GPUMemNet (the paper's MLP and Transformer ensembles) on the B200.

Host mirror of the estimator interface for the neural EstimatorKind next to
the k-NN (`GpuKnn`): a per-family model bank (Manager::set_learned_estimators,
manager.hpp:77) whose predict returns bins and upper-edge bytes like
estimate_learned (estimators.cpp:540-551), with FamilyMismatch rows as
bin -1 / no estimate (manager.cpp:99-105). The compute is carma_nn_*
(include/carma_gpu.h, csrc/cuda/gpumemnet.cu); there is no CPU path.

The reference artifact ships only the k-NN; the network
structure follows PAPER.md:436-442 and the weights come from
scripts/train_gpumemnet.py (committed under weights/).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Dict, List, Optional

import numpy as np

from . import abi
from .abi import check, lib, ptr

WEIGHTS_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "weights")
FAMILY_NAMES = {0: "mlp", 1: "cnn", 2: "transformer"}

# Features whose raw values are counts / sizes: log1p before standardising.
# 0-6 tallies, batch, params, activations; 10, 11, 13, 14, 16, 17 the layer
# tuples' activations and params; 18 the 16P + 4BA footprint proxy.
LOG_DIMS = (0, 1, 2, 3, 4, 5, 6, 10, 11, 13, 14, 16, 17, 18)
LOG_MASK = sum(1 << d for d in LOG_DIMS)
ARCH_MLP, ARCH_TRANSFORMER = 0, 1


@dataclasses.dataclass
class NnModel:
    family: int
    bucket_range: int
    classes: int
    depth: List[int]            # hidden layers per member
    width: List[List[int]]      # hidden widths per member
    shift: np.ndarray           # 19 fp32
    scale: np.ndarray           # 19 fp32
    params: np.ndarray          # flat fp32, layout of carma_nn_set_model
    log_mask: int = LOG_MASK
    holdout_accuracy: float = float("nan")
    arch: int = ARCH_MLP        # ARCH_TRANSFORMER: depth = encoder layers, width[e] = [d]

    @property
    def members(self) -> int:
        return len(self.depth)

    def spec(self) -> np.ndarray:
        s = np.zeros(1, abi.nn_spec_dtype)
        s["members"] = self.members
        s["classes"] = self.classes
        s["bucket_range"] = self.bucket_range
        for e, (d, w) in enumerate(zip(self.depth, self.width)):
            s["depth"][0][e] = d
            s["width"][0][e][: len(w)] = w
        s["log_mask"] = self.log_mask
        s["arch"] = self.arch
        s["shift"][0] = self.shift
        s["scale"][0] = self.scale
        return s

    def save(self, path: str) -> None:
        width = np.zeros((self.members, abi.NN_MAX_DEPTH), np.int32)
        for e, w in enumerate(self.width):
            width[e, : len(w)] = w
        np.savez(path, family=self.family, bucket_range=self.bucket_range, classes=self.classes,
                 depth=np.asarray(self.depth, np.int32), width=width, shift=self.shift, scale=self.scale,
                 params=self.params, log_mask=self.log_mask, holdout_accuracy=self.holdout_accuracy, arch=self.arch)

    @staticmethod
    def load(path: str) -> "NnModel":
        z = np.load(path)
        depth = [int(d) for d in z["depth"]]
        arch = int(z["arch"]) if "arch" in z else ARCH_MLP
        if arch == ARCH_TRANSFORMER:
            width = [[int(z["width"][e][0])] for e in range(len(depth))]
        else:
            width = [[int(v) for v in z["width"][e][:d]] for e, d in enumerate(depth)]
        return NnModel(int(z["family"]), int(z["bucket_range"]), int(z["classes"]), depth, width,
                       z["shift"].astype(np.float32), z["scale"].astype(np.float32), z["params"].astype(np.float32),
                       int(z["log_mask"]), float(z["holdout_accuracy"]), arch)


def load_default_models(arch: int = ARCH_MLP) -> Dict[int, NnModel]:
    """The committed GPUMemNet ensembles (MLP or Transformer), one per family."""
    out = {}
    pre = "gpumemnet_tf_" if arch == ARCH_TRANSFORMER else "gpumemnet_"
    for f, name in FAMILY_NAMES.items():
        path = os.path.join(WEIGHTS_DIR, f"{pre}{name}.npz")
        if os.path.exists(path):
            out[f] = NnModel.load(path)
    return out


def param_count(m: NnModel) -> int:
    return int(lib.carma_nn_param_count(ptr(m.spec())))


class GpuMemNet:
    """A device-resident bank of neural GPUMemNet ensembles, one per family."""

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        check(lib.carma_nn_create(device, ctypes.byref(h)))
        self._h = h
        self.models: Dict[int, NnModel] = {}

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def set_model(self, m: NnModel) -> None:
        params = np.ascontiguousarray(m.params, np.float32)
        check(lib.carma_nn_set_model(self._h, m.family, ptr(m.spec()), ptr(params), len(params)))
        self.models[m.family] = m

    def predict(self, rows: np.ndarray, family=None, default_family: Optional[int] = None):
        """Bins and upper-edge bytes for feature rows (host buffers)."""
        q = len(rows)
        bucket = np.zeros(q, np.int32)
        nbytes = np.zeros(q, np.uint64)
        fam = None if family is None else np.ascontiguousarray(family, np.int8)
        dflt = default_family if default_family is not None else next(iter(self.models))
        rows = np.ascontiguousarray(rows, abi.feature_row_dtype)
        check(lib.carma_nn_predict(self._h, ptr(rows), ptr(fam), dflt, q, ptr(bucket), ptr(nbytes)))
        return bucket, nbytes

    def predict_bitpacked(self, words: np.ndarray, schema: np.ndarray, q: int):
        bucket = np.zeros(q, np.int32)
        nbytes = np.zeros(q, np.uint64)
        check(lib.carma_nn_predict_bitpacked(self._h, ptr(np.ascontiguousarray(words)), ptr(schema), q,
                                             ptr(bucket), ptr(nbytes)))
        return bucket, nbytes

    def predict_device(self, rows, fmt: int, q: int, bucket, nbytes, family=None, default_family: int = 0,
                       probs=None, logits=None, stream=None) -> None:
        """Device-resident predict (torch tensors or raw device pointers) on
        `stream` (torch stream or cudaStream_t; None = torch's current stream)."""
        check(lib.carma_nn_predict_device(self._h, ptr(rows), fmt, ptr(family), default_family, q, ptr(bucket),
                                          ptr(nbytes), ptr(probs), ptr(logits), abi.stream_arg(stream, self.device)))

    def set_path(self, path: int) -> None:
        """MLP ensembles: 0 auto (CUDA cores), 1 tcgen05 tensor cores, 2 CUDA cores."""
        check(lib.carma_nn_set_path(self._h, path))

    def set_act_table(self, table: np.ndarray) -> None:
        check(lib.carma_nn_set_act_table(self._h, ptr(np.ascontiguousarray(table, np.float64))))

    def set_bit_schema(self, schema: np.ndarray) -> None:
        check(lib.carma_nn_set_bit_schema(self._h, ptr(schema)))

    def last_timing(self):
        k, c = ctypes.c_double(), ctypes.c_double()
        la, mm = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.carma_nn_last_timing(self._h, ctypes.byref(k), ctypes.byref(c), ctypes.byref(la),
                                       ctypes.byref(mm)))
        return {"kernel_ms": k.value, "call_ms": c.value, "launches": la.value, "mmas": mm.value}

    def close(self) -> None:
        if self._h:
            check(lib.carma_nn_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
