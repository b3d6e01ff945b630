"""B200-native CARMA hot path: GPUMemNet (k-NN) inference and trace replay.

The compute lives in libcarma_b200.so (sm_100a kernels behind the C ABI in
include/carma_gpu.h, plus host provisioning behind include/carma_host.h).
"""
from . import abi  # noqa: F401  (raises ImportError when the library is missing)
from .carma import *  # noqa: F401,F403

__all__ = ["abi"]
