"""Multi-GPU sharding for the two stages (one process per GPU).

Both stages are embarrassingly parallel: estimator rows and
replay jobs are independent, so a multi-GPU run shards them contiguously,
runs each shard on the local device with no data-path collective, and
gathers the per-shard results to rank 0 over the process group (NCCL on the
GPU box, gloo in the CPU tests). This mirrors run_sweep's job pool
(runner.cpp:196-249) spread over devices instead of host threads.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np


def balanced_shards(weights: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Contiguous [begin, end) ranges, one per rank, balancing the summed weight
    (rows: 1 each; replay jobs: their task counts). The rule is the native
    multi-device driver's (carma_shard_ranges), so a rank of a multi-process
    run and a device of the one-process driver get the same units."""
    from . import abi
    w = np.ascontiguousarray(weights, np.uint64)
    world = max(1, int(world))
    bounds = np.zeros(world + 1, np.uint64)
    abi.check(abi.lib.carma_shard_ranges(w.ctypes.data if len(w) else None, len(w), world, bounds.ctypes.data))
    return [(int(bounds[r]), int(bounds[r + 1])) for r in range(world)]


def balanced_shards_count(n: int, world: int) -> List[Tuple[int, int]]:
    """balanced_shards for n unit weights without materialising them: cut p
    at ceil(n * p / world), the same rule."""
    world = max(1, int(world))
    cut = [(n * p + world - 1) // world for p in range(world)] + [n]
    return [(cut[r], cut[r + 1]) for r in range(world)]


def gather_to_root(local: np.ndarray, rank: int, world: int, dist=None) -> np.ndarray | None:
    """Concatenates every rank's structured array in rank order on rank 0."""
    if world <= 1 or dist is None:
        return local
    objs = [None] * world if rank == 0 else None
    dist.gather_object(local, objs, dst=0)
    return np.concatenate(objs) if rank == 0 else None


def run_sharded(n_units: int, weights: Sequence[float], run_shard: Callable[[int, int], np.ndarray],
                rank: int, world: int, dist=None) -> np.ndarray | None:
    """Runs `run_shard(begin, end)` for this rank's shard and gathers to rank 0."""
    assert len(weights) == n_units
    b, e = balanced_shards(weights, world)[rank]
    local = run_shard(b, e)
    return gather_to_root(local, rank, world, dist)


def sweep_sharded(cfgs: np.ndarray, tasks: np.ndarray, offsets: np.ndarray, jobs: np.ndarray, rank: int,
                  world: int, device: int, dist=None):
    """run_sweep across ranks: jobs sharded by task count, each rank replays
    its shard on `device`; rank 0 receives the per-job trace results in job
    order (per-task and per-GPU results stay on the owning rank)."""
    from . import carma as cb

    counts = np.diff(offsets.astype(np.int64))[jobs["trace"]]

    def shard(b: int, e: int) -> np.ndarray:
        from . import abi
        if e <= b:
            return np.zeros(0, abi.trace_result_dtype)
        plan = cb.ReplayPlan(cfgs, tasks, offsets, jobs[b:e], device=device)
        try:
            plan.run()
            return plan.results(tasks=False).traces
        finally:
            plan.close()

    return run_sharded(len(jobs), counts, shard, rank, world, dist)
