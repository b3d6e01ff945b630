"""The N>1 path on CPU: world_size-2 gloo process group; sharding + gather must
equal the single-process result (the replay/k-NN shard runners are replaced
by the oracle, since there is no GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_19073_b200.dist import balanced_shards, run_sharded


def test_balanced_shards_cover_and_balance():
    w = np.random.default_rng(0).integers(50, 130, 1000)
    for world in (1, 2, 3, 8):
        sh = balanced_shards(w, world)
        assert sh[0][0] == 0 and sh[-1][1] == len(w)
        assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
        loads = [w[b:e].sum() for b, e in sh]
        assert max(loads) - min(loads) <= 2 * w.max()
    assert balanced_shards([], 4) == [(0, 0)] * 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import paper_2508_19073_b200 as cb
    from oracle_bind import load_oracle, oracle_replay

    olib = load_oracle()
    lists = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in range(1, 13)]
    cfg = cb.make_config(cb.PolicyConfig(policy="magm"), cb.SimConstants())

    def shard(b, e):
        from paper_2508_19073_b200 import abi
        out = np.zeros(e - b, abi.trace_result_dtype)
        for k, t in enumerate(range(b, e)):
            out[k] = oracle_replay(olib, cfg, lists[t])[2]
        return out

    res = run_sharded(len(lists), [len(t) for t in lists], shard, rank, world, dist)
    if rank == 0:
        np.save(out_path, res)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sweep_equals_single_process(tmp_path, olib):
    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    import paper_2508_19073_b200 as cb
    from oracle_bind import oracle_replay
    cfg = cb.make_config(cb.PolicyConfig(policy="magm"), cb.SimConstants())
    want = np.concatenate([[oracle_replay(olib, cfg, cb.materialize_trace(cb.generate_trace("t90", s)).tasks)[2]]
                           for s in range(1, 13)])
    assert got.tobytes() == want.tobytes()


def _nn_worker(rank, world, port, out_path):
    """Estimator rows sharded over ranks (the neural GPUMemNet's shard runner
    replaced by its numpy oracle: no GPU here)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import gpumemnet_oracle
    import paper_2508_19073_b200 as cb
    from paper_2508_19073_b200 import gpumemnet as gm

    m = gm.load_default_models()[1]
    raw = cb.scalar_features(cb.generate_synthetic_dataset(1, 1001, 9).rows)

    def shard(b, e):
        return gpumemnet_oracle.forward(m.spec()[0], m.params, raw[b:e])[3]

    res = run_sharded(len(raw), np.ones(len(raw)), shard, rank, world, dist)
    if rank == 0:
        np.save(out_path, res)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_neural_estimates_equal_single_process(tmp_path):
    out = str(tmp_path / "nn.npy")
    mp.spawn(_nn_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import gpumemnet_oracle
    import paper_2508_19073_b200 as cb
    from paper_2508_19073_b200 import gpumemnet as gm
    m = gm.load_default_models()[1]
    raw = cb.scalar_features(cb.generate_synthetic_dataset(1, 1001, 9).rows)
    assert np.array_equal(got, gpumemnet_oracle.forward(m.spec()[0], m.params, raw)[3])


def test_native_shard_rule_matches_restatement():
    """carma_shard_ranges (the native multi-device driver's rule, also used by
    dist.balanced_shards) against a numpy restatement of the rule."""
    rng = np.random.default_rng(3)
    for n, world in ((0, 3), (1, 4), (7, 8), (1000, 3), (400_000, 8), (33, 33)):
        w = rng.integers(1, 200, n)
        cum = np.concatenate([[0.0], np.cumsum(w.astype(np.float64))])
        cuts = [0] + [min(int(np.searchsorted(cum, cum[-1] * r / world, side="left")), n)
                      for r in range(1, world)] + [n]
        cuts = np.maximum.accumulate(cuts)
        assert balanced_shards(w, world) == [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def _bench_worker(rank, world, port, out_path):
    """bench.py's N>1 orchestration on gloo: Dist (barrier, max, sum), the row
    and job shard rules, shard_jobs' per-rank inputs and timed_host_steps;
    the GPU shard runners are replaced by the oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import bench
    import paper_2508_19073_b200 as cb
    from oracle_bind import load_oracle, oracle_replay
    from paper_2508_19073_b200 import abi
    from paper_2508_19073_b200 import dist as cdist

    d = bench.Dist(world, backend="gloo")
    assert d.n == world and d.rank == rank
    olib = load_oracle()
    cfgs, tasks, offs, jobs = bench.sweep_inputs(cb, 30)
    counts = np.diff(offs.astype(np.int64))[jobs["trace"]]
    b, e = cdist.balanced_shards(counts, d.n)[d.rank]
    st, so, sj = bench.shard_jobs(tasks, offs, jobs, b, e)
    so = so.astype(np.int64)
    out = np.zeros(len(sj), abi.trace_result_dtype)
    for k, j in enumerate(sj):
        out[k] = oracle_replay(olib, cfgs[j["config"]: j["config"] + 1], st[so[j["trace"]]: so[j["trace"] + 1]])[2]
    placed = int(np.diff(so)[sj["trace"]].sum())
    assert d.sum(placed) == int(counts.sum())
    assert d.max(float(rank)) == world - 1
    dt = bench.timed_host_steps(lambda: None, 1, 2, d)
    assert dt >= 0.0
    rb, re_ = cdist.balanced_shards_count(1001, world)[rank]
    assert d.sum(re_ - rb) == 1001
    res = cdist.gather_to_root(out, rank, world, d.pg)
    if rank == 0:
        np.save(out_path, res)
    d.barrier()
    d.close()


def test_bench_orchestration_gloo_equals_single_process(tmp_path, olib):
    out = str(tmp_path / "bench.npy")
    mp.spawn(_bench_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    import bench
    import paper_2508_19073_b200 as cb
    from paper_2508_19073_b200 import abi
    from oracle_bind import oracle_replay
    cfgs, tasks, offs, jobs = bench.sweep_inputs(cb, 30)
    o = offs.astype(np.int64)
    want = np.zeros(len(jobs), abi.trace_result_dtype)
    for k, j in enumerate(jobs):
        want[k] = oracle_replay(olib, cfgs[j["config"]: j["config"] + 1], tasks[o[j["trace"]]: o[j["trace"] + 1]])[2]
    assert got.tobytes() == want.tobytes()
