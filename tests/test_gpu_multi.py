"""The one-process multi-device driver (carma_*_multi): shards over several
handles / plans, one host thread each, gathered into one host buffer at the
shard offsets, must equal the single-device call bit for bit. On the
one-GPU box the "devices" are several handles / plans on device 0, which
exercises the same shard, thread and gather code."""
import numpy as np
import pytest

import paper_2508_19073_b200 as cb
from cases import model

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_knn_predict_multi_equals_single(gpu, parts):
    rows = np.concatenate([cb.generate_synthetic_dataset(f, 30001, 70 + f).rows for f in (0, 1, 2)])
    fam = np.repeat(np.array([0, 1, 2], np.int8), 30001)
    knns = []
    for _ in range(parts):
        k = cb.GpuKnn(gpu)
        for f in (0, 1, 2):
            k.set_model(model(f))
        knns.append(k)
    b1, by1 = knns[0].predict(rows, family=fam)
    bm, bym = cb.predict_multi(knns, rows, family=fam)
    for k in knns:
        k.close()
    assert np.array_equal(b1, bm) and np.array_equal(by1, bym)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0, 0]])
def test_replay_multi_equals_single(gpu, devices):
    lists = [cb.materialize_trace(cb.generate_trace("t90", s)).tasks for s in range(1, 41)]
    lists += [cb.materialize_trace(cb.generate_trace("t60", s)).tasks for s in range(1, 21)]
    offs = np.concatenate([[0], np.cumsum([len(t) for t in lists])]).astype(np.uint64)
    tasks = np.concatenate(lists)
    cfgs = np.concatenate([cb.make_config(cb.PolicyConfig(policy=p, max_smact=0.8), cb.SimConstants())
                           for p in ("exclusive", "rr", "magm", "lug")])
    from paper_2508_19073_b200 import abi
    jobs = np.zeros(len(lists) * 4, abi.job_dtype)
    jobs["trace"] = np.tile(np.arange(len(lists), dtype=np.uint32), 4)
    jobs["config"] = np.repeat(np.arange(4, dtype=np.uint32), len(lists))
    plan = cb.ReplayPlan(cfgs, tasks, offs, jobs, device=gpu)
    plan.run()
    want = plan.results()
    plan.close()
    got = cb.replay_multi(devices, cfgs, tasks, offs, jobs)
    assert got.tasks.tobytes() == want.tasks.tobytes()
    assert got.traces.tobytes() == want.traces.tobytes()
    assert got.gpus.tobytes() == want.gpus.tobytes()
