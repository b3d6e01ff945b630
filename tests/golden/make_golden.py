"""Regenerates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

  make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the oracle and the GPU path to the reference's own outputs
on boxes where /root/reference (and hence oracle/_ref) is absent:
  knn.npz     estimate_learned buckets/bytes for 2000 dataset rows per family,
              models trained like provision_estimators (runner.cpp:17-38)
  replay.npz  run_simulation outputs (per task / per GPU / report) for a grid
              of policies, mixes, seeds, estimators, platforms and MIG tables
Inputs are not stored: they are regenerated bit-identically by the product's
host provisioning (checked by tests/test_oracle_vs_ref.py).
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_bind import load_ref, ref_config, ref_run  # noqa: E402

KNN_CASES = [  # (family, model seed, query seed, n)
    (0, 11, 12345, 2000), (1, 112, 2024, 2000), (2, 213, 2025, 2000)]

REPLAY_CASES = []
for mix in ("t90", "t60"):
    for seed in (1, 2, 3):
        for pol in ("exclusive", "rr", "magm", "lug", "mug"):
            REPLAY_CASES.append(dict(mix=mix, seed=seed, policy=pol, estimator="none"))
        REPLAY_CASES.append(dict(mix=mix, seed=seed, policy="magm", estimator="learned"))
        REPLAY_CASES.append(dict(mix=mix, seed=seed, policy="magm", estimator="oracle"))
        REPLAY_CASES.append(dict(mix=mix, seed=seed, policy="rr", estimator="none", mode="streams"))
        REPLAY_CASES.append(dict(mix=mix, seed=seed, policy="magm", estimator="none", min_free=2 << 30))
        REPLAY_CASES.append(dict(mix=mix, seed=seed, policy="lug", estimator="learned", gpu_count=8, window=5.0))
        # MIG (instance 0 holds the largest catalog task so every run terminates)
        REPLAY_CASES.append(dict(mix=mix, seed=seed, policy="magm", estimator="none", mode="mig", mig=(0.75, 0.25)))
        REPLAY_CASES.append(dict(mix=mix, seed=seed, policy="rr", estimator="oracle", mode="mig",
                                 mig=(0.8, 0.1, 0.1), rr_pre=True))


def main():
    ref = load_ref()
    if ref is None:
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    knn = {}
    for fam, mseed, qseed, n in KNN_CASES:
        b = np.zeros(n, np.int32)
        by = np.zeros(n, np.uint64)
        assert ref.ref_predict_dataset(fam, 4000, mseed, 5, n, qseed, b.ctypes.data, by.ctypes.data) == 0
        knn[f"bucket_{fam}"] = b
        knn[f"bytes_{fam}"] = by
    knn["cases"] = np.array(KNN_CASES, np.int64)
    # holdout report of train_learned_estimator (estimators.cpp:396-434):
    # accuracy, macro_f1, underestimate_rate per case model
    for fam, mseed, _, _ in KNN_CASES:
        lo, hi = np.zeros(19), np.zeros(19)
        pts, lab = np.zeros((4000, 19)), np.zeros(4000, np.int32)
        n, br, h = ctypes.c_uint64(), ctypes.c_uint64(), np.zeros(3)
        assert ref.ref_train(fam, 4000, mseed, 5, b"/tmp/carma_golden_model.json", lo.ctypes.data, hi.ctypes.data,
                             pts.ctypes.data, lab.ctypes.data, 4000, ctypes.byref(n), ctypes.byref(br),
                             h.ctypes.data) == 0
        knn[f"holdout_{fam}"] = h
    np.savez_compressed(os.path.join(HERE, "knn.npz"), **knn)

    out = {}
    for i, case in enumerate(REPLAY_CASES):
        kw = {k: v for k, v in case.items() if k not in ("mix", "seed")}
        cfg = ref_config(**kw)
        tout, rout, ge, gs, gp = ref_run(ref, cfg, mix=case["mix"], seed=case["seed"])
        out[f"tasks_{i}"] = tout
        out[f"report_{i}"] = np.array([rout])
        out[f"gpu_energy_{i}"] = ge
        out[f"gpu_smact_{i}"] = gs
        out[f"gpu_peak_{i}"] = gp
    out["cases"] = np.array([repr(c) for c in REPLAY_CASES])
    np.savez_compressed(os.path.join(HERE, "replay.npz"), **out)
    print(f"wrote {len(KNN_CASES)} knn cases and {len(REPLAY_CASES)} replay cases")


if __name__ == "__main__":
    main()
