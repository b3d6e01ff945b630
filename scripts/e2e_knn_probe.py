import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi
ds = [cb.generate_synthetic_dataset(f, 8388608, s) for f, s in ((1, 2024), (2, 2025))]
rows = np.concatenate([d.rows for d in ds]); fam = np.concatenate([np.full(8388608, 1, np.int8), np.full(8388608, 2, np.int8)])
knn = cb.GpuKnn(0)
for f, s in ((1, 112), (2, 213)): knn.set_model(cb.fit_knn(f, 4000, s, 5))
words, schema = cb.pack_features_bits(rows, fam)
Q = len(rows)
h_rows = torch.from_numpy(words.view(np.uint8)).pin_memory().numpy().view(np.uint32)
h_b = torch.empty(Q, dtype=torch.int32).pin_memory().numpy()
h_by = torch.empty(Q, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
def step():
    abi.check(abi.lib.carma_knn_predict_bitpacked(knn.handle, h_rows.ctypes.data, schema.ctypes.data, Q, h_b.ctypes.data, h_by.ctypes.data))
for _ in range(3): step()
ts = []
for _ in range(5):
    t = time.perf_counter(); step(); ts.append(time.perf_counter() - t)
print("e2e ms", [round(x * 1e3, 2) for x in ts], "best", round(min(ts) * 1e3, 2), "est/s", Q / np.mean(ts) / 1e6)
