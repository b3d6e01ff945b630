"""Times the device dataset generator on the c2 inputs (8,388,608 rows per
family) against the host generator, and prints the per-round stats."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_19073_b200 as cb
from paper_2508_19073_b200 import abi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_388_608
for family, seed in ((1, 2024), (2, 2025), (0, 7)):
    rows = torch.empty(n * 136, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    m = torch.empty(n, dtype=torch.int64, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = cb.generate_synthetic_dataset_device(family, n, seed, rows, b, m)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"family {family}: device {dt*1e3:.1f} ms  stats {st}", flush=True)
    t0 = time.perf_counter(); h = cb.generate_synthetic_dataset(family, n, seed); dh = time.perf_counter() - t0
    ok = rows.cpu().numpy().tobytes() == h.rows.tobytes() and np.array_equal(b.cpu().numpy(), h.bucket)
    print(f"family {family}: host {dh*1e3:.1f} ms  identical={ok}", flush=True)
