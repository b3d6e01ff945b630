"""Host-side probes for the e2e design: memory read bandwidth with T threads,
and the cost of the row packers (carma_pack_features / _bits) per row."""
import os, sys, threading, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

n = 1 << 28  # 2 GiB of u64
a = np.ones(n, np.uint64)
for T in (1, 2, 4, 8, 16):
    parts = np.array_split(a, T)
    out = [0] * T
    def f(i):
        out[i] = int(np.bitwise_xor.reduce(parts[i][::1]))
    t0 = time.perf_counter()
    th = [threading.Thread(target=f, args=(i,)) for i in range(T)]
    [t.start() for t in th]; [t.join() for t in th]
    dt = time.perf_counter() - t0
    print(f"read T={T}: {a.nbytes / dt / 1e9:.1f} GB/s", flush=True)
b = np.empty_like(a)
t0 = time.perf_counter(); np.copyto(b, a); dt = time.perf_counter() - t0
print(f"copy T=1: {a.nbytes / dt / 1e9:.1f} GB/s (read+write bytes x2)", flush=True)
import paper_2508_19073_b200 as cb
ds = cb.generate_synthetic_dataset(1, 1 << 20, 2024)
for name, fn in (("pack64", cb.pack_features), ("packbits", cb.pack_features_bits)):
    t0 = time.perf_counter(); fn(ds.rows, default_family=1); dt = time.perf_counter() - t0
    print(f"{name}: {dt * 1e3 / 1.048576:.1f} ns/row (1 thread)", flush=True)
print("cpus", os.cpu_count(), flush=True)
