"""Times the reference (oracle/_ref) on the FULL c5 trace: 10^6 rows, MAGM +
learned, 64 GPUs, W = 5 s, one run_simulation on one core. Too slow for
bench.py's bounded CPU sample (~20 min); run once per round and recorded in
DESIGN.md / profiles/."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ref = bench.ref_lib()
t = time.time()
rate, sample = bench.cpu_fused_baseline(ref, n)
print(json.dumps({"tasks": n, "seconds": n / rate, "placed_tasks_per_s": rate, "cores": 1,
                  "host": os.uname().nodename, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")}))
