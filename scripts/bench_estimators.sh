# estimator stages of bench.py only (k-NN + neural), summarised
timeout 600 python bench.py --skip-replay --skip-fused --skip-small --skip-scoring --skip-cpu --steps ${STEPS:-10} > gpurun_out/bench_est.json 2> gpurun_out/bench_est.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_est.json").read().strip().splitlines()[-1])
m = d["neural"]["mlp"]
print("knn", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"] / 1e6, 1),
      "| mlp ms", round(m["ms_per_step"], 3), round(m["value"] / 1e6, 1), "e2e", round(m["e2e"] / 1e6, 1))
PY
