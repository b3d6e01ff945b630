# host-buffer e2e A/B: which chunks ship raw (CARMA_E2E_RAW_FIRST), two runs each
set -u
run() { timeout 600 python bench.py --skip-replay --skip-fused --skip-small --skip-scoring --skip-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('knn e2e', round(d['e2e']['value']/1e6,1), 'h2d', d['e2e']['h2d_bytes_per_step'], 'mlp e2e', round(d['neural']['mlp']['e2e']/1e6,1))"; }
for r in 1 2; do
  for f in 0 1; do echo "== raw first $f"; CARMA_E2E_RAW_FIRST=$f run; done
done
