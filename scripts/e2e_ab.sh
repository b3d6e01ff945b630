# host-buffer e2e A/B: share of chunks shipped raw (CARMA_E2E_RAW_EVERY)
for k in 0 2 3 4; do
  echo "== raw every $k"
  CARMA_E2E_RAW_EVERY=$k timeout 600 python bench.py --skip-replay --skip-fused --skip-small --skip-scoring --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('knn e2e', d['e2e']['value']/1e6, 'mlp e2e', d['neural']['mlp']['e2e']/1e6)"
done
