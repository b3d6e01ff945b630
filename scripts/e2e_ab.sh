# host-buffer e2e A/B: compact 40-B rows on/off (CARMA_E2E_COMPACT) x share
# of chunks shipped raw (CARMA_E2E_RAW_EVERY); AB_CFGS="1 2,1 4" selects
CFGS=("1 2" "0 2" "1 3" "1 0" "1 4")
[ -n "${AB_CFGS:-}" ] && IFS=, read -ra CFGS <<< "$AB_CFGS"
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  echo "== compact $1 raw every $2"
  CARMA_E2E_COMPACT=$1 CARMA_E2E_RAW_EVERY=$2 timeout 600 python bench.py --skip-replay --skip-fused --skip-small --skip-scoring --skip-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('knn e2e', d['e2e']['value']/1e6, 'h2d', d['e2e']['h2d_bytes_per_step'], 'mlp e2e', d['neural']['mlp']['e2e']/1e6)"
done
