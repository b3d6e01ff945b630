# A/B of neural builds (ab/libcarma_nn_*.so): MLP ensemble c2 timing (bench's
# own neural stage) + parity
set -u
run() { timeout 600 python bench.py --skip-replay --skip-fused --skip-small --skip-scoring --skip-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['neural']['mlp']; print('mlp ms', m['ms_per_step'], 'value', m['value']/1e6)"; }
echo "== base"; run
for v in ab/libcarma_nn_*.so; do
  echo "== $v"
  CARMA_B200_LIB=$PWD/$v run
  CARMA_B200_LIB=$PWD/$v timeout 600 python -m pytest tests/test_gpumemnet.py -m gpu -x -q --timeout 300 2>&1 | tail -1
done
echo "== base again"; run
