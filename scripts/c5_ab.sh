# A/B of long-trace replay builds (ab/libcarma_pf*.so): c5 timing + parity
set -u
echo "== base"; timeout 300 python scripts/profile_driver.py fused --tasks 1000000 --reps 2 2>&1 | tail -2
for v in ab/libcarma_pf*.so; do
  echo "== $v"
  CARMA_B200_LIB=$PWD/$v timeout 300 python scripts/profile_driver.py fused --tasks 1000000 --reps 2 2>&1 | tail -2
done
v=$(ls ab/libcarma_pf*.so | tail -1)
CARMA_B200_LIB=$PWD/$v timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_fullsize.py -m gpu -x -q --timeout 600 2>&1 | tail -1
