# A/B of replay builds (ab/libcarma_minctas*.so): c4 timing (+ replay parity)
set -u
echo "== base"; timeout 300 python scripts/profile_driver.py replay --traces 100000 --reps 3 2>&1 | tail -2
for v in ab/libcarma_minctas*.so; do
  echo "== $v"
  CARMA_B200_LIB=$PWD/$v timeout 300 python scripts/profile_driver.py replay --traces 100000 --reps 3 2>&1 | tail -2
  CARMA_B200_LIB=$PWD/$v timeout 600 python -m pytest tests/test_gpu_replay.py -m gpu -x -q --timeout 300 2>&1 | tail -1
done
echo "== base again"; timeout 300 python scripts/profile_driver.py replay --traces 100000 --reps 3 2>&1 | tail -2
