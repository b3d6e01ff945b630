# A/B of k-NN search builds (ab/libcarma_knn_*.so): parity + c2 timing each
set -u
echo "== base"; timeout 300 python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 3 2>&1 | tail -2
for sp in ${AB_SPLITS:-}; do
  echo "== base CARMA_KNN_SPLIT=$sp"
  CARMA_KNN_SPLIT=$sp timeout 300 python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 3 2>&1 | tail -2
done
for v in ab/libcarma_knn_*.so; do
  echo "== $v"
  CARMA_B200_LIB=$PWD/$v timeout 600 python -m pytest tests/test_gpu_knn.py -m gpu -x -q 2>&1 | tail -1
  CARMA_B200_LIB=$PWD/$v timeout 300 python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 3 2>&1 | tail -2
done
