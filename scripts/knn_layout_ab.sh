# k-NN fp32-path layouts A/B: parity tests and c2 timing per layout (CARMA_KNN_LAYOUT)
set -u
for L in 0 3; do
  echo "== layout $L"
  CARMA_KNN_LAYOUT=$L timeout 600 python -m pytest tests/test_gpu_knn.py -m gpu -x -q 2>&1 | tail -1
  CARMA_KNN_LAYOUT=$L timeout 300 python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 4 2>&1 | tail -2
done
CARMA_KNN_LAYOUT=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 0 -c 12 --csv --log-file gpurun_out/knn_pipeline_l3.csv python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 1 > /dev/null 2>&1
