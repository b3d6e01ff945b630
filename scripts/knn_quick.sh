# k-NN parity tests + the c2 search timing (profile_driver, 136-B rows)
set -u
timeout 600 python -m pytest tests/test_gpu_knn.py -m gpu -x -q > gpurun_out/knn_t.log 2>&1; echo rc=$? >> gpurun_out/knn_t.log
tail -2 gpurun_out/knn_t.log
timeout 300 python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 4 2>&1 | tail -3
