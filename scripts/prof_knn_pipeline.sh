# Per-kernel duration + DRAM bytes of every kernel in one c2 k-NN call
# (136-B rows), for the traffic accounting of the pipeline.
set -u
mkdir -p gpurun_out/prof
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 0 -c 12 --csv --log-file gpurun_out/prof/knn_pipeline.csv \
    python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 1 > gpurun_out/prof/ncu_knn_pipe.log 2>&1
