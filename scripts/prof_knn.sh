set -u
mkdir -p gpurun_out/prof
python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 4 > gpurun_out/prof/knn_time.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_search_f32 -s 1 -c 1 \
    -o gpurun_out/prof/knn_search_full -f python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 2 > gpurun_out/prof/ncu_knn.log 2>&1
python scripts/profile_summary.py report gpurun_out/prof/knn_search_full.ncu-rep > gpurun_out/prof/ncu_knn_search.txt 2>&1
python scripts/ncu_lines.py gpurun_out/prof/knn_search_full.ncu-rep paper_2508_19073_b200/csrc/build/knn.cu.o "knn_search_f32ILi5ELi0" paper_2508_19073_b200/csrc/cuda/knn.cu 60 > gpurun_out/prof/knn_lines.txt 2>&1
ls -la gpurun_out/prof
