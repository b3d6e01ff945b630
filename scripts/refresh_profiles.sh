#!/bin/bash
# One GPU call that regenerates the round's measurement artefacts (run via gpurun):
#   bench line, launch list of the same bench command, ncu --set full of the
#   dominant kernels. Summaries are written here afterwards with
#   scripts/profile_summary.py (no GPU needed).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
cp gpurun_out/bench_detail_n1.json $OUT/bench_detail_n1.json 2>/dev/null  # before the ncu runs overwrite it
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-cpu --skip-small --skip-fused > $OUT/launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_search -s 1 -c 1 \
    -o $OUT/knn_search_full -f python scripts/profile_driver.py knn --rows 16777216 --format rows --reps 2 > $OUT/ncu_knn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 2 -c 1 \
    -o $OUT/replay_kernel_full -f python scripts/profile_driver.py replay --traces 100000 --reps 2 > $OUT/ncu_replay.log 2>&1
tail -2 $OUT/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pick_kernel -s 1 -c 1 \
    -o $OUT/pick_kernel_full -f python scripts/profile_driver.py scoring --reps 2 > $OUT/ncu_pick.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
    -o $OUT/replay_c5_full -f python scripts/profile_driver.py fused --tasks 100000 --reps 1 > $OUT/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nn_ensemble -s 1 -c 1 \
    -o $OUT/nn_ensemble_full -f python scripts/profile_driver.py nn --path 1 --rows 16777216 --reps 2 > $OUT/ncu_nn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_ffma -s 1 -c 1 \
    -o $OUT/mlp_ffma_full -f python scripts/profile_driver.py nn --path 2 --rows 16777216 --reps 2 > $OUT/ncu_ffma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tf_ensemble -s 1 -c 1 \
    -o $OUT/tf_ensemble_full -f python scripts/profile_driver.py nn --arch transformer --rows 4194304 --reps 2 > $OUT/ncu_tf.log 2>&1
