# c5 replay (one long trace, one warp): source-level stall profile of the
# large shared-memory tier on a 100k-task prefix.
set -u
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
    -o gpurun_out/prof/replay_c5_full -f python scripts/profile_driver.py fused --tasks 100000 --reps 1 > gpurun_out/prof/ncu_c5.log 2>&1
python scripts/profile_summary.py report gpurun_out/prof/replay_c5_full.ncu-rep > gpurun_out/prof/ncu_replay_c5.txt 2>&1
python scripts/ncu_lines.py gpurun_out/prof/replay_c5_full.ncu-rep paper_2508_19073_b200/csrc/build/replay.cu.o \
    "LayoutILi64ELi1024" paper_2508_19073_b200/csrc/cuda/replay_kernel.cuh 70 > gpurun_out/prof/c5_lines.txt 2>&1
