# replay parity (all replay / sweep / timeline / bridge / full-size tests) + c5 and c4 timings
set -u
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_sweep.py tests/test_gpu_timeline.py tests/test_gpu_acceptance.py tests/test_gpu_fullsize.py tests/test_gpu_bridge.py -m gpu -x -q > gpurun_out/replay_t.log 2>&1; echo rc=$? >> gpurun_out/replay_t.log
tail -3 gpurun_out/replay_t.log
timeout 300 python scripts/profile_driver.py fused --tasks 1000000 --reps 2 2>&1 | tail -3
timeout 300 python scripts/profile_driver.py replay --traces 100000 --reps 3 2>&1 | tail -3
if [ -f ab/libcarma_prof.so ]; then CARMA_B200_LIB=$PWD/ab/libcarma_prof.so timeout 300 python scripts/profile_driver.py fused --tasks 200000 --reps 1 2>&1 | tail -10; fi
