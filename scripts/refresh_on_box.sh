#!/bin/bash
# refresh_profiles.sh with the ncu reports kept on the box (they exceed
# gpurun's 64 MiB copy-back): the summaries committed under profiles/ are
# written here, on the box, into gpurun_out/profiles/.
set -u
R=${ROUND:-r02}
export OUT=/tmp/prof
mkdir -p $OUT gpurun_out/profiles
bash scripts/refresh_profiles.sh
P=gpurun_out/profiles
cp $OUT/bench.json $OUT/bench.err $OUT/launches.csv $OUT/bench_detail_n1.json $P/ 2>/dev/null
tail -1 $OUT/bench.json > $P/bench_${R}_n1.json
python scripts/profile_summary.py launches $OUT/launches.csv > $P/launches_${R}.txt 2>&1
python scripts/profile_summary.py traffic $OUT/knn_search_full.ncu-rep:knn_search \
    $OUT/replay_kernel_full.ncu-rep:replay_kernel $OUT/pick_kernel_full.ncu-rep:pick_kernel \
    $OUT/nn_ensemble_full.ncu-rep:nn_ensemble $OUT/tf_ensemble_full.ncu-rep:tf_ensemble \
    $OUT/mlp_ffma_full.ncu-rep:mlp_ffma > $P/traffic.json 2>&1
for k in knn_search:knn_search_full replay_kernel:replay_kernel_full pick_kernel:pick_kernel_full \
         replay_c5:replay_c5_full nn_ensemble:nn_ensemble_full tf_ensemble:tf_ensemble_full mlp_ffma:mlp_ffma_full; do
    n=${k%%:*}; f=${k##*:}
    python scripts/profile_summary.py report $OUT/$f.ncu-rep > $P/ncu_${n}_${R}.txt 2>&1
done
O=paper_2508_19073_b200/csrc/build/gpumemnet.cu.o
{ echo "  SASS of gpumemnet.cu.o (cuobjdump -sass | tcgen05 mnemonics):"
  cuobjdump -sass $O | grep -oE "UTCHMMA|UTCBAR|LDTM|STTM|UTCATOMSWS" | sort | uniq -c | sed 's/^/   /'
  echo "  stall samples by source line (scripts/ncu_lines.py):"
  python scripts/ncu_lines.py $OUT/nn_ensemble_full.ncu-rep $O "nn_ensembleILi3ELi3ELi8ELb0E" \
      paper_2508_19073_b200/csrc/cuda/gpumemnet.cu 15 2>/dev/null | sed 's/^/   /'; } >> $P/ncu_nn_ensemble_${R}.txt
ls -la $P
