# k-NN host-buffer e2e A/B over chunk sizes (ab/libcarma_e2e_c*.so), two runs each
set -u
run() { timeout 600 python bench.py --skip-replay --skip-fused --skip-small --skip-scoring --skip-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('knn e2e', d['e2e']['value']/1e6)"; }
for r in 1 2; do
  echo "== base (2^21)"; run
  for v in ab/libcarma_e2e_c*.so; do echo "== $v"; CARMA_B200_LIB=$PWD/$v run; done
done
