#!/bin/bash
# Interleaved A/B of diag/libpsso_$V.so against the product build on one box:
# REPS alternations per workload, kernel ms per iteration of each run.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
PSSO_LIB=$PWD/diag/libpsso_$V.so timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_$V.log 2>&1; echo "pytest[$V] rc=$?"
fi
for w in ${WORKLOADS:-c3 c3f32 c4}; do
  for rep in $(seq ${REPS:-3}); do
    for lib in product $V; do
      L=$PWD/paper_2110_01470_b200/libpsso.so; [ $lib != product ] && L=$PWD/diag/libpsso_$V.so
      PSSO_LIB=$L timeout 300 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu --workload $w > gpurun_out/ab.log 2>&1
      python -c "
import json
for l in open('gpurun_out/ab.log'):
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$w', '$lib', 'kernel ms %.4f'%r['kernel_ms_per_iteration'], 'step ms %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'])
" || tail -3 gpurun_out/ab.log
    done
  done
done
