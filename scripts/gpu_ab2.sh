#!/bin/bash
# Interleaved A/B of diag/libpsso_$V.so against the product build on one box.
#   V=name CASES="c3;c3f32 --rng philox;c4" REPS=3 bash scripts/gpu_ab2.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
IFS=';' read -ra LIST <<< "${CASES:-c3;c4}"
for args in "${LIST[@]}"; do
  for rep in $(seq ${REPS:-3}); do
    for lib in product $V; do
      L=$PWD/paper_2110_01470_b200/libpsso.so; [ $lib != product ] && L=$PWD/diag/libpsso_$V.so
      PSSO_LIB=$L timeout 300 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu --workload $args > gpurun_out/ab.log 2>&1
      python -c "
import json
for l in open('gpurun_out/ab.log'):
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$args', '$lib', 'kernel ms %.4f'%r['kernel_ms_per_iteration'], 'step ms %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], d['clocks']['reasons'])
" || tail -3 gpurun_out/ab.log
    done
  done
done
