#!/bin/bash
# Persistent-grid SM count sweep under the board's power cap (PSSO_FUSED_SMS).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for w in ${WORKLOADS:-c4 c3}; do
  for n in ${SMS:-148 140 132 124 116}; do
    PSSO_FUSED_SMS=$n timeout 300 python bench.py --steps ${STEPS:-300} --warmup 5 --no-cpu --workload $w > gpurun_out/sm.log 2>&1
    python -c "
import json
for l in open('gpurun_out/sm.log'):
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$w', 'sms $n', 'k %.4f'%r['kernel_ms_per_iteration'], 'step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])
" || tail -3 gpurun_out/sm.log
  done
done
done
