#!/bin/bash
# whole-run kernel tuning: C1/C2 per-iteration time vs row groups per CTA, plus one ncu capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in ${GPCS:-1 2 4 8 16}; do
  for w in c2 c1; do
    PSSO_SWARM_GPC=$g timeout 120 python bench.py --steps 200 --warmup 5 --no-cpu --workload $w > gpurun_out/sw_${w}_$g.log 2>&1
    python -c "
import json
for l in open('gpurun_out/sw_${w}_$g.log'):
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('gpc=$g', '$w', 'us/iter %.2f'%(1e3*r['kernel_ms_per_iteration']), r['kernel'])
" || tail -3 gpurun_out/sw_${w}_$g.log
  done
done
if [ -n "$NCU" ]; then
PSSO_SWARM_GPC=${NCU} timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_swarm -c 1 -o /tmp/prof_sw python bench.py --steps 30 --warmup 3 --no-cpu --workload c2 > gpurun_out/ncu_sw.log 2>&1
tail -1 gpurun_out/ncu_sw.log
python scripts/ncu_summary.py report /tmp/prof_sw.ncu-rep > gpurun_out/ncu_summary_sw.txt 2>&1
ncu -i /tmp/prof_sw.ncu-rep --page source --csv --print-source sass > gpurun_out/sw_sass.csv 2>/dev/null
fi
