#!/bin/bash
# Steady-state ncu captures (launch ~SKIP of the iteration kernel) of named
# bench configurations, summarised on the box (scripts/ncu_summary.py).
#   CASES="c3f32p:c3f32 --rng philox  c4:c4" SKIP=250 bash scripts/gpu_ncu2.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
units() { case $1 in c3|c3f32|c3sphere) echo $((1048576*128));; c4) echo $((16777216*64));; c5) echo $((65536*4096));; esac; }
IFS=';' read -ra LIST <<< "${CASES:-c3:c3;c3f32p:c3f32 --rng philox;c4:c4;c5:c5}"
for item in "${LIST[@]}"; do
  name=${item%%:*}; args=${item#*:}; wl=${args%% *}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain|k_rows|k_fused|k_tile" -s ${SKIP:-250} -c 1 -o /tmp/prof_$name python bench.py --steps $(( ${SKIP:-250} + 10 )) --warmup 3 --no-cpu --workload $args > gpurun_out/ncu_$name.log 2>&1
  tail -1 gpurun_out/ncu_$name.log
  python scripts/ncu_summary.py report /tmp/prof_$name.ncu-rep --units $(units $wl) > gpurun_out/ncu_summary_$name.txt 2>&1
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv > gpurun_out/ncu_source_$name.csv 2>/dev/null
done
for k in ${KEEP:-}; do cp /tmp/prof_$k.ncu-rep gpurun_out/ 2>/dev/null; done
