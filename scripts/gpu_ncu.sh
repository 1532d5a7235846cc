#!/bin/bash
# Full ncu captures (steady state: launch ~250 of the iteration kernel) of the
# main workloads, summarised ON THE BOX (scripts/ncu_summary.py) so only text
# and one report come back (gpurun_out is capped at 64 MiB).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
units() { case $1 in c3|c3f32|c3sphere) echo $((1048576*128));; c4) echo $((16777216*64));; c5) echo $((65536*4096));; esac; }
for w in ${NCU_WORKLOADS:-c3 c3f32 c4 c5}; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --workload $w > gpurun_out/bench_$w.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain|k_rows|k_fused|k_tile" -s ${SKIP:-250} -c 1 -o /tmp/prof_$w python bench.py --steps $(( ${SKIP:-250} + 10 )) --warmup 3 --no-cpu --workload $w > gpurun_out/ncu_$w.log 2>&1
  tail -1 gpurun_out/ncu_$w.log
  python scripts/ncu_summary.py report /tmp/prof_$w.ncu-rep --units $(units $w) > gpurun_out/ncu_summary_$w.txt 2>&1
  python scripts/ncu_summary.py traffic /tmp/prof_$w.ncu-rep --workload $w --bench-log gpurun_out/bench_$w.log >> gpurun_out/ncu_summary_$w.txt 2>&1
  cp bench_traffic.json gpurun_out/bench_traffic.json
done
cp /tmp/prof_${KEEP:-c3}.ncu-rep gpurun_out/ 2>/dev/null
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_c3.csv > gpurun_out/launches_c3.txt
fi
