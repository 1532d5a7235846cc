#!/bin/bash
# ncu capture of the whole-run kernel on C2 (one launch of 30 iterations)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_swarm -s 1 -c 1 -o /tmp/prof_sw python bench.py --steps 30 --warmup 3 --no-cpu --workload ${W:-c2} > gpurun_out/ncu_sw.log 2>&1
tail -1 gpurun_out/ncu_sw.log
python scripts/ncu_summary.py report /tmp/prof_sw.ncu-rep > gpurun_out/ncu_summary_sw.txt 2>&1
ncu -i /tmp/prof_sw.ncu-rep --page source --csv --print-source sass > gpurun_out/sw_sass.csv 2>/dev/null
ncu -i /tmp/prof_sw.ncu-rep --page source --csv --print-source cuda > gpurun_out/sw_cuda.csv 2>/dev/null
