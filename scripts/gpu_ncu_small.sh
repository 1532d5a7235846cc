#!/bin/bash
# ncu captures of the latency-bound kernels: the whole-run k_swarm (C2 f5) and
# the sequential-schedule k_seq (C2 shape, 1024 x 100 f5), summarised on the box.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_swarm -s 1 -c 1 -o /tmp/prof_sw python bench.py --steps 30 --warmup 3 --no-cpu --workload c2 > gpurun_out/ncu_sw.log 2>&1
python scripts/ncu_summary.py report /tmp/prof_sw.ncu-rep > gpurun_out/ncu_summary_c2_swarm.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_seq -c 1 -o /tmp/prof_seq python -c "
import sys; sys.path.insert(0, '.')
import paper_2110_01470_b200 as psso
fn = psso.make_function('f5', 100)
p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max, nsol=1024, nvar=100, niter=100)
print(psso.run_sequential(p, fn, 0).best_fitness)
" > gpurun_out/ncu_seq.log 2>&1
python scripts/ncu_summary.py report /tmp/prof_seq.ncu-rep > gpurun_out/ncu_summary_c2_seq.txt 2>&1
tail -n 1 gpurun_out/ncu_sw.log gpurun_out/ncu_seq.log
