#!/bin/bash
# full ncu captures of the fused kernel for several workloads (WORKLOADS, KERNEL regex)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for w in ${WORKLOADS:-c4 c5 c3f32}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KERNEL:-k_chain|k_rows}" -s 5 -c 1 -o gpurun_out/prof_$w python bench.py --steps 5 --warmup 3 --no-cpu --workload $w > gpurun_out/ncu_$w.log 2>&1
  tail -1 gpurun_out/ncu_$w.log
done
