#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in ${GS:-1 2 4 8 16}; do
  for w in c2 c1; do
    echo "G=$g $w: $(PSSO_LIB=$PWD/diag/libpsso_trace.so PSSO_SWARM_G=$g timeout 120 python bench.py --steps 200 --warmup 5 --no-cpu --workload $w 2>&1 | grep 'swarm trace' | tail -1)"
  done
done
