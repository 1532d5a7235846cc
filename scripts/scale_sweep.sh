#!/bin/bash
# Strong-scaling sweep on a multi-GPU node (not runnable on the one-GPU boxes of
# this build): the default C4 workload at N = 1, 2, 4, 8 GPUs with the NCCL graph
# exchange and with the device-initiated P2P exchange; prints pvu/s and the
# efficiency value(N) / (N * value(1)).
cd ${GRAFT_REPO_ROOT:-$(dirname "$0")/..}; mkdir -p gpurun_out
ngpu=$(nvidia-smi -L | wc -l)
for ex in nccl p2p; do
  base=""
  for n in 1 2 4 8; do
    [ $n -gt $ngpu ] && break
    python bench.py --gpus $n --steps ${STEPS:-50} --warmup 5 --no-cpu --workload ${WORKLOAD:-c4} \
      --exchange $ex > gpurun_out/scale_${ex}_$n.log 2>&1
    v=$(python -c "
import json
for l in open('gpurun_out/scale_${ex}_$n.log'):
  if l.startswith('{'): print(json.loads(l)['value'])")
    [ -z "$base" ] && base=$v
    python -c "print('$ex', 'N=$n', '%.4g pvu/s' % $v, 'efficiency %.3f' % ($v / ($n * $base)))"
  done
done
