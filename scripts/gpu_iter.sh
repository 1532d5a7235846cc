#!/bin/bash
# One development iteration on the GPU: correctness, the workload benches and
# (NCU=<workload>) one full ncu capture of the chain/fused kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
fi
for w in ${WORKLOADS:-c3 c3f32 c4 c5 c3sphere}; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --workload $w $BENCH_ARGS > gpurun_out/bench_$w.log 2>&1
  python -c "
import json
for l in open('gpurun_out/bench_$w.log'):
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$w', '%.4g pvu/s'%d['value'], 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f ms'%r['kernel_ms_per_iteration'], 'frac %.3f'%r['frac'], 'e2e %.4g'%d['e2e']['value'])
" || tail -5 gpurun_out/bench_$w.log
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_chain} -s 5 -c 1 -o gpurun_out/prof_$NCU python bench.py --steps 5 --warmup 3 --no-cpu --workload $NCU > gpurun_out/ncu_$NCU.log 2>&1
  tail -1 gpurun_out/ncu_$NCU.log
fi
