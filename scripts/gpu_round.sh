#!/bin/bash
# One full GPU pass: smoke, gpu tests, the contract bench (+ reference arm), the
# other BASELINE workloads, the ncu launch list and full captures (steady state,
# iteration ~250) of the iteration kernel of the main workloads.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
for w in ${WORKLOADS:-c3f32 c4 c5 c2 c2f4 c2f6 c2f7 c1 c3sphere}; do
  timeout 400 python bench.py --steps ${STEPS:-200} --warmup 5 --no-cpu --workload $w > gpurun_out/bench_$w.log 2>&1
  python -c "
import json
for l in open('gpurun_out/bench_$w.log'):
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$w', '%.4g pvu/s'%d['value'], 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f ms'%r['kernel_ms_per_iteration'], 'frac %.3f'%r['frac'], 'e2e %.4g'%d['e2e']['value'], r['kernel'])
" || tail -5 gpurun_out/bench_$w.log
done
if [ -z "$SKIP_NCU" ]; then LAUNCHES=1 bash scripts/gpu_ncu.sh; fi
