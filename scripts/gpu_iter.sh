# one development iteration on the GPU: correctness, benches, one ncu capture
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-c3 c3sphere c3f32 c4 c5}; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --workload $w > gpurun_out/bench_$w.log 2>&1
  python -c "
import json
for l in open('gpurun_out/bench_$w.log'):
  if l.startswith('{'):
    d=json.loads(l); print('$w', '%.3g pvu/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f ms'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'])
" || tail -5 gpurun_out/bench_$w.log
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_$NCU python bench.py --steps 5 --warmup 3 --no-cpu --workload $NCU > gpurun_out/ncu_$NCU.log 2>&1
  tail -2 gpurun_out/ncu_$NCU.log
fi
