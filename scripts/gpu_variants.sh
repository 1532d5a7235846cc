# correctness of the current kernel + throughput of each tuning variant
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for lib in variants/*.so; do
  for w in c3 c3sphere c3f32 c5 c4; do
    PSSO_LIB=$PWD/$lib timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --workload $w > gpurun_out/v_$(basename $lib .so)_$w.log 2>&1
    python -c "
import json
for l in open('gpurun_out/v_$(basename $lib .so)_$w.log'):
  if l.startswith('{'):
    d=json.loads(l); print('$(basename $lib .so)', '$w', '%.3g pvu/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])
"
  done
done
