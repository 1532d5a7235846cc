# profiling pass: launch list + one full ncu capture of the fused kernel + bench variants
cd $GRAFT_REPO_ROOT
for w in c3 c3sphere c3f32 c3sphere32 c5 c4; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --workload $w > gpurun_out/bench_$w.log 2>&1
done
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --workload c3 --rng philox > gpurun_out/bench_c3_philox.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -o gpurun_out/prof_c3 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -o gpurun_out/prof_c3sphere python bench.py --steps 5 --warmup 3 --no-cpu --workload c3sphere > gpurun_out/ncu_c3sphere.log 2>&1
for f in gpurun_out/bench_*.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
  if l.startswith('{'):
    d=json.loads(l); print(d['config']['workload'], '%.3g pvu/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['clocks'])
" ; done
tail -3 gpurun_out/ncu_c3.log
