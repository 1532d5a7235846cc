cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
run() { # label, env..., workload
  label=$1; shift; w=$1; shift
  env "$@" timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --workload $w > gpurun_out/b_${label}_$w.log 2>&1
  python -c "
import json
for l in open('gpurun_out/b_${label}_$w.log'):
  if l.startswith('{'):
    d=json.loads(l); print('$label', '$w', '%.3g pvu/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f ms'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'])
" || tail -3 gpurun_out/b_${label}_$w.log
}
for w in c3 c3sphere c3f32 c4 c5; do run main $w; done
for w in c3 c3sphere c3f32 c4; do run cm3 $w PSSO_LIB=$PWD/variants/libpsso_cm3.so; run cm4 $w PSSO_LIB=$PWD/variants/libpsso_cm4.so; run nochain $w PSSO_NO_CHAIN=1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 3 -c 1 -o gpurun_out/prof_chain_c3 python bench.py --steps 5 --warmup 3 --no-cpu --workload c3 > gpurun_out/ncu_chain_c3.log 2>&1
tail -1 gpurun_out/ncu_chain_c3.log
