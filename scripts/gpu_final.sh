#!/bin/bash
# The round's committed measurements, one box: smoke, GPU tests, the default
# bench line + reference arm, every workload, the ncu launch list of the
# default bench and steady-state full captures (summaries + bench_traffic.json).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,memory.total --format=csv > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$?" >> $O/bench_default.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference_arm.log 2>&1
: > $O/bench_workloads.jsonl
IFS=';' read -ra LIST <<< "${WORKLOADS:-c3;c3 --rng philox;c3f32;c3f32 --rng philox;c4 --rng philox;c5;c5 --rng philox;c2;c2f4;c2f6;c2f7;c1}"
for a in "${LIST[@]}"; do
  timeout 600 python bench.py --steps ${STEPS:-200} --warmup 5 --no-cpu --workload $a > $O/bw.log 2>&1
  grep '^{' $O/bw.log >> $O/bench_workloads.jsonl || (echo "FAILED $a"; tail -5 $O/bw.log)
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python bench.py --steps 20 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1
python scripts/ncu_summary.py launches $O/launches_c4.csv > $O/launches_c4.txt
units() { case $1 in c3|c3f32) echo $((1048576*128));; c4) echo $((16777216*64));; c5) echo $((65536*4096));; esac; }
IFS=';' read -ra CAP <<< "${CASES:-c4:c4;c3:c3;c3f32_philox:c3f32 --rng philox;c5:c5;c3f32:c3f32;c5_philox:c5 --rng philox}"
for item in "${CAP[@]}"; do
  name=${item%%:*}; args=${item#*:}; wl=${args%% *}
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --workload $args > $O/bench_$name.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain|k_rows" -s ${SKIP:-250} -c 1 -o /tmp/prof_$name python bench.py --steps $(( ${SKIP:-250} + 10 )) --warmup 3 --no-cpu --workload $args > $O/ncu_$name.log 2>&1
  python scripts/ncu_summary.py report /tmp/prof_$name.ncu-rep --units $(units $wl) > $O/ncu_full_$name.txt 2>&1
  python scripts/ncu_summary.py traffic /tmp/prof_$name.ncu-rep --workload $name --bench-log $O/bench_$name.log >> $O/ncu_full_$name.txt 2>&1
done
cp bench_traffic.json $O/bench_traffic.json
cp /tmp/prof_c4.ncu-rep $O/ 2>/dev/null
echo done
