#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/san_$tool.log | tail -4
done
PSSO_SWARM_NO_CLUSTER=1 timeout 900 compute-sanitizer --tool racecheck python scripts/sanitize_run.py > gpurun_out/san_race_nocluster.log 2>&1
echo "== racecheck (global swarm exchange) rc=$?"; grep -E "SUMMARY" gpurun_out/san_race_nocluster.log | tail -2
