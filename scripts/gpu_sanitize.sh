cd $GRAFT_REPO_ROOT
timeout 300 compute-sanitizer --tool memcheck python scripts/repro_fused.py f4 16384 64 2 > gpurun_out/san_memcheck.log 2>&1
tail -40 gpurun_out/san_memcheck.log
timeout 300 python scripts/repro_fused.py f4 16384 64 3 > gpurun_out/repro.log 2>&1; tail -8 gpurun_out/repro.log
