cd $GRAFT_REPO_ROOT
timeout 300 compute-sanitizer --tool memcheck python scripts/repro_fused.py f4 16384 64 2 > gpurun_out/san_memcheck.log 2>&1
tail -4 gpurun_out/san_memcheck.log
timeout 300 compute-sanitizer --tool synccheck python scripts/repro_fused.py f5 8192 128 2 > gpurun_out/san_synccheck.log 2>&1
tail -4 gpurun_out/san_synccheck.log
bash scripts/gpu_iter.sh
