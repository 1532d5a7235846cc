"""Timing of the sequential schedule (run_sequential) on device vs the CPU oracle.

    python scripts/seq_timing.py
One JSON line per configuration: device loop time (CUDA events, one k_seq
launch), speculative passes, and the oracle's single-thread serial loop.
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (CPU baseline only)
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

CONFIGS = [("f1", 100, 30, 1000), ("f5", 1024, 100, 1000), ("f4", 1024, 100, 1000),
           ("f6", 1024, 100, 1000), ("f5", 16384, 128, 100)]

for fid, nsol, nvar, niter in CONFIGS:
    fn = psso.make_function(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=niter)
    best = None
    for _ in range(3):
        eng = DeviceEngine(p, fn, 0)
        eng.initialize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        eng.run_sequential(0, niter)
        b.record(eng.stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        passes = eng.sequential_passes
        gf = float(eng.g_f.cpu()[0])
        eng.close()
        best = ms if best is None else min(best, ms)
    # parallel schedule on the same shape, for scale
    rec = psso.run_parallel(p, fn, 0)
    o = O.Oracle.from_params(p, fid, 0)
    sw = o.initialize()
    n_cpu = max(1, min(niter, int(2e7 // (nsol * nvar))))
    t0 = time.perf_counter()
    o.run_sequential(sw, 0, n_cpu)
    cpu_s = (time.perf_counter() - t0) * niter / n_cpu
    print(json.dumps({"fn": fid, "nsol": nsol, "nvar": nvar, "niter": niter,
                      "seq_device_ms": round(best, 3), "passes": passes,
                      "passes_per_iteration": round(passes / niter, 3),
                      "seq_pvu_per_s": nsol * nvar * niter / (best * 1e-3),
                      "parallel_device_ms": round(rec.wall_time_s * 1e3, 3),
                      "oracle_seq_1thread_s": round(cpu_s, 3),
                      "oracle_iters_timed": n_cpu, "final_g_f": gf}), flush=True)
