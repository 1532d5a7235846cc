"""The paper's Table 3.10 setup on the B200.

f4 Rosenbrock, P = Nvar = 50, 1000 iterations, Nsol = 100 / 200 / 300 / 350:
CPU-SSO 48.8 / 193.1 / 434.9 / 582.7 s (i7-4770K), PSSO 0.139 / 0.154 / 0.164 /
0.170 s (GTX 1080).  Here: loop-only device time per run of both schedules,
single runs and 20-seed batches (per-run share), one JSON line per Nsol.
    python scripts/paper_table.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2110_01470_b200 as psso  # noqa: E402

PAPER = {100: (48.8263, 0.13875), 200: (193.10285, 0.154), 300: (434.8518, 0.1638),
         350: (582.71855, 0.1695)}
fn = psso.make_function("f4", 50)
for nsol, (cpu_s, gpu_s) in PAPER.items():
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=50, niter=1000)
    best = {}
    for name, call in (("parallel", lambda: psso.run_parallel(p, fn, 0).wall_time_s),
                       ("sequential", lambda: psso.run_sequential(p, fn, 0).wall_time_s),
                       ("parallel_batch20", lambda: psso.run_parallel_batch(p, fn, range(20))[0].wall_time_s / 20),
                       ("sequential_batch20", lambda: psso.run_sequential_batch(p, fn, range(20))[0].wall_time_s / 20)):
        best[name] = min(call() for _ in range(3))
    print(json.dumps({"fn": "f4", "nsol": nsol, "nvar": 50, "niter": 1000,
                      "b200_s_per_run": {k: round(v, 6) for k, v in best.items()},
                      "paper_cpu_sso_s": cpu_s, "paper_psso_gtx1080_s": gpu_s,
                      "vs_paper_psso": round(gpu_s / best["parallel"], 1)}), flush=True)
