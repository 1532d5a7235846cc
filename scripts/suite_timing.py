"""The C2 benchmark suite as one harness experiment (4 functions x both schedules x 30
seeds, N=1024, D=100, 1000 iterations), cells serial vs concurrent (parallel_cells)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2110_01470_b200 import harness as H  # noqa: E402
from paper_2110_01470_b200.records import ScheduleKind  # noqa: E402

kw = dict(functions=["f5", "f4", "f6", "f7"], schedules=[ScheduleKind.SEQUENTIAL, ScheduleKind.PARALLEL],
          replications=30, nsol=1024, nvar=100, niter=1000)
H.run_experiment(H.ExperimentConfig(**{**kw, "replications": 2, "niter": 10}))  # warm
for par in (False, True, False, True):
    t0 = time.perf_counter()
    rep = H.run_experiment(H.ExperimentConfig(parallel_cells=par, **kw))
    el = time.perf_counter() - t0
    print(json.dumps({"parallel_cells": par, "cells": 8, "runs": len(rep.records), "wall_s": round(el, 3),
                      "per_run_ms": round(1e3 * el / len(rep.records), 3)}), flush=True)
