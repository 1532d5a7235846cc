"""Generate tests/golden/seq_runs.npz by running the REFERENCE's sequential schedule.

Test infrastructure only.  Run in the build container, where the reference
package is importable from /root/reference/pkg/src (it does not exist on the GPU
box, which only reads the committed fixture):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_seq_golden.py

``run_sequential`` (reference core.py:213-258) keeps its final swarm local, so the
end state is captured by replaying its loop body (core.py:224-243) with the
reference's own helpers and checking the replay against the returned record.
"""

from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from sso.benchmarks import make_function  # noqa: E402
from sso.core import (  # noqa: E402
    SsoParams,
    _compose_update,
    _draw_update_fields,
    _eval_rows,
    initialize,
    run_sequential,
)
from sso.rng import RngStream  # noqa: E402

# (fid, nsol, nvar, niter, seed, thresholds or None)
RUNS = [
    ("f1", 100, 30, 1000, 0, None),    # C1 shape (10.383304882651581)
    ("f1", 100, 30, 200, 1, None),
    ("f2", 23, 7, 60, 4, None),
    ("f3", 19, 9, 60, 5, None),
    ("f4", 40, 10, 80, 42, None),
    ("f4", 64, 64, 40, 12, None),      # C4 row shape
    ("f5", 33, 20, 60, 6, None),
    ("f5", 64, 128, 30, 11, None),     # C3 row shape
    ("f6", 17, 12, 60, 7, (0.1, 0.3, 0.5)),
    ("f7", 14, 9, 40, 3, None),
    ("f8", 21, 16, 60, 8, None),
    ("f8", 12, 10, 30, 9, None),       # truncated form (uses 8 of 10)
    ("f9", 25, 13, 60, 10, None),
    ("f1", 1, 12, 40, 17, None),       # nsol = 1
    ("f1", 7, 1, 30, 2, None),         # nvar = 1
    ("f1", 300, 20, 30, 21, None),     # more rows than one pass of the CTA
    ("f1", 30, 20, 15, 1, (1.0, 1.0, 1.0)),   # all-keep thresholds
    ("f1", 30, 20, 15, 1, (0.0, 0.0, 0.0)),   # all-fresh thresholds
    ("f5", 30, 20, 15, 1, (0.0, 0.5, 0.5)),   # no gbest branch
    ("f4", 30, 20, 25, 3, (0.0, 0.0, 1.0)),   # every coordinate from gbest
]


def _params(fn, nsol, nvar, niter, thr):
    cw, cp, cg = thr if thr is not None else (0.3, 0.6, 0.8)
    return SsoParams(cw=cw, cp=cp, cg=cg, var_min=fn.var_min, var_max=fn.var_max,
                     nsol=nsol, nvar=nvar, niter=niter)


def replay(p, fn, seed):
    """core.py:219-243 verbatim in structure, keeping the swarm and the event count."""
    rng = RngStream(seed)
    sw = initialize(p, fn, rng)
    traj = np.empty(p.niter)
    moves = 0
    for t in range(p.niter):
        u, fresh = _draw_update_fields(rng, p, t, 0, p.nsol)
        for i in range(p.nsol):
            row = _compose_update(u[i], fresh[i], sw.sol[i], sw.pbests[i], sw.gbest, p)
            sw.sol[i] = row
            fx = float(_eval_rows(fn, row[None, :])[0])
            sw.sol_f[i] = fx
            if fx <= sw.p_f[i]:
                sw.pbests[i] = row
                sw.p_f[i] = fx
                if fx <= sw.g_f:
                    sw.gbest[:] = sw.pbests[i]
                    sw.g_f = fx
                    moves += 1
        traj[t] = sw.g_f
    return sw, traj, moves


def main():
    arrays, index = {}, []
    for k, (fid, nsol, nvar, niter, seed, thr) in enumerate(RUNS):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            fn = make_function(fid, nvar)
        p = _params(fn, nsol, nvar, niter, thr)
        rec = run_sequential(p, fn, seed)
        sw, traj, moves = replay(p, fn, seed)
        assert np.array_equal(traj, rec.trajectory) and np.array_equal(sw.gbest, rec.best_position)
        key = f"seq{k}"
        arrays[f"{key}_traj"] = rec.trajectory
        arrays[f"{key}_gbest"] = rec.best_position
        arrays[f"{key}_sol"] = sw.sol
        arrays[f"{key}_pbests"] = sw.pbests
        arrays[f"{key}_sol_f"] = sw.sol_f
        arrays[f"{key}_p_f"] = sw.p_f
        index.append(dict(key=key, fid=fid, nsol=nsol, nvar=nvar, niter=niter, seed=seed,
                          cw=p.cw, cp=p.cp, cg=p.cg, var_min=p.var_min, var_max=p.var_max,
                          best_fitness=rec.best_fitness, gbest_moves=moves))
        print(key, fid, nsol, nvar, niter, seed, rec.best_fitness, "gbest moves", moves,
              f"{rec.wall_time_s:.2f}s")
    np.savez_compressed(HERE / "seq_runs.npz", **arrays)
    (HERE / "seq_runs.json").write_text(json.dumps(index, indent=1) + "\n")


if __name__ == "__main__":
    main()
