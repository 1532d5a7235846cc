"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Test infrastructure only.  Run in the build container, where the reference
package is importable from /root/reference/pkg/src (it does not exist on the GPU
box, which only reads the committed .npz files):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array is stored bit-exactly (float64 / uint64 in .npz).  Inputs for the
fitness fixtures are NOT stored: they are regenerated from the keyed INIT stream
(``var_min + span * u(INIT, 0, i, j)``, reference core.py:198-199), which is itself
pinned bit-for-bit by ``rng.npz``.
"""

from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import sso  # noqa: E402  (the reference package)
from sso.benchmarks import make_function  # noqa: E402
from sso.core import SsoParams, initialize, run_sequential  # noqa: E402
from sso.parallel import (  # noqa: E402
    evaluate_phase,
    run_parallel,
    search_phase,
    update_gbest_phase,
    update_pbests_phase,
)
from sso.rng import RngStream, SubStream  # noqa: E402

DEFAULTS = dict(cw=0.3, cp=0.6, cg=0.8)

# (fid, nsol, nvar, niter, seed, thresholds or None, store_state)
RUNS = [
    ("f1", 100, 30, 1000, 0, None, False),   # C1 (BASELINE.json configs[0])
    ("f1", 100, 30, 1000, 1, None, False),
    ("f5", 1024, 100, 1000, 0, None, False),  # C2 suite
    ("f4", 1024, 100, 1000, 0, None, False),
    ("f6", 1024, 100, 1000, 0, None, False),
    ("f7", 1024, 100, 1000, 0, None, False),
    ("f1", 16, 10, 40, 3, None, True),
    ("f2", 23, 7, 40, 4, None, True),
    ("f3", 19, 9, 40, 5, None, True),
    ("f4", 23, 10, 25, 42, None, True),
    ("f5", 33, 20, 40, 6, None, True),
    ("f6", 17, 12, 40, 7, (0.1, 0.3, 0.5), True),
    ("f7", 14, 9, 20, 3, None, True),
    ("f8", 21, 16, 40, 8, None, True),
    ("f8", 12, 10, 20, 9, None, True),        # truncated form (uses 8 of 10)
    ("f9", 25, 13, 40, 10, None, True),
    ("f1", 1, 12, 40, 17, None, True),        # nsol = 1
    ("f4", 1, 12, 40, 17, None, True),
    ("f1", 7, 1, 30, 2, None, True),          # nvar = 1
    ("f5", 64, 128, 30, 11, None, True),      # C3 row shape, short
    ("f4", 64, 64, 30, 12, None, True),       # C4 row shape, short
    ("f6", 8, 4096, 8, 13, None, False),      # C5 row shape, short
    ("f2", 40, 300, 20, 14, None, False),     # multi-leaf pairwise plan
    ("f3", 10, 129, 20, 15, None, True),
    ("f1", 30, 20, 15, 1, (1.0, 1.0, 1.0), True),   # all-keep thresholds
    ("f1", 30, 20, 15, 1, (0.0, 0.0, 0.0), True),   # all-fresh thresholds
    ("f5", 30, 20, 15, 1, (0.0, 0.5, 0.5), True),   # no gbest branch
]

FIT_DIMS = [1, 2, 3, 4, 7, 8, 9, 16, 30, 48, 50, 63, 64, 100, 127, 128, 129, 256,
            300, 1000, 4095, 4096]
FIT_ROWS = 6


def _params(fn, nsol, nvar, niter, thr):
    cw, cp, cg = thr if thr is not None else (DEFAULTS["cw"], DEFAULTS["cp"], DEFAULTS["cg"])
    return SsoParams(cw=cw, cp=cp, cg=cg, var_min=fn.var_min, var_max=fn.var_max,
                     nsol=nsol, nvar=nvar, niter=niter)


def gen_rng():
    seeds = np.array([0, 1, 42, 7, 0xDEADBEEFCAFEF00D, (1 << 64) - 1], dtype=np.uint64)
    streams = np.array([int(s) for s in SubStream], dtype=np.uint64)
    iters = np.array([0, 1, 7, 999, 123456], dtype=np.uint64)
    parts = np.array([0, 1, 5, 1000, (1 << 20) - 1, (1 << 24) + 3], dtype=np.uint64)
    vars_ = np.array([0, 1, 2, 3, 127, 4095], dtype=np.uint64)
    out = np.empty((len(seeds), len(streams), len(iters), len(parts), len(vars_)), np.float64)
    for a, s in enumerate(seeds):
        r = RngStream(int(s))
        for b, st in enumerate(SubStream):
            for c, t in enumerate(iters):
                out[a, b, c] = r.uniform(st, int(t), parts[:, None], vars_[None, :])
    # seed masking (rng.py:68)
    wide = RngStream((1 << 64) + 42).uniform(SubStream.BRANCH, 0, 0, 0)
    np.savez(HERE / "rng.npz", seeds=seeds, streams=streams, iters=iters, parts=parts,
             vars=vars_, u=out, wide_seed_u=np.float64(wide))


def gen_fitness():
    arrays = {}
    for fid in sso.FUNCTION_IDS:
        for d in FIT_DIMS:
            if fid == "f4" and d < 2:
                continue
            if fid == "f8" and d < 4:
                continue
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                fn = make_function(fid, d)
            lo, hi = fn.bounds
            u = RngStream(1000 + d).matrix(SubStream.INIT, 0, 0, FIT_ROWS, d)
            x = lo + (hi - lo) * u
            arrays[f"{fid}_{d}"] = fn(x)
            arrays[f"{fid}_{d}_refpt"] = np.float64(fn(fn.reference_point))
    np.savez(HERE / "fitness.npz", **arrays)


def gen_runs():
    arrays = {}
    index = []
    for k, (fid, nsol, nvar, niter, seed, thr, store) in enumerate(RUNS):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            fn = make_function(fid, nvar)
        p = _params(fn, nsol, nvar, niter, thr)
        rec = run_parallel(p, fn, seed)
        init = initialize(p, fn, RngStream(seed))
        key = f"run{k}"
        arrays[f"{key}_traj"] = rec.trajectory
        arrays[f"{key}_gbest"] = rec.best_position
        arrays[f"{key}_init_p_f"] = init.p_f
        arrays[f"{key}_init_g_f"] = np.float64(init.g_f)
        if store:
            # replay the phased loop to capture the final swarm state
            rng = RngStream(seed)
            sw = initialize(p, fn, rng)
            for t in range(niter):
                search_phase(sw, p, rng, t)
                evaluate_phase(sw, fn, t)
                update_pbests_phase(sw)
                update_gbest_phase(sw)
            assert np.array_equal(sw.gbest, rec.best_position)
            arrays[f"{key}_sol"] = sw.sol
            arrays[f"{key}_pbests"] = sw.pbests
            arrays[f"{key}_sol_f"] = sw.sol_f
            arrays[f"{key}_p_f"] = sw.p_f
        cw, cp, cg = (p.cw, p.cp, p.cg)
        index.append(dict(key=key, fid=fid, nsol=nsol, nvar=nvar, niter=niter, seed=seed,
                          cw=cw, cp=cp, cg=cg, var_min=p.var_min, var_max=p.var_max,
                          state=store, best_fitness=rec.best_fitness,
                          init_best=int(np.argmin(init.p_f))))
        print(key, fid, nsol, nvar, niter, seed, rec.best_fitness, f"{rec.wall_time_s:.2f}s")
    # per-iteration state dump of one small run (step-wise comparison)
    fn = make_function("f4", 10)
    p = _params(fn, 12, 10, 12, None)
    rng = RngStream(5)
    sw = initialize(p, fn, rng)
    xs, ps, pfs, gs = [], [], [], []
    for t in range(p.niter):
        search_phase(sw, p, rng, t)
        evaluate_phase(sw, fn, t)
        update_pbests_phase(sw)
        update_gbest_phase(sw)
        xs.append(sw.sol.copy()); ps.append(sw.pbests.copy())
        pfs.append(sw.p_f.copy()); gs.append(sw.gbest.copy())
    arrays["steps_sol"] = np.stack(xs)
    arrays["steps_pbests"] = np.stack(ps)
    arrays["steps_p_f"] = np.stack(pfs)
    arrays["steps_gbest"] = np.stack(gs)
    # sequential schedule, for the nsol=1 coincidence and C1 oracle value
    fn = make_function("f1", 30)
    seq = run_sequential(_params(fn, 100, 30, 1000, None), fn, 0)
    arrays["seq_c1_traj"] = seq.trajectory
    np.savez_compressed(HERE / "runs.npz", **arrays)
    (HERE / "runs.json").write_text(json.dumps(index, indent=1) + "\n")


if __name__ == "__main__":
    gen_rng()
    gen_fitness()
    gen_runs()
