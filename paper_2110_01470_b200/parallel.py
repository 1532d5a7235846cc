"""Barrier-synchronized phased engine (reference parallel.py) on the B200.

``run_parallel`` keeps the reference signature (parallel.py:152-158) and
returns the same ``RunRecord``; the iteration loop runs as one fused sm_100a
kernel (search + evaluate + pBest + per-CTA gBest candidate) plus a one-CTA
gBest stage-2 kernel per iteration, replayed from a CUDA graph, with the
swarm resident in HBM.  ``workers`` and ``layout`` are validated and then
have no effect, exactly as in the reference (they never change the output);
the device layout is particle-major.

The phase functions operate on a host ``Swarm`` like the reference's
(parallel.py:120-144): the swarm is uploaded, the phase runs as a device
kernel, and the fields that phase owns are written back in place.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .benchmarks import make_function
from .core import SsoParams, Swarm
from .records import RunRecord, ScheduleKind

__all__ = [
    "LayoutMode",
    "Schedule",
    "convert_layout",
    "search_phase",
    "evaluate_phase",
    "update_pbests_phase",
    "update_gbest_phase",
    "run_parallel",
    "run_parallel_batch",
    "run_sequential_batch",
]


class LayoutMode(str, enum.Enum):
    """Storage order of the (nsol, nvar) matrices; no semantic effect (parallel.py:53-60)."""

    PARTICLE_MAJOR = "particle-major"
    INTERLEAVED = "interleaved"

    def __str__(self) -> str:
        return self.value


@dataclass(frozen=True)
class Schedule:
    """Which engine to run and, for the phased one, how many workers (parallel.py:63-72)."""

    kind: ScheduleKind
    workers: int = 1

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")


def convert_layout(data: np.ndarray, src: LayoutMode, dst: LayoutMode) -> np.ndarray:
    """Re-store a host matrix in the requested order; indexing unchanged (parallel.py:75-84)."""
    data = np.asarray(data)
    if data.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {data.shape}")
    if src == dst:
        return data
    if dst is LayoutMode.INTERLEAVED:
        return np.asfortranarray(data)
    return np.ascontiguousarray(data)


# ------------------------------------------------------------------ phases --

def _phase_params(swarm: Swarm, f=None, params: SsoParams = None) -> SsoParams:
    if params is not None:
        return params
    lo, hi = (f.var_min, f.var_max) if f is not None else (-1.0, 1.0)
    return SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=lo, var_max=hi,
                     nsol=swarm.nsol, nvar=swarm.nvar, niter=1)


def _engine_for(swarm: Swarm, params: SsoParams, f, seed: int):
    from .engine import DeviceEngine

    eng = DeviceEngine(params, f, seed, keep_sol_f=True)
    eng.load(swarm)
    return eng


def _write_back(swarm: Swarm, host: Swarm, fields) -> None:
    for name in fields:
        if name == "g_f":
            swarm.g_f = host.g_f
        else:
            getattr(swarm, name)[...] = getattr(host, name)


def search_phase(swarm: Swarm, params: SsoParams, rng, iteration: int) -> Swarm:
    """Rewrite every position from the phase-entry personal/global bests (parallel.py:120-124)."""
    fn = make_function("f1", swarm.nvar)  # search evaluates nothing; any objective works
    eng = _engine_for(swarm, params, fn, rng.seed)
    try:
        eng.search(iteration)
        _write_back(swarm, eng.to_host(), ("sol",))
    finally:
        eng.close()
    return swarm


def evaluate_phase(swarm: Swarm, f, iteration=None) -> Swarm:
    """Refresh ``sol_f`` from the current positions on device (parallel.py:127-129)."""
    eng = _engine_for(swarm, _phase_params(swarm, f), f, 0)
    try:
        eng.evaluate(iteration)
        eng.check()
        _write_back(swarm, eng.to_host(), ("sol_f",))
    finally:
        eng.close()
    return swarm


def update_pbests_phase(swarm: Swarm) -> Swarm:
    """Row-independent paired comparison; ties refresh the incumbent (parallel.py:132-135)."""
    eng = _engine_for(swarm, _phase_params(swarm), make_function("f1", swarm.nvar), 0)
    try:
        eng.update_pbests()
        _write_back(swarm, eng.to_host(), ("pbests", "p_f"))
    finally:
        eng.close()
    return swarm


def update_gbest_phase(swarm: Swarm) -> Swarm:
    """Min-reduce over (p_f, index); incumbent survives only if strictly better (parallel.py:138-144)."""
    eng = _engine_for(swarm, _phase_params(swarm), make_function("f1", swarm.nvar), 0)
    try:
        eng.update_gbest()
        _write_back(swarm, eng.to_host(), ("gbest", "g_f"))
    finally:
        eng.close()
    return swarm


# -------------------------------------------------------------- run_parallel --

def run_parallel(
    params: SsoParams,
    f,
    seed: int,
    workers: int = 1,
    layout: LayoutMode = LayoutMode.PARTICLE_MAJOR,
    *,
    dtype: str = "float64",
    rng: str = "reference",
    shards: int = 1,
    device=None,
) -> RunRecord:
    """Run the phased schedule on the GPU; the result depends only on (params, f, seed).

    Extra keyword-only knobs: ``dtype`` ("float64" | "float32"), ``rng``
    ("reference" = the reference's keyed SplitMix64, bit-exact; "philox" =
    benchmark mode), ``shards`` (>1 splits the particles into contiguous
    shards on this GPU, exchanging gBest candidates like the multi-GPU path;
    bit-identical to ``shards=1``).  ``wall_time_s`` is the loop-only device
    time (CUDA events), excluding initialization like parallel.py:190,216.
    """
    import torch

    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    LayoutMode(layout)
    if shards > 1:
        from .sharded import run_virtual_shards

        return run_virtual_shards(params, f, seed, shards, dtype=dtype, rng=rng, device=device)
    from .engine import DeviceEngine

    eng = DeviceEngine(params, f, seed, dtype=dtype, rng=rng, device=device)
    try:
        eng.initialize()
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(eng.stream)
        eng.run(0, params.niter)
        stop.record(eng.stream)
        eng.check()
        wall = start.elapsed_time(stop) * 1e-3
        trajectory = eng.traj.cpu().numpy()
        best_position = eng.gbest.to(torch.float64).cpu().numpy()
        best = float(eng.g_f.cpu()[0])
    finally:
        eng.close()
    return RunRecord(
        run_id=0,
        schedule=ScheduleKind.PARALLEL,
        function=getattr(f, "id", "custom"),
        nsol=params.nsol,
        nvar=params.nvar,
        niter=params.niter,
        cw=params.cw,
        cp=params.cp,
        cg=params.cg,
        seed=seed,
        best_fitness=best,
        wall_time_s=wall,
        best_position=best_position,
        trajectory=trajectory,
    )


def run_parallel_batch(
    params: SsoParams,
    f,
    seeds,
    *,
    dtype: str = "float64",
    rng: str = "reference",
    run_id_base: int = 0,
) -> list:
    """Many independent runs of ``run_parallel`` (one per seed) as one device job.

    The reference's experiment protocol runs the same configuration for many
    seeds (harness.py:148-163, 217-263, seed = base_seed + run_id); here all
    swarms run side by side in one whole-run kernel launch (psso_solve_batch).
    Record k is bit-identical to ``run_parallel(params, f, seeds[k])``;
    ``wall_time_s`` is the loop-only device time of the whole batch.  Needs
    ``nvar <= 128`` and ``nsol * nvar <= 2**22``.
    """
    return _solve_batch(params, f, seeds, dtype, rng, run_id_base, sequential=False)


def run_sequential_batch(
    params: SsoParams,
    f,
    seeds,
    *,
    dtype: str = "float64",
    rng: str = "reference",
    run_id_base: int = 0,
) -> list:
    """Many independent runs of ``run_sequential`` (core.py:213-258) as one device job.

    All swarms are initialized together and their sequential loops run in one
    k_seq launch, one CTA per swarm (psso_solve_sequential_batch).  Record k is
    bit-identical to ``run_sequential(params, f, seeds[k])``; ``wall_time_s``
    is the loop-only device time of the whole batch.  Same limits as
    ``run_parallel_batch``.
    """
    return _solve_batch(params, f, seeds, dtype, rng, run_id_base, sequential=True)


def _solve_batch(params, f, seeds, dtype, rng, run_id_base, sequential) -> list:
    import ctypes

    from . import _lib
    from .core import NonFiniteFitnessError
    from .engine import make_config

    seeds = [int(s) for s in seeds]
    if not seeds:
        raise ValueError("need at least one seed")
    _lib.require_device()
    L = _lib.load()
    cfg = make_config(params, f, seeds[0], dtype=dtype, rng=rng)
    B, n, D = len(seeds), params.niter, params.nvar
    arr = (ctypes.c_uint64 * B)(*[s & ((1 << 64) - 1) for s in seeds])
    traj = np.empty((B, n), dtype=np.float64)
    best = np.empty((B, D), dtype=np.float64 if dtype == "float64" else np.float32)
    bestf = np.empty(B, dtype=np.float64)
    wall = ctypes.c_double()
    solve = L.psso_solve_sequential_batch if sequential else L.psso_solve_batch
    rc = solve(ctypes.byref(cfg), arr, B, n, traj.ctypes.data, best.ctypes.data,
               bestf.ctypes.data, ctypes.byref(wall))
    if rc == _lib.PSSO_E_NONFINITE:  # the failing swarm's (iteration, particle, value)
        sw, it, i, v = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        L.psso_batch_failure(ctypes.byref(sw), ctypes.byref(it), ctypes.byref(i), ctypes.byref(v))
        raise NonFiniteFitnessError(float(v.value), int(i.value),
                                    None if it.value < 0 else int(it.value))
    _lib.check(rc)
    kind = ScheduleKind.SEQUENTIAL if sequential else ScheduleKind.PARALLEL
    return [
        RunRecord(run_id=run_id_base + k, schedule=kind,
                  function=getattr(f, "id", "custom"), nsol=params.nsol, nvar=D, niter=n,
                  cw=params.cw, cp=params.cp, cg=params.cg, seed=seeds[k],
                  best_fitness=float(bestf[k]), wall_time_s=wall.value,
                  best_position=best[k].astype(np.float64), trajectory=traj[k].copy())
        for k in range(B)
    ]
