"""Core types of the swarm engine (reference core.py), host side.

``SsoParams``, ``Swarm``, ``NonFiniteFitnessError`` and the scalar
``step_update_variable`` keep the reference's names, fields, validation and
error messages (core.py:43-135).  ``initialize`` runs the device init kernel
(psso_init; core.py:196-210) and returns a host ``Swarm``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = [
    "SsoParams",
    "Swarm",
    "NonFiniteFitnessError",
    "step_update_variable",
    "initialize",
    "run_sequential",
]


class NonFiniteFitnessError(RuntimeError):
    """The objective produced NaN or infinity; coordinates identify the call (core.py:43-53)."""

    def __init__(self, value: float, particle: int, iteration: Optional[int] = None):
        self.value = value
        self.particle = particle
        self.iteration = iteration
        where = "during initialization" if iteration is None else f"at iteration {iteration}"
        super().__init__(
            f"objective returned non-finite value {value!r} for particle {particle} {where}"
        )


@dataclass(frozen=True)
class SsoParams:
    """Algorithm constants: cumulative branch thresholds, box bounds, sizes (core.py:56-85)."""

    cw: float
    cp: float
    cg: float
    var_min: float
    var_max: float
    nsol: int
    nvar: int
    niter: int

    def __post_init__(self):
        if not (0.0 <= self.cw <= self.cp <= self.cg <= 1.0):
            raise ValueError(
                f"thresholds must satisfy 0 <= cw <= cp <= cg <= 1, "
                f"got ({self.cw}, {self.cp}, {self.cg})"
            )
        if not self.var_min < self.var_max:
            raise ValueError(
                f"need var_min < var_max, got [{self.var_min}, {self.var_max}]"
            )
        for label, n in (("nsol", self.nsol), ("nvar", self.nvar), ("niter", self.niter)):
            if not isinstance(n, (int, np.integer)) or n < 1:
                raise ValueError(f"{label} must be a positive integer, got {n!r}")

    @property
    def span(self) -> float:
        return self.var_max - self.var_min


@dataclass(eq=False)
class Swarm:
    """Positions, personal bests, and the global best with cached fitnesses (core.py:88-115)."""

    sol: np.ndarray
    pbests: np.ndarray
    gbest: np.ndarray
    sol_f: np.ndarray
    p_f: np.ndarray
    g_f: float

    @property
    def nsol(self) -> int:
        return self.sol.shape[0]

    @property
    def nvar(self) -> int:
        return self.sol.shape[1]

    def copy(self) -> "Swarm":
        return Swarm(
            sol=self.sol.copy(),
            pbests=self.pbests.copy(),
            gbest=self.gbest.copy(),
            sol_f=self.sol_f.copy(),
            p_f=self.p_f.copy(),
            g_f=self.g_f,
        )


def step_update_variable(x: float, p: float, g: float, u: float, fresh: float,
                         params: SsoParams) -> float:
    """The per-coordinate four-way update rule, scalar form (core.py:118-135).

    The device kernels apply the same rule as an integer compare of the branch
    hash against ceil(c * 2^53) (exactly equivalent to ``u < c``).
    """
    if not 0.0 <= u < 1.0:
        raise ValueError(f"branch deviate must lie in [0, 1), got {u!r}")
    if u < params.cw:
        return x
    if u < params.cp:
        return p
    if u < params.cg:
        return g
    return fresh


def initialize(params: SsoParams, f, rng, *, dtype: str = "float64") -> Swarm:
    """Draw the initial population on the device and score it (core.py:196-210)."""
    from .engine import DeviceEngine

    eng = DeviceEngine(params, f, rng.seed, dtype=dtype)
    try:
        eng.initialize()
        return eng.to_host()
    finally:
        eng.close()


def run_sequential(params: SsoParams, f, seed: int, *, dtype: str = "float64",
                   rng: str = "reference", device=None):
    """The per-particle asynchronous schedule (core.py:213-258) on the GPU.

    Particles are updated in index order against the live gBest, which moves
    as soon as a particle's new pBest is ``<=`` g_f (core.py:236-241); same
    keyed draws as ``run_parallel``.  Each iteration runs as speculative passes
    over the remaining particles, committing the prefix up to the first gBest
    move, so the result is bit-identical to the serial loop: for rows of up to
    128 variables the whole loop is ONE kernel launch (k_seq), longer rows run
    the same passes as a loop of device kernels over the resident swarm
    (``psso_run_sequential`` either way).  ``wall_time_s`` is the loop-only
    device time (core.py:222,245).
    """
    import torch

    from .engine import DeviceEngine
    from .records import RunRecord, ScheduleKind

    eng = DeviceEngine(params, f, seed, dtype=dtype, rng=rng, device=device)
    try:
        eng.initialize()
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(eng.stream)
        eng.run_sequential(0, params.niter)  # k_seq, or the device pass loop for nvar > 128
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
        schedule=ScheduleKind.SEQUENTIAL,
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
