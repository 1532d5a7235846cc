"""DeviceEngine: one libpsso context plus its HBM-resident swarm.

Owns the torch tensors that hold the swarm (particle-major X and P, p_f,
gbest, g_f, trajectory) on one CUDA device and a private non-default stream
(so the iteration loop can be replayed from a CUDA graph).  Everything here
is plumbing around the C ABI; all compute is in libpsso.so.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .benchmarks import device_code_of
from .core import NonFiniteFitnessError, SsoParams, Swarm

__all__ = ["DeviceEngine", "make_config", "DTYPES", "RNG_MODES"]

DTYPES = {"float64": _lib.PSSO_F64, "float32": _lib.PSSO_F32}
RNG_MODES = {"reference": _lib.PSSO_RNG_REFERENCE, "philox": _lib.PSSO_RNG_PHILOX}
_MASK64 = (1 << 64) - 1


def make_config(params: SsoParams, f, seed: int, *, dtype="float64", rng="reference",
                row_lo=0, row_hi=None, keep_sol_f=False) -> _lib.PssoConfig:
    code = device_code_of(f)
    if params.nvar != f.dimension:
        raise ValueError(f"{f.id} expects dimension {f.dimension}, got {params.nvar}")
    if dtype not in DTYPES:
        raise ValueError(f"dtype must be one of {tuple(DTYPES)}, got {dtype!r}")
    if rng not in RNG_MODES:
        raise ValueError(f"rng must be one of {tuple(RNG_MODES)}, got {rng!r}")
    return _lib.PssoConfig(
        fn_id=code, dtype=DTYPES[dtype], rng_mode=RNG_MODES[rng],
        flags=1 if keep_sol_f else 0, nsol=params.nsol, nvar=params.nvar,
        row_lo=row_lo, row_hi=params.nsol if row_hi is None else row_hi,
        cw=params.cw, cp=params.cp, cg=params.cg, var_min=params.var_min,
        var_max=params.var_max, seed=int(seed) & _MASK64, probe_level=float(f.probe_level))


class DeviceEngine:
    """A swarm shard [row_lo, row_hi) resident in HBM with its psso context."""

    def __init__(self, params: SsoParams, f, seed: int, *, dtype="float64", rng="reference",
                 row_lo=0, row_hi=None, device=None, keep_sol_f=False, traj_len=None,
                 stream=None):
        import torch

        _lib.require_device()
        self.params, self.f, self.seed, self.dtype = params, f, int(seed), dtype
        self.cfg = make_config(params, f, seed, dtype=dtype, rng=rng, row_lo=row_lo,
                               row_hi=row_hi, keep_sol_f=keep_sol_f)
        self.row_lo, self.row_hi = self.cfg.row_lo, self.cfg.row_hi
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._lib = _lib.load()
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
            ctx = ctypes.c_void_p()
            _lib.check(self._lib.psso_create(ctypes.byref(self.cfg), ctypes.byref(ctx)))
            self.ctx = ctx
            rows, D = self.row_hi - self.row_lo, params.nvar
            tdt = torch.float64 if dtype == "float64" else torch.float32
            kw = dict(device=self.device)
            self.sol = torch.empty((rows, D), dtype=tdt, **kw)
            self.pbests = torch.empty((rows, D), dtype=tdt, **kw)
            self.sol_f = torch.full((rows,), float("nan"), dtype=torch.float64, **kw)
            self.p_f = torch.empty((rows,), dtype=torch.float64, **kw)
            self.gbest = torch.empty((D,), dtype=tdt, **kw)
            self.g_f = torch.zeros((1,), dtype=torch.float64, **kw)
            self.traj = torch.full((traj_len or params.niter,), float("nan"), dtype=torch.float64, **kw)
        torch.cuda.synchronize(self.device)  # allocations visible to the library's stream
        self._bind()

    # -- plumbing --------------------------------------------------------------
    def _bind(self):
        b = _lib.PssoBuffers(
            sol=self.sol.data_ptr(), pbests=self.pbests.data_ptr(), sol_f=self.sol_f.data_ptr(),
            p_f=self.p_f.data_ptr(), gbest=self.gbest.data_ptr(), g_f=self.g_f.data_ptr(),
            traj=self.traj.data_ptr())
        _lib.check(self._lib.psso_bind(self.ctx, ctypes.byref(b), self.stream.cuda_stream), self.ctx)

    def _call(self, name, *args):
        _lib.check(getattr(self._lib, name)(self.ctx, *args), self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.stream.synchronize()
            self._lib.psso_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self._lib.psso_launch_count(self.ctx))

    def synchronize(self):
        self.stream.synchronize()

    # -- reference operations --------------------------------------------------
    def initialize(self):
        """core.initialize (core.py:196-210) on device."""
        self._call("psso_init")
        self.check(init=True)

    def step(self, t: int):
        self._call("psso_step", int(t))

    def run(self, t0: int, niter: int):
        """The run_parallel loop (parallel.py:192-212), asynchronous on self.stream."""
        self._call("psso_run", int(t0), int(niter))

    def run_sequential(self, t0: int, niter: int):
        """The run_sequential loop (core.py:222-244), asynchronous on self.stream."""
        self._call("psso_run_sequential", int(t0), int(niter))

    @property
    def sequential_passes(self) -> int:
        """Speculative passes of the last run_sequential (iterations + gBest moves)."""
        n = ctypes.c_int64(0)
        self._call("psso_sequential_passes", ctypes.byref(n))
        return int(n.value)

    def search(self, t):
        self._call("psso_search", int(t))

    def evaluate(self, t=None):
        self._call("psso_evaluate", -1 if t is None else int(t))

    def update_pbests(self):
        self._call("psso_update_pbests")

    def update_gbest(self):
        self._call("psso_update_gbest")

    def check(self, init=False):
        """Raise NonFiniteFitnessError for the first non-finite fitness (core.py:190-193)."""
        bt, bi, v = ctypes.c_int64(0), ctypes.c_int64(-1), ctypes.c_double()
        rc = self._lib.psso_nonfinite(self.ctx, ctypes.byref(bt), ctypes.byref(bi), ctypes.byref(v))
        if rc == _lib.PSSO_E_NONFINITE:
            iteration = None if bt.value < 0 else int(bt.value)
            raise NonFiniteFitnessError(float(v.value), int(bi.value), iteration)
        _lib.check(rc, self.ctx)

    def result(self) -> tuple[float, int]:
        """(g_f, gBest particle index) -- the argmin of parallel.py:208-211 / core.py:202.

        Synchronizes; raises NonFiniteFitnessError like :meth:`check`."""
        gf, gi = ctypes.c_double(), ctypes.c_int64(-1)
        bt, bi = ctypes.c_int64(0), ctypes.c_int64(-1)
        rc = self._lib.psso_result(self.ctx, ctypes.byref(gf), ctypes.byref(gi), ctypes.byref(bt),
                                   ctypes.byref(bi))
        if rc == _lib.PSSO_E_NONFINITE:
            self.check()
        _lib.check(rc, self.ctx)
        return float(gf.value), int(gi.value)

    @property
    def best_index(self) -> int:
        """Global index of the particle whose pBest row is gbest (-1 before initialization)."""
        return self.result()[1]

    # -- sharded iteration (see sharded.py) -----------------------------------
    @property
    def candidate_bytes(self) -> int:
        return int(self._lib.psso_candidate_bytes(ctypes.byref(self.cfg)))

    def new_candidate(self):
        import torch

        return torch.zeros(self.candidate_bytes, dtype=torch.uint8, device=self.device)

    def init_local(self, cand):
        self._call("psso_init_local", cand.data_ptr())

    def step_local(self, t, cand):
        self._call("psso_step_local", int(t), cand.data_ptr())

    def apply(self, t, cands, ncand, is_init=False):
        self._call("psso_apply_candidates", int(t), cands.data_ptr(), int(ncand), int(bool(is_init)))

    def publish_p2p(self, cand, peer_table, nranks, rank, epoch):
        """This shard's record into slot ``rank`` of every rank's exchange buffer (psso_publish_p2p)."""
        self._call("psso_publish_p2p", cand.data_ptr(), peer_table.data_ptr(), int(nranks), int(rank),
                   int(epoch))

    def apply_p2p(self, t, my_buf, nranks, epoch, is_init=False):
        """Wait for the epoch's records in this shard's buffer, then select (psso_apply_p2p)."""
        self._call("psso_apply_p2p", int(t), int(my_buf), int(nranks), int(epoch), int(bool(is_init)))

    # -- host <-> device -------------------------------------------------------
    def to_host(self) -> Swarm:
        self.stream.synchronize()
        f64 = lambda t: t.to(dtype=__import__("torch").float64).cpu().numpy()  # noqa: E731
        return Swarm(sol=f64(self.sol), pbests=f64(self.pbests), gbest=f64(self.gbest),
                     sol_f=self.sol_f.cpu().numpy(), p_f=self.p_f.cpu().numpy(),
                     g_f=float(self.g_f.cpu()[0]))

    def load(self, swarm: Swarm, best_index: int | None = None):
        """Upload a host Swarm (any storage order) into this engine's buffers.

        ``best_index``: the gBest particle (psso_result); default = the lowest
        index whose p_f equals g_f (the parallel schedule's argmin), -1 if none.
        """
        import torch

        if best_index is None:
            hit = np.flatnonzero(np.asarray(swarm.p_f) == swarm.g_f)
            best_index = int(hit[0]) if hit.size else -1

        lo, hi = self.row_lo, self.row_hi
        tdt = self.sol.dtype
        with torch.cuda.stream(self.stream):
            self.sol.copy_(torch.as_tensor(np.ascontiguousarray(swarm.sol[lo:hi])).to(tdt))
            self.pbests.copy_(torch.as_tensor(np.ascontiguousarray(swarm.pbests[lo:hi])).to(tdt))
            self.gbest.copy_(torch.as_tensor(np.ascontiguousarray(swarm.gbest)).to(tdt))
            self.sol_f.copy_(torch.as_tensor(np.ascontiguousarray(swarm.sol_f[lo:hi], dtype=np.float64)))
            self.p_f.copy_(torch.as_tensor(np.ascontiguousarray(swarm.p_f[lo:hi], dtype=np.float64)))
            self.g_f.fill_(float(swarm.g_f))
        self._call("psso_set_gbest_index", int(best_index))
        self.stream.synchronize()

    # -- checkpoint / resume ---------------------------------------
    def _identity(self) -> dict:
        """Everything a checkpoint must match for a bitwise continuation."""
        c = self.cfg
        return {"seed": np.uint64(self.seed & _MASK64), "dtype": np.str_(self.dtype),
                "rows": np.int64([self.row_lo, self.row_hi]), "fn_id": np.int64(c.fn_id),
                "rng_mode": np.int64(c.rng_mode), "nsol": np.int64(c.nsol), "nvar": np.int64(c.nvar),
                "thresholds": np.float64([c.cw, c.cp, c.cg]),
                "box": np.float64([c.var_min, c.var_max])}

    def save_state(self, path, t_next: int) -> None:
        """Checkpoint the swarm before iteration ``t_next``.

        The keyed RNG makes ``(X, P, p_f, gbest, g_f, t)`` the whole state of a
        run (reference test_core.py:186-191: a shorter run is an exact prefix),
        so a run restored from this file continues bit for bit.  A run with a
        pending non-finite fitness raises NonFiniteFitnessError instead of
        being checkpointed.
        """
        self.check()
        g_f, g_idx = self.result()
        sw = self.to_host()
        np.savez(path, sol=sw.sol, pbests=sw.pbests, sol_f=sw.sol_f, p_f=sw.p_f, gbest=sw.gbest,
                 g_f=np.float64(g_f), g_idx=np.int64(g_idx), t_next=np.int64(t_next),
                 traj=self.traj.cpu().numpy(), **self._identity())

    def restore_state(self, path) -> int:
        """Load a checkpoint written by :meth:`save_state`; returns the next iteration.

        Rejects (ValueError) a checkpoint of another configuration: seed, dtype,
        row range, objective, RNG mode, thresholds, box, nsol or nvar."""
        import torch

        z = np.load(path)
        want = self._identity()
        bad = [k for k, v in want.items() if k not in z or not np.array_equal(z[k], v)]
        if bad or z["sol"].shape != tuple(self.sol.shape):
            raise ValueError("checkpoint does not match this engine ("
                             + ", ".join(bad or ["shape"]) + ")")
        self.load(Swarm(sol=z["sol"], pbests=z["pbests"], gbest=z["gbest"], sol_f=z["sol_f"],
                        p_f=z["p_f"], g_f=float(z["g_f"])), best_index=int(z["g_idx"]))
        n = min(len(z["traj"]), self.traj.numel())
        with torch.cuda.stream(self.stream):
            self.traj[:n].copy_(torch.as_tensor(z["traj"][:n]))
        self.stream.synchronize()
        return int(z["t_next"])
