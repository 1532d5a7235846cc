"""Particle-sharded PSSO: contiguous row shards + one gBest exchange per iteration.

Sharding follows the reference's worker partition (``_partition``,
parallel.py:147-149: contiguous ranges from ``linspace``).  Every deviate is
keyed by the *global* particle index, rows are disjoint, and the gBest step
is a lexicographic (p_f, index) min -- so any shard count reproduces the
unsharded run bit for bit, the property the reference pins as worker
invariance (test_parallel.py:185-193).

Per iteration each shard runs the fused kernel over its rows and reduces its
own candidate record (p_f, global index, row); the records of all shards are
gathered in rank order (one all-gather of R * (32 + D * sizeof(T)) bytes --
the per-slice candidates + ``min(candidates)`` of parallel.py:199-208) and
every shard applies the same deterministic selection (parallel.py:209-212).

Exchanges:
  * ``NcclExchange``         -- the default across GPUs: the library owns an
                                NCCL communicator (psso_comm) and runs
                                whole chunks of iterations -- fused kernel,
                                candidate record, ncclAllGather, apply -- from
                                one captured CUDA graph per 16 iterations
                                (psso_run_sharded): no host round trip per
                                iteration.
  * ``LocalExchange``        -- all shards live in this process (virtual
                                shards on one GPU); gather = concatenation.
  * ``ProcessGroupExchange`` -- one shard per process over torch.distributed
                                (NCCL over NVLink on B200; gloo on CPU tests).
  * ``P2PExchange``          -- device-initiated (SURVEY §8 f #3): each shard's
                                kernel stores its record straight into every
                                shard's exchange buffer (CUDA-IPC mappings over
                                NVLink P2P across processes; plain pointers for
                                virtual shards) and raises an epoch flag; each
                                shard's apply kernel waits on the flags.  No
                                host synchronization, no collective library.
"""

from __future__ import annotations

import numpy as np

from .core import SsoParams
from .records import RunRecord, ScheduleKind

__all__ = [
    "partition",
    "NcclComm",
    "NcclExchange",
    "LocalExchange",
    "ProcessGroupExchange",
    "P2PExchange",
    "ShardedDriver",
    "run_virtual_shards",
    "run_parallel_distributed",
]


def partition(nsol: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous particle ranges, the reference's ``_partition`` (parallel.py:147-149)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    edges = np.linspace(0, nsol, parts + 1).astype(int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


class NcclComm:
    """A library-owned NCCL communicator (psso_comm) for this process's rank and device.

    Made once per (process group, device) and cached: creating a communicator
    is a collective bootstrap costing far more than a run's iterations, so it
    is a session resource like torch's process group.  The group is used once,
    to hand rank 0's ncclUniqueId to every rank.
    """

    ID_BYTES = 128
    _cache: dict = {}

    def __init__(self, group, device):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib

        self.L = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = (ctypes.c_ubyte * self.ID_BYTES)()
        if self.rank == 0:
            _lib.check(self.L.psso_nccl_unique_id(uid))
        box = [bytes(uid)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(box, src=src, group=group)
        uid = (ctypes.c_ubyte * self.ID_BYTES).from_buffer_copy(box[0])
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.check(self.L.psso_comm_create(uid, self.world, self.rank, ctypes.byref(h)))
        self.handle = h

    @classmethod
    def get(cls, group, device):
        key = (id(group), str(device))
        if key not in cls._cache:
            cls._cache[key] = cls(group, device)
        return cls._cache[key]

    def __del__(self):
        try:
            if self.handle:
                self.L.psso_comm_destroy(self.handle)
        except Exception:
            pass


class NcclExchange:
    """Library-owned NCCL communicator; iterations run as graph-replayed device loops.

    One shard per process (rank = rank in the torch.distributed ``group``).
    The iteration path is psso_run_sharded: fused kernel, candidate record,
    ncclAllGather and apply, captured in a CUDA graph of 16 iterations.
    """

    device_loop = True

    def __init__(self, engine, group=None):
        from . import _lib

        self.L = _lib.load()
        self.comm = NcclComm.get(group, engine.device)
        self.world, self.rank = self.comm.world, self.comm.rank
        _lib.check(self.L.psso_attach_comm(engine.ctx, self.comm.handle), engine.ctx)

    def initialize(self, engines):
        from . import _lib

        for e in engines:
            _lib.check(self.L.psso_init_sharded(e.ctx), e.ctx)

    def run(self, engines, t0: int, niter: int):
        from . import _lib

        for e in engines:
            _lib.check(self.L.psso_run_sharded(e.ctx, int(t0), int(niter)), e.ctx)


class LocalExchange:
    """All shards in this process: the gathered buffer is the rank-ordered concatenation."""

    def gather(self, cands):
        import torch

        return torch.cat(list(cands))


class ProcessGroupExchange:
    """One shard per process: ``all_gather_into_tensor`` of the candidate records."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def gather(self, cands):
        import torch.distributed as dist

        (c,) = cands
        if c.is_cuda and dist.get_backend(self.group) != "nccl":  # gloo: stage through the host
            out = c.new_empty(self.world * c.numel(), device="cpu")
            dist.all_gather_into_tensor(out, c.cpu(), group=self.group)
            return out.to(c.device)
        out = c.new_empty(self.world * c.numel())
        dist.all_gather_into_tensor(out, c, group=self.group)
        return out


class P2PExchange:
    """Device-initiated record exchange through per-rank exchange buffers (psso_publish_p2p).

    ``engines``: the shards this process owns.  ``distributed=False``: they
    are all the ranks (virtual shards, rank = position).  ``distributed=True``:
    this process owns exactly one shard (rank = rank in the torch.distributed
    ``group``, None = default group) and the buffers of the other ranks are
    mapped through CUDA IPC handles exchanged over the group.  Call
    :meth:`close` to unmap and free.
    """

    HANDLE_BYTES = 64

    def __init__(self, engines, group=None, distributed=False):
        import ctypes

        import numpy as np
        import torch

        from . import _lib

        self.L = _lib.load()
        self.engines = list(engines)
        self.group = group
        self.epoch = 0
        first = self.engines[0]
        self.distributed = bool(distributed)
        if not self.distributed:
            self.world, self.ranks = len(self.engines), list(range(len(self.engines)))
        else:
            import torch.distributed as dist

            if len(self.engines) != 1:
                raise ValueError("a process-group P2P exchange drives exactly one shard per process")
            self.world, self.ranks = dist.get_world_size(group), [dist.get_rank(group)]
        nbytes = int(self.L.psso_p2p_buffer_bytes(ctypes.byref(first.cfg), self.world))
        self.own = []
        for e in self.engines:  # each buffer on its shard's device
            ptr = ctypes.c_void_p()
            with torch.cuda.device(e.device):
                _lib.check(self.L.psso_p2p_alloc(nbytes, ctypes.byref(ptr)))
            self.own.append(ptr.value)
        self.opened = []
        if not self.distributed:
            table = self.own
        else:
            import torch.distributed as dist

            h = (ctypes.c_ubyte * self.HANDLE_BYTES)()
            _lib.check(self.L.psso_p2p_handle(ctypes.c_void_p(self.own[0]), h))
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h), group=group)
            table = []
            for r, hb in enumerate(handles):
                if r == self.ranks[0]:
                    table.append(self.own[0])
                    continue
                ptr = ctypes.c_void_p()
                buf = (ctypes.c_ubyte * self.HANDLE_BYTES).from_buffer_copy(hb)
                with torch.cuda.device(first.device):
                    _lib.check(self.L.psso_p2p_open(buf, ctypes.byref(ptr)))
                self.opened.append(ptr.value)
                table.append(ptr.value)
        self.table = torch.tensor(np.array(table, dtype=np.uint64).view(np.int64), device=first.device)

    @property
    def device_loop(self) -> bool:
        # one shard per process: whole chunks of iterations run as a graph-replayed
        # device loop (psso_run_p2p).  Virtual shards share one stream, where one
        # shard's loop would wait on records the next shard publishes later.
        return self.distributed

    def exchange_and_apply(self, engines, cands, t: int, is_init: bool):
        # epoch 1 = initialization, t + 2 = iteration t: the same numbering the
        # device loop derives from its iteration counter
        self.epoch = 1 if is_init else t + 2
        for e, c, r in zip(engines, cands, self.ranks):
            e.publish_p2p(c, self.table, self.world, r, self.epoch)
        for e, buf in zip(engines, self.own):
            e.apply_p2p(t, buf, self.world, self.epoch, is_init)

    def initialize(self, engines, cands):
        for e, c in zip(engines, cands):
            e.init_local(c)
        self.exchange_and_apply(engines, cands, -1, True)

    def run(self, engines, t0: int, niter: int):
        from . import _lib

        for e, buf, r in zip(engines, self.own, self.ranks):
            _lib.check(self.L.psso_run_p2p(e.ctx, int(t0), int(niter), self.table.data_ptr(), buf,
                                           self.world, r), e.ctx)

    def close(self):
        import ctypes

        for e in self.engines:
            e.synchronize()
        for p in self.opened:
            self.L.psso_p2p_close(ctypes.c_void_p(p))
        for p in self.own:
            self.L.psso_p2p_free(ctypes.c_void_p(p))
        self.opened, self.own = [], []


class ShardedDriver:
    """Drives shard engines through init / iterations around the exchange.

    ``engines`` are the shards owned by this process, in rank order; each must
    provide ``new_candidate()``, ``init_local(cand)``, ``step_local(t, cand)``,
    ``apply(t, cands, ncand, is_init)`` and ``check(init=...)`` (DeviceEngine
    does, over the C ABI).  ``ncand`` is the total number of shards.
    """

    def __init__(self, engines, exchange, ncand: int):
        self.engines = list(engines)
        self.exchange = exchange
        self.ncand = int(ncand)
        self.cands = [e.new_candidate() for e in self.engines]

    def _exchange_and_apply(self, t: int, is_init: bool):
        if hasattr(self.exchange, "exchange_and_apply"):  # device-initiated exchange
            self.exchange.exchange_and_apply(self.engines, self.cands, t, is_init)
            return None
        gathered = self.exchange.gather(self.cands)
        for e in self.engines:
            e.apply(t, gathered, self.ncand, is_init)
        return gathered

    def initialize(self):
        if isinstance(self.exchange, P2PExchange):
            self.exchange.initialize(self.engines, self.cands)
        elif getattr(self.exchange, "device_loop", False):
            self.exchange.initialize(self.engines)
        else:
            for e, c in zip(self.engines, self.cands):
                e.init_local(c)
            self._exchange_and_apply(-1, True)
        for e in self.engines:
            e.check(init=True)

    def step(self, t: int):
        if getattr(self.exchange, "device_loop", False):
            self.exchange.run(self.engines, t, 1)
            return
        for e, c in zip(self.engines, self.cands):
            e.step_local(t, c)
        self._exchange_and_apply(t, False)

    def run(self, t0: int, niter: int):
        if getattr(self.exchange, "device_loop", False):
            self.exchange.run(self.engines, t0, niter)  # graph-replayed on the device
            return
        for t in range(t0, t0 + niter):
            self.step(t)

    def check(self):
        for e in self.engines:
            e.check()


def _record(params, f, seed, best, wall, traj, best_position) -> RunRecord:
    return RunRecord(
        run_id=0, schedule=ScheduleKind.PARALLEL, function=getattr(f, "id", "custom"),
        nsol=params.nsol, nvar=params.nvar, niter=params.niter, cw=params.cw, cp=params.cp,
        cg=params.cg, seed=seed, best_fitness=best, wall_time_s=wall,
        best_position=best_position, trajectory=traj)


def run_virtual_shards(params: SsoParams, f, seed: int, shards: int, *, dtype="float64",
                       rng="reference", device=None, exchange: str = "gather") -> RunRecord:
    """``shards`` contiguous shards on one GPU with the candidate exchange (tests sharding).

    ``exchange``: "gather" (concatenate records, like the NCCL all-gather) or
    "p2p" (the device-initiated exchange through per-shard buffers).
    """
    import torch

    from .engine import DeviceEngine

    ranges = partition(params.nsol, shards)
    first = DeviceEngine(params, f, seed, dtype=dtype, rng=rng, row_lo=ranges[0][0],
                         row_hi=ranges[0][1], device=device)
    engines = [first] + [
        DeviceEngine(params, f, seed, dtype=dtype, rng=rng, row_lo=lo, row_hi=hi,
                     device=device, stream=first.stream)
        for lo, hi in ranges[1:]
    ]
    ex = P2PExchange(engines) if exchange == "p2p" else LocalExchange()
    try:
        drv = ShardedDriver(engines, ex, len(engines))
        with torch.cuda.stream(first.stream):
            drv.initialize()
            start = torch.cuda.Event(enable_timing=True)
            stop = torch.cuda.Event(enable_timing=True)
            start.record(first.stream)
            drv.run(0, params.niter)
            stop.record(first.stream)
        drv.check()
        wall = start.elapsed_time(stop) * 1e-3
        return _record(params, f, seed, float(first.g_f.cpu()[0]), wall, first.traj.cpu().numpy(),
                       first.gbest.to(torch.float64).cpu().numpy())
    finally:
        if exchange == "p2p":
            ex.close()
        for e in engines:
            e.close()


def run_parallel_distributed(params: SsoParams, f, seed: int, *, group=None, dtype="float64",
                             rng="reference", exchange: str = "nccl") -> RunRecord:
    """One shard per torch.distributed rank (one process per GPU, NCCL over NVLink).

    Every rank returns the same RunRecord.  ``wall_time_s`` is this rank's
    loop time; callers wanting the job time take the max over ranks.
    ``exchange``: "nccl" (default: the library's own communicator, iterations
    replayed from CUDA graphs with the all-gather inside), "collective"
    (all-gather over the torch process group, one host-issued exchange per
    iteration; works over gloo) or "p2p" (device-initiated stores into
    CUDA-IPC-mapped peer buffers; the group only exchanges the IPC handles).
    """
    import torch
    import torch.distributed as dist

    from .engine import DeviceEngine

    pg = ProcessGroupExchange(group)
    ranges = partition(params.nsol, pg.world)
    if len(ranges) != pg.world:
        raise ValueError(f"nsol={params.nsol} cannot give every one of {pg.world} ranks a particle")
    lo, hi = ranges[pg.rank]
    eng = DeviceEngine(params, f, seed, dtype=dtype, rng=rng, row_lo=lo, row_hi=hi)
    if exchange not in ("nccl", "collective", "p2p"):
        raise ValueError(f"exchange must be 'nccl', 'collective' or 'p2p', got {exchange!r}")
    ex = (P2PExchange([eng], group=group, distributed=True) if exchange == "p2p"
          else NcclExchange(eng, group=group) if exchange == "nccl" else pg)
    try:
        drv = ShardedDriver([eng], ex, pg.world)
        with torch.cuda.stream(eng.stream):
            drv.initialize()
            dist.barrier(group)
            start = torch.cuda.Event(enable_timing=True)
            stop = torch.cuda.Event(enable_timing=True)
            start.record(eng.stream)
            drv.run(0, params.niter)
            stop.record(eng.stream)
        drv.check()
        wall = start.elapsed_time(stop) * 1e-3
        return _record(params, f, seed, float(eng.g_f.cpu()[0]), wall, eng.traj.cpu().numpy(),
                       eng.gbest.to(torch.float64).cpu().numpy())
    finally:
        if exchange == "p2p":
            dist.barrier(group)  # every rank done reading before buffers are unmapped
            ex.close()
        eng.close()
