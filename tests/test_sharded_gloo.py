"""World-size-2 (and 3) gloo test of the multi-rank path on CPU.

The product's ShardedDriver + ProcessGroupExchange (the code that runs over
NCCL on the GPU box) drive per-rank shard engines through init, per-iteration
candidate all-gathers and the gBest apply.  Here each rank's shard engine is
the oracle (test infrastructure) packing the same candidate record layout the
device writes (float64 p_f, int64 global index, non-finite key and value, the row) -- so the partition,
the exchange ordering and the record format are exercised end to end, and the
result must equal the unsharded oracle run bit for bit (the reference's worker
invariance, test_parallel.py:185-193).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleShardEngine:
    """Shard engine with DeviceEngine's sharded interface, computed by the oracle."""

    def __init__(self, fid, nsol, nvar, thr, bounds, seed, lo, hi, niter):
        self.lo, self.hi, self.D = lo, hi, nvar
        self.o = O.Oracle(fid, hi - lo, nvar, *thr, *bounds, seed, row_lo=lo)
        self.seed, self.bounds = seed, bounds
        self.rec_bytes = 32 + ((nvar * 8 + 15) // 16) * 16
        self.traj = np.full(niter, np.nan)
        self.sw = None
        self.last = (float("inf"), lo)

    def new_candidate(self):
        return torch.zeros(self.rec_bytes, dtype=torch.uint8)

    def _pack(self, cand, f, i):
        buf = cand.numpy()
        buf[:8] = np.frombuffer(np.float64(f).tobytes(), np.uint8)
        buf[8:16] = np.frombuffer(np.int64(i).tobytes(), np.uint8)
        self._pack_key(buf)
        row = self.sw.pbests[i - self.lo]
        buf[32:32 + 8 * self.D] = np.frombuffer(row.tobytes(), np.uint8)

    def init_local(self, cand):
        u = O.u_batch(self.seed, "INIT", 0, np.arange(self.lo, self.hi)[:, None],
                      np.arange(self.D)[None, :])
        x = self.bounds[0] + (self.bounds[1] - self.bounds[0]) * u
        n = self.hi - self.lo
        self.sw = O.OracleSwarm(x, x.copy(), np.zeros(self.D), np.empty(n), np.empty(n), 0.0)
        f, i = self.o.step_local(self.sw, -1)
        self._pack(cand, f, i)

    # the device protocol for a non-finite fitness (psso_api.cu k_local_cand /
    # adopt_nonfinite): the shard's first key (t+1) << 40 | i and the value ride in
    # the record header, applying the records adopts the smallest key, and a shard
    # with a key set stops iterating
    key = (1 << 64) - 1
    bad_value = 0.0

    def step_local(self, t, cand):
        if self.key == (1 << 64) - 1:
            try:
                f, i = self.o.step_local(self.sw, t)
            except O.OracleNonFinite as e:
                self.key = ((t + 1) << 40) | e.particle
                self.bad_value = float(self.sw.sol_f[e.particle - self.lo])
                f, i = float("inf"), self.lo
            self.last = (f, i)
        self._pack(cand, *self.last)

    def _pack_key(self, buf):
        buf[16:24] = np.frombuffer(np.uint64(self.key).tobytes(), np.uint8)
        buf[24:32] = np.frombuffer(np.float64(self.bad_value).tobytes(), np.uint8)

    def apply(self, t, cands, ncand, is_init=False):
        recs = cands.numpy().reshape(ncand, self.rec_bytes)
        for r in recs:  # adopt the run's first non-finite event
            k = int(np.frombuffer(r[16:24].tobytes(), np.uint64)[0])
            if k < self.key:
                self.key, self.bad_value = k, float(np.frombuffer(r[24:32].tobytes(), np.float64)[0])
        best = None
        for r in recs:
            f = float(np.frombuffer(r[:8].tobytes(), np.float64)[0])
            i = int(np.frombuffer(r[8:16].tobytes(), np.int64)[0])
            if best is None or (f, i) < best[:2]:
                best = (f, i, np.frombuffer(r[32:32 + 8 * self.D].tobytes(), np.float64).copy())
        if is_init or best[0] <= self.sw.g_f:
            self.sw.g_f = best[0]
            self.sw.gbest[:] = best[2]
        if t >= 0:
            self.traj[t] = self.sw.g_f

    def check(self, init=False):
        if self.key != (1 << 64) - 1:
            from paper_2110_01470_b200.core import NonFiniteFitnessError

            t = (self.key >> 40) - 1
            raise NonFiniteFitnessError(self.bad_value, self.key & ((1 << 40) - 1),
                                        None if t < 0 else t)


# f1 in one variable on [0, B] with B just above sqrt(DBL_MAX): x*x overflows to
# +inf for ~0.7 % of the draws -- a naturally non-finite objective for the oracle
OVERFLOW_BOX = (0.0, 1.35e154)

CASES = {
    "f4": ("f4", 23, 10, 25, (0.3, 0.6, 0.8), (-2.048, 2.048), 42),
    "f5": ("f5", 64, 17, 30, (0.3, 0.6, 0.8), (-5.12, 5.12), 3),
}


def _worker(rank, world, port, case, outdir):
    from paper_2110_01470_b200.sharded import ProcessGroupExchange, ShardedDriver, partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fid, nsol, nvar, niter, thr, bounds, seed = CASES[case]
        lo, hi = partition(nsol, world)[rank]
        eng = OracleShardEngine(fid, nsol, nvar, thr, bounds, seed, lo, hi, niter)
        ex = ProcessGroupExchange()
        assert ex.world == world and ex.rank == rank
        drv = ShardedDriver([eng], ex, world)
        drv.initialize()
        drv.run(0, niter)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), traj=eng.traj, gbest=eng.sw.gbest,
                 sol=eng.sw.sol, lo=lo, hi=hi)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,case", [(2, "f4"), (2, "f5"), (3, "f5")])
def test_gloo_sharded_driver_matches_unsharded_oracle(world, case):
    fid, nsol, nvar, niter, thr, bounds, seed = CASES[case]
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), case, d), nprocs=world,
                           join=True, start_method="spawn")
        outs = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(world)]
        o = O.Oracle(fid, nsol, nvar, *thr, *bounds, seed)
        sw = o.initialize()
        traj = o.run(sw, 0, niter)
        for r, out in enumerate(outs):
            assert np.array_equal(out["traj"], traj), r
            assert np.array_equal(out["gbest"], sw.gbest), r
            assert np.array_equal(out["sol"], sw.sol[int(out["lo"]):int(out["hi"])]), r


def _nonfinite_worker(rank, world, port, seed, nsol, niter, outdir):
    from paper_2110_01470_b200.core import NonFiniteFitnessError
    from paper_2110_01470_b200.sharded import ProcessGroupExchange, ShardedDriver, partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = partition(nsol, world)[rank]
        eng = OracleShardEngine("f1", nsol, 1, (0.3, 0.6, 0.8), OVERFLOW_BOX, seed, lo, hi, niter)
        drv = ShardedDriver([eng], ProcessGroupExchange(), world)
        drv.initialize()
        drv.run(0, niter)
        try:
            drv.check()
            out = None
        except NonFiniteFitnessError as e:
            out = (e.iteration, e.particle, e.value)
        np.save(os.path.join(outdir, f"nf{rank}.npy"), np.array(out, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_gloo_sharded_nonfinite_stops_every_rank_at_the_first_event():
    """A non-finite fitness in one shard: every rank reports the unsharded run's first
    (iteration, particle, value) (core.py:190-193), through the record header protocol."""
    nsol, niter, world = 60, 40, 2
    seed = None
    for s in range(200):  # a seed whose init is finite and whose first event is in rank 1's rows
        o = O.Oracle("f1", nsol, 1, 0.3, 0.6, 0.8, *OVERFLOW_BOX, s)
        try:
            sw = o.initialize()
        except O.OracleNonFinite:
            continue
        try:
            o.run(sw, 0, niter)
        except O.OracleNonFinite as e:
            if e.particle >= nsol // 2 and e.iteration > 0:
                seed, want = s, (e.iteration, e.particle)
                break
    assert seed is not None
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_nonfinite_worker, args=(world, _free_port(), seed, nsol, niter, d),
                           nprocs=world, join=True, start_method="spawn")
        got = [tuple(np.load(os.path.join(d, f"nf{r}.npy"), allow_pickle=True)) for r in range(world)]
    assert got[0] == got[1]
    assert got[0][:2] == want and np.isinf(got[0][2])
