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

    def new_candidate(self):
        return torch.zeros(self.rec_bytes, dtype=torch.uint8)

    def _pack(self, cand, f, i):
        buf = cand.numpy()
        buf[:8] = np.frombuffer(np.float64(f).tobytes(), np.uint8)
        buf[8:16] = np.frombuffer(np.int64(i).tobytes(), np.uint8)
        buf[16:24] = 0xFF  # no non-finite fitness (the oracle raises instead)
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

    def step_local(self, t, cand):
        f, i = self.o.step_local(self.sw, t)
        self._pack(cand, f, i)

    def apply(self, t, cands, ncand, is_init=False):
        recs = cands.numpy().reshape(ncand, self.rec_bytes)
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
        pass


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
