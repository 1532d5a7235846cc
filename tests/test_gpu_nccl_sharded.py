"""The default multi-GPU path at world size 1: library-owned NCCL communicator,
fused kernel + candidate record + ncclAllGather + apply replayed from CUDA graphs
(psso_run_sharded), against the unsharded run (parallel.py:199-212; worker
invariance, reference test_parallel.py:185-193).

Only one GPU is available to the tests, and NCCL refuses two ranks on one GPU,
so the collective runs with one rank here; the record format, graph capture
with the collective inside, device iteration counter, non-finite adoption and
communicator reuse are all exercised.  The multi-rank host logic is covered by
the gloo tests (tests/test_sharded_gloo.py) and the 2-rank bench test.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200.sharded import run_parallel_distributed  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def process_group():
    if dist.is_initialized():
        yield
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _params(fn, nsol, niter):
    return psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                          nsol=nsol, nvar=fn.dimension, niter=niter)


@pytest.mark.parametrize("fid,nsol,nvar,niter,dtype", [
    ("f4", 5000, 64, 40, "float64"),     # 2 graph replays + 8 direct iterations
    ("f5", 3000, 128, 37, "float64"),
    ("f1", 4096, 100, 16, "float32"),    # exactly one replay, ragged rows
    ("f6", 64, 4096, 20, "float64"),     # k_rows
])
def test_nccl_sharded_equals_unsharded(fid, nsol, nvar, niter, dtype):
    fn = psso.make_function(fid, nvar)
    p = _params(fn, nsol, niter)
    rec = run_parallel_distributed(p, fn, 7, dtype=dtype, exchange="nccl")
    ref = psso.run_parallel(p, fn, seed=7, dtype=dtype)
    assert np.array_equal(rec.trajectory, ref.trajectory)
    assert np.array_equal(rec.best_position, ref.best_position)
    assert rec.best_fitness == ref.best_fitness


def test_nccl_sharded_matches_oracle_and_reuses_the_communicator():
    from paper_2110_01470_b200.sharded import NcclComm

    fn = psso.make_function("f4", 64)
    p = _params(fn, 2000, 48)
    o = O.Oracle.from_params(p, "f4", 3)
    sw = o.initialize()
    otraj = o.run(sw, 0, p.niter)
    n0 = len(NcclComm._cache)
    for _ in range(3):
        rec = run_parallel_distributed(p, fn, 3, exchange="nccl")
        assert np.array_equal(rec.trajectory, otraj)
        assert np.array_equal(rec.best_position, sw.gbest)
    assert len(NcclComm._cache) == max(n0, 1)


def test_nccl_sharded_nonfinite_names_the_first_particle():
    level = float(O.init_positions(0, 40, 4, -1.0, 1.0)[:, 0].max())  # init stays finite
    fn = psso.probe_function(4, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=40, nvar=4, niter=200)
    with pytest.raises(psso.NonFiniteFitnessError) as ref:
        psso.run_parallel(p, fn, seed=0)
    with pytest.raises(psso.NonFiniteFitnessError) as got:
        run_parallel_distributed(p, fn, 0, exchange="nccl")
    assert (got.value.iteration, got.value.particle, got.value.value) == \
        (ref.value.iteration, ref.value.particle, ref.value.value)
