"""gBest index at the boundary (psso_result): SURVEY §8 b's `g_idx` output.

The reference selects gbest as the lexicographic `(p_f, index)` minimum over
the slice candidates (parallel.py:199-211) and, at initialization, `argmin`
of p_f (core.py:202).  In the parallel schedule the incumbent is always taken
again (the new minimum of the monotone p_f is `<=` g_f), so after every
iteration the gBest index is the lowest index of the minimum p_f -- what the
oracle's `np.argmin` gives.  In the sequential schedule the index is the last
particle that moved gbest (core.py:236-241): its pBest row and fitness are
gbest's.  Checked for every iteration kernel (k_chain + k_gbest, k_rows,
k_swarm, k_seq), sharded applies (gather and P2P) and the phase API.
"""

import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200 import _lib  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402
from paper_2110_01470_b200.sharded import (  # noqa: E402
    LocalExchange, P2PExchange, ShardedDriver, partition)


def _fn(fid, d):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return psso.make_function(fid, d)


def _params(fn, nsol, niter, **kw):
    return psso.SsoParams(cw=kw.get("cw", 0.3), cp=kw.get("cp", 0.6), cg=kw.get("cg", 0.8),
                          var_min=fn.var_min, var_max=fn.var_max, nsol=nsol, nvar=fn.dimension,
                          niter=niter)


@pytest.mark.parametrize("key", [f"run{k}" for k in range(27)])
def test_index_against_reference_runs(key, golden_runs):
    """init index == the reference's init argmin; final index == argmin of the final p_f."""
    index, arr = golden_runs
    e = {x["key"]: x for x in index}[key]
    fn = _fn(e["fid"], e["nvar"])
    p = psso.SsoParams(cw=e["cw"], cp=e["cp"], cg=e["cg"], var_min=e["var_min"],
                       var_max=e["var_max"], nsol=e["nsol"], nvar=e["nvar"], niter=e["niter"])
    eng = DeviceEngine(p, fn, e["seed"])
    try:
        assert eng.result()[1] == -1, "no index before initialization"
        eng.initialize()
        gf, gi = eng.result()
        assert gi == e["init_best"], "initialization argmin (core.py:202)"
        eng.run(0, e["niter"])
        gf, gi = eng.result()
        sw = eng.to_host()
    finally:
        eng.close()
    assert gi == int(np.argmin(sw.p_f)), "final lexicographic (p_f, index) minimum"
    assert gf == sw.p_f[gi] and np.array_equal(sw.gbest, sw.pbests[gi])
    if e["state"]:  # the reference's own final p_f
        assert gi == int(np.argmin(arr[key + "_p_f"]))


@pytest.mark.parametrize("fid,nsol,nvar,niter,kernel", [
    ("f1", 100, 30, 200, "k_swarm"),
    ("f5", 1024, 100, 100, "k_swarm"),
    ("f4", 20000, 64, 40, "k_chain"),
    ("f5", 6000, 100, 40, "k_chain"),
    ("f6", 64, 4096, 12, "k_rows"),
    ("f3", 700, 200, 12, "k_"),        # general tile path
])
def test_index_every_kernel_every_iteration(fid, nsol, nvar, niter, kernel):
    """Per step (psso_step) and per run (psso_run): the index tracks the oracle's argmin."""
    fn = _fn(fid, nvar)
    p = _params(fn, nsol, niter)
    o = O.Oracle.from_params(p, fid, 11, threads=O.max_threads())
    osw = o.initialize()
    L = _lib.load()
    eng = DeviceEngine(p, fn, 11)
    try:
        assert L.psso_kernel_name(eng.ctx).decode().startswith(kernel)
        eng.initialize()
        assert eng.result()[1] == int(np.argmin(osw.p_f))
        for t in range(niter // 2):
            eng.step(t)
            o.step(osw, t)
            assert eng.result()[1] == int(np.argmin(osw.p_f)), t
        eng.run(niter // 2, niter - niter // 2)      # graph / whole-run kernel
        o.run(osw, niter // 2, niter - niter // 2)
        assert eng.result()[1] == int(np.argmin(osw.p_f))
    finally:
        eng.close()


@pytest.mark.parametrize("exchange", ["gather", "p2p"])
def test_index_sharded(exchange):
    fn = _fn("f4", 64)
    p = _params(fn, 3001, 30)
    ranges = partition(p.nsol, 3)
    engines = []
    first = DeviceEngine(p, fn, 4, row_lo=ranges[0][0], row_hi=ranges[0][1])
    engines = [first] + [DeviceEngine(p, fn, 4, row_lo=lo, row_hi=hi, stream=first.stream)
                         for lo, hi in ranges[1:]]
    ex = P2PExchange(engines) if exchange == "p2p" else LocalExchange()
    o = O.Oracle.from_params(p, "f4", 4)
    osw = o.initialize()
    try:
        drv = ShardedDriver(engines, ex, 3)
        with torch.cuda.stream(first.stream):
            drv.initialize()
            idx = {e.result()[1] for e in engines}
            assert idx == {int(np.argmin(osw.p_f))}
            drv.run(0, p.niter)
        o.run(osw, 0, p.niter)
        assert {e.result()[1] for e in engines} == {int(np.argmin(osw.p_f))}
    finally:
        if exchange == "p2p":
            ex.close()
        for e in engines:
            e.close()


def test_index_phase_api():
    fn = _fn("f5", 20)
    p = _params(fn, 40, 10)
    eng = DeviceEngine(p, fn, 8, keep_sol_f=True)
    o = O.Oracle.from_params(p, "f5", 8)
    osw = o.initialize()
    try:
        eng.initialize()
        for t in range(p.niter):
            eng.search(t)
            eng.evaluate(t)
            eng.update_pbests()
            eng.update_gbest()
            o.step(osw, t)
            assert eng.result()[1] == int(np.argmin(osw.p_f)), t
    finally:
        eng.close()


@pytest.mark.parametrize("fid,nsol,nvar", [("f1", 100, 30), ("f5", 1024, 100)])
def test_index_sequential_schedule(fid, nsol, nvar):
    """k_seq: the last particle that moved gbest (core.py:236-241), against the oracle's state."""
    fn = _fn(fid, nvar)
    p = _params(fn, nsol, 200)
    eng = DeviceEngine(p, fn, 2)
    o = O.Oracle.from_params(p, fid, 2)
    osw = o.initialize()
    try:
        eng.initialize()
        eng.run_sequential(0, p.niter)
        gf, gi = eng.result()
        sw = eng.to_host()
    finally:
        eng.close()
    o.run_sequential(osw, 0, p.niter)
    assert np.array_equal(sw.gbest, osw.gbest) and gf == osw.g_f
    # the index names a particle whose pBest is gbest; with no exact fitness
    # ties (Appendix A) that particle is unique
    hits = np.flatnonzero((osw.p_f == osw.g_f) & np.all(osw.pbests == osw.gbest, axis=1))
    assert list(hits) == [gi]


def test_result_abi_reports_nonfinite():
    level = float(O.init_positions(0, 40, 4, -1.0, 1.0)[:, 0].max())  # init stays finite
    fn = psso.probe_function(4, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=40, nvar=4, niter=200)
    eng = DeviceEngine(p, fn, 0)
    try:
        eng.initialize()
        assert eng.result()[1] >= 0
        eng.run(0, p.niter)
        with pytest.raises(psso.NonFiniteFitnessError):
            eng.result()
    finally:
        eng.close()


@pytest.mark.parametrize("exchange", ["gather", "p2p"])
def test_sharded_nonfinite_stops_every_shard_at_the_first_event(exchange):
    """A non-finite fitness in one shard stops all shards; every shard reports the
    unsharded run's first (iteration, particle, value) (core.py:190-193)."""
    level = float(O.init_positions(0, 40, 4, -1.0, 1.0)[:, 0].max())  # init stays finite
    fn = psso.probe_function(4, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=40, nvar=4, niter=200)
    with pytest.raises(psso.NonFiniteFitnessError) as ref:
        psso.run_parallel(p, fn, seed=0)
    ranges = partition(p.nsol, 3)
    first = DeviceEngine(p, fn, 0, row_lo=ranges[0][0], row_hi=ranges[0][1])
    engines = [first] + [DeviceEngine(p, fn, 0, row_lo=lo, row_hi=hi, stream=first.stream)
                         for lo, hi in ranges[1:]]
    ex = P2PExchange(engines) if exchange == "p2p" else LocalExchange()
    try:
        drv = ShardedDriver(engines, ex, 3)
        with torch.cuda.stream(first.stream):
            drv.initialize()
            drv.run(0, p.niter)
        seen = []
        for e in engines:
            with pytest.raises(psso.NonFiniteFitnessError) as ei:
                e.check()
            seen.append((ei.value.iteration, ei.value.particle, ei.value.value))
        want = (ref.value.iteration, ref.value.particle, ref.value.value)
        assert seen == [want] * 3
    finally:
        if exchange == "p2p":
            ex.close()
        for e in engines:
            e.close()
