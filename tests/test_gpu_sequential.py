"""GPU parity of the sequential schedule (reference core.py:213-258) on device.

``run_sequential`` runs ONE k_seq launch (speculative passes with rollback,
psso_seq.cuh).  Checked against fixtures made by the reference's own
run_sequential (tests/golden/make_seq_golden.py) and against the oracle's C
restatement: positions, pBests and gBest bitwise, fitness bitwise for f1-f4 and
within RTOL for the transcendental objectives.
"""

import json
import math
import warnings

import numpy as np
import pytest

from conftest import BITWISE_FIDS, GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU runs deselect -m gpu
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

RTOL = 1e-12

SEQ_INDEX = {e["key"]: e for e in json.loads((GOLDEN / "seq_runs.json").read_text())}


def _fn(fid, d):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return psso.make_function(fid, d)


def _close(a, b, fid):
    a, b = np.asarray(a), np.asarray(b)
    if fid in BITWISE_FIDS:
        return np.array_equal(a, b)
    return np.allclose(a, b, rtol=RTOL, atol=0.0)


def _params_of(e):
    return psso.SsoParams(cw=e["cw"], cp=e["cp"], cg=e["cg"], var_min=e["var_min"],
                          var_max=e["var_max"], nsol=e["nsol"], nvar=e["nvar"], niter=e["niter"])


@pytest.mark.parametrize("key", sorted(SEQ_INDEX, key=lambda k: int(k[3:])))
def test_run_sequential_against_reference_golden(key, golden_seq_runs):
    e = SEQ_INDEX[key]
    _, arr = golden_seq_runs
    fn = _fn(e["fid"], e["nvar"])
    p = _params_of(e)
    rec = psso.run_sequential(p, fn, seed=e["seed"])
    assert rec.schedule == psso.ScheduleKind.SEQUENTIAL and rec.function == e["fid"]
    assert np.array_equal(rec.best_position, arr[key + "_gbest"]), "gbest position (bitwise)"
    assert _close(rec.trajectory, arr[key + "_traj"], e["fid"]), "trajectory"
    assert rec.best_fitness == rec.trajectory[-1]
    # end state, and the pass count of the rollback scheme: one pass per
    # iteration plus one per gbest move
    eng = DeviceEngine(p, fn, e["seed"])
    try:
        eng.initialize()
        eng.run_sequential(0, p.niter)
        eng.check()
        sw = eng.to_host()
        passes = eng.sequential_passes
    finally:
        eng.close()
    assert np.array_equal(sw.sol, arr[key + "_sol"])
    assert np.array_equal(sw.pbests, arr[key + "_pbests"])
    assert _close(sw.p_f, arr[key + "_p_f"], e["fid"])
    assert _close(sw.sol_f, arr[key + "_sol_f"], e["fid"])
    assert passes <= p.niter + e["gbest_moves"]
    assert passes >= p.niter


def test_c1_sequential_appendix_value():
    fn = psso.make_function("f1", 30)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-5.12, var_max=5.12, nsol=100, nvar=30,
                       niter=1000)
    rec = psso.run_sequential(p, fn, seed=0)
    assert rec.best_fitness == 10.383304882651581  # SURVEY appendix A (reference run_sequential)


@pytest.mark.parametrize("fid,nsol,nvar,niter", [
    ("f1", 1000, 32, 30), ("f2", 517, 50, 20), ("f3", 300, 64, 15), ("f4", 2000, 64, 10),
    ("f5", 700, 128, 12), ("f6", 333, 100, 12), ("f7", 400, 77, 12), ("f8", 250, 40, 12),
    ("f9", 600, 13, 15),
])
def test_sequential_against_oracle(fid, nsol, nvar, niter):
    fn = _fn(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=niter)
    o = O.Oracle.from_params(p, fid, 23)
    osw = o.initialize()
    otraj = o.run_sequential(osw, 0, niter)
    eng = DeviceEngine(p, fn, 23)
    try:
        eng.initialize()
        eng.run_sequential(0, niter)
        eng.check()
        sw = eng.to_host()
        traj = eng.traj.cpu().numpy()
    finally:
        eng.close()
    assert np.array_equal(sw.sol, osw.sol)
    assert np.array_equal(sw.pbests, osw.pbests)
    assert np.array_equal(sw.gbest, osw.gbest)
    assert _close(traj, otraj, fid)
    assert _close(sw.p_f, osw.p_f, fid)


def test_sequential_continues_across_calls():
    """Two psso_run_sequential calls == one call over the whole range."""
    fn = psso.make_function("f4", 20)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=150, nvar=20, niter=40)
    outs = []
    for split in (None, 17):
        eng = DeviceEngine(p, fn, 4)
        try:
            eng.initialize()
            if split is None:
                eng.run_sequential(0, 40)
            else:
                eng.run_sequential(0, split)
                eng.run_sequential(split, 40 - split)
            outs.append((eng.to_host(), eng.traj.cpu().numpy()))
        finally:
            eng.close()
    assert np.array_equal(outs[0][0].sol, outs[1][0].sol)
    assert np.array_equal(outs[0][1], outs[1][1])


def test_sequential_nonfinite_names_first_particle():
    """The first (iteration, particle) in serial order whose probe fitness is +inf."""
    level = float(O.init_positions(0, 40, 4, -1.0, 1.0)[:, 0].max())  # init stays finite
    fn = psso.probe_function(4, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=40, nvar=4, niter=200)
    with pytest.raises(psso.NonFiniteFitnessError) as ei:
        psso.run_sequential(p, fn, seed=0)
    err = ei.value
    assert err.iteration is not None and math.isinf(err.value)
    # the probe is Sphere until it fires: replay with the oracle's f1 sequential step
    o = O.Oracle("f1", 40, 4, 0.3, 0.6, 0.8, -1.0, 1.0, 0)
    sw = o.initialize()
    for t in range(p.niter):
        o.step_sequential(sw, t)
        bad = np.nonzero(sw.sol[:, 0] > level)[0]
        if bad.size:
            assert (t, int(bad[0])) == (err.iteration, err.particle)
            break
    else:
        pytest.fail("oracle replay never hit the probe")


def test_sequential_long_rows_run_on_the_device_state_resident():
    """nvar > 128: psso_run_sequential's device pass loop, stepwise == the oracle's serial
    loop iteration by iteration (state, gBest index, pass count), no host state round trips."""
    fn = psso.make_function("f5", 300)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max, nsol=70,
                       nvar=300, niter=6)
    eng = DeviceEngine(p, fn, 4, keep_sol_f=True)
    o = O.Oracle.from_params(p, "f5", 4)
    osw = o.initialize()
    try:
        eng.initialize()
        for t in range(p.niter):
            eng.run_sequential(t, 1)
            eng.check()
            o.step_sequential(osw, t)
            sw = eng.to_host()
            assert np.array_equal(sw.sol, osw.sol) and np.array_equal(sw.pbests, osw.pbests), t
            assert np.array_equal(sw.gbest, osw.gbest), t
            assert np.allclose(sw.p_f, osw.p_f, rtol=1e-12, atol=0), t
            gf, gi = eng.result()  # the last particle that moved gbest holds it as its pBest
            assert np.array_equal(osw.pbests[gi], osw.gbest), t
            assert eng.sequential_passes >= 1
    finally:
        eng.close()


def test_sequential_long_rows_nonfinite_names_particle():
    level = float(O.init_positions(0, 40, 200, -1.0, 1.0)[:, 0].max())
    fn = psso.probe_function(200, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=40, nvar=200, niter=100)
    with pytest.raises(psso.NonFiniteFitnessError) as ei:
        psso.run_sequential(p, fn, seed=0)
    o = O.Oracle("f1", 40, 200, 0.3, 0.6, 0.8, -1.0, 1.0, 0)
    sw = o.initialize()
    for t in range(p.niter):
        o.step_sequential(sw, t)
        bad = np.nonzero(sw.sol[:, 0] > level)[0]
        if bad.size:
            assert (t, int(bad[0])) == (ei.value.iteration, ei.value.particle)
            return
    pytest.fail("oracle replay never hit the probe")


@pytest.mark.parametrize("fid,nsol,nvar,niter", [("f1", 60, 200, 12), ("f5", 40, 300, 10),
                                                  ("f4", 30, 512, 8), ("f7", 25, 129, 10),
                                                  ("f6", 300, 4096, 4), ("f3", 50, 130, 6)])
def test_sequential_long_rows_against_oracle(fid, nsol, nvar, niter):
    fn = _fn(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=niter)
    rec = psso.run_sequential(p, fn, 31)
    o = O.Oracle.from_params(p, fid, 31)
    osw = o.initialize()
    otraj = o.run_sequential(osw, 0, niter)
    assert rec.schedule == psso.ScheduleKind.SEQUENTIAL
    assert np.array_equal(rec.best_position, osw.gbest)
    assert _close(rec.trajectory, otraj, fid)


def test_sequential_fp32_and_philox_modes_run():
    fn = psso.make_function("f5", 64)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-5.12, var_max=5.12, nsol=256, nvar=64,
                       niter=50)
    for dtype, rng in (("float32", "reference"), ("float64", "philox")):
        rec = psso.run_sequential(p, fn, seed=3, dtype=dtype, rng=rng)
        assert np.all(np.diff(rec.trajectory) <= 0)
        assert np.all(np.abs(rec.best_position) <= 5.12)
        assert rec.best_fitness == pytest.approx(fn(rec.best_position[None, :].astype(np.float64))[0],
                                                 rel=1e-5)


@pytest.mark.parametrize("fid,nsol,nvar,niter,nseeds", [
    ("f1", 100, 30, 200, 5), ("f4", 64, 64, 50, 3), ("f7", 40, 100, 30, 4), ("f5", 300, 128, 20, 2),
])
def test_sequential_batch_equals_single_runs(fid, nsol, nvar, niter, nseeds):
    fn = _fn(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=niter)
    seeds = [3 + 7 * k for k in range(nseeds)]
    recs = psso.run_sequential_batch(p, fn, seeds)
    for rec, s in zip(recs, seeds):
        one = psso.run_sequential(p, fn, s)
        assert rec.schedule == psso.ScheduleKind.SEQUENTIAL and rec.seed == s
        assert np.array_equal(rec.best_position, one.best_position)
        assert np.array_equal(rec.trajectory, one.trajectory)


def test_sequential_batch_c1_appendix_value():
    fn = psso.make_function("f1", 30)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-5.12, var_max=5.12, nsol=100, nvar=30,
                       niter=1000)
    recs = psso.run_sequential_batch(p, fn, [1, 0])
    assert recs[1].best_fitness == 10.383304882651581


def test_sequential_nonfinite_on_a_cluster_names_first_particle():
    """300 rows -> a 5-CTA cluster: the first serial-order probe hit, across CTA boundaries."""
    level = float(O.init_positions(1, 300, 4, -1.0, 1.0)[:, 0].max())
    fn = psso.probe_function(4, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=300, nvar=4, niter=300)
    with pytest.raises(psso.NonFiniteFitnessError) as ei:
        psso.run_sequential(p, fn, seed=1)
    err = ei.value
    o = O.Oracle("f1", 300, 4, 0.3, 0.6, 0.8, -1.0, 1.0, 1)
    sw = o.initialize()
    for t in range(p.niter):
        o.step_sequential(sw, t)
        bad = np.nonzero(sw.sol[:, 0] > level)[0]
        if bad.size:
            assert (t, int(bad[0])) == (err.iteration, err.particle)
            break
    else:
        pytest.fail("oracle replay never hit the probe")


def test_sequential_batch_nonfinite_names_particle():
    fn = psso.probe_function(8, level=0.999, bounds=(-1.0, 1.0))  # +inf once x[0] > 0.999
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=64, nvar=8, niter=400)
    with pytest.raises(psso.NonFiniteFitnessError) as ei:
        psso.run_sequential_batch(p, fn, [0, 1, 2])
    assert ei.value.particle >= 0 and ei.value.iteration is not None


@pytest.mark.parametrize("g", ["1", "3", "16"])
def test_sequential_cluster_size_does_not_change_results(g, monkeypatch):
    fn = psso.make_function("f5", 40)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=500, nvar=40, niter=25)
    ref = psso.run_sequential(p, fn, 9)
    monkeypatch.setenv("PSSO_SEQ_G", g)
    rec = psso.run_sequential(p, fn, 9)
    assert np.array_equal(rec.best_position, ref.best_position)
    assert np.array_equal(rec.trajectory, ref.trajectory)


@pytest.mark.parametrize("schedule", ["parallel", "sequential"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_checkpoint_resume_is_bitwise(schedule, dtype, tmp_path):
    """save_state at t=25, restore into a fresh engine, run 20 more == 45 straight."""
    fn = psso.make_function("f4", 64)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=3000, nvar=64, niter=45)

    def go(e, t0, n):
        (e.run if schedule == "parallel" else e.run_sequential)(t0, n)

    a = DeviceEngine(p, fn, 5, dtype=dtype)
    a.initialize()
    go(a, 0, 25)
    a.save_state(tmp_path / "ck.npz", 25)
    a.close()
    b = DeviceEngine(p, fn, 5, dtype=dtype)
    t = b.restore_state(tmp_path / "ck.npz")
    go(b, t, 45 - t)
    b.check()
    c = DeviceEngine(p, fn, 5, dtype=dtype)
    c.initialize()
    go(c, 0, 45)
    try:
        sb, sc = b.to_host(), c.to_host()
        assert t == 25
        assert np.array_equal(sb.sol, sc.sol) and np.array_equal(sb.pbests, sc.pbests)
        assert np.array_equal(sb.gbest, sc.gbest) and sb.g_f == sc.g_f
        assert np.array_equal(b.traj.cpu().numpy(), c.traj.cpu().numpy())
        assert b.result() == c.result(), "gBest fitness and index survive the checkpoint"
    finally:
        b.close()
        c.close()
    import dataclasses

    others = [(p, fn, 6, {}), (p, fn, 5, {"rng": "philox"}),
              (dataclasses.replace(p, cg=0.9), fn, 5, {}),
              (dataclasses.replace(p, var_min=-2.0), fn, 5, {})]
    for q, f, seed, kw in others:  # another seed, RNG mode, thresholds, box
        other = DeviceEngine(q, f, seed, dtype=dtype, **kw)
        try:
            with pytest.raises(ValueError, match="does not match"):
                other.restore_state(tmp_path / "ck.npz")
        finally:
            other.close()


def test_checkpoint_refuses_pending_nonfinite(tmp_path):
    level = float(O.init_positions(0, 40, 4, -1.0, 1.0)[:, 0].max())  # init stays finite
    fn = psso.probe_function(4, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=40, nvar=4, niter=200)
    eng = DeviceEngine(p, fn, 0)
    try:
        eng.initialize()
        eng.run(0, p.niter)
        with pytest.raises(psso.NonFiniteFitnessError):
            eng.save_state(tmp_path / "bad.npz", p.niter)
        assert not (tmp_path / "bad.npz").exists()
    finally:
        eng.close()


@pytest.mark.parametrize("fid,nsol,nvar", [("f5", 1024, 100), ("f7", 300, 77), ("f3", 200, 64)])
def test_sequential_resident_rows_equal_global_rows(fid, nsol, nvar, monkeypatch):
    """k_seq with the CTA's rows in shared memory == rows in global memory, bit for bit."""
    fn = _fn(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=30)
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PSSO_SEQ_NO_RES", flag)
        eng = DeviceEngine(p, fn, 12)
        try:
            eng.initialize()
            eng.run_sequential(0, 30)
            eng.check()
            outs.append((eng.to_host(), eng.traj.cpu().numpy()))
        finally:
            eng.close()
    (a, ta), (b, tb) = outs
    assert np.array_equal(a.sol, b.sol) and np.array_equal(a.pbests, b.pbests)
    assert np.array_equal(a.p_f, b.p_f) and np.array_equal(ta, tb)


@pytest.mark.parametrize("dtype,rng", [("float32", "reference"), ("float64", "philox"),
                                       ("float32", "philox")])
def test_sequential_long_rows_other_modes(dtype, rng):
    """The device pass loop (nvar > 128) in fp32 and benchmark modes: a valid run --
    monotone trajectory, positions in the box, gbest consistent with its fitness."""
    fn = psso.make_function("f5", 300)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max, nsol=50,
                       nvar=300, niter=20)
    rec = psso.run_sequential(p, fn, seed=5, dtype=dtype, rng=rng)
    assert np.all(np.diff(rec.trajectory) <= 0) and np.isfinite(rec.trajectory).all()
    assert np.all(np.abs(rec.best_position) <= 5.12)
    assert rec.best_fitness == pytest.approx(
        fn(rec.best_position[None, :].astype(np.float64))[0], rel=1e-5 if dtype == "float32" else 1e-12)
