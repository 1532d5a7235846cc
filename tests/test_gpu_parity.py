"""GPU parity: the CUDA path (through libpsso.so) against the reference's goldens and the oracle.

Bit-exact for indices, selections, positions and f1-f4 fitness (pure +,-,* in
numpy order, no FMA).  f5-f9 use transcendentals (CUDA libdevice vs glibc /
numpy SIMD): their fitness values must agree within RTOL = 1e-12 relative
(north-star tolerance for fp64) while positions and selections stay bitwise.
"""

import ctypes
import math
import warnings

import numpy as np
import pytest

from conftest import BITWISE_FIDS, BOUNDS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU runs deselect -m gpu
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200 import _lib  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

RTOL = 1e-12     # fp64 fitness tolerance for transcendental objectives
RTOL32 = 1e-5    # fp32 fitness tolerance


def _fn(fid, d):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return psso.make_function(fid, d)


def _params(fn, nsol, niter, cw=0.3, cp=0.6, cg=0.8, var_min=None, var_max=None):
    return psso.SsoParams(cw=cw, cp=cp, cg=cg,
                          var_min=fn.var_min if var_min is None else var_min,
                          var_max=fn.var_max if var_max is None else var_max,
                          nsol=nsol, nvar=fn.dimension, niter=niter)


def _close(a, b, fid, rtol=RTOL):
    a, b = np.asarray(a), np.asarray(b)
    if fid in BITWISE_FIDS:
        return np.array_equal(a, b)
    return np.allclose(a, b, rtol=rtol, atol=0.0)


# ------------------------------------------------------------------- RNG ----

def test_rng_bitwise_against_reference_golden(golden_rng):
    g = golden_rng
    for a, seed in enumerate(g["seeds"]):
        r = psso.RngStream(int(seed))
        for b, st in enumerate(g["streams"]):
            for c, t in enumerate(g["iters"]):
                u = r.uniform(psso.SubStream(int(st)), int(t), g["parts"][:, None], g["vars"][None, :])
                assert np.array_equal(u, g["u"][a, b, c]), (seed, st, t)
    wide = psso.RngStream((1 << 64) + 42).uniform(psso.SubStream.BRANCH, 0, 0, 0)
    assert wide == g["wide_seed_u"]


def test_rng_matrix_slices_and_range():
    r = psso.RngStream(9)
    full = r.matrix(psso.SubStream.BRANCH, 3, 0, 100, 17)
    assert np.array_equal(full[30:40], r.matrix(psso.SubStream.BRANCH, 3, 30, 40, 17))
    u = psso.RngStream(1).matrix(psso.SubStream.INIT, 0, 0, 1000, 100)
    assert u.min() >= 0.0 and u.max() < 1.0
    assert np.array_equal(u, O.u_batch(1, "INIT", 0, np.arange(1000)[:, None], np.arange(100)[None, :]))


# --------------------------------------------------------------- fitness ----

@pytest.mark.parametrize("fid", psso.FUNCTION_IDS)
def test_fitness_against_reference_golden(fid, golden_fitness):
    for key in golden_fitness.files:
        if not key.startswith(fid + "_") or key.endswith("refpt"):
            continue
        d = int(key.split("_")[1])
        fn = _fn(fid, d)
        x = O.init_positions(1000 + d, 6, d, *BOUNDS[fid])
        got = fn(x)
        assert _close(got, golden_fitness[key], fid), (key, got, golden_fitness[key])
        ref = fn(fn.reference_point)
        assert _close(ref, golden_fitness[key + "_refpt"], fid) or abs(ref) <= 1e-12, key


@pytest.mark.parametrize("fid", psso.FUNCTION_IDS)
def test_batch_equals_rows_and_storage_order(fid):
    fn = _fn(fid, 48)
    rng = np.random.default_rng(abs(hash(fid)) % 2**32)
    block = rng.uniform(fn.var_min, fn.var_max, size=(37, 48))
    rows = np.array([fn(r) for r in block])
    assert np.array_equal(fn(block), rows)
    assert np.array_equal(fn(np.asfortranarray(block)), rows)
    assert _close(rows, O.evaluate(fid, block), fid)


def test_known_values():
    origin50 = np.zeros(50)
    for fid in ("f1", "f2", "f3", "f5", "f7"):
        assert psso.make_function(fid, 50)(origin50) == 0.0
    assert psso.make_function("f4", 50)(np.ones(50)) == 0.0
    assert abs(psso.make_function("f6", 50)(origin50)) <= 1e-12
    assert abs(psso.make_function("f9", 50)(origin50) - 20949.145) <= 1e-9
    assert psso.make_function("f2", 3)(np.ones(3)) == pytest.approx(6.0, abs=1e-12)
    assert psso.make_function("f3", 8)(np.ones(8)) == pytest.approx(204.0, abs=1e-12)
    assert psso.make_function("f1", 2)(np.array([3.0, 4.0])) == pytest.approx(25.0)
    fn = _fn("f8", 50)
    x = np.zeros(50)
    x[-2:] = 3.0
    assert fn(x) == 0.0
    y = np.random.default_rng(7).uniform(-4, 5, size=50)
    assert fn(y) == psso.make_function("f8", 48)(y[:48])


@pytest.mark.parametrize("fid", psso.FUNCTION_IDS)
def test_fp32_fitness_within_tolerance(fid):
    d = 64
    fn = _fn(fid, d)
    x = O.init_positions(77, 64, d, *BOUNDS[fid]).astype(np.float32)
    from paper_2110_01470_b200.benchmarks import evaluate_rows

    got = evaluate_rows(fn, x, dtype="float32")
    ref = O.evaluate(fid, x.astype(np.float64))
    rel = np.abs(got - ref) / np.abs(ref)  # no objective is near 0 at in-box random points
    assert rel.max() <= RTOL32, (fid, rel.max())


# ----------------------------------------------------------- whole runs ----

def _run_ids(golden):
    index, _ = golden
    return [e["key"] for e in index]


@pytest.fixture(scope="module")
def runs_index():
    import json

    from conftest import GOLDEN

    return {e["key"]: e for e in json.loads((GOLDEN / "runs.json").read_text())}


RUN_KEYS = [f"run{k}" for k in range(27)]


@pytest.mark.parametrize("key", RUN_KEYS)
def test_run_parallel_against_reference_golden(key, runs_index, golden_runs):
    e = runs_index[key]
    _, arr = golden_runs
    fn = _fn(e["fid"], e["nvar"])
    p = psso.SsoParams(cw=e["cw"], cp=e["cp"], cg=e["cg"], var_min=e["var_min"],
                       var_max=e["var_max"], nsol=e["nsol"], nvar=e["nvar"], niter=e["niter"])
    rec = psso.run_parallel(p, fn, seed=e["seed"])
    assert rec.schedule == psso.ScheduleKind.PARALLEL and rec.function == e["fid"]
    assert np.array_equal(rec.best_position, arr[key + "_gbest"]), "gbest position (bitwise)"
    assert _close(rec.trajectory, arr[key + "_traj"], e["fid"]), "trajectory"
    assert rec.best_fitness == rec.trajectory[-1]
    if e["state"]:
        eng = DeviceEngine(p, fn, e["seed"], keep_sol_f=True)
        try:
            eng.initialize()
            assert _close(eng.p_f.cpu().numpy(), arr[key + "_init_p_f"], e["fid"])
            eng.run(0, e["niter"])
            eng.check()
            sw = eng.to_host()
        finally:
            eng.close()
        assert np.array_equal(sw.sol, arr[key + "_sol"])
        assert np.array_equal(sw.pbests, arr[key + "_pbests"])
        assert _close(sw.p_f, arr[key + "_p_f"], e["fid"])
        assert _close(sw.sol_f, arr[key + "_sol_f"], e["fid"])


def test_stepwise_state_against_reference_golden(golden_runs):
    _, arr = golden_runs
    fn = psso.make_function("f4", 10)
    p = _params(fn, 12, 12)
    eng = DeviceEngine(p, fn, 5, keep_sol_f=True)
    try:
        eng.initialize()
        for t in range(p.niter):
            eng.step(t)
            sw = eng.to_host()
            assert np.array_equal(sw.sol, arr["steps_sol"][t]), t
            assert np.array_equal(sw.pbests, arr["steps_pbests"][t]), t
            assert np.array_equal(sw.p_f, arr["steps_p_f"][t]), t
            assert np.array_equal(sw.gbest, arr["steps_gbest"][t]), t
    finally:
        eng.close()


def test_c1_appendix_values():
    fn = psso.make_function("f1", 30)
    rec = psso.run_parallel(_params(fn, 100, 1000), fn, seed=0)
    assert rec.best_fitness == 8.542836016810329
    import hashlib

    assert hashlib.sha256(rec.trajectory.tobytes()).hexdigest()[:16] == "767e5860d9ad62e6"
    assert hashlib.sha256(rec.best_position.tobytes()).hexdigest()[:16] == "586dba8e667ca007"


# ------------------------------------------------------------- phase API ----

def test_phase_api_composes_to_fused_step():
    fn = psso.make_function("f5", 20)
    p = _params(fn, 15, 40)
    rng = psso.RngStream(99)
    swarm = psso.initialize(p, fn, rng)
    o = O.Oracle.from_params(p, "f5", 99)
    osw = o.initialize()
    assert np.array_equal(swarm.sol, osw.sol)
    g_prev = swarm.g_f
    for t in range(p.niter):
        psso.search_phase(swarm, p, rng, t)
        psso.evaluate_phase(swarm, fn, t)
        psso.update_pbests_phase(swarm)
        psso.update_gbest_phase(swarm)
        o.step(osw, t)
        assert np.array_equal(swarm.sol, osw.sol), t
        assert np.array_equal(swarm.pbests, osw.pbests), t
        assert np.array_equal(swarm.gbest, osw.gbest), t
        assert np.all(swarm.p_f <= swarm.sol_f)
        assert np.all(swarm.g_f <= swarm.p_f)
        assert swarm.g_f <= g_prev
        g_prev = swarm.g_f
    rec = psso.run_parallel(p, fn, seed=99)
    assert np.array_equal(rec.best_position, swarm.gbest)


def test_search_phase_keeps_untouched_fields_and_box():
    fn = psso.make_function("f6", 12)
    p = _params(fn, 50, 5, cw=0.1, cp=0.3, cg=0.5)
    swarm = psso.initialize(p, fn, psso.RngStream(2))
    before = swarm.copy()
    for t in range(5):
        psso.search_phase(swarm, p, psso.RngStream(2), t)
        assert swarm.sol.min() >= p.var_min and swarm.sol.max() <= p.var_max
    assert np.array_equal(swarm.pbests, before.pbests)
    assert np.array_equal(swarm.gbest, before.gbest)


def test_all_keep_thresholds_leave_positions():
    fn = psso.make_function("f1", 6)
    p = _params(fn, 10, 5, cw=1.0, cp=1.0, cg=1.0)
    swarm = psso.initialize(p, fn, psso.RngStream(1))
    before = swarm.sol.copy()
    psso.search_phase(swarm, p, psso.RngStream(1), 0)
    assert np.array_equal(swarm.sol, before)


def test_update_phases_edge_semantics():
    fn = psso.make_function("f1", 3)
    p = _params(fn, 2, 1)
    swarm = psso.initialize(p, fn, psso.RngStream(6))
    swarm.sol[0] = [1.0, 2.0, 3.0]
    swarm.sol_f[0] = swarm.p_f[0]  # tie refreshes the incumbent
    psso.update_pbests_phase(swarm)
    assert np.array_equal(swarm.pbests[0], [1.0, 2.0, 3.0])
    # gbest: lowest index wins ties; incumbent survives only if strictly better
    swarm = psso.initialize(_params(fn, 3, 1), fn, psso.RngStream(0))
    swarm.pbests = np.arange(9, dtype=float).reshape(3, 3)
    swarm.p_f = np.array([5.0, 3.0, 3.0])
    swarm.gbest = np.array([-1.0, -1.0, -1.0])
    swarm.g_f = 4.0
    psso.update_gbest_phase(swarm)
    assert swarm.g_f == 3.0 and np.array_equal(swarm.gbest, swarm.pbests[1])
    swarm.p_f = np.array([5.0, 6.0, 7.0])
    swarm.g_f = 4.0
    swarm.gbest = np.array([-1.0, -1.0, -1.0])
    psso.update_gbest_phase(swarm)
    assert swarm.g_f == 4.0 and np.array_equal(swarm.gbest, [-1.0, -1.0, -1.0])


# ------------------------------------------------------ sharding / layout ----

@pytest.mark.parametrize("shards", [2, 3, 7, 23])
def test_virtual_shards_bitwise(shards):
    fn = psso.make_function("f4", 10)
    p = _params(fn, 23, 25)
    base = psso.run_parallel(p, fn, seed=42)
    rec = psso.run_parallel(p, fn, seed=42, shards=shards)
    assert rec.best_fitness == base.best_fitness
    assert np.array_equal(rec.best_position, base.best_position)
    assert np.array_equal(rec.trajectory, base.trajectory)


def test_workers_and_layout_have_no_effect():
    fn = psso.make_function("f7", 9)
    p = _params(fn, 14, 20)
    a = psso.run_parallel(p, fn, seed=3, workers=1, layout=psso.LayoutMode.PARTICLE_MAJOR)
    b = psso.run_parallel(p, fn, seed=3, workers=8, layout=psso.LayoutMode.INTERLEAVED)
    assert a.best_fitness == b.best_fitness and np.array_equal(a.trajectory, b.trajectory)
    with pytest.raises(ValueError, match="workers"):
        psso.run_parallel(p, fn, seed=0, workers=0)


# ---------------------------------------------------------- fault paths ----

def test_nonfinite_during_iterations_names_particle():
    level = float(O.init_positions(0, 40, 4, -1.0, 1.0)[:, 0].max())  # init stays finite
    fn = psso.probe_function(4, level=level, bounds=(-1.0, 1.0))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=40, nvar=4, niter=200)
    with pytest.raises(psso.NonFiniteFitnessError) as ei:
        psso.run_parallel(p, fn, seed=0)
    err = ei.value
    assert err.iteration is not None and math.isinf(err.value)
    assert f"particle {err.particle}" in str(err)
    # replay through the phase API: the same (iteration, particle) is the first failure
    rng = psso.RngStream(0)
    swarm = psso.initialize(p, fn, rng)
    for t in range(err.iteration + 1):
        psso.search_phase(swarm, p, rng, t)
        bad = np.nonzero(swarm.sol[:, 0] > level)[0]
        if bad.size:
            assert t == err.iteration and bad[0] == err.particle
            with pytest.raises(psso.NonFiniteFitnessError, match=f"particle {err.particle}"):
                psso.evaluate_phase(swarm, fn, t)
            break
        psso.evaluate_phase(swarm, fn, t)
        psso.update_pbests_phase(swarm)
        psso.update_gbest_phase(swarm)
    else:
        pytest.fail("phase replay never hit the probe")


def test_nonfinite_during_initialization():
    fn = psso.probe_function(3, level=-2.0)  # every particle is +inf
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=5, nvar=3, niter=2)
    with pytest.raises(psso.NonFiniteFitnessError, match="particle 0 during initialization"):
        psso.run_parallel(p, fn, seed=1)


def test_plain_callables_rejected():
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=5, nvar=3, niter=2)
    with pytest.raises(TypeError, match="registry objectives"):
        psso.run_parallel(p, lambda x: 0.0, seed=1)


# ------------------------------------------------------ C ABI host entry ----

def test_psso_solve_host_buffers_match_run_parallel():
    fn = psso.make_function("f2", 40)
    p = _params(fn, 300, 60)
    rec = psso.run_parallel(p, fn, seed=5)
    from paper_2110_01470_b200.engine import make_config

    cfg = make_config(p, fn, 5)
    traj = np.empty(p.niter)
    best = np.empty(p.nvar)
    bf, wall = ctypes.c_double(), ctypes.c_double()
    rc = _lib.load().psso_solve(ctypes.byref(cfg), p.niter, traj.ctypes.data, best.ctypes.data,
                                ctypes.byref(bf), ctypes.byref(wall))
    assert rc == 0, _lib.last_error()
    assert np.array_equal(traj, rec.trajectory) and np.array_equal(best, rec.best_position)
    assert bf.value == rec.best_fitness and wall.value > 0


# ------------------------------------------------- full-size properties ----

def _oracle_run(fid, p, seed, niter, threads=None):
    o = O.Oracle.from_params(p, fid, seed, threads=threads or O.max_threads())
    sw = o.initialize()
    traj = o.run(sw, 0, niter)
    return sw, traj


@pytest.mark.parametrize("fid,nsol,nvar,niter", [
    ("f5", 1 << 17, 128, 4),   # C3 row shape
    ("f4", 1 << 17, 64, 4),    # C4 row shape
    ("f6", 1024, 4096, 3),     # C5 row shape (multi-leaf rows)
    ("f7", 4096, 100, 5),      # C2 shape (sequential product, aux table)
    # chain kernel, compile-time row shapes (D = 8M) with ragged last groups
    ("f5", 4099, 32, 6), ("f4", 4099, 32, 6), ("f1", 1003, 64, 6), ("f9", 515, 128, 5),
    ("f2", 1001, 128, 5),
    # row-split kernel k_rows: D = 512 W, W = 1, 2, 4, 8, rows not a multiple of 8 / W
    ("f6", 1021, 512, 4), ("f2", 257, 1024, 3), ("f5", 130, 2048, 3), ("f9", 77, 4096, 3),
    ("f1", 333, 512, 4),
])
def test_large_shapes_against_oracle(fid, nsol, nvar, niter):
    fn = psso.make_function(fid, nvar)
    p = _params(fn, nsol, niter)
    eng = DeviceEngine(p, fn, 0, keep_sol_f=True)
    try:
        eng.initialize()
        eng.run(0, niter)
        eng.check()
        sw = eng.to_host()
        traj = eng.traj.cpu().numpy()
    finally:
        eng.close()
    osw, otraj = _oracle_run(fid, p, 0, niter)
    assert np.array_equal(sw.sol, osw.sol)
    assert np.array_equal(sw.pbests, osw.pbests)
    assert np.array_equal(sw.gbest, osw.gbest)
    assert _close(sw.p_f, osw.p_f, fid) and _close(traj, otraj, fid)


def test_c3_full_size_invariants_and_determinism():
    """BASELINE config C3 at full size: 2^20 x 128 Rastrigin, size-independent properties."""
    fn = psso.make_function("f5", 128)
    p = _params(fn, 1 << 20, 12)
    outs = []
    for shards in (1, 2):
        if shards == 1:
            eng = DeviceEngine(p, fn, 0, keep_sol_f=True)
            try:
                eng.initialize()
                eng.run(0, p.niter)
                eng.check()
                traj = eng.traj.cpu().numpy()
                p_f = eng.p_f.cpu().numpy()
                sol_f = eng.sol_f.cpu().numpy()
                gb = eng.gbest.cpu().numpy()
                P = eng.pbests
                X = eng.sol
                assert float(X.min()) >= p.var_min and float(X.max()) <= p.var_max
                assert np.all(p_f <= sol_f)
                b = int(np.argmin(p_f))
                assert traj[-1] == p_f[b] and np.array_equal(gb, P[b].cpu().numpy())
                assert np.all(np.diff(traj) <= 0)
                xs = float(X.double().sum())
            finally:
                eng.close()
            outs.append((traj, gb, xs))
        else:
            rec = psso.run_parallel(p, fn, seed=0, shards=shards)
            outs.append((rec.trajectory, rec.best_position, None))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_fp32_mode_positions_are_rounded_reference_positions():
    fn = psso.make_function("f5", 128)
    p = _params(fn, 4096, 30)
    eng = DeviceEngine(p, fn, 3, dtype="float32", keep_sol_f=True)
    try:
        eng.initialize()
        x32 = eng.sol.cpu().numpy()
        eng.run(0, p.niter)
        eng.check()
        traj = eng.traj.cpu().numpy()
    finally:
        eng.close()
    x64 = O.Oracle.from_params(p, "f5", 3).initialize().sol
    assert np.array_equal(x32, x64.astype(np.float32))
    assert np.all(np.diff(traj) <= 0) and np.isfinite(traj).all()
    # fp32 fitness of the fp32 positions vs the fp64 oracle on the same inputs
    ref = O.evaluate("f5", x32.astype(np.float64))
    from paper_2110_01470_b200.benchmarks import evaluate_rows

    got = evaluate_rows(fn, x32, dtype="float32")
    assert np.all(np.abs(got - ref) <= RTOL32 * np.abs(ref))


def test_philox_mode_distribution_matches_reference():
    """Benchmark mode: final-fitness distribution over 30 seeds vs the oracle (reference RNG)."""
    from scipy import stats

    fn = psso.make_function("f1", 30)
    p = _params(fn, 100, 1000)
    gpu = np.array([psso.run_parallel(p, fn, seed=s, rng="philox").best_fitness for s in range(30)])
    ref = np.array([_oracle_run("f1", p, s, p.niter, threads=1)[1][-1] for s in range(30)])
    assert abs(gpu.mean() - ref.mean()) <= 0.10 * ref.mean(), (gpu.mean(), ref.mean())
    assert stats.kruskal(gpu, ref).pvalue > 0.01
    assert stats.ttest_ind(gpu, ref).pvalue > 0.01


# ------------------------------------------- whole-run kernel (k_swarm) ----

def _engine_run(fid, nsol, nvar, niter, monkeypatch, env=None, dtype="float64", rng="reference",
                seed=3):
    for k in ("PSSO_NO_SWARM", "PSSO_NO_CHAIN"):
        monkeypatch.delenv(k, raising=False)
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    fn = _fn(fid, nvar)
    p = _params(fn, nsol, niter)
    eng = DeviceEngine(p, fn, seed, dtype=dtype, rng=rng, keep_sol_f=True)
    try:
        eng.initialize()
        eng.run(0, 7)            # two launches: the loop state carries across calls
        eng.run(7, niter - 7)
        eng.check()
        sw = eng.to_host()
        traj = eng.traj.cpu().numpy()
    finally:
        eng.close()
    return sw, traj


@pytest.mark.parametrize("fid,nsol,nvar,niter", [
    ("f1", 100, 30, 60),      # C1 shape: one CTA
    ("f5", 1024, 100, 40),    # C2 shape: 32 CTAs and a swarm barrier
    ("f7", 1024, 100, 30),    # sequential product through the smem rows
    ("f4", 1001, 64, 30), ("f3", 333, 20, 30), ("f8", 515, 128, 30), ("f6", 4099, 33, 25),
])
def test_whole_run_kernel_matches_streaming_path(fid, nsol, nvar, niter, monkeypatch):
    """k_swarm (one launch, swarm barrier) == fused+gBest launches per iteration, bitwise."""
    a, ta = _engine_run(fid, nsol, nvar, niter, monkeypatch)
    b, tb = _engine_run(fid, nsol, nvar, niter, monkeypatch, env={"PSSO_NO_SWARM": "1"})
    assert np.array_equal(ta, tb)
    for name in ("sol", "pbests", "gbest", "p_f"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
    assert a.g_f == b.g_f


@pytest.mark.parametrize("dtype,rng", [("float32", "reference"), ("float64", "philox"),
                                       ("float32", "philox")])
def test_whole_run_kernel_other_modes(dtype, rng, monkeypatch):
    a, ta = _engine_run("f5", 1024, 100, 30, monkeypatch, dtype=dtype, rng=rng)
    b, tb = _engine_run("f5", 1024, 100, 30, monkeypatch, env={"PSSO_NO_SWARM": "1"},
                        dtype=dtype, rng=rng)
    assert np.array_equal(ta, tb) and np.array_equal(a.gbest, b.gbest)
    assert np.array_equal(a.sol, b.sol) and np.array_equal(a.pbests, b.pbests)


# ------------------------------------------------ multi-seed batch runs ----

@pytest.mark.parametrize("fid,nsol,nvar,niter,nseeds", [
    ("f1", 100, 30, 200, 5),    # C1 shape, co-resident swarms with a swarm barrier each
    ("f5", 1024, 100, 30, 3),   # C2 shape
    ("f7", 256, 100, 20, 4),
    ("f4", 60, 16, 50, 300),    # 300 clusters of 2 CTAs
    ("f5", 4096, 128, 10, 3),   # too big for one cluster: global-memory exchange, rows in HBM
])
def test_batch_runs_equal_single_runs(fid, nsol, nvar, niter, nseeds):
    fn = _fn(fid, nvar)
    p = _params(fn, nsol, niter)
    seeds = [11 + 7 * k for k in range(nseeds)]
    recs = psso.run_parallel_batch(p, fn, seeds)
    assert [r.seed for r in recs] == seeds and [r.run_id for r in recs] == list(range(nseeds))
    for k in sorted({0, nseeds // 2, nseeds - 1}):
        one = psso.run_parallel(p, fn, seeds[k])
        assert np.array_equal(recs[k].trajectory, one.trajectory)
        assert np.array_equal(recs[k].best_position, one.best_position)
        assert recs[k].best_fitness == one.best_fitness
        # and directly against the oracle (the checker), not only the streaming path
        sw, otraj = _oracle_run(fid, p, seeds[k], niter)
        assert _close(recs[k].trajectory, otraj, fid)
        assert np.array_equal(recs[k].best_position, sw.gbest)


def test_batch_c1_appendix_values():
    """Config C1 for seeds 0 and 1 in one launch: the reference's final values bitwise."""
    fn = _fn("f1", 30)
    p = _params(fn, 100, 1000)
    r0, r1 = psso.run_parallel_batch(p, fn, [0, 1])
    assert r0.best_fitness == 8.542836016810329
    assert r1.best_fitness == 8.834077304158543


def test_batch_nonfinite_names_particle():
    fn = psso.probe_function(8, level=0.999, bounds=(-1.0, 1.0))  # +inf once x[0] > 0.999
    p = _params(fn, 64, 400)
    with pytest.raises(psso.NonFiniteFitnessError) as ei:
        psso.run_parallel_batch(p, fn, [0, 1, 2])
    assert ei.value.particle >= 0 and math.isinf(ei.value.value)
    for seed in (0, 1, 2):  # the first failing seed's own run names the same event
        try:
            psso.run_parallel(p, fn, seed=seed)
        except psso.NonFiniteFitnessError as one:
            assert (one.iteration, one.particle, one.value) == \
                (ei.value.iteration, ei.value.particle, ei.value.value)
            break
    else:
        pytest.fail("no single run failed")


# ------------------------------------------------- kernel dispatch paths ----

@pytest.mark.parametrize("fid,nsol,nvar,box,kernel", [
    ("f5", 1 << 16, 128, None, "k_chain"),       # streaming, register rows
    ("f5", 1000, 100, None, "k_swarm"),          # small swarm: whole run in one launch
    ("f6", 300, 1024, None, "k_rows"),           # long rows D = 512 W
    ("f5", 300, 300, None, "k_fused"),           # D > 128, not 512 W: TMA tile ring
    ("f5", 200, 301, None, "k_tile"),            # odd row length: register tiles
    ("f5", 1 << 16, 128, 1e13, "k_fused"),       # box beyond the branch-free trig range
    ("f9", 500, 63, 1e13, "k_tile"),
])
def test_dispatch_paths_against_oracle(fid, nsol, nvar, box, kernel):
    """Every iteration-kernel family, selected by shape, against the oracle."""
    fn = _fn(fid, nvar)
    niter = 4
    p = _params(fn, nsol, niter, var_min=None if box is None else -box,
                var_max=None if box is None else box)
    eng = DeviceEngine(p, fn, 5, keep_sol_f=True)
    try:
        name = _lib.load().psso_kernel_name(eng.ctx).decode()
        assert name.startswith(kernel), name
        eng.initialize()
        eng.run(0, niter)
        eng.check()
        sw = eng.to_host()
        traj = eng.traj.cpu().numpy()
    finally:
        eng.close()
    o = O.Oracle.from_params(p, fid, 5, threads=O.max_threads())
    osw = o.initialize()
    otraj = o.run(osw, 0, niter)
    assert np.array_equal(sw.sol, osw.sol) and np.array_equal(sw.pbests, osw.pbests)
    assert np.array_equal(sw.gbest, osw.gbest)
    assert _close(sw.p_f, osw.p_f, fid) and _close(traj, otraj, fid)


# ------------------------------------------ reference test-strategy gaps ----

def test_rng_uniformity_seed_masking_and_key_sensitivity():
    """reference test_rng.py:23-53 -- chi^2 per substream, 64-bit seed masking, key sensitivity."""
    n_i, n_j = 1000, 1000  # 10^6 draws per substream
    i = np.arange(n_i, dtype=np.uint64)[:, None]
    j = np.arange(n_j, dtype=np.uint64)[None, :]
    rng = psso.RngStream(12345)
    for stream in psso.SubStream:
        u = rng.uniform(stream, 3, i, j).ravel()
        assert u.min() >= 0.0 and u.max() < 1.0
        counts = np.bincount(np.minimum((u * 100).astype(int), 99), minlength=100)
        chi2 = float(((counts - u.size / 100) ** 2 / (u.size / 100)).sum())
        assert chi2 < 160.0, (stream, chi2)  # 99 dof: p ~ 1e-4
    a = psso.RngStream(7).uniform(psso.SubStream.BRANCH, 1, i[:10], j[:, :10])
    b = psso.RngStream(7 + (1 << 64)).uniform(psso.SubStream.BRANCH, 1, i[:10], j[:, :10])
    assert np.array_equal(a, b)  # seeds are masked to 64 bits
    for other in (psso.RngStream(8).uniform(psso.SubStream.BRANCH, 1, i[:10], j[:, :10]),
                  psso.RngStream(7).uniform(psso.SubStream.BRANCH, 2, i[:10], j[:, :10]),
                  psso.RngStream(7).uniform(psso.SubStream.FRESH, 1, i[:10], j[:, :10])):
        assert np.mean(a == other) < 0.01  # every key component changes the draws


def test_branch_law_on_a_million_draws():
    """Acceptance C3 (reference test_acceptance.py:101-113): branch frequencies follow the thresholds."""
    cw, cp, cg = 0.3, 0.6, 0.8
    u = psso.RngStream(0).uniform(psso.SubStream.BRANCH, 5, np.arange(1000, dtype=np.uint64)[:, None],
                                  np.arange(1000, dtype=np.uint64)[None, :]).ravel()
    freq = np.array([np.mean(u < cw), np.mean((u >= cw) & (u < cp)), np.mean((u >= cp) & (u < cg)),
                     np.mean(u >= cg)])
    assert np.allclose(freq, [0.3, 0.3, 0.2, 0.2], atol=0.003), freq


@pytest.mark.parametrize("fid,nsol,nvar", [("f1", 100, 30), ("f5", 1 << 16, 128)])
def test_shorter_run_is_a_prefix(fid, nsol, nvar):
    """reference test_core.py:186-191: the keyed RNG makes a shorter run an exact prefix."""
    fn = _fn(fid, nvar)
    short = psso.run_parallel(_params(fn, nsol, 20), fn, 4)
    long_ = psso.run_parallel(_params(fn, nsol, 45), fn, 4)
    assert np.array_equal(long_.trajectory[:20], short.trajectory)
    assert np.all(np.diff(long_.trajectory) <= 0)  # g_f is monotone (parallel.py:209)


# ------------------------------- device-initiated gBest exchange (P2P) ----

@pytest.mark.parametrize("shards", [2, 3, 7])
def test_p2p_exchange_virtual_shards_bitwise(shards):
    """Records stored straight into every shard's buffer + epoch flags == one shard."""
    fn = _fn("f5", 64)
    p = _params(fn, 4096 + 5, 30)
    one = psso.run_parallel(p, fn, 9)
    from paper_2110_01470_b200.sharded import run_virtual_shards

    rec = run_virtual_shards(p, fn, 9, shards, exchange="p2p")
    assert np.array_equal(rec.trajectory, one.trajectory)
    assert np.array_equal(rec.best_position, one.best_position)
    sw, otraj = _oracle_run("f5", p, 9, p.niter)  # the checker itself
    assert _close(rec.trajectory, otraj, "f5") and np.array_equal(rec.best_position, sw.gbest)


def _p2p_rank(rank, world, port, q):
    import os

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    import paper_2110_01470_b200 as P

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fn = P.make_function("f4", 64)
    p = P.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                    nsol=5000, nvar=64, niter=25)
    rec = P.run_parallel_distributed(p, fn, 11, exchange="p2p")
    q.put((rank, rec.trajectory.tobytes(), rec.best_position.tobytes()))
    dist.destroy_process_group()


def test_p2p_exchange_across_processes_via_cuda_ipc():
    """Two processes (gloo only for the one-time IPC-handle exchange) on one GPU."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_rank, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    fn = _fn("f4", 64)
    one = psso.run_parallel(_params(fn, 5000, 25), fn, 11)
    for _, traj, best in out:
        assert traj == one.trajectory.tobytes() and best == one.best_position.tobytes()


def test_more_than_2_31_coordinates():
    """2^25 + 3 particles x 64 = 2.1e9 coordinates per matrix (32 GiB of X + P): 64-bit indexing.

    The last particle (coordinates beyond 2^31) is checked exactly against the
    keyed RNG: its initial row (core.py:198-199) and its first search step
    (core.py:129-135), recomputed on the host from RngStream draws.
    """
    fn = _fn("f4", 64)
    n = (1 << 25) + 3
    p = _params(fn, n, 2)
    eng = DeviceEngine(p, fn, 21)
    rng = psso.RngStream(21)
    j = np.arange(64, dtype=np.uint64)
    span = p.var_max - p.var_min
    try:
        eng.initialize()
        eng.check()
        x0 = eng.sol[-1].cpu().numpy()
        u0 = rng.uniform(psso.SubStream.INIT, 0, n - 1, j)
        assert np.array_equal(x0, p.var_min + span * u0)
        g = eng.gbest.cpu().numpy()
        eng.run(0, 1)
        eng.check()
        x1 = eng.sol[-1].cpu().numpy()
        ub = rng.uniform(psso.SubStream.BRANCH, 0, n - 1, j)
        uf = rng.uniform(psso.SubStream.FRESH, 0, n - 1, j)
        want = np.where(ub < p.cw, x0, np.where(ub < p.cp, x0, np.where(ub < p.cg, g,
                                                                          p.var_min + span * uf)))
        assert np.array_equal(x1, want)  # pbest == initial row after initialization
        torch.cuda.synchronize()
        X, P, p_f = eng.sol, eng.pbests, eng.p_f
        assert float(X.min()) >= p.var_min and float(X.max()) <= p.var_max
        b = int(torch.argmin(p_f))
        assert float(eng.g_f[0]) == float(p_f[b]) == float(p_f.min())
        assert torch.equal(eng.gbest, P[b])
    finally:
        eng.close()
