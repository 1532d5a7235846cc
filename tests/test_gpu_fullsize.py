"""Full-size verification of the BASELINE configs against the oracle (SURVEY §8 c, §7 H1).

Each test runs the bench configuration of a BASELINE config (C3, C4, C5) on
the device through the product path (DeviceEngine.run: graph-replayed
iteration kernel + k_gbest) and the oracle (the C restatement of the
reference, all host threads) side by side, comparing in chunks of
iterations:

* trajectory within the fitness tolerance, gBest index equal every chunk;
* X and P bitwise, p_f within the tolerance (f4: bitwise everywhere);
* at any divergence the chunk is replayed one iteration at a time from the
  chunk's start state until the first iteration whose state differs, and
  every differing selection is CLASSIFIED: a pBest `<=` (parallel.py:108-112)
  or gBest `<=` (parallel.py:209) decision flipped by fitness values that
  agree within the tolerance (device cos/exp vs glibc/numpy SIMD)
  is a near-tie -- counted, reported, and the device resynchronized from the
  oracle's state; anything else fails with the row, the iteration and both
  fitness values.  For bitwise objectives (f4) any divergence fails.

The oracle is the checker only (tests/ may import it); the product path never
touches it.  Runtime on the GPU box (16 host threads): C3 fp64 ~2.5 min, C4
~1 min, C5 ~2 min, C3 fp32 ~1 min.
"""

import copy
import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200 import _lib  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

RTOL = 1e-12      # fp64 fitness, transcendental objectives (north star)
RTOL32 = 1e-5     # fp32 fitness on identical inputs (north star)
BLOCK = 1 << 17   # rows per host comparison block


def _fn(fid, d):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return psso.make_function(fid, d)


def _params(fn, nsol, niter):
    return psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                          nsol=nsol, nvar=fn.dimension, niter=niter)


def _close(a, b, rtol):
    return np.array_equal(a, b) if rtol == 0 else np.allclose(a, b, rtol=rtol, atol=0.0)


def _diff_rows(eng, osw, rtol):
    """Rows whose X or P differ bitwise, or whose p_f differ beyond rtol (block-wise)."""
    n = eng.sol.shape[0]
    bad = []
    for a in range(0, n, BLOCK):
        b = min(n, a + BLOCK)
        x = eng.sol[a:b].to(torch.float64).cpu().numpy()
        pb = eng.pbests[a:b].to(torch.float64).cpu().numpy()
        pf = eng.p_f[a:b].cpu().numpy()
        d = np.any(x != osw.sol[a:b], axis=1) | np.any(pb != osw.pbests[a:b], axis=1)
        if rtol == 0:
            d |= pf != osw.p_f[a:b]
        else:
            d |= ~np.isclose(pf, osw.p_f[a:b], rtol=rtol, atol=0.0)
        bad.extend((a + np.flatnonzero(d)).tolist())
    return bad


def _gbest_ok(eng, osw, rtol):
    gf, gi = eng.result()
    g = eng.gbest.to(torch.float64).cpu().numpy()
    return (gi == int(np.argmin(osw.p_f)) and np.array_equal(g, osw.gbest)
            and _close(np.array([gf]), np.array([osw.g_f]), rtol))


def _classify_iteration(p, fn, seed, snap, t, rtol, dtype):
    """Replay iteration t from `snap` (equal start states) with sol_f kept on both sides.

    Returns (oracle state after t, list of near-tie records); raises AssertionError
    for an unclassified divergence."""
    o = O.Oracle.from_params(p, fn.id, seed, threads=O.max_threads())
    osw = copy.deepcopy(snap)
    rep = DeviceEngine(p, fn, seed, dtype=dtype, keep_sol_f=True)
    try:
        rep.load(snap)
        rep.step(t)
        rep.check()
        o.step(osw, t)
        x = rep.sol.to(torch.float64).cpu().numpy()
        assert np.array_equal(x, osw.sol), (
            f"iteration {t}: new positions differ from equal start states -- the search "
            "(keyed draws + four-way select) is not a near-tie")
        fd, fo = rep.sol_f.cpu().numpy(), osw.sol_f
        assert _close(fd, fo, rtol), f"iteration {t}: fitness beyond rtol {rtol}"
        ties = []
        imp_d, imp_o = fd <= snap.p_f, fo <= snap.p_f     # parallel.py:108-112
        for r in np.flatnonzero(imp_d != imp_o).tolist():
            ties.append({"kind": "pbest", "t": t, "row": r, "f_device": float(fd[r]),
                         "f_oracle": float(fo[r]), "p_f": float(snap.p_f[r])})
        pf_d = np.where(imp_d, fd, snap.p_f)
        gd, go = int(np.argmin(pf_d)), int(np.argmin(osw.p_f))
        if gd != go:                                      # parallel.py:208-211
            assert np.isclose(pf_d[gd], osw.p_f[go], rtol=rtol, atol=0.0), (
                f"iteration {t}: gBest {gd} ({pf_d[gd]!r}) vs oracle {go} ({osw.p_f[go]!r})")
            ties.append({"kind": "gbest", "t": t, "device": gd, "oracle": go,
                         "f_device": float(pf_d[gd]), "f_oracle": float(osw.p_f[go])})
        for r in ties:
            if r["kind"] == "pbest":  # the flipped decision straddles p_f within the tolerance
                assert abs(r["f_device"] - r["p_f"]) <= rtol * abs(r["p_f"]) + 0.0, r
    finally:
        rep.close()
    return osw, ties


def verify(fid, nsol, nvar, niter, chunk, seed=0, rtol=RTOL):
    fn = _fn(fid, nvar)
    p = _params(fn, nsol, niter)
    o = O.Oracle.from_params(p, fid, seed, threads=O.max_threads())
    eng = DeviceEngine(p, fn, seed)
    ties, compared = [], 0
    try:
        name = _lib.load().psso_kernel_name(eng.ctx).decode()
        eng.initialize()
        osw = o.initialize()
        assert eng.result()[1] == int(np.argmin(osw.p_f)), "init gBest index"
        assert _diff_rows(eng, osw, rtol) == [], "initialization state"
        t = 0
        while t < niter:
            k = min(chunk, niter - t)
            snap = copy.deepcopy(osw) if rtol else None
            eng.run(t, k)
            otraj = o.run(osw, t, k)
            eng.check()
            gtraj = eng.traj[t:t + k].cpu().numpy()
            rows = _diff_rows(eng, osw, rtol)
            ok = not rows and _gbest_ok(eng, osw, rtol) and _close(gtraj, otraj, rtol)
            compared += 1
            if not ok:
                assert rtol, (f"{name}: bitwise objective {fid} diverged in iterations "
                              f"[{t}, {t + k}): rows {rows[:8]} (any divergence is a failure)")
                # first divergent iteration: replay the chunk step by step from its start
                cur = snap
                for s in range(t, t + k):
                    nxt, found = _classify_iteration(p, fn, seed, cur, s, rtol, "float64")
                    cur = nxt
                    if found:
                        ties.extend(found)
                o_state = cur
                assert _close(o_state.p_f, osw.p_f, 0) and np.array_equal(o_state.sol, osw.sol)
                eng.load(osw)                     # resync the device from the oracle
                with torch.cuda.stream(eng.stream):
                    eng.traj[t:t + k].copy_(torch.as_tensor(otraj))
                assert ties, f"{name}: divergence in [{t}, {t + k}) without a classified near-tie"
            t += k
        traj = eng.traj.cpu().numpy()
    finally:
        eng.close()
    return {"kernel": name, "chunks": compared, "near_ties": ties, "final": float(traj[-1])}


def test_c3_rastrigin_fp64_500_iterations():
    """C3: f5, N=2^20, D=128, 500 iterations, fp64 (BASELINE configs[2])."""
    r = verify("f5", 1 << 20, 128, 500, chunk=50)
    print("C3 fp64", r["kernel"], "near-ties:", r["near_ties"])
    assert r["kernel"].startswith("k_chain")
    assert len(r["near_ties"]) <= 8, r["near_ties"]


def test_c4_rosenbrock_2p24_bitwise():
    """C4: f4, N=2^24, D=64, fp64 -- pure + - *, so every value is bitwise (BASELINE configs[3])."""
    r = verify("f4", 1 << 24, 64, 20, chunk=10, rtol=0.0)
    assert r["kernel"].startswith("k_chain")


def test_c5_ackley_4096_200_iterations():
    """C5: f6, N=65536, D=4096, 200 iterations, fp64 (BASELINE configs[4])."""
    r = verify("f6", 65536, 4096, 200, chunk=50)
    print("C5", r["kernel"], "near-ties:", r["near_ties"])
    assert r["kernel"].startswith("k_rows")
    assert len(r["near_ties"]) <= 8, r["near_ties"]


def test_c3_rastrigin_fp32_fitness_on_identical_inputs():
    """C3 fp32 (BASELINE configs[2]): the run's own states at t = 0, 250, 499.

    From each device state, one more iteration on the device (sol_f kept) and
    on the oracle (the fp32 state widened to fp64): positions must be the
    oracle's rounded to fp32 (selections exact), fitness within 1e-5 of the
    oracle's fitness OF THE SAME fp32 positions, and pBest decisions equal
    except where that fitness is within 1e-5 of p_f (classified near-ties).
    """
    fn = _fn("f5", 128)
    N, niter = 1 << 20, 500
    p = _params(fn, N, niter)
    eng = DeviceEngine(p, fn, 0, dtype="float32")
    o = O.Oracle.from_params(p, "f5", 0, threads=O.max_threads())
    try:
        eng.initialize()
        done = 0
        for t in (0, 250, 499):
            eng.run(done, t - done)
            done = t
            eng.check()
            sw = eng.to_host()                        # fp32 state, widened exactly
            rep = DeviceEngine(p, fn, 0, dtype="float32", keep_sol_f=True)
            try:
                rep.load(sw)
                rep.step(t)
                rep.check()
                x32 = rep.sol.cpu().numpy()
                fd = rep.sol_f.cpu().numpy()
                pf_d = rep.p_f.cpu().numpy()
            finally:
                rep.close()
            osw = copy.deepcopy(sw)
            o.search(osw, t)                          # oracle draws + select on the same state
            assert np.array_equal(x32, osw.sol.astype(np.float32)), f"t={t}: positions"
            fo = O.evaluate("f5", x32.astype(np.float64), threads=O.max_threads())
            rel = np.abs(fd - fo) / np.maximum(np.abs(fo), 1e-300)
            assert rel.max() <= RTOL32, f"t={t}: fp32 fitness rel err {rel.max():.3g}"
            imp_d, imp_o = fd <= sw.p_f, fo <= sw.p_f
            flips = np.flatnonzero(imp_d != imp_o)
            assert np.all(np.abs(fo[flips] - sw.p_f[flips]) <= RTOL32 * np.abs(sw.p_f[flips])), \
                f"t={t}: unclassified pBest flips {flips[:8]}"
            assert np.array_equal(pf_d, np.where(imp_d, fd, sw.p_f)), f"t={t}: p_f update"
            print(f"C3 fp32 t={t}: max rel fitness err {rel.max():.3g}, near-tie flips {flips.size}")
    finally:
        eng.close()
