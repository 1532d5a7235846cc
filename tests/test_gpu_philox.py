"""Benchmark mode (on-device Philox4x32-10): the stream is pinned to the Random123
known answers through the oracle's Philox (tests/test_oracle_golden.py), and the
final-fitness distribution over 30 seeds matches the reference's (reference RNG,
the oracle) on the C2 suite -- the north star's benchmark-mode criterion, with
the reference harness's protocol (harness.py:217-263: seeds 0..29) and
statistics (stats.py:129-151: mean within 10 %, Kruskal-Wallis and Welch t-test
p > 0.01).

Keying (psso_device.cuh philox_pair): coordinates {16a+b, 16a+b+8} of particle
i share one call, counter (pair, i_lo, i_hi, t) -- t = 0xFFFFFFFF for the
INIT draw -- and key = seed; half h = (j >> 3) & 1 takes word h (branch) and
word 2 + h (fresh), or words 2h, 2h+1 as one 64-bit INIT draw.
"""

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

M32 = 0xFFFFFFFF


def _words(seed, i, j, t):
    pair = ((j >> 4) << 3) | (j & 7)
    return O.philox([pair, i & M32, (i >> 32) & M32, t & M32], [seed & M32, (seed >> 32) & M32])


def _k32(c):
    return min(1 << 32, max(0, math.ceil(c * 4294967296.0)))


@pytest.mark.parametrize("fid,nsol,nvar", [("f1", 6, 40), ("f5", 5, 64), ("f4", 4, 100),
                                           ("f6", 2, 512)])
def test_philox_stream_matches_random123_keying(fid, nsol, nvar):
    fn = psso.make_function(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=3)
    seed = (1 << 40) + 12345
    span = p.var_max - p.var_min
    eng = DeviceEngine(p, fn, seed, rng="philox")
    try:
        eng.initialize()
        x0 = eng.sol.cpu().numpy().copy()
        for i in range(nsol):
            for j in range(nvar):
                w = _words(seed, i, j, M32)
                h = (j >> 3) & 1
                u = ((((w[2 * h] << 32) | w[2 * h + 1]) >> 11)) * 2.0 ** -53
                assert x0[i, j] == p.var_min + span * u, (i, j)
        sw = eng.to_host()
        eng.step(0)
        x1 = eng.sol.cpu().numpy()
    finally:
        eng.close()
    K = [_k32(p.cw), _k32(p.cp), _k32(p.cg)]
    for i in range(nsol):
        for j in range(nvar):
            w = _words(seed, i, j, 0)
            h = (j >> 3) & 1
            kb, raw = w[h], w[2 + h] * 2.0 ** -32
            want = (sw.sol[i, j] if kb < K[0] else sw.pbests[i, j] if kb < K[1]
                    else sw.gbest[j] if kb < K[2] else p.var_min + span * raw)
            assert x1[i, j] == want, (i, j)


def _oracle_final(args):
    fid, nsol, nvar, niter, seed = args[:5]
    sequential = len(args) > 5 and args[5]
    fn_box = {"f4": (-2.048, 2.048), "f5": (-5.12, 5.12), "f6": (-32.768, 32.768),
              "f7": (-600.0, 600.0)}[fid]
    o = O.Oracle(fid, nsol, nvar, 0.3, 0.6, 0.8, *fn_box, seed, threads=1)
    sw = o.initialize()
    return (o.run_sequential if sequential else o.run)(sw, 0, niter)[-1]


@pytest.fixture(scope="module")
def reference_finals():
    """The reference's final fitness (oracle, reference keyed RNG) for seeds 0..29 of the C2 suite."""
    jobs = [(fid, 1024, 100, 1000, s) for fid in ("f5", "f4", "f6", "f7") for s in range(30)]
    with ThreadPoolExecutor(max_workers=O.max_threads()) as ex:  # ctypes releases the GIL; no fork of a CUDA process
        out = list(ex.map(_oracle_final, jobs))
    return {fid: np.array(out[k * 30:(k + 1) * 30]) for k, fid in enumerate(("f5", "f4", "f6", "f7"))}


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("fid", ["f5", "f4", "f6", "f7"])
def test_philox_c2_suite_distribution_matches_reference(fid, dtype, reference_finals):
    from scipy import stats

    fn = psso.make_function(fid, 100)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=1024, nvar=100, niter=1000)
    recs = psso.run_parallel_batch(p, fn, list(range(30)), dtype=dtype, rng="philox")  # one launch
    gpu = np.array([r.best_fitness for r in recs])
    ref = reference_finals[fid]
    assert np.isfinite(gpu).all()
    assert abs(gpu.mean() - ref.mean()) <= 0.10 * abs(ref.mean()), (gpu.mean(), ref.mean())
    assert stats.kruskal(gpu, ref).pvalue > 0.01, (gpu, ref)
    assert stats.ttest_ind(gpu, ref, equal_var=False).pvalue > 0.01, (gpu, ref)


@pytest.fixture(scope="module")
def reference_finals_sequential():
    """The same for the reference's sequential schedule (core.py:213-258)."""
    jobs = [(fid, 1024, 100, 1000, s, True) for fid in ("f5", "f4", "f6", "f7") for s in range(30)]
    with ThreadPoolExecutor(max_workers=O.max_threads()) as ex:  # ctypes releases the GIL
        out = list(ex.map(_oracle_final, jobs))
    return {fid: np.array(out[k * 30:(k + 1) * 30]) for k, fid in enumerate(("f5", "f4", "f6", "f7"))}


@pytest.mark.parametrize("fid", ["f5", "f4", "f6", "f7"])
def test_philox_sequential_schedule_distribution_matches_reference(fid, reference_finals_sequential):
    """Benchmark mode for the other schedule: run_sequential_batch (one k_seq
    launch for 30 seeds) in Philox mode against the reference sequential
    schedule's final fitness (oracle, reference RNG), same criteria."""
    from scipy import stats

    fn = psso.make_function(fid, 100)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=1024, nvar=100, niter=1000)
    recs = psso.run_sequential_batch(p, fn, list(range(30)), rng="philox")
    gpu = np.array([r.best_fitness for r in recs])
    ref = reference_finals_sequential[fid]
    assert np.isfinite(gpu).all()
    assert abs(gpu.mean() - ref.mean()) <= 0.10 * abs(ref.mean()), (gpu.mean(), ref.mean())
    assert stats.kruskal(gpu, ref).pvalue > 0.01, (gpu, ref)
    assert stats.ttest_ind(gpu, ref, equal_var=False).pvalue > 0.01, (gpu, ref)
