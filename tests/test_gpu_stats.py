"""Per-iteration device statistics (psso_iteration_stats): the improved-row count the
roofline's rho term uses (pBest write-back, parallel.py:108-112) equals the
oracle's count of `sol_f <= p_f` rows, iteration by iteration, and every
iteration of a graph-replayed run is timed on the device."""

import ctypes

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


def _stats(eng, t0, n):
    L = _lib.load()
    ms, imp, cnt = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(L.psso_iteration_stats(eng.ctx, t0, n, ctypes.byref(ms), ctypes.byref(imp),
                                      ctypes.byref(cnt)), eng.ctx)
    return ms.value, imp.value, cnt.value


@pytest.mark.parametrize("fid,nsol,nvar,niter,dtype,kernel", [
    ("f4", 30000, 64, 40, "float64", "k_chain"),
    ("f5", 9000, 128, 35, "float32", "k_chain"),
    ("f6", 300, 4096, 20, "float64", "k_rows"),
])
def test_improved_rows_match_oracle_and_every_iteration_is_timed(fid, nsol, nvar, niter, dtype,
                                                                 kernel):
    fn = psso.make_function(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=niter)
    eng = DeviceEngine(p, fn, 5, dtype=dtype)
    try:
        assert _lib.load().psso_kernel_name(eng.ctx).decode().startswith(kernel)
        eng.initialize()
        eng.step(0)                     # direct launch
        eng.run(1, niter - 1)           # graph replays (+ direct tail)
        eng.check()
        per_t = [_stats(eng, t, 1) for t in range(niter)]
        total = _stats(eng, 0, niter)
    finally:
        eng.close()
    assert all(c == 1 and ms > 0 for ms, _, c in per_t)
    assert total[2] == niter and total[1] == sum(i for _, i, _ in per_t)
    if dtype == "float64":  # improved rows of the reference run (same inputs, same decisions)
        o = O.Oracle.from_params(p, fid, 5, threads=O.max_threads())
        sw = o.initialize()
        for t in range(niter):
            pf_old = sw.p_f.copy()
            o.step(sw, t)
            assert per_t[t][1] == int(np.count_nonzero(sw.sol_f <= pf_old)), t
    rho0 = per_t[0][1] / nsol
    assert 0.2 < rho0 < 0.8  # rho ~ 0.5 in the first iterations
