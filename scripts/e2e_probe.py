"""Where does psso_solve's end-to-end time go? (diagnostic)"""
import ctypes, time, sys
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2110_01470_b200 as psso
from paper_2110_01470_b200 import _lib
from paper_2110_01470_b200.engine import make_config

L = _lib.load()
torch.cuda.init()
fn = psso.make_function("f5", 128)
for steps in (1, 1, 50, 500, 500):
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max, nsol=1 << 20, nvar=128, niter=steps)
    cfg = make_config(p, fn, 0)
    traj = np.empty(steps); best = np.empty(128); bf, wall = ctypes.c_double(), ctypes.c_double()
    t0 = time.perf_counter()
    rc = L.psso_solve(ctypes.byref(cfg), steps, traj.ctypes.data, best.ctypes.data, ctypes.byref(bf), ctypes.byref(wall))
    el = time.perf_counter() - t0
    print(f"steps={steps} rc={rc} wall(host)={el*1e3:.1f} ms  loop(device)={wall.value*1e3:.1f} ms  overhead={el*1e3 - wall.value*1e3:.1f} ms", flush=True)
