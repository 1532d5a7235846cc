"""Small repro for the fused kernel with several tiles per CTA (stage refills)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2110_01470_b200 as psso
from paper_2110_01470_b200.engine import DeviceEngine
from oracle import oracle as O

fid, N, D, it = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
fn = psso.make_function(fid, D)
p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max, nsol=N, nvar=D, niter=it)
eng = DeviceEngine(p, fn, 0, keep_sol_f=True)
eng.initialize()
for t in range(it):
    eng.step(t)
    eng.synchronize()
    print("step", t, "ok", flush=True)
eng.check()
sw = eng.to_host()
o = O.Oracle.from_params(p, fid, 0, threads=O.max_threads())
osw = o.initialize(); o.run(osw, 0, it)
print("sol equal", np.array_equal(sw.sol, osw.sol), "pbests equal", np.array_equal(sw.pbests, osw.pbests))
