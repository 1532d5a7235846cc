"""Whole-run kernel (k_swarm) vs streaming kernels per iteration, by swarm size (diagnostic).

    python scripts/swarm_crossover.py            (on a GPU box)
"""
import os
import sys
import json

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_01470_b200 as psso  # noqa: E402
from paper_2110_01470_b200 import _lib  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

torch.cuda.set_device(0)
L = _lib.load()
K = 200
for fid, D in (("f5", 128), ("f4", 64), ("f5", 100)):
    for N in (1024, 4096, 8192, 16384, 32768):
        res = {}
        for mode in ("swarm", "stream"):
            if mode == "stream":
                os.environ["PSSO_NO_SWARM"] = "1"
            else:
                os.environ.pop("PSSO_NO_SWARM", None)
            fn = psso.make_function(fid, D)
            p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                               nsol=N, nvar=D, niter=K + 20)
            eng = DeviceEngine(p, fn, 0)
            name = L.psso_kernel_name(eng.ctx).decode()
            eng.initialize()
            eng.run(0, 20)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(eng.stream)
            eng.run(20, K)
            b.record(eng.stream)
            torch.cuda.synchronize()
            res[mode] = (a.elapsed_time(b) * 1e3 / K, name)
            eng.close()
        print(json.dumps({"fn": fid, "nsol": N, "nvar": D, "elems": N * D,
                          "swarm_us": round(res["swarm"][0], 2), "stream_us": round(res["stream"][0], 2),
                          "swarm_kernel": res["swarm"][1], "stream_kernel": res["stream"][1]}), flush=True)
