"""Per-iteration cost of the multi-GPU exchange path, measured on ONE GPU.

    torchrun --nproc-per-node 1 --master-addr 127.0.0.1 scripts/exchange_overhead.py

For each per-rank shard shape, times K iterations of (a) the plain
single-context loop and (b) the sharded loop -- psso_step_local, NCCL
all_gather of the candidate records, psso_apply_candidates -- with world size
1.  (b) - (a) is the fixed per-iteration cost of the exchange path that an
N-GPU run pays on top of its shard's compute (the NVLink transfer of
R * (16 + D * 8) bytes is negligible next to it).
"""
import os
import sys
import json

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_01470_b200 as psso  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402
from paper_2110_01470_b200.sharded import ProcessGroupExchange, ShardedDriver  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
K = 50
for fid, rows, D, label in (("f4", 1 << 21, 64, "C4 share of 8 GPUs (2^24/8 rows)"),
                            ("f4", 1 << 24, 64, "C4 full per GPU (weak scaling)"),
                            ("f6", 8192, 4096, "C5 share of 8 GPUs (65536/8 rows)"),
                            ("f5", 1 << 20, 128, "C3 per rank (bench --gpus N)")):
    fn = psso.make_function(fid, D)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=rows, nvar=D, niter=K + 10)
    res = {}
    for mode in ("plain", "sharded"):
        eng = DeviceEngine(p, fn, 0, keep_sol_f=False, row_lo=0, row_hi=rows)
        drv = ShardedDriver([eng], ProcessGroupExchange(), 1) if mode == "sharded" else None
        with torch.cuda.stream(eng.stream):
            (drv.initialize() if drv else eng.initialize())
            (drv.run(0, 5) if drv else eng.run(0, 5))
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(eng.stream)
            (drv.run(5, K) if drv else eng.run(5, K))
            b.record(eng.stream)
        torch.cuda.synchronize()
        res[mode] = a.elapsed_time(b) / K
        eng.close()
    print(json.dumps({"shape": label, "rows": rows, "nvar": D,
                      "plain_ms": res["plain"], "sharded_ms": res["sharded"],
                      "exchange_overhead_us": 1e3 * (res["sharded"] - res["plain"])}), flush=True)
dist.destroy_process_group()
