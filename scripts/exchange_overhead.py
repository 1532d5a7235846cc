"""Per-iteration cost of the multi-GPU exchange path, measured on ONE GPU.

    torchrun --nproc-per-node 1 --master-addr 127.0.0.1 scripts/exchange_overhead.py

For each per-rank shard shape, times K iterations of (a) the plain
single-context loop, (b) the sharded loop -- psso_step_local, NCCL
all_gather of the candidate records, psso_apply_candidates -- and (c) the
sharded loop with the device-initiated P2P exchange (psso_publish_p2p /
psso_apply_p2p), with world size 1.  (b) - (a) and (c) - (a) are the fixed
per-iteration costs of the exchange paths that an N-GPU run pays on top of
its shard's compute (the NVLink transfer of R * (16 + D * 8) bytes is
negligible next to them).
"""
import os
import sys
import json

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_01470_b200 as psso  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402
from paper_2110_01470_b200.sharded import P2PExchange, ProcessGroupExchange, ShardedDriver  # noqa: E402

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
    for mode in ("plain", "sharded", "p2p"):
        eng = DeviceEngine(p, fn, 0, keep_sol_f=False, row_lo=0, row_hi=rows)
        ex = None
        if mode == "sharded":
            ex = ProcessGroupExchange()
        elif mode == "p2p":
            ex = P2PExchange([eng], distributed=True)
        drv = ShardedDriver([eng], ex, 1) if ex is not None else None
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
        if mode == "p2p":
            ex.close()
        eng.close()
    print(json.dumps({"shape": label, "rows": rows, "nvar": D,
                      "plain_ms": res["plain"], "sharded_ms": res["sharded"], "p2p_ms": res["p2p"],
                      "exchange_overhead_us": 1e3 * (res["sharded"] - res["plain"]),
                      "p2p_overhead_us": 1e3 * (res["p2p"] - res["plain"])}), flush=True)
dist.destroy_process_group()
