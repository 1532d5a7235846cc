"""Per-iteration cost of the multi-GPU exchange paths, measured on ONE GPU.

    torchrun --nproc-per-node 1 --master-addr 127.0.0.1 scripts/exchange_overhead.py

For each per-rank shard shape, times K iterations of (a) the plain
single-context loop (psso_run: graph-replayed kernel + k_gbest), (b) "nccl":
the default sharded loop -- fused kernel, candidate record, ncclAllGather,
apply, all replayed from CUDA graphs (psso_run_sharded), (c) "collective":
the host-driven loop over torch.distributed (psso_step_local, all_gather,
psso_apply_candidates), (d) "p2p": the device-initiated exchange as a
graph-replayed device loop (psso_run_p2p), each with world size 1.  The
modes are interleaved over REPS repetitions and the median per-iteration
time is reported, so clock / power-cap drift between runs does not show up
as an exchange cost.  (x) - (a) is the fixed per-iteration cost an N-GPU run
pays on top of its shard's compute (the NVLink transfer of R * (32 + D * 8)
bytes is negligible next to it).
"""
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_01470_b200 as psso  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402
from paper_2110_01470_b200.sharded import (NcclExchange, P2PExchange, ProcessGroupExchange,  # noqa: E402
                                           ShardedDriver)

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
K = int(os.environ.get("K", "64"))
REPS = int(os.environ.get("REPS", "5"))
MODES = ("plain", "nccl", "collective", "p2p")
for fid, rows, D, label in (("f4", 1 << 21, 64, "C4 share of 8 GPUs (2^24/8 rows)"),
                            ("f6", 8192, 4096, "C5 share of 8 GPUs (65536/8 rows)"),
                            ("f5", 1 << 17, 128, "C3 share of 8 GPUs (2^20/8 rows)"),
                            ("f4", 1 << 24, 64, "C4 full per GPU")):
    fn = psso.make_function(fid, D)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=rows, nvar=D, niter=K + 10)
    res = {m: [] for m in MODES}
    for rep in range(REPS):
        for mode in MODES:
            eng = DeviceEngine(p, fn, 0, keep_sol_f=False, row_lo=0, row_hi=rows)
            ex = {"nccl": lambda: NcclExchange(eng), "collective": ProcessGroupExchange,
                  "p2p": lambda: P2PExchange([eng], distributed=True)}.get(mode, lambda: None)()
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
            res[mode].append(a.elapsed_time(b) / K)
            if mode == "p2p":
                ex.close()
            eng.close()
    med = {m: statistics.median(v) for m, v in res.items()}
    out = {"shape": label, "rows": rows, "nvar": D, "iterations": K, "reps": REPS}
    out.update({f"{m}_ms": med[m] for m in MODES})
    out.update({f"{m}_overhead_us": 1e3 * (med[m] - med["plain"]) for m in MODES[1:]})
    out["spread_plain_us"] = 1e3 * (max(res["plain"]) - min(res["plain"]))
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
