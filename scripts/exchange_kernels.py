"""Per-kernel view of one exchange iteration at world size 1 (for ncu's launch list).

    ncu --metrics gpu__time_duration.sum --csv --log-file k.csv \
        torchrun --nproc-per-node 1 --master-addr 127.0.0.1 scripts/exchange_kernels.py
    python scripts/ncu_summary.py launches k.csv

Runs 32 iterations of the NCCL graph loop and of the P2P device loop (direct
launches: psso_profile on, so every kernel is its own launch) at the C3 shard
shape of 8 GPUs (2^17 x 128).
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_01470_b200 as psso  # noqa: E402
from paper_2110_01470_b200 import _lib  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402
from paper_2110_01470_b200.sharded import NcclExchange, P2PExchange, ShardedDriver  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
L = _lib.load()
fn = psso.make_function("f5", 128)
p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                   nsol=1 << 17, nvar=128, niter=64)
for mode in ("nccl", "p2p"):
    eng = DeviceEngine(p, fn, 0)
    ex = NcclExchange(eng) if mode == "nccl" else P2PExchange([eng], distributed=True)
    drv = ShardedDriver([eng], ex, 1)
    with torch.cuda.stream(eng.stream):
        drv.initialize()
        L.psso_profile(eng.ctx, 1)  # direct launches: one ncu row per kernel
        drv.run(0, 32)
        L.psso_profile(eng.ctx, 0)
    torch.cuda.synchronize()
    if mode == "p2p":
        ex.close()
    eng.close()
    print("done", mode, flush=True)
dist.destroy_process_group()
