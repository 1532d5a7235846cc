"""Small runs of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_01470_b200 as psso  # noqa: E402
from paper_2110_01470_b200 import _lib  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

CASES = [("f5", 1 << 16, 128, 2), ("f4", 70000, 64, 2), ("f5", 50000, 100, 2),  # k_chain
         ("f5", 1 << 14, 128, 3), ("f4", 4099, 64, 3), ("f6", 66, 4096, 2), ("f2", 130, 1024, 2),
         ("f5", 300, 300, 2), ("f9", 200, 301, 2), ("f5", 1024, 100, 4), ("f7", 256, 100, 3),
         ("f1", 100, 30, 5)]
torch.cuda.set_device(0)
L = _lib.load()
for fid, n, d, it in CASES:
    fn = psso.make_function(fid, d)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=n, nvar=d, niter=it)
    eng = DeviceEngine(p, fn, 1, keep_sol_f=True)
    name = L.psso_kernel_name(eng.ctx).decode()
    eng.initialize()
    eng.run(0, it)
    eng.check()
    torch.cuda.synchronize()
    eng.close()
    print("ok", name, flush=True)
recs = psso.run_parallel_batch(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-5.12, var_max=5.12,
                                              nsol=64, nvar=16, niter=5),
                               psso.make_function("f5", 16), [1, 2, 3])
print("ok batch", len(recs), flush=True)
recs = psso.run_parallel_batch(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-5.12, var_max=5.12,
                                              nsol=4096, nvar=128, niter=3),
                               psso.make_function("f5", 128), [1, 2, 3])
print("ok batch (global-memory exchange)", len(recs), flush=True)
from paper_2110_01470_b200.sharded import run_virtual_shards  # noqa: E402

fn = psso.make_function("f4", 64)
rec = run_virtual_shards(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min,
                                        var_max=fn.var_max, nsol=3000, nvar=64, niter=4),
                         fn, 2, 3, exchange="p2p")
print("ok virtual shards, P2P exchange", flush=True)
for fid, n, d, it in (("f1", 100, 30, 20), ("f7", 70, 20, 10), ("f5", 300, 128, 5)):  # k_seq
    fn = psso.make_function(fid, d)
    rec = psso.run_sequential(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min,
                                             var_max=fn.var_max, nsol=n, nvar=d, niter=it), fn, 2)
    print("ok sequential", fid, n, d, flush=True)
for fid, n, d, it in (("f5", 40, 300, 3), ("f6", 20, 4096, 2)):  # long-row sequential pass loop
    fn = psso.make_function(fid, d)
    rec = psso.run_sequential(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min,
                                             var_max=fn.var_max, nsol=n, nvar=d, niter=it), fn, 2)
    print("ok sequential (device pass loop)", fid, n, d, flush=True)
for fid, n, d, dt in (("f5", 5000, 128, "float32"), ("f6", 40, 4096, "float64")):  # Philox mode
    fn = psso.make_function(fid, d)
    rec = psso.run_parallel(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min,
                                           var_max=fn.var_max, nsol=n, nvar=d, niter=3), fn, 2,
                            dtype=dt, rng="philox")
    print("ok philox", fid, dt, flush=True)
# library NCCL communicator + graph-replayed sharded loop, and the P2P device loop (world size 1)
import torch.distributed as dist  # noqa: E402

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ.get("SAN_PORT", "29561"), RANK="0",
                  WORLD_SIZE="1")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_2110_01470_b200.sharded import run_parallel_distributed  # noqa: E402

fn = psso.make_function("f4", 64)
p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max, nsol=3000,
                   nvar=64, niter=20)
for ex in ("nccl", "p2p"):
    rec = run_parallel_distributed(p, fn, 2, exchange=ex)
    print("ok distributed", ex, flush=True)
dist.destroy_process_group()
