#!/usr/bin/env python
"""Benchmark of the fused PSSO iteration (BASELINE.json metric) -- one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c3f32|c4|c5|c2]

A "step" is one PSSO iteration (search + evaluate + pBest + gBest) over the
whole synthetic swarm.  Default workload = BASELINE config C3 (Rastrigin,
N = 2^20 particles x Nvar = 128, fp64, reference keyed RNG: results
bit-identical in positions/selections to the reference).  The swarm is the
reference's own synthetic init (uniform in the box from the INIT stream).

Under torchrun (N > 1) every rank owns a 2^20-particle shard (weak scaling,
global N = 2^20 * ranks) and the ranks exchange gBest candidates through one
NCCL all-gather per iteration; time = max over ranks of the device time.

--impl reference times the reference algorithm on the host CPU cores: the C
restatement in oracle/ (kind "port"; the reference itself is Python/numpy and
is not shipped to the GPU box), all host threads, on a bounded sample of the
workload's rows.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-variable updates/s and HBM GB/s vs peak at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "pvu/s"
L2_BYTES = 126 * 1024 * 1024

WORKLOADS = {
    # name: (fid, nsol per rank, nvar, dtype, BASELINE config)
    "c1": ("f1", 100, 30, "float64", "C1 Sphere N=100 Nvar=30 fp64"),
    "c3": ("f5", 1 << 20, 128, "float64", "C3 Rastrigin N=2^20 Nvar=128 fp64"),
    "c3f32": ("f5", 1 << 20, 128, "float32", "C3 Rastrigin N=2^20 Nvar=128 fp32"),
    "c4": ("f4", 1 << 24, 64, "float64", "C4 Rosenbrock N=2^24 Nvar=64 fp64"),
    "c5": ("f6", 65536, 4096, "float64", "C5 Ackley N=65536 Nvar=4096 fp64"),
    "c2": ("f5", 1024, 100, "float64", "C2 Rastrigin N=1024 Nvar=100 fp64"),
    "c2f4": ("f4", 1024, 100, "float64", "C2 Rosenbrock N=1024 Nvar=100 fp64"),
    "c2f6": ("f6", 1024, 100, "float64", "C2 Ackley N=1024 Nvar=100 fp64"),
    "c2f7": ("f7", 1024, 100, "float64", "C2 Griewank N=1024 Nvar=100 fp64"),
    # diagnostics (not BASELINE configs): C3 shape with the cheapest objective
    "c3sphere": ("f1", 1 << 20, 128, "float64", "diagnostic: Sphere N=2^20 Nvar=128 fp64"),
    "c3sphere32": ("f1", 1 << 20, 128, "float32", "diagnostic: Sphere N=2^20 Nvar=128 fp32"),
}


def _traffic(workload, kernel):
    """DRAM bytes per launch of this workload's kernel from the committed ncu capture
    (bench_traffic.json, written by scripts/ncu_summary.py traffic), else None."""
    p = ROOT / "bench_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(workload)
    if not d or d.get("kernel") != kernel:
        return None
    return d["dram_bytes_per_launch"]


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline(fid, nvar, steps_budget_s=12.0, sample_rows=1 << 16, dtype="float64"):
    """Oracle (C restatement, all host threads) on a bounded row sample; pvu/s."""
    from oracle import oracle as O

    threads = O.max_threads()
    lo, hi = {"f1": (-5.12, 5.12), "f5": (-5.12, 5.12), "f4": (-2.048, 2.048),
              "f6": (-32.768, 32.768)}[fid]
    o = O.Oracle(fid, sample_rows, nvar, 0.3, 0.6, 0.8, lo, hi, 0, threads=threads)
    sw = o.initialize()
    o.run(sw, 0, 1)  # warm
    n, t0 = 0, time.perf_counter()
    while True:
        o.run(sw, 1 + n, 1)
        n += 1
        el = time.perf_counter() - t0
        if el >= steps_budget_s or n >= 2000:
            break
    return {"value": sample_rows * nvar * n / el, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample_rows} of the workload's particles x Nvar={nvar}, {n} iterations "
                      f"({el:.1f} s), oracle/psso_oracle.c with {threads} OpenMP threads"}


def run_reference(args, wl):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    fid, nsol, nvar, dtype, desc = WORKLOADS[wl]
    from oracle import oracle as O

    threads = O.max_threads()
    sample = min(nsol, 1 << 16) if nvar <= 256 else min(nsol, 1 << 11)
    lo, hi = {"f1": (-5.12, 5.12), "f5": (-5.12, 5.12), "f4": (-2.048, 2.048),
              "f6": (-32.768, 32.768)}[fid]
    o = O.Oracle(fid, sample, nvar, 0.3, 0.6, 0.8, lo, hi, 0, threads=threads)
    sw = o.initialize()
    o.run(sw, 0, args.warmup)
    t0 = time.perf_counter()
    o.run(sw, args.warmup, args.steps)
    el = time.perf_counter() - t0
    value = sample * nvar * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference INIT-stream swarm)",
        "config": {"workload": desc + f" (host sample: {sample} particles)", "fn": fid,
                   "nsol_sample": sample, "nvar": nvar, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} particles x Nvar={nvar} per step, oracle/psso_oracle.c "
                                   f"(C restatement of the reference, numpy order) with {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, wl):
    import torch

    ws, rank, local = _dist()
    fid, nsol_rank, nvar, dtype, desc = WORKLOADS[wl]
    if ws > 1:
        import torch.distributed as dist

        # PSSO_BENCH_BACKEND=gloo (tests only): ranks may share a GPU, so the
        # multi-rank path can be exercised on a one-GPU box; runs use NCCL
        backend = os.environ.get("PSSO_BENCH_BACKEND", "nccl")
        local = local % torch.cuda.device_count() if backend == "gloo" else local
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    import paper_2110_01470_b200 as psso
    from paper_2110_01470_b200 import _lib
    from paper_2110_01470_b200.engine import DeviceEngine, make_config
    from paper_2110_01470_b200.sharded import (P2PExchange, ProcessGroupExchange, ShardedDriver,
                                               partition)

    fn = psso.make_function(fid, nvar)
    nsol = nsol_rank * ws
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=args.warmup + args.steps + 1)
    lo, hi = partition(nsol, ws)[rank]
    eng = DeviceEngine(p, fn, 0, dtype=dtype, rng=args.rng, row_lo=lo, row_hi=hi)
    L = _lib.load()
    es = 8 if dtype == "float64" else 4
    if ws > 1:
        ex = (P2PExchange([eng], distributed=True) if args.exchange == "p2p"
              else ProcessGroupExchange())
        drv = ShardedDriver([eng], ex, ws)
        with torch.cuda.stream(eng.stream):
            drv.initialize()
            drv.run(0, args.warmup)
    else:
        eng.initialize()
        eng.run(0, args.warmup)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()

    # ---- timed region: K iterations, CUDA events on the engine's stream, kernel
    # events around every fused tile launch (roofline), clocks sampled live
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    L.psso_profile(eng.ctx, 1)
    l0 = eng.launches
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record(eng.stream)
    if ws > 1:
        with torch.cuda.stream(eng.stream):
            drv.run(args.warmup, args.steps)
    else:
        eng.run(args.warmup, args.steps)
    stop.record(eng.stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = eng.launches - l0
    kname = L.psso_kernel_name(eng.ctx).decode()
    kms, kn = ctypes.c_double(), ctypes.c_int64()
    _lib.check(L.psso_profile_read(eng.ctx, ctypes.byref(kms), ctypes.byref(kn)))
    L.psso_profile(eng.ctx, 0)
    clocks = sampler.stop() if sampler else None
    eng.check()
    ms = start.elapsed_time(stop)
    if ws > 1:
        t = torch.tensor([ms, kms.value / max(kn.value, 1)], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_ms = float(t[0]), float(t[1])
    else:
        kern_ms = kms.value / max(kn.value, 1)  # per iteration
    if ws > 1 and args.exchange == "p2p":
        dist.barrier()  # every rank finished reading peer buffers before unmapping
        ex.close()
    eng.close()
    del eng
    torch.cuda.empty_cache()

    pvu_step = nsol * nvar
    value = pvu_step * args.steps / (ms * 1e-3)
    peak, peak_src = _peaks()
    rows_rank = hi - lo
    alg_bytes = 3 * es * rows_rank * nvar  # read X, read P, write X per pvu
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9

    # ---- e2e through the C ABI with host buffers (psso_solve = run_parallel)
    e2e = None
    if rank == 0:
        cfg = make_config(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min,
                                         var_max=fn.var_max, nsol=nsol_rank, nvar=nvar,
                                         niter=args.steps), fn, 0, dtype=dtype, rng=args.rng)
        import numpy as np

        traj = np.empty(args.steps)
        best = np.empty(nvar, dtype=np.float64 if dtype == "float64" else np.float32)
        bf, wall = ctypes.c_double(), ctypes.c_double()
        times = []
        for rep in range(4):  # first call warms module load / allocator; best of the other 3
            t0 = time.perf_counter()
            _lib.check(L.psso_solve(ctypes.byref(cfg), args.steps, traj.ctypes.data,
                                    best.ctypes.data, ctypes.byref(bf), ctypes.byref(wall)))
            times.append(time.perf_counter() - t0)
        el = min(times[1:])
        e2e = {"value": nsol_rank * nvar * args.steps / el, "unit": UNIT,
               "h2d_bytes_per_step": ctypes.sizeof(cfg) / args.steps,
               "d2h_bytes_per_step": (8 * args.steps + best.nbytes + 8) / args.steps,
               "note": "psso_solve(config) -> host trajectory/best position; includes device "
                       "alloc, init, all iterations and copy-back; the reference API takes no "
                       "array inputs (the swarm is generated from the seed); best of 3 calls "
                       "after a warm-up call (host-side API latency on the box varies; "
                       "PSSO_SOLVE_TRACE=1 prints the phases)",
               "calls_s": [round(x, 4) for x in times]}
        if ws > 1:
            e2e["note"] += "; measured on rank 0's shard size (single GPU)"

    if rank != 0:
        dist.destroy_process_group()
        return
    cpu = cpu_baseline(fid, nvar) if ws == 1 and not args.no_cpu else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if dtype == "float64" else "f32",
        "data": "synthetic (reference INIT-stream swarm, seed 0)",
        "config": {"workload": desc + (f" per rank, global N={nsol}" if ws > 1 else ""),
                   "fn": fid, "nsol": nsol, "nvar": nvar, "rng": args.rng,
                   "evals_per_s": nsol * args.steps / (ms * 1e-3),
                   "hbm_gbs_per_gpu": 3 * es * nsol * nvar * args.steps / (ms * 1e-3) / 1e9 / ws,
                   "l2": f"inputs larger than L2: X+P = {2 * es * rows_rank * nvar / 2**30:.2f} GiB "
                         f"per GPU vs 126 MB L2",
                   "parallelism": f"particle shards x{ws}" + (
                       (" + NCCL all-gather of gBest candidates per iteration" if args.exchange == "collective"
                        else " + device-initiated P2P stores of gBest candidates per iteration")
                       if ws > 1 else "")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(wl, kname), "peak_source": peak_src,
                     "kernel": kname, "kernel_ms_per_iteration": kern_ms,
                     "alg_bytes_per_launch": alg_bytes, "alg_bytes_per_pvu": 3 * es,
                     "note": ("per iteration: one fused launch (streaming path)" if "k_swarm" not in kname
                              else "whole-run kernel: all timed iterations in one launch; L2/SMEM-"
                                   "resident swarm, so the HBM roofline does not bind")},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--rng", default="reference", choices=["reference", "philox"])
    ap.add_argument("--exchange", default="collective", choices=["collective", "p2p"],
                    help="N > 1: gBest records by NCCL all-gather or device-initiated P2P stores")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (diagnostics)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args, args.workload)
    else:
        run_ours(args, args.workload)


if __name__ == "__main__":
    main()
