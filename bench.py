#!/usr/bin/env python
"""Benchmark of the fused PSSO iteration (BASELINE.json metric) -- one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c3|c3f32|c5|c2|...] [--scaling strong|weak]
                    [--exchange nccl|collective|p2p] [--rng reference|philox]

A "step" is one PSSO iteration (search + evaluate + pBest + gBest) over the
whole synthetic swarm.  Default workload = BASELINE config C4 (Rosenbrock,
N = 2^24 particles x Nvar = 64, fp64, reference keyed RNG: positions,
selections and fitness bit-identical to the reference), the config BASELINE
quotes at 1/2/4/8 GPUs.  The swarm is the reference's own synthetic init
(uniform in the box from the INIT stream).

--gpus N > 1: one rank per GPU.  Without torchrun's WORLD_SIZE in the
environment bench.py launches itself under torch.distributed.run with N ranks.
Rank r owns the contiguous rows of the reference partition (parallel.py:147-
149); per iteration the ranks exchange gBest candidate records -- by default
through the library's own NCCL communicator, kernels and all-gather replayed
from CUDA graphs (psso_run_sharded).  --scaling strong (default) keeps the
workload's global N fixed (C4: 2^24 rows / N per GPU); weak gives every rank
the workload's N.  Time = max over ranks of the device time.

--impl reference times the reference algorithm on the host CPU cores: the C
restatement in oracle/ (kind "port"; the reference itself is Python/numpy and
is not shipped to the GPU box), all host threads, on the FULL workload when
it fits in host memory (else a row sample, stated in the line).
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

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
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
        import datetime

        for line in self.proc.stdout:  # (nvidia-smi's own sample time, the sample)
            ts, _, rest = line.strip().partition(",")
            try:
                when = datetime.datetime.strptime(ts.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                when = None
            self.lines.append((when, rest))

    def mark(self, begin: bool):
        """Bracket the timed region (host wall clock, after the device syncs)."""
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

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
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        inside = [ln for ts, ln in self.lines
                  if ts is not None and t0 is not None and t1 is not None and t0 <= ts <= t1]
        # samples taken during the timed region; a region shorter than the sampling
        # period keeps the samples of the whole sampling window (stated in "window")
        window = "timed region" if inside else "timed region + 0.3 s lead-in + kernel-timing pass"
        for ln in inside or [ln for _, ln in self.lines]:
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
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


BOXES = {"f1": (-5.12, 5.12), "f5": (-5.12, 5.12), "f4": (-2.048, 2.048), "f6": (-32.768, 32.768),
         "f7": (-600.0, 600.0)}


def _host_rows(nsol, nvar, want_full=True):
    """Rows the host oracle can hold: the full workload when X, P (fp64) and the
    oracle's temporaries fit in half the available host memory, else a sample."""
    need = nsol * nvar * 8 * 2 + nsol * 8 * 4
    avail = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                avail = int(ln.split()[1]) * 1024
    except OSError:
        pass
    if want_full and (avail is None or need <= avail // 2):
        return nsol
    per_row = nvar * 8 * 2 + 32
    return max(1024, min(nsol, (avail // 2) // per_row if avail else 1 << 16))


def cpu_baseline(fid, nsol, nvar, budget_s=12.0):
    """Oracle (C restatement, all host threads) on the workload's own rows for ~budget_s; pvu/s."""
    from oracle import oracle as O

    threads = O.max_threads()
    rows = _host_rows(nsol, nvar)
    lo, hi = BOXES[fid]
    o = O.Oracle(fid, rows, nvar, 0.3, 0.6, 0.8, lo, hi, 0, threads=threads)
    sw = o.initialize()
    n, t0 = 0, time.perf_counter()
    while True:
        o.run(sw, n, 1)
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s or n >= 2000:
            break
    what = "all" if rows == nsol else f"{rows} of the"
    return {"value": rows * nvar * n / el, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{what} {nsol} particles x Nvar={nvar}, {n} iterations ({el:.1f} s), "
                      f"oracle/psso_oracle.c with {threads} OpenMP threads"}


def _global_nsol(args, wl, ws):
    fid, nsol, nvar, dtype, desc = WORKLOADS[wl]
    return nsol * ws if args.scaling == "weak" else nsol


def run_reference(args, wl):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    fid, _, nvar, dtype, desc = WORKLOADS[wl]
    nsol = _global_nsol(args, wl, ws)
    from oracle import oracle as O

    threads = O.max_threads()
    rows = _host_rows(nsol, nvar)
    lo, hi = BOXES[fid]
    o = O.Oracle(fid, rows, nvar, 0.3, 0.6, 0.8, lo, hi, 0, threads=threads)
    sw = o.initialize()
    o.run(sw, 0, args.warmup)
    t0 = time.perf_counter()
    o.run(sw, args.warmup, args.steps)
    el = time.perf_counter() - t0
    value = rows * nvar * args.steps / el
    full = rows == nsol
    what = "the full workload" if full else f"a sample of {rows} of the {nsol} particles"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference INIT-stream swarm, seed 0)",
        "config": {"workload": desc + ("" if full else f" (host sample: {rows} particles)"),
                   "fn": fid, "nsol": nsol, "nsol_host": rows, "nvar": nvar, "same_config": full,
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{what} x Nvar={nvar} per step, oracle/psso_oracle.c (C "
                                   f"restatement of the reference, numpy order) with {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _max_over_ranks(vals, ws):
    import torch.distributed as dist

    if not dist.is_initialized():
        return vals
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def _sum_over_ranks(v, ws):
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return v
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.cpu()[0])


def run_ours(args, wl):
    import torch

    ws, rank, local = _dist()
    fid, _, nvar, dtype, desc = WORKLOADS[wl]
    dist = None
    sharded = ws > 1 or args.force_sharded
    if sharded:
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
    from paper_2110_01470_b200.sharded import (NcclExchange, P2PExchange, ProcessGroupExchange,
                                               ShardedDriver, partition, run_parallel_distributed)

    fn = psso.make_function(fid, nvar)
    nsol = _global_nsol(args, wl, ws)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                       nsol=nsol, nvar=nvar, niter=args.warmup + 2 * args.steps + 1)
    lo, hi = partition(nsol, ws)[rank]
    eng = DeviceEngine(p, fn, 0, dtype=dtype, rng=args.rng, row_lo=lo, row_hi=hi)
    L = _lib.load()
    es = 8 if dtype == "float64" else 4
    drv = ex = None
    if sharded:
        if args.exchange == "nccl":
            try:
                ex = NcclExchange(eng)
            except Exception as e:  # e.g. no loadable libnccl: every rank falls back alike
                print(f"bench: library NCCL communicator unavailable ({e}); using the "
                      "torch.distributed all-gather", file=sys.stderr, flush=True)
                args.exchange = "collective"
        if ex is None:
            ex = (P2PExchange([eng], distributed=True) if args.exchange == "p2p"
                  else ProcessGroupExchange())
        drv = ShardedDriver([eng], ex, ws)

    def run(t0, n):
        if drv is not None:
            with torch.cuda.stream(eng.stream):
                drv.run(t0, n)
        else:
            eng.run(t0, n)

    if drv is not None:
        with torch.cuda.stream(eng.stream):
            drv.initialize()
    else:
        eng.initialize()
    run(0, args.warmup)
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()

    # ---- timed region: K iterations as the product runs them (graph-replayed
    # iteration kernels, + the exchange for N > 1), CUDA events on the engine's
    # stream, clocks sampled live; max over ranks
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    l0 = eng.launches
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    if sampler:
        sampler.mark(True)
    start.record(eng.stream)
    run(args.warmup, args.steps)
    stop.record(eng.stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.mark(False)
    if sharded:
        dist.barrier()
    launches = eng.launches - l0
    ms = start.elapsed_time(stop)
    # ---- the iteration kernel's duration over the timed region: the streaming
    # kernels (k_chain, k_rows) time themselves on the device (first CTA start
    # to last CTA end, %globaltimer) and count improved rows, per iteration,
    # inside the graph replays (psso_iteration_stats)
    sk_ms, s_imp, s_n = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    nstat = min(args.steps, 1024)
    _lib.check(L.psso_iteration_stats(eng.ctx, args.warmup + args.steps - nstat, nstat,
                                      ctypes.byref(sk_ms), ctypes.byref(s_imp), ctypes.byref(s_n)))
    # ---- cross-check / fallback: the same K iterations again with every
    # iteration-kernel launch bracketed by CUDA events on the engine's stream
    # (psso_profile: direct launches instead of the graph)
    L.psso_profile(eng.ctx, 1)
    run(args.warmup + args.steps, args.steps)
    kms, kn = ctypes.c_double(), ctypes.c_int64()
    _lib.check(L.psso_profile_read(eng.ctx, ctypes.byref(kms), ctypes.byref(kn)))
    L.psso_profile(eng.ctx, 0)
    clocks = sampler.stop() if sampler else None
    eng.check()
    kname = L.psso_kernel_name(eng.ctx).decode()
    dev_timed = s_n.value == nstat and nstat > 0
    kern_dev = sk_ms.value / nstat if dev_timed else float("nan")
    imp_rows = float(s_imp.value) if dev_timed else float("nan")
    ms, kern_ev, kern_dev = _max_over_ranks([ms, kms.value / max(kn.value, 1), kern_dev], ws)
    imp_rows = _sum_over_ranks(imp_rows, ws)
    kern_ms = kern_dev if dev_timed else kern_ev
    if sharded and args.exchange == "p2p":
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
    # rho: fraction of rows whose pBest improved, counted by the kernel;
    # with it the pBest write-back (rho*T per pvu) and p_f traffic ((8 + 8 rho)/D)
    rho = imp_rows / (nstat * nsol) if dev_timed else None
    bpv_rho = (3 * es + rho * es + (8 + 8 * rho) / nvar) if rho is not None else None

    # ---- e2e through the public API with host buffers: N = 1 psso_solve (C ABI:
    # config in, trajectory + best position out); N > 1 every rank calls
    # run_parallel_distributed (the multi-GPU public API) -- device allocation,
    # init, K iterations, copy-back inside the wall-clock region; max over ranks
    import numpy as np

    cfg = make_config(psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min,
                                     var_max=fn.var_max, nsol=nsol, nvar=nvar, niter=args.steps),
                      fn, 0, dtype=dtype, rng=args.rng)
    times = []
    if not sharded:
        traj = np.empty(args.steps)
        best = np.empty(nvar, dtype=np.float64 if dtype == "float64" else np.float32)
        bf, wall = ctypes.c_double(), ctypes.c_double()
        for rep in range(4):  # first call warms module load / allocator; best of the other 3
            t0 = time.perf_counter()
            _lib.check(L.psso_solve(ctypes.byref(cfg), args.steps, traj.ctypes.data,
                                    best.ctypes.data, ctypes.byref(bf), ctypes.byref(wall)))
            times.append(time.perf_counter() - t0)
        note = ("psso_solve(config) -> host trajectory/best position; includes device alloc, "
                "init, all iterations and copy-back")
    else:
        pe = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                            nsol=nsol, nvar=nvar, niter=args.steps)
        ex_e2e = "collective" if args.exchange == "collective" else args.exchange
        for rep in range(4):
            dist.barrier()
            t0 = time.perf_counter()
            rec = run_parallel_distributed(pe, fn, 0, dtype=dtype, rng=args.rng, exchange=ex_e2e)
            el = time.perf_counter() - t0
            times.append(_max_over_ranks([el], ws)[0])
            del rec
        note = (f"run_parallel_distributed on every rank (exchange={ex_e2e}) -> host trajectory/"
                "best position; includes device alloc, init, all iterations and copy-back; "
                "max over ranks")
    el = min(times[1:])
    e2e = {"value": nsol * nvar * args.steps / el, "unit": UNIT,
           "h2d_bytes_per_step": ctypes.sizeof(cfg) / args.steps,
           "d2h_bytes_per_step": (8 * args.steps + es * nvar + 8) / args.steps,
           "note": note + "; the reference API takes no array inputs (the swarm is generated "
                          "from the seed); best of 3 calls after a warm-up call",
           "calls_s": [round(x, 4) for x in times]}

    if rank != 0:
        dist.destroy_process_group()
        return
    cpu = cpu_baseline(fid, nsol, nvar) if ws == 1 and not args.no_cpu else None
    exch = {"nccl": " + library NCCL all-gather of gBest candidate records per iteration "
                    "(CUDA-graph replayed)",
            "collective": " + torch.distributed all-gather of gBest candidates per iteration",
            "p2p": " + device-initiated P2P stores of gBest candidates per iteration"}[args.exchange]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64" if dtype == "float64" else "f32",
        "data": "synthetic (reference INIT-stream swarm, seed 0)",
        "config": {"workload": desc + (f", global N={nsol} over {ws} GPUs ({args.scaling} scaling)"
                                       if ws > 1 else ""),
                   "fn": fid, "nsol": nsol, "nsol_per_gpu": rows_rank, "nvar": nvar, "rng": args.rng,
                   "evals_per_s": nsol * args.steps / (ms * 1e-3),
                   "hbm_gbs_per_gpu": 3 * es * nsol * nvar * args.steps / (ms * 1e-3) / 1e9 / ws,
                   "l2": f"inputs larger than L2: X+P = {2 * es * rows_rank * nvar / 2**30:.2f} GiB "
                         f"per GPU vs 126 MB L2",
                   "parallelism": f"particle shards x{ws}" + (exch if sharded else "")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": _traffic(wl + ("_philox" if args.rng == "philox" else ""), kname),
                     "peak_source": peak_src,
                     "kernel": kname, "kernel_ms_per_iteration": kern_ms,
                     "alg_bytes_per_launch": alg_bytes, "alg_bytes_per_pvu": 3 * es,
                     "rho": rho, "bytes_per_pvu_with_rho": bpv_rho,
                     "achieved_with_rho": (bpv_rho * rows_rank * nvar / (kern_ms * 1e-3) / 1e9
                                           if bpv_rho is not None else None),
                     "kernel_ms_events": kern_ev,
                     "note": ("kernel_ms_per_iteration: the iteration kernel timed on the device "
                              "(first CTA start to last CTA end, %globaltimer) for every iteration "
                              "of the timed region, graph replays included (psso_iteration_stats); "
                              "kernel_ms_events: CUDA events around every launch of a second "
                              "K-iteration pass with direct launches; rho = improved rows / rows "
                              "per iteration over the timed region, counted by the kernel; max "
                              "over ranks" if dev_timed else
                              "whole-run kernel: all timed iterations in one launch; L2/SMEM-"
                              "resident swarm, so the HBM roofline does not bind"
                              if "k_swarm" in kname else
                              "kernel duration from CUDA events around every launch of a second "
                              "K-iteration pass (this kernel records no device statistics)")},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


def _spawn(args):
    """--gpus N > 1 without torchrun: relaunch this script with N ranks."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: fixed global N (strong) or the workload's N per GPU (weak)")
    ap.add_argument("--rng", default="reference", choices=["reference", "philox"])
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "collective", "p2p"],
                    help="N > 1: gBest records by the library's NCCL all-gather in CUDA graphs, "
                         "a torch.distributed all-gather, or device-initiated P2P stores")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (diagnostics)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="tests: the multi-rank path (process group + exchange) even at one rank")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference(args, args.workload)
    else:
        run_ours(args, args.workload)


if __name__ == "__main__":
    main()
