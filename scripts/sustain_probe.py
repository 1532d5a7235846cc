"""Per-iteration kernel time over a long C3 run, beside live clocks and power.

Diagnostic for the gap between a single ncu-timed launch and the sustained
bench number: if the per-iteration time creeps up while power sits at the cap
and the clocks drop, the gap is the board's power management.
    python scripts/sustain_probe.py [--workload c3|c3f32] [--iters 600]
"""
import argparse
import json
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2110_01470_b200 as psso  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--iters", type=int, default=600)
args = ap.parse_args()
dtype = "float32" if args.workload.endswith("f32") else "float64"
fn = psso.make_function("f5", 128)
p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max,
                   nsol=1 << 20, nvar=128, niter=args.iters)
eng = DeviceEngine(p, fn, 0, dtype=dtype)
eng.initialize()
torch.cuda.synchronize()

Q = ("timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,"
     "clocks_event_reasons.sw_power_cap")
proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={Q}", "--format=csv,noheader,nounits",
                         "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
samples = []


def _read():
    for ln in proc.stdout:
        samples.append((time.perf_counter(), ln.strip()))


th = threading.Thread(target=_read, daemon=True)
th.start()
time.sleep(0.5)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
       for _ in range(args.iters)]
t_host0 = time.perf_counter()
for t in range(args.iters):
    a, b = evs[t]
    a.record(eng.stream)
    eng.step(t)
    b.record(eng.stream)
torch.cuda.synchronize()
t_host1 = time.perf_counter()
time.sleep(0.3)
proc.terminate()
ms = [a.elapsed_time(b) for a, b in evs]
eng.check()
eng.close()

blk = 50
rows = []
for k in range(0, args.iters, blk):
    seg = ms[k:k + blk]
    rows.append({"iters": f"{k}-{k + len(seg) - 1}", "ms_mean": round(sum(seg) / len(seg), 4),
                 "ms_min": round(min(seg), 4)})
pw = []
for ts, ln in samples:
    parts = [x.strip() for x in ln.split(",")]
    if len(parts) >= 7 and t_host0 <= ts <= t_host1:
        try:
            pw.append({"sm": float(parts[1]), "mem": float(parts[2]), "W": float(parts[3]),
                       "T": parts[4], "Tmem": parts[5], "cap": parts[6]})
        except ValueError:
            pass


def med(v):
    v = sorted(v)
    return v[len(v) // 2] if v else None


out = {"workload": args.workload, "dtype": dtype, "per_50": rows, "samples": len(pw),
       "sm_mhz": med(s["sm"] for s in pw), "sm_mhz_min": min((s["sm"] for s in pw), default=None),
       "mem_mhz": med(s["mem"] for s in pw), "power_w_median": med(s["W"] for s in pw),
       "power_w_max": max((s["W"] for s in pw), default=None),
       "power_cap_active_frac": (sum(1 for s in pw if s["cap"].lower().startswith("active")) / len(pw))
       if pw else None,
       "temps_first_last": [(pw[0]["T"], pw[0]["Tmem"]), (pw[-1]["T"], pw[-1]["Tmem"])] if pw else None}
print(json.dumps(out))
