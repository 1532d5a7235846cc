#!/usr/bin/env python
"""Summarise ncu output into the text files kept under profiles/.

    python scripts/ncu_summary.py report  prof.ncu-rep [--units N] > profiles/x.txt
    python scripts/ncu_summary.py launches launches.csv            > profiles/y.txt
    python scripts/ncu_summary.py traffic prof.ncu-rep --workload c3 --bench-log b.log

`report`: one `ncu --set full` capture -> duration, DRAM bytes and
throughput, issue/occupancy, pipe utilisation, warp-stall samples and the
executed SASS mix (per unit of work when --units gives the pvu count of the
launch).  `launches`: a `--metrics gpu__time_duration.sum` launch list ->
per-kernel launch count, mean duration and share of the profiled time.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess
import sys

RAW_KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path, units):
    raw = ncu_csv([path, "--page", "raw"])
    hdr, unit, val = raw[0], raw[1], raw[2]
    name = val[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"kernel: {name}")
    d = dict(zip(hdr, zip(unit, val)))
    for key, label in RAW_KEYS:
        if key in d:
            u, v = d[key]
            print(f"  {label:28s} {v} {u}")
    if "dram__bytes_read.sum" in d and "gpu__time_duration.sum" in d:
        def to_bytes(uv):
            u, v = uv
            return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        def to_s(uv):
            u, v = uv
            return float(v.replace(",", "")) * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(u, 1)
        tb = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
        t = to_s(d["gpu__time_duration.sum"])
        print(f"  {'dram traffic (r+w)':28s} {tb / 1e9:.4f} GB  -> {tb / t / 1e9:.1f} GB/s")
        if units:
            print(f"  {'dram bytes per unit':28s} {tb / units:.3f} B   ({units} units in the launch)")
    stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v[1].replace(",", "") or 0)
              for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1
    print("  warp-state samples: " + ", ".join(
        f"{k} {100 * v / tot:.0f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]))
    src = ncu_csv([path, "--page", "source", "--print-source", "sass"])
    h = src[1]
    iE, iS = h.index("Instructions Executed"), h.index("Source")
    mix, n = collections.Counter(), 0
    for row in src[2:]:
        op = row[iS].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        ex = int(row[iE] or 0)
        mix[o.split(".")[0]] += ex
        n += ex
    per = (units / 32) if units else None
    print(f"  executed warp instructions: {n}" + (f"  ({n / per:.1f} per warp-unit, i.e. per unit per thread)" if per else ""))
    print("  mix: " + " ".join(f"{k}:{(v / per if per else v):.1f}" for k, v in mix.most_common(22)))


def launches(path):
    rows = list(csv.reader(open(path)))
    # skip ncu's preamble lines (==PROF== ...) before the header
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    iU = h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iU], 1.0)
        agg[r[iK].split("(")[0]].append(float(r[iV].replace(",", "")) * scale)
    total = sum(sum(v) for v in agg.values()) or 1
    print(f"{'kernel':70s} {'launches':>8s} {'mean us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:70]:70s} {len(v):8d} {sum(v) / len(v):10.2f} {100 * sum(v) / total:6.1f}%")


def traffic(path, workload, bench_log):
    """Record the capture's DRAM bytes per launch in bench_traffic.json for bench.py."""
    import json
    import pathlib

    raw = ncu_csv([path, "--page", "raw"])
    d = dict(zip(raw[0], zip(raw[1], raw[2])))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tb = sum(float(d[k][1].replace(",", "")) * scale.get(d[k][0], 1)
             for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    kernel = None
    for line in open(bench_log):
        if line.startswith("{"):
            kernel = json.loads(line)["roofline"]["kernel"]
    out = pathlib.Path(__file__).resolve().parent.parent / "bench_traffic.json"
    db = json.loads(out.read_text()) if out.exists() else {}
    db[workload] = {"kernel": kernel, "dram_bytes_per_launch": tb,
                    "source": f"ncu --set full capture {pathlib.Path(path).name} "
                              f"({d.get('Kernel Name', ('', '?'))[1]})"}
    out.write_text(json.dumps(db, indent=1, sort_keys=True) + "\n")
    print(f"{workload}: {kernel} {tb / 1e9:.4f} GB per launch -> {out.name}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["report", "launches", "traffic"])
    ap.add_argument("path")
    ap.add_argument("--units", type=int, default=0, help="work units (pvu) in the captured launch")
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--bench-log", default=None)
    a = ap.parse_args()
    if a.mode == "report":
        report(a.path, a.units)
    elif a.mode == "traffic":
        traffic(a.path, a.workload, a.bench_log)
    else:
        launches(a.path)


if __name__ == "__main__":
    sys.exit(main())
