"""Golden CSV rows from the REFERENCE experiment harness (run here, not on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_harness_golden.py

Runs `sso.harness.run_experiment` (parallel schedule; and both schedules for
the harness_seq_* files) on small cells and
stores its results CSV and summary CSV with the wall-time column blanked (the
only machine-dependent field), so tests can check that the B200 harness
writes the same rows.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from sso.harness import ExperimentConfig, run_experiment  # noqa: E402
from sso.records import ScheduleKind  # noqa: E402

CELLS = dict(functions=["f1", "f4", "f5", "f7"], schedules=[ScheduleKind.PARALLEL],
             replications=4, base_seed=7, nsol=64, nvar=16, niter=60)
# both schedules, sequential first (harness_seq_*.csv)
SEQ_CELLS = dict(functions=["f1", "f4", "f6"],
                 schedules=[ScheduleKind.SEQUENTIAL, ScheduleKind.PARALLEL],
                 replications=3, base_seed=11, nsol=48, nvar=20, niter=40)


def _write(cells, stem):
    with tempfile.TemporaryDirectory() as d:
        out, summ = Path(d) / "r.csv", Path(d) / "s.csv"
        run_experiment(ExperimentConfig(**cells), out=out, summary_out=summ)
        rows = out.read_text().splitlines()
        blank = [rows[0]] + [",".join(r.split(",")[:-1] + [""]) for r in rows[1:]]
        (HERE / f"{stem}_records.csv").write_text("\n".join(blank) + "\n")
        (HERE / f"{stem}_summary.csv").write_text(summ.read_text())
    print(f"wrote {stem}_records.csv, {stem}_summary.csv")


def main():
    _write(CELLS, "harness")
    _write(SEQ_CELLS, "harness_seq")


if __name__ == "__main__":
    main()
