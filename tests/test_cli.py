"""CLI of the B200 engine: the reference's flag/config/exit-code contract (cli.py:44-69, 355-386)."""

import json

import pytest

from paper_2110_01470_b200 import cli


def test_usage_errors_exit_1(tmp_path, capsys):
    assert cli.main(["run", "--function", "f42"]) == cli.EXIT_USAGE
    bad = tmp_path / "c.json"
    bad.write_text(json.dumps({"nsol": 10, "bogus": 1}))
    assert cli.main(["run", "--config", str(bad)]) == cli.EXIT_USAGE
    assert "unknown config key 'bogus'" in capsys.readouterr().err
    assert cli.main(["run", "--config", str(tmp_path / "missing.json")]) == cli.EXIT_USAGE
    assert cli.main(["run", "--cw", "0.9", "--cp", "0.1"]) == cli.EXIT_USAGE  # thresholds
    assert cli.main(["sweep", "--triples", str(tmp_path / "nope.txt")]) == cli.EXIT_USAGE


def test_config_layering():
    args = cli._build_parser().parse_args(["run", "--nsol", "7"])
    merged = cli._merged(args, {"nsol": 100, "nvar": 50})
    assert merged == {"nsol": 7, "nvar": 50}


def test_triples_file(tmp_path):
    f = tmp_path / "t.txt"
    f.write_text("# comment\n0.1,0.3,0.7\n0.2 0.4 0.6\n")
    assert cli._parse_triples(str(f)) == ((0.1, 0.3, 0.7), (0.2, 0.4, 0.6))
    assert cli._parse_triples("builtin")[5] == (0.3, 0.6, 0.8)


@pytest.mark.gpu
def test_run_and_sweep_on_device(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "r.csv"
    rc = cli.main(["run", "--function", "f5", "--schedule", "sequential", "--nsol", "40",
                   "--nvar", "16", "--iters", "30", "--runs", "3", "--out", str(out), "--trajectory"])
    assert rc == cli.EXIT_OK
    rows = out.read_text().splitlines()
    assert rows[0].startswith("run_id,schedule,function") and len(rows) == 4
    assert rows[1].split(",")[1] == "sequential"
    side = tmp_path / "r.csv.trajectories.dat"
    assert len(side.read_text().splitlines()) == 1 + 3 * 30
    rc = cli.main(["sweep", "--function", "f1", "--runs", "2", "--nsol", "32", "--nvar", "8",
                   "--iters", "20", "--out", str(tmp_path / "s.csv")])
    assert rc == cli.EXIT_OK
    assert len((tmp_path / "s.csv").read_text().splitlines()) == 1 + 6 * 2
