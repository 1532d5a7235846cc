"""bench.py keeps the driver's JSON contract (CPU-side pieces: the reference arm)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--workload", "c1", "--steps", "3", "--warmup", "3")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "pvu/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "pvu/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1


def test_gpus_flag_spawns_its_own_ranks():
    """--gpus 2 without torchrun: bench.py relaunches itself with 2 ranks (rank 0 prints)."""
    d = _run("--impl", "reference", "--workload", "c1", "--gpus", "2", "--steps", "3",
             "--warmup", "3")
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["scaling"] == "strong"
    assert d["config"]["nsol"] == 100 and d["config"]["same_config"] is True


def test_weak_scaling_grows_the_global_swarm():
    d = _run("--impl", "reference", "--workload", "c1", "--gpus", "2", "--scaling", "weak",
             "--steps", "3", "--warmup", "3")
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["nsol"] == 200


def test_warmup_floor_enforced():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--warmup", "2"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode != 0 and "warmup" in out.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["collective", "p2p"])
def test_bench_multi_rank_path_runs_under_torchrun(exchange):
    """bench.py --gpus 2 under torchrun: the sharded path end to end.  Both ranks
    share the one GPU of the box (gloo process group; runs use NCCL)."""
    import json
    import os
    import socket
    import subprocess
    import sys

    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, PSSO_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "6", "--warmup", "3", "--workload", "c3sphere",
           "--exchange", exchange, "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["nsol"] == 1 << 20 and d["config"]["nsol_per_gpu"] == 1 << 19
    assert d["gpu_launches"] > 0 and d["roofline"]["achieved"] > 0
    assert d["e2e"]["value"] > 0 and len(d["e2e"]["calls_s"]) == 4


@pytest.mark.gpu
def test_bench_sharded_nccl_graph_path_world_size_1():
    """torchrun with one rank and --force-sharded: the default multi-GPU path (library NCCL
    communicator, kernels + all-gather replayed from CUDA graphs) on the C4 strong workload."""
    import os
    import socket

    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--gpus", "1", "--steps", "20", "--warmup", "3", "--workload", "c4",
           "--scaling", "strong", "--force-sharded", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ), capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = lines[0]
    assert d["config"]["nsol"] == 1 << 24 and "NCCL" in d["config"]["parallelism"]
    assert d["roofline"]["kernel"].startswith("k_chain") and d["roofline"]["frac"] > 0.5
    assert d["e2e"]["value"] > 0


@pytest.mark.gpu
def test_bench_gpus_2_self_spawns_and_bootstraps_the_nccl_communicator():
    """bench.py --gpus 2 without torchrun (self-spawn) on the one GPU of the box, gloo
    process group: both ranks run the library's communicator bootstrap (rank 0's
    ncclUniqueId over the process group, collective ncclCommInitRank), which NCCL
    refuses for two ranks on one device -- every rank then falls back to the
    torch.distributed all-gather alike and the run completes with n_gpus 2."""
    import os

    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, PSSO_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "6",
                          "--warmup", "3", "--workload", "c3sphere", "--no-cpu"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert out.stderr.count("library NCCL communicator unavailable") == 2  # both ranks, alike
    assert "torch.distributed all-gather" in d["config"]["parallelism"]


def test_clock_samples_are_restricted_to_the_timed_region():
    """ClockSampler keeps the samples nvidia-smi stamped inside [t0, t1] (the timed
    region) and reports throttle reasons seen there; with none inside it falls back
    to every sample and says so."""
    import datetime
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)

    def stamp(ts):
        return datetime.datetime.fromtimestamp(ts).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]

    cs = bench.ClockSampler(0)
    base = 1_800_000_000.0
    rows = [(base - 1.0, "1000, 1965, 300, Not Active, Not Active, Not Active, Not Active"),
            (base + 0.10, "1700, 1965, 990, Not Active, Not Active, Not Active, Active"),
            (base + 0.12, "1650, 1965, 995, Not Active, Not Active, Not Active, Active"),
            (base + 5.0, "1965, 1965, 100, Not Active, Not Active, Not Active, Not Active")]
    import io

    class P:  # a stand-in for the nvidia-smi process
        stdout = io.StringIO("".join(f"{stamp(t)}, {r}\n" for t, r in rows))

        def terminate(self):
            pass

        def wait(self, timeout=None):
            pass

    cs.proc = P()
    cs._read()
    cs.thread = type("T", (), {"join": lambda self, timeout=None: None})()
    cs.t0, cs.t1 = base, base + 1.0
    out = cs.stop()
    assert out["window"] == "timed region" and out["samples"] == 2
    assert out["sm_mhz"] == 1700.0 and out["reasons"] == ["sw_power_cap"]
    cs2 = bench.ClockSampler(0)
    cs2.lines = [(base + 9.0, rows[0][1])]
    cs2.proc, cs2.thread = P(), cs.thread
    cs2.t0, cs2.t1 = base, base + 1.0
    out2 = cs2.stop()
    assert out2["samples"] == 1 and out2["window"].startswith("timed region +")
