"""The driver's bench.py invocations (README "bench contract"): one JSON line
from rank 0, exit code 0 on every rank, for the reference arm (CPU, runs
here) and for our arm under torchrun with two ranks sharing cuda:0 (gloo
plumbing, CUDA-IPC push between the two processes)."""

import json
import os
import socket
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _torchrun(nproc, args, env=None, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", *args]
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(cmd, cwd=REPO, env=e, capture_output=True, text=True, timeout=timeout)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return r.returncode, lines, r.stderr


def test_reference_arm_under_torchrun_prints_one_line():
    rc, lines, err = _torchrun(2, ["--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "3",
                                   "--config", "C1"])
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    # the reference itself (baseline/_ref), not the port, with 2 simulated ranks
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["ranks"] == 2, cb
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_default_is_c3():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3"],
                       cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["config"]["workload"].startswith("C3:") and d["config"]["domain"] == [512, 512, 512]
    assert d["config"]["ghost_bytes_per_step"] == 830734336
    assert d["cpu_baseline"]["kind"] == "reference" and d["steps"] == 3


@pytest.mark.gpu
def test_our_arm_one_gpu_default_c3():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--e2e-steps", "2",
                        "--cpu-seconds", "2", "--no-port"], cwd=REPO, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["config"]["workload"].startswith("C3:") and d["n_gpus"] == 1 and d["scaling"] == "strong"
    assert d["verified"] is True and d["gpu_launches"] == 5
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.2
    sp = d["roofline"]["direction_split"]  # the floors measured in the same run
    assert sp["x_row_seams"] == 64 * 8 * 128 * 128 and sp["x_only_ms"] > 0 and sp["yz_only_ms"] > 0
    assert 0.5 < sp["frac_of_additive_floor_same_layout"] < 2.0
    assert d["e2e"]["exec"]["phased"] == 1 and d["e2e"]["exec"]["ring_tasks"] > 0  # the host-memory path
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["bit_exact_vs_ours_fab0"] is True, cb
    assert d["e2e"]["verified"] is True and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.gpu
def test_our_arm_two_ranks_on_one_gpu():
    rc, lines, err = _torchrun(2, ["--gpus", "2", "--steps", "5", "--warmup", "3", "--no-cpu", "--e2e-steps", "2"],
                               env={"GHX_BENCH_BACKEND": "gloo", "GHX_BARRIER_TIMEOUT_S": "30"})
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 5 and d["warmup"] == 3 and d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("C3:")
    assert d["verified"] is True and d["value"] > 0 and d["gpu_launches"] > 0
    # C3 over 2 GPUs: 142.7 MB per GPU each way over NVLink bounds the step
    nv = d["roofline"]
    assert nv["bound"] == "nvlink" and nv["frac"] > 0 and nv["peak"] == 770.0
    assert nv["bytes_per_gpu_max_send_recv"] == 142737408 and "hbm" in nv
    assert d["e2e"]["verified"] is True and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.gpu
def test_our_arm_two_ranks_device_sync():
    """The path a multi-GPU box takes (device sync: READY/DONE inside the
    copy kernel, enqueue-only timing loop), forced on two processes that
    share one GPU (time-sliced: the timing means nothing, the result is
    verified)."""
    rc, lines, err = _torchrun(2, ["--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "2"],
                               env={"GHX_BENCH_BACKEND": "gloo", "GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "60"})
    assert rc == 0, err[-2000:]
    d = json.loads(lines[0])
    assert d["config"]["sync"] == "device" and d["config"]["transport"] == "p2p"
    assert d["verified"] is True and d["e2e"]["verified"] is True
    bd = d["multi_gpu_breakdown"]  # per-rank push and unpack kernels, max over ranks
    assert bd["push_kernel_ms"] > 0 and bd["unpack_or_wait_ms"] > 0 and bd["remote"] == "packed"
