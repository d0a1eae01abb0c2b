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
                                   "--cpu-seconds", "1"])
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_two_ranks_on_one_gpu():
    rc, lines, err = _torchrun(2, ["--gpus", "2", "--steps", "5", "--warmup", "3", "--no-cpu", "--e2e-steps", "2"],
                               env={"GHX_BENCH_BACKEND": "gloo", "GHX_BARRIER_TIMEOUT_S": "30"})
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 5 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["verified"] is True and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] in ("hbm", "nvlink") and d["roofline"]["frac"] > 0
    assert d["e2e"]["verified"] is True and d["e2e"]["h2d_bytes_per_step"] > 0
