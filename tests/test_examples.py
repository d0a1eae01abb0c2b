"""The README's quickstart runs end to end on the GPU (FillBoundary blocking
and enqueue-only, fill_patch, average_down, the CUDA-graph heat loop)."""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_quickstart_runs():
    r = subprocess.run([sys.executable, os.path.join(REPO, "examples", "quickstart.py")], cwd=REPO,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "quickstart ok" in r.stdout
