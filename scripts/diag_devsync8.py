"""Diagnostic: C3 across N processes (DIAG_WORLD, default 8) on one GPU with
the in-kernel device sync -- the one-kernel packed exchange (pushes, local
tags and unpacks in one launch), the push-then-unpack pair, direct remote
stores -- through tests/test_gpu_process.py's workers; pass variant names
(repeats allowed) to choose."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

VARIANTS = {
    "one-kernel": {},
    "two-kernels": {"GHX_ONE_KERNEL": "0"},
    "direct": {"GHX_REMOTE": "direct"},
}

if __name__ == "__main__":
    import test_gpu_process as T
    world = int(os.environ.get("DIAG_WORLD", "8"))
    for name in (sys.argv[1:] or VARIANTS):
        env = {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": os.environ.get("DIAG_TIMEOUT", "60"), **VARIANTS[name]}
        t0 = time.time()
        try:
            T._run(("C3", 512, 128, 8, 2, f"C3_x{world}", env), world)
            r = "ok"
        except BaseException as e:  # noqa: BLE001
            r = "FAIL " + str(e).strip().splitlines()[-1][-200:]
        print(f"{name}: {r} ({time.time() - t0:.1f} s)", flush=True)
