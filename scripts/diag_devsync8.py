"""Diagnostic: C3 across 8 processes on one GPU with device sync -- the
serial unpack, the concurrent unpack with end-of-kernel DONE, and the
concurrent unpack with per-peer DONE (tests/test_gpu_process.py workers)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

VARIANTS = {
    "serial-unpack": {"GHX_UNPACK_OVERLAP": "0"},
    "overlap-kernel-done": {"GHX_UNPACK_OVERLAP": "1", "GHX_PEER_DONE": "0"},
    "overlap-peer-done": {"GHX_UNPACK_OVERLAP": "1"},
    "serial-unpack-peer-done": {"GHX_UNPACK_OVERLAP": "0", "GHX_PEER_DONE": "1"},
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
