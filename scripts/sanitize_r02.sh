#!/usr/bin/env bash
# compute-sanitizer pass over the round-2 code paths -> gpurun_out/sanitizer_r02.txt
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
O=gpurun_out/sanitizer_r02.txt
{
echo "== memcheck tests/test_gpu_random.py (36 layouts, every variant incl. phased + tile ring, pinned)"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_random.py 2>&1 | tail -3
echo "== memcheck golden FillBoundary, phased variants"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_parity.py -k "golden and phased" 2>&1 | tail -3
echo "== racecheck golden FillBoundary, phased_ring variant"
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -q -x tests/test_gpu_parity.py -k "golden and phased_ring" 2>&1 | tail -3
echo "== memcheck reference binding (plain C ABI on the reference's objects)"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_reference_binding.py 2>&1 | tail -3
echo "== memcheck debug mode + arena"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x -m gpu tests/test_debug_mode.py tests/test_arena.py 2>&1 | tail -3
echo "== synccheck tests/test_gpu_random.py"
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -q -x tests/test_gpu_random.py 2>&1 | tail -3
} > $O 2>&1
cat $O
