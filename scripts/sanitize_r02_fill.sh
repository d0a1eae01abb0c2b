#!/usr/bin/env bash
# compute-sanitizer over the sector-fill unpack -> gpurun_out/sanitizer_r02_fill.txt
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
O=gpurun_out/sanitizer_r02_fill.txt
{
echo "== memcheck tests/test_gpu_sector_fill.py (sector fills vs plain unpack, aligned and 16-B-offset fab bases)"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x -m gpu tests/test_gpu_sector_fill.py 2>&1 | tail -3
echo "== racecheck tests/test_gpu_sector_fill.py"
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -q -x -m gpu tests/test_gpu_sector_fill.py 2>&1 | tail -3
echo "== initcheck tests/test_gpu_sector_fill.py"
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest -q -x -m gpu tests/test_gpu_sector_fill.py 2>&1 | tail -3
} > $O 2>&1
cat $O
