#!/usr/bin/env bash
# One GPU session: smoke, GPU tests, bench, ncu launch list + full capture.
# Usage (from the repo root, under gpurun):  bash scripts/gpu_round.sh [steps...]
# steps: smoke tests bench ncu (default: all)
set -u
mkdir -p gpurun_out
STEPS="${*:-smoke tests bench ncu}"
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
for s in $STEPS; do
  case "$s" in
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?" ;;
    tests)
      timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
      echo "tests rc=$?"; tail -5 gpurun_out/pytest_gpu.log ;;
    bench)
      for c in ${BENCH_CONFIGS:-C3}; do
        timeout 900 python bench.py --config $c --steps ${BENCH_STEPS:-200} --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.log
        echo "bench $c rc=$?"; cat gpurun_out/bench_$c.json
      done ;;
    ncu)
      for c in ${NCU_CONFIGS:-C3}; do
        timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu \
          > gpurun_out/ncu_launch_$c.log 2>&1
        echo "ncu launches $c rc=$?"
        timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ghx_copy_kernel -s 4 -c 1 \
          -f -o gpurun_out/prof_$c python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu \
          > gpurun_out/ncu_full_$c.log 2>&1
        echo "ncu full $c rc=$?"
      done ;;
  esac
done
