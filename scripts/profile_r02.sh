#!/usr/bin/env bash
# Round-2 profiling pass on one GPU (run under gpurun from the repo root):
# bench lines (default = C3 with the direction split), the reference arm,
# the ncu launch list of the default bench command, ncu --set full of the
# top kernel (C3, C2), per-direction DRAM metrics (x only / y-z only / all)
# for C2 and C3, and compute-sanitizer racecheck / memcheck of the
# FillBoundary task mix.  Output: gpurun_out/prof2/
mkdir -p gpurun_out/prof2
O=gpurun_out/prof2
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.log; echo "bench default rc=$?"
for c in C2 C4 C5 C1; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.log; echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference_C3.json 2> $O/bench_reference_C3.log
echo "bench reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_C3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-split > $O/launches_C3.log 2>&1
echo "launch list rc=$?"
for c in C3 C2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ghx_copy_kernel -s 4 -c 1 -f \
    -o $O/full_$c python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-split > $O/full_$c.log 2>&1
  echo "full $c rc=$?"
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__maximum_warps_per_active_cycle_pct
for c in C3 C2 C4 C5 C1; do
  for g in all x yz; do
    case $g in all) a="";; x) a="--ngrow 2,0,0";; yz) a="--ngrow 0,2,2";; esac
    [ "$c" = C5 ] && [ "$g" != all ] && continue
    [ "$c" = C1 ] && [ "$g" != all ] && continue
    timeout 900 ncu --metrics $M --clock-control none --csv -k regex:ghx_copy_kernel -s 4 -c 1 \
      python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-split $a > $O/split_${c}_$g.csv 2> $O/split_${c}_$g.err
    echo "split $c $g rc=$?"
  done
done
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
{
for t in "tests/test_gpu_random.py" "tests/test_gpu_parity.py -k golden"; do
  echo "== racecheck $t"; timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -q -x $t 2>&1 | tail -4
done
echo "== racecheck ring_check (tile ring tasks)"; GHX_RING=1 timeout 900 compute-sanitizer --tool racecheck python scripts/ring_check.py 2>&1 | tail -4
echo "== memcheck ring_check (tile ring tasks)"; GHX_RING=1 timeout 900 compute-sanitizer --tool memcheck python scripts/ring_check.py 2>&1 | tail -4
echo "== memcheck tests/test_gpu_random.py"; timeout 1500 compute-sanitizer --tool memcheck python -m pytest -q -x tests/test_gpu_random.py 2>&1 | tail -3
} > $O/sanitizer.txt 2>&1
echo "sanitizer done"
