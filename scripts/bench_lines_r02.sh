#!/usr/bin/env bash
# Final round-2 bench lines (every config, the reference arm) -> gpurun_out/prof2/
mkdir -p gpurun_out/prof2
O=gpurun_out/prof2
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.log; echo "bench default rc=$?"
for c in C2 C4 C5 C1; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.log; echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference_C3.json 2> $O/bench_reference_C3.log
echo "bench reference rc=$?"
timeout 900 python bench.py --impl reference --config C2 --steps 20 --warmup 3 > $O/bench_reference_C2.json 2> $O/bench_reference_C2.log
echo "bench reference C2 rc=$?"
for op in fill_patch average_down heat heat2; do
  timeout 600 python bench_amr.py --op $op > $O/bench_amr_$op.json 2> $O/bench_amr_$op.log
  echo "bench_amr $op rc=$?"
done
