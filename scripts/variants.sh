#!/usr/bin/env bash
# Kernel-variant sweep on one GPU.  Usage: variants.sh CFG "ENVSET1" "ENVSET2" ...
mkdir -p gpurun_out
CFG=$1; shift
for envs in "$@"; do
  r=$(env $envs timeout 300 python bench.py --config $CFG --steps 100 --warmup 5 --no-e2e --no-cpu 2>>gpurun_out/variants.err)
  echo "$CFG [$envs] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["verified"])' 2>&1 | tail -1)"
done
