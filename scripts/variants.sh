#!/usr/bin/env bash
# Kernel-variant sweep on one GPU.  Usage: variants.sh CFG "ENVSET1[|bench args]" "ENVSET2[|bench args]" ...
mkdir -p gpurun_out
CFG=$1; shift
for spec in "$@"; do
  envs=${spec%%|*}; args=""; [[ "$spec" == *"|"* ]] && args=${spec#*|}
  r=$(env $envs timeout 300 python bench.py --config $CFG --steps ${VSTEPS:-100} --warmup 5 --no-e2e --no-cpu $args 2>>gpurun_out/variants.err)
  echo "$CFG [$spec] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["verified"])' 2>&1 | tail -1)"
done
