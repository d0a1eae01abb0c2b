#!/usr/bin/env bash
# ncu --set full of ghx_copy_kernel for one config + env set: ncu_one.sh CFG TAG "ENVS"
mkdir -p gpurun_out
env $3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ghx_copy_kernel -s 4 -c 1 \
  -f -o gpurun_out/prof_$1_$2 python bench.py --config $1 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$1_$2.log 2>&1
echo "ncu $1 $2 rc=$?"
