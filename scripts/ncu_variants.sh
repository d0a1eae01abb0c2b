#!/usr/bin/env bash
mkdir -p gpurun_out
CFG=${1:-C3}
for v in mirror nomirror; do
  envs=""; [ $v = nomirror ] && envs="GHX_NO_MIRROR=1"
  env $envs timeout 900 ncu --set full --clock-control none --import-source on -k regex:ghx_copy_kernel -s 4 -c 1 \
    -f -o gpurun_out/prof_${CFG}_$v python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_${CFG}_$v.log 2>&1
  echo "ncu $v rc=$?"
done
