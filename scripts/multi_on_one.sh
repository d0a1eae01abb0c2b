#!/usr/bin/env bash
# N>1 code paths with every rank on the single GPU of a gpurun box (gloo plumbing).
for envs in "GHX_SYNC=device" "GHX_SYNC=host" "GHX_TRANSPORT=nccl"; do
  env GHX_BENCH_BACKEND=gloo GHX_BARRIER_TIMEOUT_S=20 $envs timeout 600 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu \
    > gpurun_out/multi_$envs.json 2> gpurun_out/multi_$envs.log
  echo "[$envs] rc=$? $(python -c "import json; d=json.load(open('gpurun_out/multi_$envs.json')); print(d['value'], d['ms_per_step'], d['verified'], d['config']['transport'], d['config']['sync'], d['e2e']['value'])" 2>&1 | tail -1)"
done
