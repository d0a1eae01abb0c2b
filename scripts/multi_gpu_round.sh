#!/usr/bin/env bash
# Multi-GPU measurement pass for a box with N >= 2 B200s (one process per
# GPU, NCCL plumbing): the north-star C3 first (BASELINE configs[2], the
# bench default), then C5 and C2, at 2/4/8 GPUs over the CUDA-IPC push
# (packed remote rows in one push + unpack launch, the same as two launches
# GHX_ONE_KERNEL=0, direct remote rows; in-kernel READY/DONE sync, plus the
# standalone-barrier sequence GHX_FUSED_SYNC=0 for comparison) and the NCCL
# pack/send/unpack fallback.
# Output: gpurun_out/multi/<config>_<transport>_<N>.json (one bench line each).
#   bash scripts/multi_gpu_round.sh [max_gpus]
set -u
mkdir -p gpurun_out/multi
export PYTHONDONTWRITEBYTECODE=1
MAXG=${1:-$(nvidia-smi -L | wc -l)}
nvidia-smi topo -m > gpurun_out/multi/topo.txt 2>&1
port=29600
for cfg in C3 C5 C2; do
  steps=100; [ "$cfg" = C5 ] && steps=20
  for n in 2 4 8; do
    [ "$n" -le "$MAXG" ] || continue
    for variant in "p2p:GHX_REMOTE=packed" "p2p2k:GHX_ONE_KERNEL=0" "p2p:GHX_REMOTE=direct" "p2pbar:GHX_FUSED_SYNC=0" \
                   "nccl:GHX_TRANSPORT=nccl"; do
      tag=${variant%%:*}; envs=${variant#*:}
      port=$((port + 1))
      env $envs GHX_BARRIER_TIMEOUT_S=30 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --config $cfg --steps $steps --warmup 5 --no-cpu --e2e-steps 2 \
        > gpurun_out/multi/${cfg}_${tag}_${envs#*=}_$n.json 2> gpurun_out/multi/${cfg}_${tag}_${envs#*=}_$n.log
      echo "$cfg n=$n $envs rc=$? $(python -c "import json,sys; d=json.load(open('gpurun_out/multi/${cfg}_${tag}_${envs#*=}_$n.json')); r=d['roofline'] or {}; print(d['value'], d['ms_per_step'], d['verified'], r.get('frac'), (r.get('nvlink') or {}).get('frac'), d['e2e']['value'])" 2>&1 | tail -1)"
    done
  done
done
