#!/usr/bin/env bash
# HBM-side cost of the multi-rank exchange kernels on ONE GPU: N processes
# (gloo plumbing, host sync) share the device, so every "remote" store lands
# in the same HBM instead of crossing NVLink; ncu times each rank's push and
# unpack launches in isolation.  -> gpurun_out/multi1/
mkdir -p gpurun_out/multi1
O=gpurun_out/multi1
export GHX_BENCH_BACKEND=gloo GHX_BARRIER_TIMEOUT_S=60 PYTHONDONTWRITEBYTECODE=1
port=29700
for n in 2 4 8; do
  for remote in packed direct; do
    port=$((port + 1))
    GHX_REMOTE=$remote timeout 900 ncu --target-processes all -k regex:ghx_copy_kernel \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus $n --steps 2 --warmup 3 --no-e2e --no-cpu > $O/C3_${remote}_$n.csv 2> $O/C3_${remote}_$n.err
    echo "n=$n $remote rc=$?"
  done
done
