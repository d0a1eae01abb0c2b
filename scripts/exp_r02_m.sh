# r02 experiment M: sector-fill unpack (GHX_SECTOR_FILL) -- parity, then the
# 8-process packed unpack per rank under ncu (HBM side, one GPU), fill on / off
set -u
mkdir -p gpurun_out/expM
O=gpurun_out/expM
timeout 900 python -m pytest tests/test_gpu_sector_fill.py tests/test_gpu_process.py tests/test_gpu_process_golden.py -q -x -m gpu > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
tail -3 $O/tests.log
for sf in 1 0; do
  GHX_SECTOR_FILL=$sf GHX_BENCH_BACKEND=gloo GHX_BARRIER_TIMEOUT_S=60 GHX_REMOTE=packed timeout 900 ncu --clock-control none --target-processes all -k regex:ghx_copy_kernel \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
      python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port $((29810 + sf)) \
      bench.py --gpus 8 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/proc8_packed_fill$sf.csv 2> $O/proc8_packed_fill$sf.err
  echo "fill=$sf rc=$?"
done
