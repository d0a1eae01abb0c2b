# r02 experiment K: remote-tag pairing (sender: thread ranks; receiver unpack: process ranks) at 8 ranks on one GPU
set -u
mkdir -p gpurun_out/expK
O=gpurun_out/expK
for pr in 0 1; do
  GHX_REMOTE_PAIR=$pr timeout 600 ncu --clock-control none -k regex:ghx_copy_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv python scripts/thread_ranks_c3.py 8 3 > $O/thread8_pair$pr.csv 2> $O/thread8_pair$pr.err
  GHX_REMOTE_PAIR=$pr timeout 600 ncu --clock-control none -k regex:ghx_copy_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv python scripts/thread_ranks_c3.py 1 3 > $O/thread1_pair$pr.csv 2> $O/thread1_pair$pr.err
  GHX_REMOTE_PAIR=$pr GHX_BENCH_BACKEND=gloo GHX_BARRIER_TIMEOUT_S=60 GHX_REMOTE=packed timeout 900 ncu --clock-control none --target-processes all -k regex:ghx_copy_kernel \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
      python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port $((29800 + pr)) \
      bench.py --gpus 8 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/proc8_packed_pair$pr.csv 2> $O/proc8_packed_pair$pr.err
  echo "pair=$pr done"
done
timeout 1200 python -m pytest tests/test_gpu_process.py tests/test_gpu_parity.py -q -x -m gpu -k "devsync or ipc or golden" 2>&1 | tail -2
