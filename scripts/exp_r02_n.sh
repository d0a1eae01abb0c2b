# r02 experiment N: host-memory seam pack / unpack tasks for remote x faces
# across processes (one GPU, gloo): parity, then e2e at 2/4/8 ranks with
# GHX_SEAM_TASKS=1 (default) and 0.  e2e of processes sharing one GPU and
# its PCIe link: every rank's kernels run in turn, so the per-step time is
# the sum of the ranks' PCIe work -- comparable between the two variants.
set -u
mkdir -p gpurun_out/expN
O=gpurun_out/expN
timeout 1500 python -m pytest tests/test_gpu_process_random.py tests/test_gpu_process.py -q -x -m gpu -k "pinned or C3x4 or two" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
tail -3 $O/tests.log
for n in 2 4 8; do
  for st in 1 0; do
    GHX_SEAM_TASKS=$st GHX_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29800 + 10 * n + st)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu \
      --e2e-steps 5 > $O/e2e_n${n}_seam$st.json 2> $O/e2e_n${n}_seam$st.err
    python -c "import json; d=json.loads(open('$O/e2e_n${n}_seam$st.json').read().strip().splitlines()[-1]); e=d['e2e']; print('n=$n seam=$st', e['value'], e['ms_per_step'], e['verified'])"
  done
done
