#!/usr/bin/env bash
# Profiling pass on one GPU (run under gpurun from the repo root):
#   ncu launch list of the headline bench command (C3), one --set full capture
#   of ghx_copy_kernel, per-config DRAM traffic, and the bench lines.
mkdir -p gpurun_out/prof
export PYTHONDONTWRITEBYTECODE=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_C2.csv python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/prof/launches_C2.log 2>&1
echo "launch list rc=$?"
for c in C2 C3 C4 C5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ghx_copy_kernel -s 4 -c 1 -f \
    -o gpurun_out/prof/full_$c python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/prof/full_$c.log 2>&1
  echo "full $c rc=$?"
done
for c in C1 C2 C3 C4 C5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv -k regex:ghx_copy_kernel -s 4 -c 1 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/prof/traffic_$c.csv 2> gpurun_out/prof/traffic_$c.err
  echo "traffic $c rc=$?"
done
for c in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps ${BENCH_STEPS:-200} --warmup 5 > gpurun_out/prof/bench_$c.json 2> gpurun_out/prof/bench_$c.log
  echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/prof/bench_ref_C2.json 2> gpurun_out/prof/bench_ref_C2.log
echo "bench ref rc=$?"
# level transfers
for op in fill_patch average_down heat heat2; do
  timeout 600 python bench_amr.py --op $op > gpurun_out/prof/bench_amr_$op.json 2> gpurun_out/prof/bench_amr_$op.log
  echo "bench_amr $op rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:"interp_kernel|avgdown_kernel" -c 2 python bench_amr.py --op fill_patch --steps 3 --warmup 3 \
  > gpurun_out/prof/traffic_interp.csv 2> gpurun_out/prof/traffic_interp.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:"avgdown_kernel" -c 2 python bench_amr.py --op average_down --steps 3 --warmup 3 \
  > gpurun_out/prof/traffic_avgdown.csv 2> gpurun_out/prof/traffic_avgdown.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:"advance_kernel" -c 2 python bench_amr.py --op heat --steps 3 --warmup 3 \
  > gpurun_out/prof/traffic_advance.csv 2> gpurun_out/prof/traffic_advance.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"advance_kernel" -c 1 -f \
  -o gpurun_out/prof/full_advance python bench_amr.py --op heat --steps 3 --warmup 3 > gpurun_out/prof/full_advance.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_fill_patch.csv python bench_amr.py --op fill_patch --steps 3 --warmup 3 \
  > gpurun_out/prof/launches_fill_patch.log 2>&1
echo "amr ncu done"
# microbenchmarks behind the roofline discussion
(cd scripts/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/seam_probe seam_probe.cu \
  && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pcie_probe pcie_probe.cu) \
  && /tmp/seam_probe 544 > gpurun_out/prof/seam_probe_544.txt && /tmp/seam_probe 1056 > gpurun_out/prof/seam_probe_1056.txt \
  && /tmp/pcie_probe > gpurun_out/prof/pcie_probe.txt
echo "probes rc=$?"
