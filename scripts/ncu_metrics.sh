#!/usr/bin/env bash
# Key memory metrics of ghx_copy_kernel: ncu_metrics.sh TAG "ENVS" bench-args...
TAG=$1; ENVS=$2; shift 2
env $ENVS timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct \
  -k regex:ghx_copy_kernel -s 4 -c 1 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu "$@" 2>&1 | grep -E "^    [a-z]" | sed "s/^/$TAG /"
