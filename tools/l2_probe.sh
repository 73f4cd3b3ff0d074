#!/bin/bash
# L2 (LTS) vs DRAM traffic of the hot kernels: is a kernel HBM-bound or
# LTS-throughput-bound?  One ncu pass with a short metric list per workload.
set -e
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum
out=${1:-gpurun_out}
ncu --metrics $M --clock-control none -k regex:k_fastfood_pair -s 2 -c 1 --csv python tools/prof_ff.py ff > $out/l2_ff.csv 2>&1
ncu --metrics $M --clock-control none -k regex:fwht_rows -s 2 -c 1 --csv python tools/prof_ff.py fwht 1024 > $out/l2_fwht1024.csv 2>&1
ncu --metrics $M --clock-control none -k regex:fwht -s 100 -c 4 --csv python tools/prof_ff.py fwht 1048576 > $out/l2_fwht2p20.csv 2>&1
ncu --metrics $M --clock-control none -k regex:fwht_cluster -s 2 -c 1 --csv python tools/prof_ff.py fwht 65536 > $out/l2_fwht2p16.csv 2>&1
ncu --metrics $M --clock-control none -k regex:k_fastfood -s 4 -c 1 --csv python tools/prof_ff.py c4 > $out/l2_c4z.csv 2>&1
