#!/bin/bash
# GEMM raster sweep under ncu: clock, tensor activity, DRAM and L2->SM bytes per raster group
M=gpc__cycles_elapsed.max.per_second,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum
for g in ${GS:-0 1 2 4 8 16 32}; do
  echo "== G=$g pair=${LEGO_GEMM_PAIR:-1}"
  G=$g timeout 120 ncu --metrics $M --clock-control none -k regex:"gemm_bf16" -s 2 -c 1 python scripts/gemm_compare.py 2>&1 \
    | grep -E "dram__|gpc__|gpu__time|xbar2l1tex|tensor" | awk '{print "   ", $1, $NF, $(NF-1)}'
done
