#!/bin/bash
# ncu evidence for every hot kernel (run under gpurun; 1 GPU; never a multi-rank command)
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
# launch list of the bench command (cold-cache, serialised -> compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/bench_under_ncu.log 2>&1
for k in transpose gather band softmax gemm nw apply_map; do
  case $k in
    gemm) pat="regex:gemm_bf16";;
    softmax) pat="regex:softmax_rows";;
    nw) pat="regex:lego_nw_tiles";;
    apply_map) pat="regex:lego_inv_map";;
    *) pat="regex:lego_remap";;
  esac
  timeout 600 ncu --set full --clock-control none --import-source on -k $pat -s 1 -c 1 \
      -o $OUT/prof_$k -f python scripts/one_kernel.py $k 2 > $OUT/ncu_$k.log 2>&1
done
ls -la $OUT
