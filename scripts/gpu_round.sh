#!/bin/bash
# one GPU session: tests, bench, headline launch list, top-kernel ncu captures
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x --durations=8 > $OUT/pytest_gpu.txt 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_headline.csv python bench.py --steps 5 --warmup 3 --no-cpu --headline-only \
    > $OUT/bench_headline_under_ncu.log 2>&1
for k in ${KERNELS:-transpose band nw}; do
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
tail -15 $OUT/pytest_gpu.txt
cat $OUT/bench.json
