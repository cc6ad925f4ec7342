#!/bin/bash
# NW compute-step ablations in micro mode (helpers idle, results garbage): block time per variant
for flags in "" "-DNW_ABL_NOSTS" "-DNW_ABL_NOPUB" "-DNW_ABL_NOLDS" "-DNW_ABL_NOSTS -DNW_ABL_NOPUB -DNW_ABL_NOLDS"; do
  LEGO_BUILD_ONLY=wavefront.cu LEGO_NVCC_FLAGS="-DLEGO_NW_DEBUG -DNW_MICRO=1 $flags" python -m paper_2505_08091_b200.build --force > /dev/null 2>&1
  echo "== micro $flags"
  timeout 60 python scripts/nw_trace.py 16384 0 2>&1 | grep -A1 "strip 0" | tail -1 | cut -c1-120
done
