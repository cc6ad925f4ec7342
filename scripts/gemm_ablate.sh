#!/bin/bash
# GEMM epilogue ablation: kernel time with and without the epilogue body (results garbage)
for flags in "" "-DLEGO_GEMM_ABL_NOEPI"; do
  LEGO_BUILD_ONLY=gemm_tcgen05.cu LEGO_NVCC_FLAGS="$flags" python -m paper_2505_08091_b200.build --force > /dev/null 2>&1
  echo "== $flags"
  GS="16" bash scripts/gemm_sweep.sh 2>&1 | grep -E "gpu__time|tensor|gpc__"
  timeout 120 python scripts/quick_gemm.py 16 16 2>&1 | tail -2 | cut -c1-60
done
LEGO_BUILD_ONLY=gemm_tcgen05.cu python -m paper_2505_08091_b200.build --force > /dev/null 2>&1
