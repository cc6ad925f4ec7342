#!/bin/bash
# GEMM epilogue TMEM-load batching sweep
for ch in 2 4 8; do
  LEGO_BUILD_ONLY=gemm_tcgen05.cu LEGO_NVCC_FLAGS="-DLEGO_GEMM_EPI_CHUNKS=$ch" python -m paper_2505_08091_b200.build --force > /dev/null 2>&1
  echo "== chunks $ch"
  GS="16" bash scripts/gemm_sweep.sh 2>&1 | grep -E "gpu__time|tensor"
  timeout 120 python scripts/quick_gemm.py 16 16 2>&1 | tail -3 | cut -c1-60
done
LEGO_BUILD_ONLY=gemm_tcgen05.cu python -m paper_2505_08091_b200.build --force > /dev/null 2>&1
