for C in 2 1 4 2 1 4; do
  LEGO_BUILD_ONLY=gemm_tcgen05.cu LEGO_NVCC_FLAGS="-DLEGO_GEMM_EPI_CHUNKS=$C" timeout 600 python -m paper_2505_08091_b200.build --force > /dev/null 2>&1
  echo "== chunks $C"
  for i in 1 2; do sleep 2; timeout 100 python scripts/quick_gemm.py 16 2>&1 | head -1 | cut -c1-60; done
done
