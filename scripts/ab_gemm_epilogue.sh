for V in 1 0 1 0; do
  LEGO_BUILD_ONLY=gemm_tcgen05.cu LEGO_NVCC_FLAGS="-DLEGO_GEMM_EARLY_RELEASE=$V" timeout 600 python -m paper_2505_08091_b200.build --force > /dev/null 2>&1
  echo "== early release $V"
  [ $V = 1 ] && timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k "gemm or matmul" 2>&1 | tail -1
  for i in 1 2 3; do sleep 3; timeout 100 python scripts/quick_gemm.py 16 2>&1 | head -1 | cut -c1-60; done
done
