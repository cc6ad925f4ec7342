"""GEMM raster-group sweep with SM clock sampling (development helper).

    python scripts/quick_gemm.py [G ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402
from bench import ClockSampler  # noqa: E402

a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
gs = [int(x) for x in sys.argv[1:]] or [16, 0, 8, 16, 32, 0]
for g in gs:
    with ClockSampler(0) as clk:
        ms = t(lambda: K.gemm(a, b, out=c, raster=g), iters=20)
    print(f"gemm raster G={g:3d} {ms*1e3:8.1f} us {2*8192**3/ms/1e9:8.1f} TFLOP/s  clocks {clk.summary()}", flush=True)
with ClockSampler(0) as clk:
    ms = t(lambda: torch.matmul(a, b.t(), out=c), iters=20)
print(f"torch.matmul (cuBLAS) {ms*1e3:8.1f} us {2*8192**3/ms/1e9:8.1f} TFLOP/s  clocks {clk.summary()}")
