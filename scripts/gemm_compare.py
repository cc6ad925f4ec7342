"""One launch each of the LEGO GEMM (pair and single-CTA kernels) and cuBLAS at 8192^3 (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_08091_b200 import kernels as K  # noqa: E402

a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    K.gemm(a, b, out=c, raster=int(os.environ.get("G", "0")))
    torch.matmul(a, b.t(), out=c)
torch.cuda.synchronize()
