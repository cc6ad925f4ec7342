"""The four Row/Col data-layout matmul variants at 8192^3 (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

n = 8192
a = torch.randn(n, n, device="cuda").to(torch.bfloat16)
b = torch.randn(n, n, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
import time  # noqa: E402

# two passes in opposite orders with a pause between variants: sustained
# back-to-back GEMMs run power-capped, so a fixed order biases the last ones
variants = [(al, bl) for al in ("row", "col") for bl in ("row", "col")]
for order in (variants, variants[::-1]):
    for al, bl in order:
        time.sleep(2)
        ms = t(lambda: K.matmul(a, b, a_layout=al, b_layout=bl, out=c), iters=20)
        print(f"matmul A={al} B={bl} {ms*1e3:8.1f} us {2*n**3/ms/1e9:8.1f} TFLOP/s", flush=True)
