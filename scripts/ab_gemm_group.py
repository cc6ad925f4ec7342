"""GEMM raster group A/B with cool-down pauses (development helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_08091_b200 import kernels as K  # noqa: E402
from bench import ClockSampler  # noqa: E402


def t(fn, iters=30, warm=5):
    """Mean time (ms) of fn over `iters` launches after `warm`, CUDA events."""
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters

a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
gs = [int(x) for x in sys.argv[1:]] or [16, 32]
res = {g: [] for g in gs}
for rep in range(4):
    for g in gs:
        time.sleep(3)
        with ClockSampler(0) as clk:
            ms = t(lambda: K.gemm(a, b, out=c, raster=g), iters=20)
        res[g].append((round(ms * 1e3, 1), clk.summary()["sm_mhz"]))
for g, v in res.items():
    print(f"G={g:3d}", " ".join(f"{us}us@{mhz}" for us, mhz in v))
