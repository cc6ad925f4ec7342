"""Transpose kernel variants on the headline layout (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402


def t(fn, iters=30, warm=5):
    """Median-free mean time (ms) of fn over `iters` launches after `warm`, CUDA events."""
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

g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
for dt in (torch.bfloat16, torch.float32):
    src = torch.randint(0, 100, (16384 * 16384,), device="cuda").to(dt)
    out = torch.empty_like(src)
    for var in (sys.argv[1:] or ["reg", "regT", "smem"]):
        for order in ("x", "y", "block"):
            K.TRANSPOSE_VARIANT = var
            K.TILE_ORDER = order
            ms = t(lambda: K.remap(src, None, g, out=out))
            ok = torch.equal(out.view(16384, 16384), src.view(16384, 16384).t())
            print(f"transpose {str(dt):15s} {var:5s} order={order:5s} {ms*1e3:8.1f} us "
                  f"{2*src.numel()*src.element_size()/ms/1e6:8.1f} GB/s ok={ok}", flush=True)
