"""Occupancy knob of the register transpose (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
for dt in (torch.bfloat16, torch.float32):
    src = torch.randint(0, 100, (16384 * 16384,), device="cuda").to(dt)
    out = torch.empty_like(src)
    for minb in (1, 4, 5, 6, 8):
        for order in ("block", "x"):
            K.TRANSPOSE_MINB = minb
            K.TILE_ORDER = order
            ms = t(lambda: K.remap(src, None, g, out=out), iters=50)
            print(f"{str(dt):15s} minb={minb} order={order:5s} {ms*1e3:8.1f} us "
                  f"{2*src.numel()*src.element_size()/ms/1e6:8.1f} GB/s", flush=True)
