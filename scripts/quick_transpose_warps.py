"""Register-transpose CTA size sweep on the headline layout (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
for dt in (torch.bfloat16, torch.float32):
    src = torch.randn(16384 * 16384, device="cuda").to(dt)
    out = torch.empty_like(src)
    ref = None
    for rep in range(2):
        for warps, order in ((8, "block"), (16, "block"), (16, "x"), (12, "block"), (24, "block"), (16, "y")):
            K.TRANSPOSE_WARPS, K.TILE_ORDER = warps, order
            ms = t(lambda: K.remap(src, None, g, out=out), iters=50)
            ref = out.clone() if ref is None else ref
            print(f"{str(dt):15s} warps={warps:2d} order={order:5s} {ms*1e3:7.1f} us "
                  f"{2*src.element_size()*16384**2/(ms*1e-3)/1e9:7.1f} GB/s ok={torch.equal(out, ref)}", flush=True)
    del src, out, ref
K.TRANSPOSE_WARPS, K.TILE_ORDER = 8, "block"
