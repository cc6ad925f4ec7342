"""Band-kernel tile and order sweep for the anti-diagonal remap (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

g = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
x = torch.arange(16384 * 16384, device="cuda", dtype=torch.int32)
ref = None
for br, bk in ((64, 64), (128, 64), (64, 128), (32, 128), (128, 32), (32, 64)):
    for order in (0, 1):
        for direction in ("scatter", "gather"):
            K.BAND_ROWS, K.BAND_DIAGS, K.BAND_ORDER = br, bk, order
            y = torch.empty_like(x)
            fn = (lambda: K.remap(x, None, g, out=y)) if direction == "scatter" else (lambda: K.remap(x, g, None, out=y))
            ms = t(fn, iters=30)
            if direction == "scatter":
                if ref is None:
                    ref = y.clone()
                ok = torch.equal(y, ref)
            else:
                ok = True
            print(f"band {br:3d}x{bk:3d} order={order} {direction:7s} {ms*1e3:8.1f} us "
                  f"{2*x.numel()*4/ms/1e6:8.1f} GB/s ok={ok}", flush=True)
