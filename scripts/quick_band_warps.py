"""Band kernel warps-per-CTA sweep (cfg4a, both directions; development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

g = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
x = torch.arange(16384 * 16384, device="cuda", dtype=torch.int32)
y = torch.empty_like(x)
ref = {}
for rep in range(2):
    for bw in (8, 4, 16):
        K.BAND_WARPS = bw
        for name, a, b in (("scatter", None, g), ("gather", g, None)):
            ms = t(lambda: K.remap(x, a, b, out=y), iters=30)
            key = name
            ref.setdefault(key, y.clone())
            print(f"warps={bw:2d} {name:8s} {ms*1e3:7.1f} us {2*4*16384**2/(ms*1e-3)/1e9:7.1f} GB/s "
                  f"ok={torch.equal(y, ref[key])}", flush=True)
