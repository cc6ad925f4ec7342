"""Staged vs per-element gather on chains with non-power-of-two tiles (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

for text in ("GroupBy([6144,6144]).OrderBy(RegP([256,24,256,24],[1,3,2,4]))"
             ".OrderBy(RegP([256,256],[2,1]), GenP([24,24], antidiag))",
             "GroupBy([6144,6144]).OrderBy(RegP([128,48,128,48],[1,3,2,4]))"
             ".OrderBy(RegP([128,128],[2,1]), GenP([48,48], rev2d))"):
    g = L.parse_layout(text)
    n = 6144 * 6144
    x = torch.arange(n, device="cuda", dtype=torch.int32)
    out = torch.empty_like(x)
    ref = None
    for box in (0, 1):
        K.BOX_STAGING = box
        ms = t(lambda: K.remap(x, None, g, out=out))
        ref = out.clone() if ref is None else ref
        print(f"box={box} {ms * 1e3:7.1f} us {2 * n * 4 / (ms * 1e-3) / 1e9:7.1f} GB/s ok={torch.equal(out, ref)} "
              f"{K.remap_plan(None, g, 4).detail[:60]}", flush=True)
