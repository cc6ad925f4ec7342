"""Cache-hint variants of the headline transpose, gather and band remaps (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

cases = [("transpose bf16", "GroupBy([16384,16384]).OrderBy(Col(16384,16384))", torch.bfloat16, 16384 * 16384),
         ("band i32", "GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))", torch.int32, 16384 * 16384),
         ("gather f32 b8", "GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))", torch.float32, 8 * 4096 * 4096)]
for name, dsl, dt, numel in cases:
    g = L.parse_layout(dsl)
    src = torch.randint(0, 100, (numel,), device="cuda").to(dt)
    out = torch.empty_like(src)
    for ldv in (0, 1, 2, 3):
        for stv in (0, 1, 2):
            K.LOAD_HINT, K.STORE_HINT = ldv, stv
            ms = t(lambda: K.remap(src, None, g, out=out), iters=50)
            print(f"{name:15s} ldv={ldv} stv={stv} {ms*1e3:8.1f} us {2*numel*src.element_size()/ms/1e6:8.1f} GB/s",
                  flush=True)
