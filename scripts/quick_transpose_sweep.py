import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K
from scripts.quick_time import t
g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
src = torch.randn(16384 * 16384, device="cuda").to(torch.bfloat16)
out = torch.empty_like(src)
for ldv in (1, 2, 0):
    for order in ("block", "x", "y"):
        for minb in (1, 2):
            K.LOAD_HINT, K.TILE_ORDER, K.TRANSPOSE_MINB = ldv, order, minb
            ms = t(lambda: K.remap(src, None, g, out=out), iters=50)
            print(f"ldv={ldv} order={order:5s} minb={minb} {ms*1e3:7.1f} us {2*2*16384**2/(ms*1e-3)/1e9:7.1f} GB/s", flush=True)
