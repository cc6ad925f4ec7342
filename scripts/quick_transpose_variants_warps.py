import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K
from scripts.quick_time import t
g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
src = torch.randint(-99, 99, (16384 * 16384,), device="cuda").to(torch.bfloat16)
out = torch.empty_like(src)
for rep in range(2):
    for var in ("regT", "reg"):
        for w in (8, 12, 16):
            K.TRANSPOSE_VARIANT, K.TRANSPOSE_WARPS = var, w
            ms = t(lambda: K.remap(src, None, g, out=out), iters=50)
            print(f"{var:5s} warps={w:2d} {ms*1e3:7.1f} us {4*16384**2/(ms*1e-3)/1e9:7.1f} GB/s", flush=True)
