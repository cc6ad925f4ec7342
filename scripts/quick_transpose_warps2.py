import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K


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
g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
for dt in (torch.bfloat16, torch.int64):
    src = torch.randint(-99, 99, (16384 * 16384,), device="cuda").to(dt)
    out = torch.empty_like(src)
    res = {}
    for rep in range(3):
        for warps in (8, 12, 16, 10, 14):
            K.TRANSPOSE_WARPS = warps
            ms = t(lambda: K.remap(src, None, g, out=out), iters=100)
            res.setdefault(warps, []).append(ms * 1e3)
    for w, v in res.items():
        print(f"{str(dt):15s} warps={w:2d} " + " ".join(f"{x:7.1f}" for x in v) +
              f"  best {2*src.element_size()*16384**2/(min(v)*1e-6)/1e9:7.1f} GB/s", flush=True)
    del src, out
