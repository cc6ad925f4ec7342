"""Quick CUDA-event timing of the hot kernels and their variants (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402


def t(fn, iters=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / iters


which = sys.argv[1:] or ["transpose", "band", "nw"]
if __name__ != "__main__":
    which = []
if "transpose" in which:
    g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
    for dt in (torch.bfloat16, torch.float32, torch.uint8):
        src = torch.randint(0, 100, (16384 * 16384,), device="cuda").to(dt)
        out = torch.empty_like(src)
        for var in ("reg", "reg2", "smem"):
            K.TRANSPOSE_VARIANT = var
            for a, b in ((None, g),):
                ms = t(lambda: K.remap(src, a, b, out=out))
                print(f"transpose {str(dt):15s} {var:5s} {'scatter' if a is None else 'gather':8s} "
                      f"{ms*1e3:8.1f} us {2*src.numel()*src.element_size()/ms/1e6:8.1f} GB/s", flush=True)
    K.TRANSPOSE_VARIANT = ""
if "band" in which:
    g = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
    for dt in (torch.int32, torch.bfloat16):
        src = torch.randint(0, 100, (16384 * 16384,), device="cuda").to(dt)
        out = torch.empty_like(src)
        for order in (0, 1):
            K.BAND_ORDER = order
            for a, b in ((None, g), (g, None)):
                ms = t(lambda: K.remap(src, a, b, out=out))
                print(f"band {str(dt):15s} order {order} {'scatter' if a is None else 'gather':8s} "
                      f"{ms*1e3:8.1f} us {2*src.numel()*src.element_size()/ms/1e6:8.1f} GB/s", flush=True)
    K.BAND_ORDER = -1
if "nw" in which:
    for n in (4096, 16384):
        sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
        score = torch.empty(n + 1, n + 1, device="cuda", dtype=torch.int32)
        ms = t(lambda: K.nw_score(sim, 10, out=score), iters=5)
        print(f"nw n={n} {ms*1e3:9.1f} us {n*n/ms/1e6:8.1f} GCUPS", flush=True)
