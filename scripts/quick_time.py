"""Quick CUDA-event timing of the remap programs (development helper)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K

def t(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(iters):
        s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

cases = [
 ("cfg1 tiled fp32", "GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))", torch.float32, 8),
 ("cfg2 transpose bf16", "GroupBy([16384,16384]).OrderBy(Col(16384,16384))", torch.bfloat16, 1),
 ("cfg2 transpose fp32", "GroupBy([16384,16384]).OrderBy(Col(16384,16384))", torch.float32, 1),
 ("cfg4 antidiag int32", "GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))", torch.int32, 1),
]
for name, dsl, dt, batch in cases:
    g = L.parse_layout(dsl)
    n = g.size
    src = torch.randn(batch, n, device="cuda").to(dt)
    out = torch.empty_like(src)
    for direction in ("scatter", "gather"):
        a, b = (None, g) if direction == "scatter" else (g, None)
        ms = t(lambda: K.remap(src, a, b, out=out))
        gbs = 2 * src.numel() * src.element_size() / ms / 1e6
        print(f"{name:24s} {direction:8s} {ms*1e3:9.1f} us  {gbs:8.1f} GB/s  plan={K.remap_plan(a, b, src.element_size())}", flush=True)
    ms = t(lambda: K.apply_map(g, out=torch.empty(n, dtype=torch.int32, device='cuda')))
    print(f"{name:24s} apply_map {ms*1e3:9.1f} us  {4*n/ms/1e6:8.1f} GB/s (write)", flush=True)
x = torch.randn(8192, 8192, device="cuda")
ms = t(lambda: K.softmax(x))
print(f"softmax 8192^2 {ms*1e3:.1f} us {2*x.numel()*4/ms/1e6:.1f} GB/s")
ms = t(lambda: src.clone())
print("copy", ms)
