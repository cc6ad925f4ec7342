"""Run ONE hot kernel a few times (for ncu captures): python scripts/one_kernel.py NAME"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if name == "transpose":
    g = L.parse_layout("GroupBy([16384,16384]).OrderBy(Col(16384,16384))")
    x = torch.randn(16384 * 16384, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    fn = lambda: K.remap(x, None, g, out=y)  # noqa: E731
elif name == "gather":
    g = L.parse_layout("GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))")
    x = torch.randn(8, 4096 * 4096, device="cuda")
    y = torch.empty_like(x)
    fn = lambda: K.remap(x, None, g, out=y)  # noqa: E731
elif name == "band":
    g = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
    x = torch.arange(16384 * 16384, device="cuda", dtype=torch.int32)
    y = torch.empty_like(x)
    fn = lambda: K.remap(x, None, g, out=y)  # noqa: E731
elif name == "softmax":
    x = torch.randn(8192, 8192, device="cuda")
    y = torch.empty_like(x)
    fn = lambda: K.softmax(x, out=y)  # noqa: E731
elif name == "gemm":
    a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
    c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
    fn = lambda: K.gemm(a, b, out=c)  # noqa: E731
elif name.startswith("gemm_"):                      # gemm_<a layout><b layout>, e.g. gemm_colrow
    al, bl = name[5:8], name[8:11]
    a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
    c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
    fn = lambda: K.matmul(a, b, a_layout=al, b_layout=bl, out=c)  # noqa: E731
elif name.startswith("nw"):
    n = int(name[2:] or 16384)
    sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
    score = torch.empty(n + 1, n + 1, device="cuda", dtype=torch.int32)
    fn = lambda: K.nw_score(sim, 10, out=score)  # noqa: E731
elif name == "apply_map":
    g = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
    out = torch.empty(16384 * 16384, device="cuda", dtype=torch.int32)
    fn = lambda: K.inv_map(g, out=out)  # noqa: E731
elif name == "staged":
    g = L.parse_layout("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
                       ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
    x = torch.arange(8192 * 8192, device="cuda", dtype=torch.int32)
    y = torch.empty_like(x)
    fn = lambda: K.remap(x, None, g, out=y)  # noqa: E731
elif name == "expand":
    g = L.parse_layout("ExpandBy([8000,8000],[8192,8192],"
                       "GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4])))")
    x = torch.arange(8000 * 8000, device="cuda", dtype=torch.int32)     # the physical buffer
    y = K.remap(x, g, None)
    fn = lambda: K.remap(x, g, None, out=y)  # noqa: E731
elif name == "scatter":
    even = L.GenP((1 << 26,), L.PermFn(lambda idx: idx[0] * 2, lambda idx: idx[0] * 2), None, name="even")
    g = L.GroupBy([1 << 26], orders=(L.OrderBy(even),), injective=True)
    x = torch.arange(1 << 26, device="cuda", dtype=torch.int32)
    y = K.remap(x, None, g)
    fn = lambda: K.remap(x, None, g, out=y, fill=0)  # noqa: E731   (fill mode: every position written)
else:
    raise SystemExit(f"unknown kernel {name}")
for _ in range(reps):
    fn()
torch.cuda.synchronize()
