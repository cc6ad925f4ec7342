"""Time the two round-1 bandwidth outliers on a B200: the anti-diagonal inverse
index map (16384^2, int32) and the f4 even-map scatter (2^26 int32, fill mode)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402


def t(fn, it=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


g4 = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
m4 = torch.empty(16384 * 16384, device="cuda", dtype=torch.int32)
us = t(lambda: K.inv_map(g4, out=m4))
print(f"antidiag inv_map  {us:8.1f} us  {m4.numel() / us / 1e3:7.1f} Gidx/s  {m4.numel() * 4 / us / 1e3:7.1f} GB/s")
ref = K.apply_map(g4)
ok = torch.equal(m4[ref.long()], torch.arange(m4.numel(), device="cuda", dtype=torch.int32))
print("inv(apply(x)) == x:", ok)
del ref
even = L.GenP((1 << 26,), L.PermFn(lambda i: i[0] * 2, lambda i: i[0] * 2), None, name="even")
f4 = L.GroupBy([1 << 26], orders=(L.OrderBy(even),), injective=True)
x = torch.arange(1 << 26, device="cuda", dtype=torch.int32)
out = K.remap(x, None, f4)
us = t(lambda: K.remap(x, None, f4, out=out, fill=0))
nb = (x.numel() + out.numel()) * 4
print(f"f4 fill scatter   {us:8.1f} us  {nb / us / 1e3:7.1f} GB/s   (unroll {os.environ.get('LEGO_FILL_UNROLL', '4')})")
print("f4 ok:", torch.equal(out[::2], x) and not out[1::2].any())
us = t(lambda: K.remap(x, None, f4, out=out))
print(f"f4 merge scatter  {us:8.1f} us")
