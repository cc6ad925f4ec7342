"""Remap throughput of irregular (non-transpose, non-contiguous) layouts (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from scripts.quick_time import t  # noqa: E402

cases = [
    "GroupBy([4096,4096]).OrderBy(RegP([64,64,64,64],[1,3,2,4])).OrderBy(Row(64,64), GenP([64,64], antidiag))",
    "GroupBy([4096,4096]).OrderBy(RegP([64,64,64,64],[1,3,2,4])).OrderBy(GenP([64,64], antidiag), GenP([64,64], antidiag))",
    "GroupBy([8192,2048]).OrderBy(RegP([8192,2048],[2,1]))",
    "GroupBy([4096,4096]).OrderBy(RegP([16,256,16,256],[3,1,4,2]))",
]
for dsl in cases:
    g = L.parse_layout(dsl)
    for dt in (torch.float32, torch.bfloat16):
        x = torch.randn(g.size, device="cuda").to(dt)
        for name, fn in (("to-layout", lambda: K.remap(x, None, g)), ("from-layout", lambda: K.remap(x, g, None))):
            ms = t(fn, iters=20)
            plan = K.remap_plan(None, g, x.element_size()) if name == "to-layout" else K.remap_plan(g, None, x.element_size())
            print(f"{dsl[:60]:60s} {str(dt)[6:]:9s} {name:11s} {ms*1e3:8.1f} us {2*x.numel()*x.element_size()/ms/1e6:7.1f} GB/s  {plan}", flush=True)
