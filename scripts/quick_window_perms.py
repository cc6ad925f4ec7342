"""Time window-local element permutations (AoS <-> AoSoA-style interleaves)
on a B200: python scripts/quick_window_perms.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402

N = 1 << 27
for dsl in ("GroupBy([1048576,32,4]).OrderBy(RegP([1048576,32,4],[1,3,2]))",
            "GroupBy([2097152,32,2]).OrderBy(RegP([2097152,32,2],[1,3,2]))",
            "GroupBy([4194304,8,4]).OrderBy(RegP([4194304,8,4],[1,3,2]))"):
    g = L.parse_layout(dsl)
    for dt in (torch.int32, torch.bfloat16, torch.int8):
        x = torch.arange(N, device="cuda", dtype=torch.int64).to(dt) if dt != torch.bfloat16 else \
            torch.randn(N, device="cuda").to(dt)
        for side in ("to", "from"):
            sl, dl = (None, g) if side == "to" else (g, None)
            y = K.remap(x, sl, dl)
            for _ in range(3):
                K.remap(x, sl, dl, out=y)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                K.remap(x, sl, dl, out=y)
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / 10 * 1e3
            plan = K.remap_plan(sl, dl, x.element_size())
            print(f"{dsl[:44]:44s} {str(dt):15s} {side:4s} {us:8.1f} us {2 * x.numel() * x.element_size() / us / 1e3:7.1f} GB/s  {repr(plan)[:70]}",
                  flush=True)
        del x, y
