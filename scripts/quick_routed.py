"""Routed (fused remap + all-to-all) transpose vs the plain transpose on one GPU:
the 8 ranks' output shards emulated as 8 buffers (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K, shard  # noqa: E402
from scripts.quick_time import t  # noqa: E402

world, n = 8, 16384
R = C = n // world
x = torch.randn(n, n, device="cuda").to(torch.bfloat16)
shards = [torch.empty(C, n, dtype=x.dtype, device="cuda") for _ in range(world)]
peers = torch.tensor([s.data_ptr() for s in shards], dtype=torch.int64, device="cuda")
routes = [shard.fused_transpose_route(R, C, world, r) for r in range(world)]


def routed_all():
    for r in range(world):
        K.remap_routed(x[r * R:(r + 1) * R].reshape(-1), None, routes[r][0], peers, routes[r][1])


ms = t(routed_all)
ok = all(torch.equal(shards[q], x.t()[q * C:(q + 1) * C]) for q in range(world))
print(f"routed, 8 ranks back to back: {ms * 1e3:.1f} us  {2 * n * n * 2 / (ms * 1e-3) / 1e9:.1f} GB/s ok={ok}")
print(K.remap_plan(None, routes[0][0], 2), "|", repr(K.plan_remap(None, routes[0][0], 2, routes[0][1])))
g = L.parse_layout(f"GroupBy([{n},{n}]).OrderBy(Col({n},{n}))")
y = torch.empty_like(x).reshape(-1)
ms = t(lambda: K.remap(x.reshape(-1), None, g, out=y))
print(f"plain transpose: {ms * 1e3:.1f} us  {2 * n * n * 2 / (ms * 1e-3) / 1e9:.1f} GB/s")
