"""NW at n = 16384 under tiled LEGO layouts of several tile heights and tile
orders (B200): python scripts/quick_nw_tiles.py"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2505_08091_b200 import kernels as K, nw  # noqa: E402
from nw_perms import skew_order  # noqa: E402

n = 16384
sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
out = torch.empty(n + 1, n + 1, device="cuda", dtype=torch.int32)
ref = K.nw_score(sim, 10).clone()
cases = [("strips", nw.nw_layout(n))]
for h in (512, 1024, 2048, 4096):
    nr = n // h
    cases += [(f"H{h} row", nw.nw_layout(n, tile_rows=h, tile_order="row")),
              (f"H{h} skew(user)", nw.nw_layout(n, tile_rows=h, tile_order=skew_order(nr, 128)))]
for name, lay in cases:
    K.nw_score(sim, 10, layout=lay, out=out)
    ok = torch.equal(out, ref)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        K.nw_score(sim, 10, layout=lay, out=out)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 3 * 1e3
    print(f"{name:18s} {us:8.1f} us {n * n / us / 1e3:7.1f} GCUPS match={ok}", flush=True)
