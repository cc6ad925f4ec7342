"""Time the NW wavefront at n = 16384 under several LEGO layouts (B200)."""
import sys
import time

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2505_08091_b200 import kernels as K, nw  # noqa: E402
from nw_perms import nw_test_layouts  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
out = torch.empty(n + 1, n + 1, device="cuda", dtype=torch.int32)
cases = [("static", None)] + nw_test_layouts(n)
for name, lay in cases:
    t0 = time.time()
    K.nw_score(sim, 10, layout=lay, out=out)
    torch.cuda.synchronize()
    setup = time.time() - t0
    ref = out.clone() if name == "static" else ref
    ok = torch.equal(out, ref)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(2):
        K.nw_score(sim, 10, layout=lay, out=out)
    evs[0].record()
    for _ in range(5):
        K.nw_score(sim, 10, layout=lay, out=out)
    evs[1].record()
    torch.cuda.synchronize()
    us = evs[0].elapsed_time(evs[1]) / 5 * 1e3
    print(f"{name:28s} {us:9.1f} us  {n * n / us / 1e3:7.1f} GCUPS  match={ok}  setup={setup:.2f}s "
          f"{nw.describe(lay) if lay is not None else ''}", flush=True)
