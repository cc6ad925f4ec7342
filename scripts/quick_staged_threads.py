"""Staged kernel CTA size / box size sweep on the f1 chain (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K, staging  # noqa: E402
from scripts.quick_time import t  # noqa: E402

f1 = L.parse_layout("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
                    ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
n = 8192 * 8192
for dt in (torch.int32, torch.bfloat16):
    x = torch.arange(n, device="cuda", dtype=torch.int64).to(dt)
    out = torch.empty_like(x)
    ref = None
    for thr in (128, 256, 512, 1024):
        for target in (8192, 16384, 32768):
            staging.BOX_THREADS, staging.BOX_TARGET = thr, target
            ms = t(lambda: K.remap(x, None, f1, out=out))
            if ref is None:
                ref = out.clone()
            gbs = 2 * n * x.element_size() / (ms * 1e-3) / 1e9
            print(f"{str(dt):15s} threads={thr:5d} target={target:6d} {ms * 1e3:7.1f} us {gbs:7.1f} GB/s "
                  f"ok={torch.equal(out, ref)} {K.remap_plan(None, f1, x.element_size()).detail[:40]}", flush=True)
