"""Box-staged gather variants on the SURVEY f1 chain (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K, staging  # noqa: E402


def t(fn, iters=30, warm=5):
    """Mean time (ms) of fn over `iters` launches after `warm`, CUDA events."""
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters

f1 = L.parse_layout("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
                    ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
n = 8192 * 8192
for dt in (torch.int32, torch.bfloat16, torch.uint8, torch.int64):
    x = torch.arange(n, device="cuda", dtype=torch.int64).to(dt)
    ref = None
    for box, target, store, bulk in ((0, 16384, "", 0), (1, 16384, "", 0), (1, 16384, "", 1),
                                     (1, 8192, "", 1), (1, 32768, "", 1), (1, 16384, "scalar", 1)):
        K.BOX_STAGING, staging.BOX_TARGET, staging.BOX_STORE, staging.BOX_BULK = box, target, store, bulk
        out = torch.empty_like(x)
        ms = t(lambda: K.remap(x, None, f1, out=out))
        if ref is None:
            ref = out.clone()
        ok = torch.equal(out, ref)
        gbs = 2 * n * x.element_size() / (ms * 1e-3) / 1e9
        print(f"{str(dt):15s} box={box} bulk={bulk} target={target:6d} store={store or 'auto':6s} {ms * 1e3:8.1f} us "
              f"{gbs:7.1f} GB/s ok={ok}  {K.remap_plan(None, f1, x.element_size()).detail}", flush=True)
    for box in (0, 1):
        K.BOX_STAGING, staging.BOX_TARGET, staging.BOX_STORE = box, 16384, ""
        y = K.remap(x, None, f1)
        out = torch.empty_like(x)
        ms = t(lambda: K.remap(y, f1, None, out=out))
        gbs = 2 * n * x.element_size() / (ms * 1e-3) / 1e9
        print(f"{str(dt):15s} from-layout box={box} {ms * 1e3:8.1f} us {gbs:7.1f} GB/s "
              f"ok={torch.equal(out, x)}  {K.remap_plan(f1, None, x.element_size()).detail}", flush=True)
    del x, out, ref, y
