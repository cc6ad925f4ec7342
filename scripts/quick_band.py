"""Band-kernel (KIND 3) knob sweep on cfg4a (16384^2 int32 row-major -> antidiag),
both directions (development helper): rows x diagonals per CTA, warps, order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402


def t(fn, iters=20, warm=5):
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


n = 16384
g = L.parse_layout(f"GroupBy([{n},{n}]).OrderBy(GenP([{n},{n}], antidiag))")
x = torch.arange(n * n, device="cuda", dtype=torch.int32)
y = torch.empty_like(x)
ref = None
variants = [v.split(",") for v in (sys.argv[1:] or ["128,32,8,1", "64,32,8,1", "128,64,8,1", "256,32,8,1",
                                                     "128,32,4,1", "128,32,16,1", "128,32,8,0", "64,64,8,1"])]
for br, bk, bw, order in variants:
    K.BAND_ROWS, K.BAND_DIAGS, K.BAND_WARPS, K.BAND_ORDER = int(br), int(bk), int(bw), int(order)
    for side in ("scatter", "gather"):
        src_l, dst_l = (None, g) if side == "scatter" else (g, None)
        try:
            ms = t(lambda: K.remap(x, src_l, dst_l, out=y))
        except Exception as exc:  # noqa: BLE001
            print(f"BR={br} BK={bk} BW={bw} order={order} {side}: {str(exc)[:80]}")
            continue
        chk = y.clone()
        print(f"BR={br:>4s} BK={bk:>3s} BW={bw:>2s} order={order} {side:7s} {ms * 1e3:7.1f} us "
              f"{2 * n * n * 4 / ms / 1e6:7.1f} GB/s  sum={int(chk.sum())}", flush=True)
