"""Debug helper: where a strip's start-up time goes (debug build:
LEGO_NVCC_FLAGS=-DLEGO_NW_DEBUG).  For strip w and its left neighbour w-1:
for each readiness check of w's compute warp in its first blocks, the rows it
needed, when w-1's lane 31 published the last of them, when w's boundary warp
marked them ready, and when the check passed."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2505_08091_b200 import kernels as K, runtime as R  # noqa: E402

n = 16384
RPS, GRP = 4, int(os.environ.get("NW_GRP", "4"))
sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
for _ in range(3):
    K.nw_score(sim, 10)
torch.cuda.synchronize()
buf = (ctypes.c_uint * (148 * 4 * 2048))()
R.lib().lego_nw_debug_trace(buf)
a = np.frombuffer(buf, dtype=np.uint32).reshape(148, 4, 2048).astype(np.int64)
strip_of = {int(a[c, 3, 2047]) - 1: c for c in range(148) if a[c, 3, 2047] > 0}
for w in [int(x) for x in (sys.argv[1:] or ["1", "64", "127"])]:
    P, C = a[strip_of[w - 1]], a[strip_of[w]]
    base = P[3, 1536]
    print(f"strip {w} (times in ns from strip {w - 1}'s first publication):")
    rows = []
    for s in range(0, 120, GRP):
        need = min(RPS * (s + GRP + 1), n)        # rows < need
        r = need - 1
        pub = P[3, 1536 + r // 4] - base if r < 512 else -1
        rdy = C[2, 1024 + r] - base if r < 512 else -1
        chk = C[0, 1536 + s] - base
        rows.append((s, need, pub, rdy, chk))
        if s % 16 == 0:
            print(f"  step {s:3d} needs rows < {need:3d}: published {pub:7d}  ready {rdy:7d} (+{rdy - pub:5d})  "
                  f"check passed {chk:7d} (+{chk - rdy:5d})")
    x = np.array(rows[4:])
    print(f"  medians: ready - published {np.median(x[:, 3] - x[:, 2]):.0f} ns, check - ready {np.median(x[:, 4] - x[:, 3]):.0f} ns")
