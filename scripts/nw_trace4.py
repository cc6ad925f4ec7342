"""Debug helper: start-up of the NW strip pipeline (debug build:
LEGO_NVCC_FLAGS=-DLEGO_NW_DEBUG).  For a few strips w, event times relative to
the left strip's compute start of block 0: compute block starts 0..3, operands
in (block 0), boundary groups 0..2 handed, and the left strip's own block starts."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2505_08091_b200 import kernels as K, runtime as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
for _ in range(3):
    K.nw_score(sim, 10)
torch.cuda.synchronize()
buf = (ctypes.c_uint * (148 * 4 * 2048))()
R.lib().lego_nw_debug_trace(buf)
a = np.frombuffer(buf, dtype=np.uint32).reshape(148, 4, 2048).astype(np.int64)
strip_of = {int(a[c, 3, 2047]) - 1: c for c in range(148) if a[c, 3, 2047] > 0}
lags = []
for w in range(1, 128):
    T = (a[strip_of[w]] - a[strip_of[w - 1], 0, 0]) / 1000.0
    P = (a[strip_of[w - 1]] - a[strip_of[w - 1], 0, 0]) / 1000.0
    lags.append(T[0, 0])
    if w in (1, 2, 3, 64, 127):
        print(f"strip {w}: left strip blocks 0..3 at {P[0, 0]:.2f} {P[0, 1]:.2f} {P[0, 2]:.2f} {P[0, 3]:.2f}; "
              f"mine {T[0, 0]:.2f} {T[0, 1]:.2f} {T[0, 2]:.2f} {T[0, 3]:.2f} (block 8 {T[0, 8]:.2f}, left's {P[0, 8]:.2f}); "
              f"operands in (blk 0) {T[0, 1024]:.2f}; bnd groups handed {T[2, 0]:.2f} {T[2, 1]:.2f} {T[2, 2]:.2f}; "
              f"landed 0/1 {T[1, 0]:.2f} {T[1, 1]:.2f}")
print(f"block-0 lag behind the left strip: median {np.median(lags):.2f} us")
