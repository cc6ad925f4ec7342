"""Debug helper: per-strip lag and block cadence of the NW strip kernel at
n = 16384 (debug build: LEGO_NVCC_FLAGS=-DLEGO_NW_DEBUG).  For every strip w:
the time its compute warp starts blocks 0 / 8 / 100 / 400; the steady lag
between neighbouring strips and the per-block cadence."""
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
ws = sorted(strip_of)
t0 = min(a[strip_of[w], 0, 0] for w in ws)
T = np.array([[(a[strip_of[w], 0, k] - t0) / 1000 for k in (0, 8, 100, 400)] for w in ws])
for i, w in enumerate(ws):
    if i % 8 == 0 or i == len(ws) - 1:
        print(f"strip {w:3d} cta {strip_of[w]:3d}: block0 {T[i, 0]:7.2f}  b8 {T[i, 1]:7.2f}  b100 {T[i, 2]:7.2f}  "
              f"b400 {T[i, 3]:7.2f} us")
lag = np.diff(T[:, 2])
print(f"lag at block 100 between neighbouring strips: mean {lag.mean():.2f} us  min {lag.min():.2f}  max {lag.max():.2f}")
for c in (2, 4, 8):
    inner = [lag[i] for i in range(len(lag)) if (i + 1) % c != 0]
    outer = [lag[i] for i in range(len(lag)) if (i + 1) % c == 0]
    print(f"  if clusters of {c}: in-cluster lag {np.mean(inner):.2f} us, cross-cluster {np.mean(outer):.2f} us")
cad = (T[:, 3] - T[:, 2]) / 300
print(f"block cadence (blocks 100..400): mean {cad.mean() * 1000:.1f} ns per 32-row block")
print(f"last strip finishes block 400 at {T[-1, 3]:.1f} us")
