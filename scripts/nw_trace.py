"""Debug helper: per-strip event timelines of the NW kernel (debug build, LEGO_NVCC_FLAGS=-DLEGO_NW_DEBUG)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_08091_b200 import kernels as K, runtime as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
show = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3]
sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
for _ in range(3):
    K.nw_score(sim, 10)
torch.cuda.synchronize()
buf = (ctypes.c_uint * (148 * 4 * 2048))()
R.lib().lego_nw_debug_trace(buf)
a = np.frombuffer(buf, dtype=np.uint32).reshape(148, 4, 2048).astype(np.int64)
strip_of = {int(a[c, 3, 2047]) - 1: c for c in range(148) if a[c, 3, 2047] > 0}
t0 = min(a[c, 0, 0] for c in strip_of.values())
nb = (n + 31) // 32 + 2
names = ["compute block start", "producer loaded", "boundary group done", "flushed"]
for w in show:
    if w not in strip_of:
        continue
    c = strip_of[w]
    print(f"strip {w} (cta {c})")
    for r in range(4):
        row = a[c, r, :min(nb, 24)]
        print(f"  {names[r]:22s}", " ".join(f"{(x - t0) / 1000:6.2f}" if x else "     -" for x in row))
ends = [(w, (a[c, 0, nb - 1] - t0) / 1000) for w, c in sorted(strip_of.items())]
print("last block start per strip (us):", " ".join(f"{w}:{t:.1f}" for w, t in ends[:: max(1, len(ends) // 20)]))
