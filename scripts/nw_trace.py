"""Debug helper: per-CTA event timelines of the NW kernel (debug build, LEGO_NVCC_FLAGS=-DLEGO_NW_DEBUG)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_08091_b200 import kernels as K, runtime as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
for _ in range(3):
    K.nw_score(sim, 10)
torch.cuda.synchronize()
buf = (ctypes.c_uint * (148 * 4 * 2048))()
R.lib().lego_nw_debug_trace(buf)
a = np.frombuffer(buf, dtype=np.uint32).reshape(148, 4, 2048).astype(np.int64)
t0 = a[a > 0].min()
nb = (n + 31) // 32 + 2
names = ["compute block start", "producer loaded", "boundary block written", "flushed"]
ctas = [c for c in range(148) if a[c, 0, 0] > 0]
# order CTAs by their first compute start (= strip order)
ctas.sort(key=lambda c: a[c, 0, 0])
for c in ctas[: int(sys.argv[2]) if len(sys.argv) > 2 else 3] + ctas[-1:]:
    print(f"cta {c}")
    for r in range(4):
        row = a[c, r, :nb]
        print(f"  {names[r]:24s}", " ".join(f"{(x - t0) / 1000:.1f}" if x else "-" for x in row[:40]))
starts = [a[c, 0, 0] - t0 for c in ctas]
ends = [a[c, 0, nb - 1] - t0 for c in ctas]
print("strip starts (us):", " ".join(f"{x/1000:.1f}" for x in starts[:: max(1, len(starts)//16)]))
print("strip last block (us):", " ".join(f"{x/1000:.1f}" for x in ends[:: max(1, len(ends)//16)]))
