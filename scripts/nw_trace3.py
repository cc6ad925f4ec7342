"""Debug helper: per-role timelines of one NW strip in the steady state
(debug build: LEGO_NVCC_FLAGS=-DLEGO_NW_DEBUG).  For strips 0, 64 and 127:
the cadence of each role over blocks 100..400 and how far each role runs
ahead of / behind the compute warp (compute block start k, producer landed
k, boundary group k complete, flusher done k)."""
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
t0 = min(a[c, 0, 0] for c in strip_of.values())
names = ["compute start", "producer landed", "boundary group", "flusher done"]
for w in (0, 64, 127):
    c = strip_of[w]
    T = (a[c] - t0) / 1000.0
    print(f"strip {w} (cta {c}): compute block 0 at {T[0, 0]:.2f} us")
    for role in range(4):
        cad = (T[role, 400] - T[role, 100]) / 300 * 1000
        rel = T[role, 100:400] - T[0, 100:400]
        print(f"  {names[role]:16s} cadence {cad:7.1f} ns/block   minus compute start (same k): "
              f"median {np.median(rel):8.2f} us  min {rel.min():8.2f}  max {rel.max():8.2f}")
    d = np.diff(T[0, 100:400]) * 1000
    print(f"  compute block durations: p10 {np.percentile(d, 10):.0f}  median {np.median(d):.0f}  p90 {np.percentile(d, 90):.0f} ns")
print()
ks = np.arange(100, 400)
for w in (0, 64, 127):
    c = strip_of[w]
    T = (a[c] - t0) / 1000.0
    comp_start, comp_in = T[0, ks], T[0, 1024 + ks]
    issued, landed = T[1, 1024 + ks], T[1, ks]
    f_start, f_done = T[3, 1024 + ks], T[3, ks]
    med = lambda x: f"{np.median(x) * 1000:7.0f}"
    print(f"strip {w}: ns medians -- compute waits for operands {med(comp_in - comp_start)}, "
          f"block k+1 issue->landed {med(T[1, ks + 1] - T[1, 1024 + ks + 1])}, "
          f"flush work {med(f_done - f_start)}, flush start - computed publication {med(f_start - T[0, ks + 2]) if False else ''}")
    print(f"   flush start(k) - compute start(k+BLAG=2) {med(f_start - T[0, ks + 2])}, (k+5) {med(f_start - T[0, ks + 5])};"
          f" issue(k) - flush done(k-12) {med(T[1, 1024 + ks] - T[3, ks - 12])}, (k-8) {med(T[1, 1024 + ks] - T[3, ks - 8])}")
print()
# strip w's lane 31 finishes rows 32m..32m+31 in its last step of compute block m + SKEW
# (~ compute start of block m + SKEW + 1); strip w+1's boundary warp has handed the
# whole group once its lane 31 logs group m
skew = int(os.environ.get("NW_SKEW", "1"))
hs = []
for w in range(1, 127):
    cw, cn = strip_of[w], strip_of[w + 1]
    Tw, Tn = (a[cw] - t0) / 1000.0, (a[cn] - t0) / 1000.0
    hs.append(np.median(Tn[2, ks] - Tw[0, ks + skew + 1]))
    if w in (1, 64, 126):
        need = Tn[0, ks] - Tn[2, ks]
        print(f"strip {w}->{w + 1}: group m handed - producer strip's compute start(m+{skew + 1}) median {hs[-1] * 1000:.0f} ns;"
              f" consumer compute start(k) - its boundary group k handed {np.median(need) * 1000:.0f} ns")
print(f"hand-off latency over strips: median {np.median(hs) * 1000:.0f} ns, mean {np.mean(hs) * 1000:.0f}")
