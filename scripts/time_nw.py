"""Time the library NW kernel (kernels.nw_score, default strip layout) at
n = 16384 and check it against the C DP: python scripts/time_nw.py [n] [reps].
Run with LEGO_B200_LIB=<an A/B build of liblego_b200.so> to compare builds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rng = np.random.default_rng(4)
sim_h = rng.integers(-10, 11, size=(n, n), dtype=np.int32)
sim = torch.from_numpy(sim_h).cuda()
out = K.nw_score(sim, 10)
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    K.nw_score(sim, 10, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ok = "unchecked"
if os.environ.get("NW_CHECK", "1") == "1":
    from oracle import oracle as O
    ok = bool(np.array_equal(out.cpu().numpy(), O.nw(sim_h, 10)))
print(f"{os.environ.get('LEGO_B200_LIB', 'in-tree lib')}: n={n} median {sorted(ts)[len(ts) // 2]:.1f} us best {min(ts):.1f} us exact={ok}")
