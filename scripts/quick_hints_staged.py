import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2505_08091_b200 as L
from paper_2505_08091_b200 import kernels as K
from scripts.quick_time import t
f1 = L.parse_layout("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4])).OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
g1 = L.parse_layout("GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))")
x = torch.arange(8192 * 8192, device="cuda", dtype=torch.int32); y = torch.empty_like(x)
x1 = torch.randn(8, 4096 * 4096, device="cuda"); y1 = torch.empty_like(x1)
for rep in range(2):
    for h in (1, 0, 2, 3):
        K.LOAD_HINT = h
        ms = t(lambda: K.remap(x, None, f1, out=y), iters=50)
        ms1 = t(lambda: K.remap(x1, None, g1, out=y1), iters=20)
        print(f"ldv={h} f1 {ms*1e3:6.1f} us {2*4*8192**2/(ms*1e-3)/1e9:7.1f} GB/s | cfg1 {ms1*1e3:6.1f} us {2*x1.numel()*4/(ms1*1e-3)/1e9:7.1f} GB/s", flush=True)
