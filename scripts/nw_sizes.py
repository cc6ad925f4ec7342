import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_08091_b200 import kernels as K
from scripts.quick_time import t
for n in (256, 512, 1024, 2048, 4096, 8192, 16384):
    sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
    score = torch.empty(n + 1, n + 1, device="cuda", dtype=torch.int32)
    ms = t(lambda: K.nw_score(sim, 10, out=score), iters=5)
    print(f"nw n={n:6d} {ms*1e3:9.1f} us {n*n/ms/1e6:8.1f} GCUPS", flush=True)
