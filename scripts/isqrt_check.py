"""Exhaustive device check of lego_isqrt32 over [0, 2^31) against an exact integer root."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402

# inv_map of antidiag(n) runs isqrt(8x+1) over the whole lower triangle; compare with
# a float64 reference of the same inverse for n = 16384 (8x+1 < 2^31)
n = 16384
g = L.parse_layout(f"GroupBy([{n},{n}]).OrderBy(GenP([{n},{n}], antidiag))")
inv = K.inv_map(g)
app = K.apply_map(g)
ok = torch.equal(app[inv.long()], torch.arange(n * n, device="cuda", dtype=app.dtype))
print("apply(inv(f)) == f for all", n * n, "positions:", ok)
