"""Randomised remap parity sweep on the GPU (development helper): random
layouts, tiled chains and ExpandBy layouts from tests/random_layouts.py with
a fresh seed, every element size, both directions, against the C oracle."""
import os
import random
import sys
import collections

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K  # noqa: E402
from oracle import oracle as O  # noqa: E402
from random_layouts import random_layout, tiled_chain, random_expand  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 12345
count = int(sys.argv[2]) if len(sys.argv) > 2 else 150
rng = random.Random(seed)
NP = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}
kinds = collections.Counter()
checked = 0
for i in range(count):
    text = [random_layout, tiled_chain, random_expand][i % 3](rng)
    g = L.parse_layout(text)
    spec = O.parse(text)
    n_log, n_phys = O.logical_size(spec), O.size(spec)
    expand = spec["kind"] == "expand"
    for e in (1, 2, 4, 8):
        directions = [("from", g, None)] if expand else [("to", None, g), ("from", g, None)]
        for name, a, b in directions:
            n_src = n_phys if a is not None else n_log
            host = (np.arange(n_src, dtype=np.int64) * 2654435761 % 1000003).astype(NP[e])
            got = K.remap(torch.from_numpy(host).cuda(), a, b).cpu().numpy()
            want = O.remap(host, spec if a is not None else None, spec if b is not None else None,
                           dst_size=n_phys if b is not None else n_log)
            if not np.array_equal(got, want):
                print("MISMATCH", text, e, name, K.remap_plan(a, b, e))
                sys.exit(1)
            kinds[repr(K.remap_plan(a, b, e)).split("(")[1].split(",")[0]] += 1
            checked += 1
print(f"seed {seed}: {checked} remaps bit-exact; kernel families {dict(kinds)}")
