"""A/B the NW kernel template's compile-time knobs at n = 16384 on one B200:
programs of the default strip layout compiled with different -D settings,
timed alternately (python scripts/ab_nw.py "NW_EARLY_SHFL=0" "NW_EARLY_SHFL=1")."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_08091_b200 import nw, runtime as R  # noqa: E402

n = 16384
variants = sys.argv[1:] or ["NW_EARLY_SHFL=0", "NW_EARLY_SHFL=1"]
# NW_AB_LAYOUT=tiles4096 / tiles128: the bench's tiled layouts (default: strips)
_which = __import__("os").environ.get("NW_AB_LAYOUT", "strips")
if _which == "tiles4096":
    sys.path.insert(0, "tests")
    from nw_perms import skew_order
    _lay = nw.nw_layout(n, tile_rows=4096, tile_order=skew_order(4, 128))
elif _which == "tiles128":
    _lay = nw.nw_layout(n, tile_rows=128, tile_order="antidiag")
elif _which in ("strips_rotate", "strips_xor"):   # strips with a user GenP cell order (NW_GEN_SLOTS)
    sys.path.insert(0, "tests")
    from nw_perms import rotate_cells, xor_cells
    _lay = nw.nw_layout(n, cell_order=(rotate_cells if _which == "strips_rotate" else xor_cells)(n))
else:
    _lay = nw.nw_layout(n)
parts = nw.nw_parts(_lay, n)
src, info, _ = nw.program_source(parts)
progs = []
for v in variants:
    kv = dict(x.split("=") for x in v.split(",") if x)
    head = "".join(f"#define {k} {val}\n" for k, val in kv.items())
    vi = R.ProgramInfo(kind=info.kind, elem_bytes=4, n=info.n, units=info.units, unit_threads=info.unit_threads,
                       block=128,
                       smem_bytes=max(nw.SMEM_BYTES, nw.smem_bytes(int(kv.get("NW_NSLOT", 12 if kv.get("NW_SKEW") == "4" else 8)),
                                                                   int(kv.get("NW_BND_ROWS", 256)))),
                       reserved=info.reserved)
    progs.append(R.Program(R.compile_cubin(head + src), vi, head + src))
sim = torch.randint(-10, 11, (n, n), device="cuda", dtype=torch.int32)
outs = [torch.empty(n + 1, n + 1, device="cuda", dtype=torch.int32) for _ in variants]


def run(p, o):
    R.check(R.lib().lego_nw_run(p.handle, sim.data_ptr(), o.data_ptr(), n, 10, 1, R.stream_handle(None)))


times = {v: [] for v in variants}
for rep in range(6):
    for v, p, o in zip(variants, progs, outs):
        run(p, o)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            run(p, o)
        b.record()
        torch.cuda.synchronize()
        times[v].append(a.elapsed_time(b) / 4 * 1e3)
for v in variants:
    t = sorted(times[v])
    print(f"{v:40s} median {t[len(t) // 2]:8.1f} us  best {t[0]:8.1f} us  equal={torch.equal(outs[0], outs[variants.index(v)])}")
