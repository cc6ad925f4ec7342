"""SASS evidence per kernel family (run here, no GPU): which Blackwell
instructions each kernel actually contains.  Writes profiles/<tag>_sass.md.

    python scripts/sass_evidence.py r02
"""
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"

import paper_2505_08091_b200 as L  # noqa: E402
from paper_2505_08091_b200 import kernels as K, nw as NW, runtime as R  # noqa: E402

# (label, opcode regex): tcgen05 MMA / TMA / TMEM, cp.async, 16-byte global and shared
# vector accesses (any cache-hint modifiers), shuffles, 3-input min/max, MUFU, barriers
WATCH = [("UTCHMMA", r"UTCHMMA"), ("UTMALDG", r"UTMALDG"), ("UTMASTG", r"UTMASTG"), ("UBLKCP", r"UBLKCP"),
         ("LDTM", r"LDTM"), ("UTCBAR", r"UTCBAR"), ("SYNCS", r"SYNCS"), ("LDGSTS", r"LDGSTS"),
         ("LDG.128", r"LDG\..*128"), ("STG.128", r"STG\..*128"), ("LDS.128", r"LDS\..*128"),
         ("STS.128", r"STS\..*128"), ("PRMT", r"PRMT"), ("SHFL", r"SHFL"), ("VIMNMX", r"VIMNMX"),
         ("MUFU.SQRT", r"MUFU\.SQRT"), ("MUFU.EX2", r"MUFU\.EX2"), ("BAR.SYNC", r"BAR\.SYNC"), ("HMMA", r"HMMA")]


def sass_of(cubin_or_so, function=None):
    args = ["cuobjdump", "-sass", cubin_or_so]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            op = m.group(1)
            funcs[cur][op] += 1
    return funcs


def summarize(counter):
    hits = []
    for label, rx in WATCH:
        n = sum(c for op, c in counter.items() if re.fullmatch(rx + r"(\..*)?", op) or re.match(rx, op))
        if n:
            hits.append(f"`{label}` x{n}")
    return ", ".join(hits) or "-"


def cubin(source):
    path = R.cubin_path(source)
    R.compile_cubin(source)
    return path


rows = []
so = os.path.join(ROOT, "paper_2505_08091_b200", "liblego_b200.so")
for fn, cnt in sass_of(so).items():
    short = re.sub(r"<unnamed>::|\(.*", "", fn)
    if any(k in fn for k in ("gemm_bf16_tcgen05", "lego_nw_tiles", "softmax_rows", "gemm_raster")):
        rows.append((f"liblego_b200.so: `{short[:70]}`", sum(cnt.values()), summarize(cnt)))
progs = {
    "headline transpose (cfg2, bf16)": K.plan_remap(None, L.parse_layout(
        "GroupBy([16384,16384]).OrderBy(Col(16384,16384))"), 2).source,
    "tiled gather (cfg1, fp32)": K.plan_remap(None, L.parse_layout(
        "GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))"), 4).source,
    "antidiag band (cfg4a, int32)": K.plan_remap(None, L.parse_layout(
        "GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))"), 4).source,
    "antidiag index maps (run-walking inverse)": K.index_map_source(L.parse_layout(
        "GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))"))[0],
    "box-staged chain (f1)": K.plan_remap(None, L.parse_layout(
        "GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
        ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))"), 4).source,
    "fill scatter (f4, int32)": K.plan_remap(None, L.GroupBy([1 << 26], orders=(L.OrderBy(L.GenP(
        (1 << 26,), L.PermFn(lambda i: 2 * i[0], lambda i: 2 * i[0]), None)),), injective=True), 4,
        fill=True).source,
    "softmax program (cfg3)": K.softmax_source(8192)[0],
    "NW program, antidiag tile order": NW.program_source(NW.nw_parts(
        NW.nw_layout(16384, tile_rows=128, tile_order="antidiag"), 16384))[0],
}
for name, src in progs.items():
    for fn, cnt in sass_of(cubin(src)).items():
        rows.append((f"{name}: `{fn}`", sum(cnt.values()), summarize(cnt)))
lines = [f"# SASS evidence ({TAG})", "",
         "`cuobjdump -sass` of the built library and of generated programs (NVRTC cubins), counting the",
         "instructions that identify each kernel family's mechanism (scripts/sass_evidence.py).", "",
         "| kernel | SASS instructions | key instructions |", "|---|---|---|"]
lines += [f"| {a} | {b} | {c} |" for a, b, c in rows]
with open(os.path.join(ROOT, "profiles", f"{TAG}_sass.md"), "w") as fh:
    fh.write("\n".join(lines) + "\n")
print("\n".join(lines))
