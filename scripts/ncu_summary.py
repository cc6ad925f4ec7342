"""Summarise ncu captures (gpurun_out/prof_*.ncu-rep) into profiles/ (run here, no GPU)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
TAG = sys.argv[2] if len(sys.argv) > 2 else "r01"
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
ALGO = {  # algorithmic bytes per launch of the captured workload (scripts/one_kernel.py)
    "transpose": 2 * 16384 * 16384 * 2, "gather": 2 * 8 * 4096 * 4096 * 4,
    "band": 2 * 16384 * 16384 * 4, "softmax": 2 * 8192 * 8192 * 4,
    "nw": 16384 * 16384 * 4 + 16385 * 16385 * 4, "apply_map": 16384 * 16384 * 4,
    "staged": 2 * 8192 * 8192 * 4, "scatter": ((1 << 26) + (1 << 27) - 1) * 4, "expand": (8192 * 8192 + 8000 * 8000) * 4,
}
KEYS = {"transpose": "remap_transpose_bf16", "gather": "remap_gather_fp32", "band": "remap_antidiag_i32",
        "softmax": "softmax_fp32", "nw": "nw_wavefront_i32", "apply_map": "inv_map_antidiag_i32",
        "gemm": "gemm_bf16", "staged": "remap_staged_f1_i32", "scatter": "remap_scatter_f4_i32",
        "expand": "remap_expand_f2_i32"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * scale


lines = [f"# ncu summaries ({TAG})", "",
         "Captured with `ncu --set full --clock-control none --import-source on -k <kernel> -s 1 -c 1`",
         "on `scripts/one_kernel.py <name>` (one B200, cold-ish cache, serialised; compare shares and",
         "traffic, not absolute times).  Algorithmic bytes = each input element read once + each",
         "output element written once.", ""]
try:
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
        traffic = json.load(fh)
except (OSError, ValueError):
    traffic = {}
for name in ["transpose", "gather", "band", "softmax", "gemm", "nw", "apply_map", "staged", "scatter", "expand"]:
    rep = os.path.join(SRC, f"prof_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    m = raw(rep)
    kname = m.get("Kernel Name", ("?", ""))[0]
    lines.append(f"## {name} — `{kname[:90]}`")
    lines.append("")
    lines.append("| metric | value |")
    lines.append("|---|---|")
    for key, label in METRICS:
        if key in m:
            v, u = m[key]
            lines.append(f"| {label} (`{key}`) | {v} {u} |")
    if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
        t = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
        traffic[KEYS[name]] = int(t)
        if name in ALGO:
            lines.append(f"| DRAM traffic / algorithmic bytes | {t / ALGO[name]:.3f} |")
    lines.append("")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", f"{TAG}_ncu_summary.md"), "w") as fh:
    fh.write("\n".join(lines) + "\n")
with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)
print("\n".join(lines))
