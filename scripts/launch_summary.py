"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into profiles/<tag>_launches.md."""
import collections
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "launches.csv")
tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
cmd = sys.argv[3] if len(sys.argv) > 3 else "python bench.py --steps 5 --warmup 3 --no-cpu"
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    us = v / 1000 if unit == "ns" else v * 1000 if unit == "ms" else v
    tot[name] = tot.get(name, 0.0) + us
    cnt[name] += 1
all_us = sum(tot.values())
out = [f"# Launch list ({tag})", "",
       f"`ncu --metrics gpu__time_duration.sum --clock-control none --csv {cmd}`",
       "(cold-cache, serialised per-launch times under ncu: compare shares, not absolute times).", "",
       "| launches | total us | mean us | share | kernel |", "|---|---|---|---|---|"]
for name, us in sorted(tot.items(), key=lambda kv: -kv[1]):
    out.append(f"| {cnt[name]} | {us:.1f} | {us / cnt[name]:.1f} | {100 * us / all_us:.1f}% | `{name[:80]}` |")
path = os.path.join(ROOT, "profiles", f"{tag}_launches.md")
open(path, "w").write("\n".join(out) + "\n")
print("\n".join(out[:20]))
