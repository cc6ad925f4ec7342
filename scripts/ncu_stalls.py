"""Summarise per-instruction warp-stall samples of an ncu report (source page, SASS view).

    python scripts/ncu_stalls.py REPORT [ADDR_LO ADDR_HI]
Prints stall-reason totals (optionally restricted to an address range) and the
top instructions by samples."""
import csv, io, subprocess, sys
rep = sys.argv[1]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0 for h in stall_cols}
inst = []
base = None
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        a = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    a -= base
    if not (lo <= a < hi):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[ix["Instructions Executed"]] or 0)
    for h in stall_cols:
        tot[h] += int(r[ix[h]] or 0)
    inst.append((s, a, r[ix["Source"]], ex, {h: int(r[ix[h]] or 0) for h in stall_cols}))
T = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{h[6:]} {v/T:.1%}" for h, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
print("instructions executed:", sum(i[3] for i in inst))
for s, a, src, ex, d in sorted(inst, reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    top = ", ".join(f"{h[6:]} {v}" for h, v in sorted(d.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{a:#06x} {s:6d} ex={ex:8d} {src[:60]:60s} {top}")
