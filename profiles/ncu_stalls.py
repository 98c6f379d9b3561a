"""Stall-reason breakdown (warp-state samples) of an ncu report's source page,
over all SASS rows or a row range, plus the top stalled instructions.
    python profiles/ncu_stalls.py report.ncu-rep [row_lo row_hi]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, data = rows[1], rows[2:]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, len(data))
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
isrc = hdr.index("Source")
tot = {hdr[i]: 0 for i in cols}
for r in data[lo:hi]:
    for i in cols:
        tot[hdr[i]] += int(r[i] or 0)
s = sum(tot.values())
print("samples", s)
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"  {k:24s} {v / s * 100:6.2f}%")
print("top instructions (row, samples, main reason):")
top = sorted(range(lo, hi), key=lambda j: -sum(int(data[j][i] or 0) for i in cols))[:20]
for j in top:
    r = data[j]
    vals = {hdr[i]: int(r[i] or 0) for i in cols}
    main = max(vals, key=vals.get)
    print(f"  {j:5d} {sum(vals.values()):6d} {main:20s} {r[isrc].strip()[:60]}")
