"""Dynamic opcode mix of one ncu report (source page, SASS view): executed
warp-instructions per opcode, optionally restricted to a row range.
    python profiles/ncu_opmix.py report.ncu-rep [row_lo row_hi]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, data = rows[1], rows[2:]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, len(data))
mix = collections.Counter()
for r in data[lo:hi]:
    src = r[isrc].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1] if " " in src else src
    op = src.split()[0] if src else "?"
    mix[op] += int(r[iex] or 0)
tot = sum(mix.values())
print("total", tot)
for op, c in mix.most_common(30):
    print(f"{op:28s} {c/tot*100:6.2f}%")
