"""Section/metric/value lines of an ncu report's details page.
    python profiles/ncu_details.py report.ncu-rep [section-regex]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
isec, iname, iunit, ival = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
for r in rows[1:]:
    if len(r) > ival and r[iname] and pat.search(r[isec]):
        print(f"{r[isec][:30]:30s} {r[iname][:42]:42s} {r[iunit]:10s} {r[ival]}")
