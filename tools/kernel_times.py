"""Per-launch gpu__time_duration of the kernels matching a regex in an ncu --csv log (stdin)."""
import csv
import re
import sys

pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
rows = list(csv.reader(sys.stdin))
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if pat.search(d["Kernel Name"]) and d.get("Metric Name") == "gpu__time_duration.sum":
            print(f'{d["Kernel Name"].split("(")[0]:40s} {float(d["Metric Value"]) / 1000:10.2f} us')
