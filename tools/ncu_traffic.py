"""Extract per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and duration from an
ncu --set full report; prints JSON {kernel: {...}} (averaged over the captured launches)."""
import collections
import csv
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "second": 1.0}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[2:]:
        k = r[col["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0].replace("lp::", "")
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            if m in col and r[col[m]] not in ("", "n/a"):
                agg[k][m].append(float(r[col[m]].replace(",", "")) * UNIT.get(units[col[m]], 1.0))
    res = {}
    for k, d in agg.items():
        rd = sum(d["dram__bytes_read.sum"]) / max(1, len(d["dram__bytes_read.sum"]))
        wr = sum(d["dram__bytes_write.sum"]) / max(1, len(d["dram__bytes_write.sum"]))
        t = sum(d["gpu__time_duration.sum"]) / max(1, len(d["gpu__time_duration.sum"]))
        res[k] = {"dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "traffic_bytes": int(rd + wr),
                  "duration_us": round(t * 1e6, 2), "launches": len(d["gpu__time_duration.sum"])}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
