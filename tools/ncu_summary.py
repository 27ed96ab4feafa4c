"""One-screen summary of an ncu --set full report (speed-of-light, occupancy, DRAM traffic)."""
import csv
import subprocess
import sys

WANT = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Avg. Active Threads Per Warp", "Executed Instructions",
        "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size", "Static Shared Memory Per Block"]


def main(rep, kernel=None):
    """First captured launch of `kernel` (substring of the name; default: the first launch)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idi = h.index("ID") if "ID" in h else None
    seen = set()
    name = None
    launch = None
    for r in rows[1:]:
        if kernel is not None and kernel not in r[ki].split("(")[0]:
            continue
        if idi is not None:
            if launch is None:
                launch = r[idi]
            elif r[idi] != launch:
                continue
        if name is None:
            name = r[ki]
            print(name[:120])
        if r[mi] in WANT and r[mi] not in seen:
            seen.add(r[mi])
            print(f"  {r[mi]:40s} {r[vi]:>16s} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
