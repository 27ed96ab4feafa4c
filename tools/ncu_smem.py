"""Per-source-line shared-memory wavefronts (total / excessive from bank conflicts) of an ncu report."""
import csv
import subprocess
import sys


def main(rep, kernel, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, data = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            wf = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
            ex = float(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
            g = float(r[hdr.index("L2 Theoretical Sectors Global")] or 0)
        except (ValueError, IndexError):
            continue
        if wf or g:
            data.append((wf, ex, g, f"{cur}:{r[0]}", r[1].strip()[:80]))
    tw = sum(d[0] for d in data) or 1
    print(f"shared wavefronts total {tw:.0f}, excessive {sum(d[1] for d in data):.0f}")
    for d in sorted(data, key=lambda d: d[0] + d[2], reverse=True)[:top]:
        print(f"{100 * d[0] / tw:5.1f}% smem wf {d[0]:11.0f} excess {d[1]:10.0f} L2 sectors {d[2]:10.0f}  {d[3]:20s} {d[4]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
