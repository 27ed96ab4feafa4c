"""Per-source-line instruction / stall summary of an ncu report (--page source --print-source cuda,sass)."""
import csv
import subprocess
import sys


def main(rep, kernel, top=40, by="inst"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, data, hdr = None, [], None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        try:
            ie = float(r[7] or 0)
            st = float(r[4] or 0)
        except ValueError:
            continue
        data.append((ie, st, f"{cur_file}:{r[0]}", r[1].strip()[:90]))
    ti = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    key = (lambda d: d[1]) if by == "stall" else (lambda d: d[0])
    for d in sorted(data, key=key, reverse=True)[:top]:
        print(f"{100 * d[0] / ti:5.1f}% inst {100 * d[1] / ts:5.1f}% stall  {d[2]:22s} {d[3]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40,
         sys.argv[4] if len(sys.argv) > 4 else "inst")
