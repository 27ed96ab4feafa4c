"""Warp-stall breakdown (cycles per issued instruction by reason) of one kernel in an ncu report."""
import csv
import subprocess
import sys


def main(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kernel, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]
    pre, post = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    got = sorted(((float(v[i]), n[len(pre):-len(post)]) for i, n in enumerate(h)
                  if n.startswith(pre) and n.endswith(post) and v[i]), reverse=True)
    print(f"{'total':24s} {sum(x for x, _ in got):6.2f}")
    for x, n in got:
        if x >= 0.05:
            print(f"{n:24s} {x:6.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
