"""Per-kernel launch averages from an ncu metrics pass over ONE bench step (--profile-step):
gpu__time_duration.sum, dram__bytes_read.sum + dram__bytes_write.sum (traffic) and
smsp__thread_inst_executed.sum (lane instructions), averaged per launch; the lp_bin_sort kernels are
also summed per view under "lp_bin_sort", the split loss's two kernels under "lp_loss_grad".  Output: JSON for profiles/<round>/ncu_kernels.json,
which bench.py reads for roofline.traffic and frac_ncu_executed."""
import collections
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}
SORT = ("k_radix_hist", "k_radix_scan", "k_radix_scatter", "k_scan_reduce", "k_scan_top", "k_scan_down", "k_emit",
        "k_ranges")


def main(path, views=8):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0].replace("lp::", "")
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        per[(k, d["ID"])][d["Metric Name"]] = v
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for (k, _), m in per.items():
        for name, v in m.items():
            agg[k][name].append(v)
    out = {}
    for k, m in agg.items():
        n = len(m["gpu__time_duration.sum"])
        avg = {name: sum(v) / len(v) for name, v in m.items()}
        out[k] = {"launches_per_step": n, "duration_us": round(avg["gpu__time_duration.sum"] * 1e6, 2),
                  "dram_read_bytes": int(avg.get("dram__bytes_read.sum", 0)),
                  "dram_write_bytes": int(avg.get("dram__bytes_write.sum", 0)),
                  "traffic_bytes": int(avg.get("dram__bytes_read.sum", 0) + avg.get("dram__bytes_write.sum", 0)),
                  "thread_inst_executed": int(avg.get("smsp__thread_inst_executed.sum", 0))}
    s = {"launches_per_step": 0, "duration_us": 0.0, "traffic_bytes": 0, "dram_read_bytes": 0, "dram_write_bytes": 0}
    for k in SORT:
        if k in out:
            o = out[k]
            s["launches_per_step"] += o["launches_per_step"]
            for f in ("duration_us", "traffic_bytes", "dram_read_bytes", "dram_write_bytes"):
                s[f] += o[f] * o["launches_per_step"] / views
    s["duration_us"] = round(s["duration_us"], 2)
    for f in ("traffic_bytes", "dram_read_bytes", "dram_write_bytes"):
        s[f] = int(s[f])
    s["note"] = "sum of the K2 kernels of one view (per-step totals / %d views)" % views
    out["lp_bin_sort"] = s
    # the split L1 + SSIM loss: its two kernels per lp_loss_grad call (one call per view)
    if "k_ssim_maps" in out and "k_ssim_grad" in out:
        a, b = out["k_ssim_maps"], out["k_ssim_grad"]
        out["lp_loss_grad"] = {"launches_per_step": a["launches_per_step"] + b["launches_per_step"],
                               "duration_us": round(a["duration_us"] + b["duration_us"], 2),
                               **{f: a[f] + b[f] for f in ("traffic_bytes", "dram_read_bytes", "dram_write_bytes",
                                                           "thread_inst_executed")},
                               "note": "k_ssim_maps + k_ssim_grad of one lp_loss_grad call (one view)"}
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1])
