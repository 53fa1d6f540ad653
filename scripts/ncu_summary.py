"""Summarise an ncu report (--set full) or a launch-list CSV into a short table.

usage: python scripts/ncu_summary.py report.ncu-rep        # per-kernel key metrics
       python scripts/ncu_summary.py launches.csv          # per-kernel share of device time
"""
import collections
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_registers"]


def short(name):
    base = name.split("(")[0]
    return base.replace("void ", "").replace("gpcg::", "")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    idx = {m: hdr.index(m) for m in RAW if m in hdr}
    ki = hdr.index("Kernel Name")
    print(f"{'kernel':38s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>8s} {'dram%':>6s} {'warps%':>6s} {'regs':>5s} {'grid':>6s} {'L2hit%':>7s}")
    for r in rows[2:]:
        def g(m, scale=1.0):
            if m not in idx:
                return float("nan")
            v = r[idx[m]].replace(",", "")
            try:
                return float(v) * scale
            except ValueError:
                return float("nan")
        tu = units[idx["gpu__time_duration.sum"]]
        t_ns = g("gpu__time_duration.sum") * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
                                               "msecond": 1e6, "ms": 1e6}.get(tu, 1)
        bsc = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}
        byt = sum(g(m) * bsc.get(units[idx[m]], 1) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        print(f"{short(r[ki])[:38]:38s} {t_ns/1e3:8.2f} {byt/1e6:9.2f} {byt/t_ns:8.1f} "
              f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} {g('launch__registers_per_thread'):5.0f} "
              f"{g('launch__grid_size'):6.0f} {g('lts__t_sector_hit_rate.pct'):7.1f}")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", "")) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
                                             "msecond": 1e6, "ms": 1e6}.get(r[ui], 1)
        d[short(r[ki]).split("(")[0]].append(v)
    tot = sum(sum(v) for v in d.values())
    print(f"{'kernel':45s} {'launches':>8s} {'mean us':>9s} {'share %':>8s}")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:45]:45s} {len(v):8d} {sum(v)/len(v)/1e3:9.2f} {100*sum(v)/tot:8.1f}")
    print(f"total device time {tot/1e6:.2f} ms over {sum(len(v) for v in d.values())} launches")


if __name__ == "__main__":
    p = sys.argv[1]
    (report if p.endswith(".ncu-rep") else launches)(p)
