"""DRAM bytes per CG iteration and per GP step of a whole solve, from an ncu launch list of the
persistent loops (profiles/traffic_<config>.json, read by bench.py's roofline `traffic`).

The launch list (`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:k6_ --csv --log-file L python scripts/diag.py CONFIG`) covers every k6_cg_loop and
k6_gp_loop launch of one solve; diag.py's line gives that solve's CG iterations and GP steps
(GP steps the host finished after a k6_gp_loop launch handed back -- rare -- are not in the
launches, so bytes per GP step is a slight overestimate).

usage: python scripts/traffic_summary.py LAUNCHES.csv DIAG.log CONFIG ROUND > profiles/traffic_CONFIG.json
"""
import csv
import json
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if "Kernel Name" in r)
i0 = rows.index(hdr)
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iu = hdr.index("Metric Unit")
iid = hdr.index("ID")
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
acc = {}
for r in rows[i0 + 1:]:
    if len(r) <= iv or not r[iid].isdigit():
        continue
    kind = "cg" if "k6_cg_loop" in r[ik] else ("gp" if "k6_gp_loop" in r[ik] else None)
    if kind is None:
        continue
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    a = acc.setdefault(kind, {"dram": 0.0, "time": 0.0, "launches": set()})
    a["launches"].add(r[iid])
    if r[im].startswith("dram__bytes"):
        a["dram"] += v
    elif r[im] == "gpu__time_duration.sum":
        a["time"] += v
diag = open(sys.argv[2]).read()
m = re.search(r"gp=(\d+) cg=(\d+)", diag)
gp_steps, cg_iters = int(m.group(1)), int(m.group(2))
out = {"config": sys.argv[3], "round": sys.argv[4], "source": "ncu launch list of one solve (scripts/traffic_summary.py)",
       "solve": diag.strip().splitlines()[-1]}
for kind, units in (("cg", cg_iters), ("gp", gp_steps)):
    a = acc.get(kind)
    if not a:
        continue
    out[kind] = {"launches": len(a["launches"]), "units": units,
                 "dram_bytes_total": a["dram"], "dram_bytes_per_launch": a["dram"] / units,
                 "ncu_time_s": a["time"], "dram_GBs_under_ncu": a["dram"] / a["time"] / 1e9 if a["time"] else None,
                 "what": ("DRAM bytes (read + write) per CG iteration" if kind == "cg" else
                          "DRAM bytes (read + write) per GP step") + ", summed over the solve's launches"}
print(json.dumps(out, indent=1))
