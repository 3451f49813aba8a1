"""Per-kernel summary of an ncu CSV launch list (gpu__time_duration.sum +
dram__bytes_read/write.sum): launches, total and mean time, share of the
step, DRAM bytes and achieved GB/s (cold-cache, serialised launches).
    python scripts/ncu_launch_summary.py launches.csv [--skip N] [--peak-gbs 6544]"""
import csv
import re
import sys
from collections import OrderedDict

path = sys.argv[1]
skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
peak = float(sys.argv[sys.argv.index("--peak-gbs") + 1]) if "--peak-gbs" in sys.argv else 6544.3
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
launch = OrderedDict()
for r in rows[1:]:
    lid = int(r[ix["ID"]])
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("void ", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"ndb::", "", name)
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
             "second": 1.0, "s": 1.0, "byte": 1, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    d = launch.setdefault(lid, {"name": name})
    d[r[ix["Metric Name"]]] = v * scale
items = list(launch.values())[skip:]
agg = OrderedDict()
for d in items:
    a = agg.setdefault(d["name"], {"n": 0, "t": 0.0, "b": 0.0})
    a["n"] += 1
    a["t"] += d.get("gpu__time_duration.sum", 0.0)
    a["b"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a["t"] for a in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'ms':>9s} {'share':>6s} {'MB':>9s} {'GB/s':>8s} {'%peak':>6s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
    gbs = a["b"] / a["t"] / 1e9 if a["t"] else 0
    print(f"{k[:60]:60s} {a['n']:5d} {a['t']*1e3:9.3f} {a['t']/tot*100:5.1f}% {a['b']/1e6:9.1f} {gbs:8.1f} {gbs/peak*100:5.1f}%")
print(f"total kernel time {tot*1e3:.3f} ms over {len(items)} launches")
