"""Print an ncu launch list (--metrics gpu__time_duration.sum --csv) as 'ns  kernel' lines.
   python scripts/launch_table.py FILE [last N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"][:80], float(d["Metric Value"].replace(",", "")), d["Metric Unit"]))
for k, v, u in out[-n:]:
    print(f"{v:14.1f} {u} {k}")
