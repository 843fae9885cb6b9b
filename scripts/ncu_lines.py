"""Top source lines of one kernel in an ncu report by warp-stall samples:
   python scripts/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[2]
idx = {k: i for i, k in enumerate(h)}
lines = []
for r in rows[3:]:
    if r and r[0]:
        try:
            lines.append(((r[0], r[1][:100]), int(r[idx["Instructions Executed"]] or 0),
                          int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)))
        except (ValueError, IndexError):
            pass
print("total instructions", sum(x[1] for x in lines), "samples", sum(x[2] for x in lines))
for l in sorted(lines, key=lambda x: -x[2])[:n]:
    print(l[2], l[1], l[0])
