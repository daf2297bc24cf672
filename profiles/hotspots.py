"""Top SASS hot spots (warp-stall samples) of one kernel in an ncu report.

    python profiles/hotspots.py <report.ncu-rep> <kernel-regex> [N]
"""
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = txt.split('"Kernel Name",')
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(kre, name):
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    ai = hdr.index("Address")
    data = []
    for r in rows[1:]:
        try:
            data.append((float(r[wi]), r[ai][-5:], r[si].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    print(f"== {name[:100]}  samples={tot:.0f}")
    for v, a, s in sorted(data, reverse=True)[:top]:
        print(f"{v / tot * 100:5.1f}%  {a}  {s[:90]}")
