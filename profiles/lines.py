"""Top CUDA source lines (warp-stall samples, instructions executed) of one kernel in an ncu report
captured with --import-source on (kernels compiled with -lineinfo).

    python profiles/lines.py <report.ncu-rep> <kernel-regex> [N]
"""
import csv
import io
import os
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
by = 1 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
data = {}   # kernel -> {(file, line): [stall, inst, src]}
fpath = fn = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = os.path.basename(r[1]); continue
    if r[0] == "Function Name":
        fn = r[1]; continue
    if r[0] == "Line No":
        hdr = r
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or not r[0] or not re.search(kre, fn or ""):
        continue
    try:
        st, ins = float(r[wi] or 0), float(r[ii] or 0)
    except (ValueError, IndexError):
        continue
    d = data.setdefault(fn, {})
    e = d.setdefault((fpath, int(r[0])), [0.0, 0.0, r[1].strip()])
    e[0] += st
    e[1] += ins
for fn, d in data.items():
    tot = sum(e[0] for e in d.values()) or 1
    toti = sum(e[1] for e in d.values()) or 1
    print(f"== {fn[:100]}  samples={tot:.0f} warp_inst={toti:.0f}")
    for (f, l), e in sorted(d.items(), key=lambda kv: -kv[1][by])[:top]:
        print(f"{e[0] / tot * 100:5.1f}% st {e[1] / toti * 100:5.1f}% in  {f}:{l:<5} {e[2][:95]}")
