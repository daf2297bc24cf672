"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = {}
for r in rows[h + 1:]:
    if len(r) <= mi:
        continue
    agg.setdefault(r[ki][:70], []).append(float(r[mi].replace(",", "")))
for k, v in agg.items():
    print(f"{k:70s} n={len(v):3d} avg={sum(v)/len(v)/1e3:10.3f} us total={sum(v)/1e6:9.3f} ms")
