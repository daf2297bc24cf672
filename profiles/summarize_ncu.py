"""Summarise ncu captures into profiles/ (run in the build container).

    python profiles/summarize_ncu.py full <report.ncu-rep> <config> <out.json>
    python profiles/summarize_ncu.py launches <launches.csv> <out.txt>

`full` writes per-kernel duration, DRAM read/write bytes and throughput, and
updates profiles/ncu_traffic.json (bench.py's `traffic` field) for the kernel
that moves the most bytes.
"""
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__block_size", "smsp__inst_executed.sum"]
SCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9,
         "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def full(rep, config, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = float(r[i].replace(",", ""))
                u = units[i]
                if u in SCALE and u not in ("byte",):
                    v *= SCALE[u]
                d[m] = v
        d["duration_s"] = d.pop("gpu__time_duration.sum")
        d["dram_bytes"] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        d["dram_GBps"] = d["dram_bytes"] / d["duration_s"] / 1e9
        res.append(d)
    with open(out, "w") as f:
        json.dump({"report": os.path.basename(rep), "config": config, "kernels": res}, f, indent=1)
    tpath = os.path.join(HERE, "ncu_traffic.json")
    t = json.load(open(tpath)) if os.path.exists(tpath) else {}
    t[config] = {}
    for d in res:  # per kernel family: the launch that did the work
        # family: the function name without return type or template arguments
        # ("void emit_kernel<0, 1>" -> "emit_kernel")
        fam = ("hash_count_kernel" if "hash_count" in d["kernel"]
               else d["kernel"].split("<")[0].split()[-1])
        if d["dram_bytes"] > t[config].get(fam, {}).get("dram_bytes_per_launch", -1):
            t[config][fam] = {"kernel": d["kernel"], "dram_bytes_per_launch": d["dram_bytes"],
                              "duration_s": d["duration_s"], "source": os.path.basename(out)}
    json.dump(t, open(tpath, "w"), indent=1)
    for d in res:
        print(f"{d['kernel'][:40]:40s} {d['duration_s']*1e6:10.1f} us  dram {d['dram_bytes']/1e9:8.3f} GB"
              f"  {d['dram_GBps']:8.1f} GB/s")


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[h + 1:]:
        if len(r) > mi:
            agg.setdefault(r[ki].split("(")[0][:60], []).append(float(r[mi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    # the sort's own kernels (the library's, not the generator's or torch's
    # checks): their shares are the ones to set beside the bench line's
    # roofline.kernels[*].share_of_step
    own = {k: v for k, v in agg.items() if "cafs::" in k and "gen_" not in k}
    tot_own = sum(sum(v) for v in own.values()) or 1.0
    with open(out, "w") as f:
        f.write(f"# per-kernel device time from `ncu --metrics gpu__time_duration.sum` ({os.path.basename(path)})\n")
        f.write("# cold-cache, serialised launches: compare shares, not absolutes\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k:60s} n={len(v):3d} avg={sum(v)/len(v)/1e3:10.3f} us  share={sum(v)/tot*100:5.1f}%\n")
        f.write("#\n# shares among the sort pipeline's kernels only (all calls of the command)\n")
        for k, v in sorted(own.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k:60s} n={len(v):3d} share_of_sort={sum(v)/tot_own*100:5.1f}%\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
