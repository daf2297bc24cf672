"""numpy (pageable) drop-in e2e vs pinned (scratch)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen
for log2n in (30,):
    n = 1 << log2n
    x0 = datagen.generate(datagen.CONFIGS["cfg4"], n, 0).cpu().numpy()
    x = x0.copy()
    cafs.cafs_sort(x)  # warm
    ts = []
    for _ in range(3):
        x[:] = x0
        t = time.perf_counter(); cafs.cafs_sort(x); ts.append(time.perf_counter() - t)
    pin = torch.from_numpy(x0).pin_memory()
    tp = []
    for _ in range(3):
        y = pin.clone().pin_memory()
        t = time.perf_counter(); cafs.cafs_sort(y.numpy()); tp.append(time.perf_counter() - t)
    print(f"n=2^{log2n}: pageable {n/min(ts)/1e9:.2f} Gkeys/s ({min(ts)*1e3:.0f} ms), pinned {n/min(tp)/1e9:.2f} Gkeys/s", flush=True)
