"""Count-kernel cost vs distinct keys (scratch): K distinct random keys, Zipf 1.1,
30M rows, through the high-cardinality (no window) count shape."""
import sys, torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen
for k in (2000, 30000, 130000):
    for dist, s in (("zipf", 1.1),):
        cfg = datagen.Config("x", 30_000_000, k, dist, s=s, seed=7)
        p = datagen.generate(cfg); x = torch.empty_like(p)
        ks = []
        for it in range(8):
            x.copy_(p); tel = cafs.SortTelemetry()
            cafs.cafs_sort(x, telemetry=tel)
            if it >= 3: ks.append(tel.kernel_ms.get("count_kernel", -1))
        torch.cuda.synchronize()
        ok = bool((x[1:] >= x[:-1]).all())
        print(f"K={k:8d} {dist:7s} count {sum(ks)/len(ks)*1e3:7.1f} us  pairs={tel.pairs} sorted={ok}", flush=True)
