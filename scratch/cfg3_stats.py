import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen
for name in sys.argv[1:]:
    cfg = datagen.CONFIGS[name]
    p = datagen.generate(cfg)
    x = torch.empty_like(p)
    for i in range(4):
        x.copy_(p)
        tel = cafs.SortTelemetry()
        cafs.cafs_sort(x, telemetry=tel)
    torch.cuda.synchronize()
    print(name, {k: getattr(tel, k) for k in ("spill_len", "global_updates", "pairs", "counted_total", "kernels_launched")})
    print(" stage", tel.stage_ms)
    print(" kern", tel.kernel_ms)
