"""Per-call overhead of the stream-ordered sharded sort at one NCCL rank, on an
eighth of cfg4 (the per-rank shard at 8 GPUs) and on the whole column (scratch)."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, ".")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen, sharded
st = torch.cuda.current_stream()
for cfgname, frac in [("cfg4", 8), ("cfg4", 1), ("cfg2", 8), ("cfg3", 8)]:
    cfg = datagen.CONFIGS[cfgname]
    n = cfg.n // frac
    p = datagen.generate(cfg, n, 0); x = torch.empty_like(p)
    res = {}
    for name, fn in [("single", lambda: cafs.cafs_sort(x)), ("sharded", lambda: sharded.cafs_sort_sharded(x))]:
        ts = []
        for it in range(13):
            x.copy_(p)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st); fn(); b.record(st); torch.cuda.synchronize()
            if it >= 3: ts.append(a.elapsed_time(b) * 1e3)
        ts.sort(); res[name] = round(ts[len(ts) // 2], 1)
    tel = cafs.SortTelemetry(); x.copy_(p); sharded.cafs_sort_sharded(x, telemetry=tel)
    print(cfgname, f"n=N/{frac}", res, "us; path", tel.sharded_path, "kernels", tel.kernels_launched, flush=True)
dist.destroy_process_group()
