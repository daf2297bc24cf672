"""Phase timing of the sharded sort at one NCCL rank (scratch)."""
import os, sys, time, collections
import torch, torch.distributed as dist
sys.path.insert(0, ".")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen, sharded
acc = collections.defaultdict(float)
def wrap(obj, name, label):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); acc[label] += time.perf_counter() - t
        return r
    setattr(obj, name, g)
for m in ["is_monotone", "estimate", "tiny_counts", "count_pairs", "merge_pairs", "emit_slice", "fallback_sort", "key_span", "partition"]:
    wrap(sharded.DeviceOps, m, "ops." + m)
for m in ["all_gather_ints", "all_reduce_sum", "all_reduce_tensor", "all_gather_pairs", "all_to_all_var", "all_gather_var"]:
    wrap(sharded.Comm, m, "comm." + m)
for name in sys.argv[1:]:
    cfg = datagen.CONFIGS[name]
    p = datagen.generate(cfg); x = torch.empty_like(p)
    for it in range(6):
        if it == 2: acc.clear()
        x.copy_(p); torch.cuda.synchronize()
        t = time.perf_counter()
        sharded.cafs_sort_sharded(x)
        torch.cuda.synchronize()
        acc["total"] += time.perf_counter() - t
    print(name, {k: round(v / 4 * 1e3, 3) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])})
dist.destroy_process_group()
