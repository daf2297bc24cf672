"""GPU-timeline and host time of each phase of the stream-ordered sharded sort
at one NCCL rank, on an eighth of cfg4 (scratch)."""
import os, sys, time, collections
import torch, torch.distributed as dist
sys.path.insert(0, ".")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29534")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_2605_25040_b200 import datagen, sharded
st = torch.cuda.current_stream()
marks = []
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True); e0.record(st); h0 = time.perf_counter()
        r = f(*a, **k)
        h1 = time.perf_counter(); e1 = torch.cuda.Event(enable_timing=True); e1.record(st)
        marks.append((name, e0, e1, h0, h1))
        return r
    setattr(obj, name, g)
for m in ["shard_begin", "shard_sample", "shard_count", "shard_finish"]:
    wrap(sharded.DeviceOps, m)
for m in ["all_gather_into", "all_reduce_inplace"]:
    wrap(sharded.Comm, m)
cfg = datagen.CONFIGS["cfg4"]
p = datagen.generate(cfg, cfg.n // 8, 0); x = torch.empty_like(p)
for it in range(6):
    x.copy_(p); torch.cuda.synchronize(); marks.clear()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st); t0 = time.perf_counter()
    sharded.cafs_sort_sharded(x)
    t1 = time.perf_counter(); b.record(st); torch.cuda.synchronize()
acc = collections.defaultdict(float)
print("total gpu", round(a.elapsed_time(b) * 1e3, 1), "us host", round((t1 - t0) * 1e6, 1))
for name, e0, e1, h0, h1 in marks:
    print(f"{name:20s} gpu {e0.elapsed_time(e1)*1e3:8.1f} us  host {(h1-h0)*1e6:8.1f} us  start@gpu {a.elapsed_time(e0)*1e3:8.1f} host {(h0-t0)*1e6:8.1f}")
dist.destroy_process_group()
