"""Per-call device time of `cafs_sort` on a column of `rows` rows of a config
(CUDA events around the call, graph replayed; median of `reps` calls), with the
count / emit / estimate kernel times of instrumented calls beside it.

    python profiles/percall.py cfg4 134217728 [reps] [sharded]

`sharded`: the native multi-GPU entry point (`cafs_sort_sharded` over an NCCL
group of one rank) on the same column.

The gap between the call and its two HBM passes is the fixed per-call cost that
caps multi-GPU scaling ("What's weak" 5).
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen


def main():
    name = sys.argv[1]
    rows = int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    sharded = len(sys.argv) > 4 and sys.argv[4] == "sharded"
    if sharded:
        import torch.distributed as dist
        from paper_2605_25040_b200.sharded import cafs_sort_sharded
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
        sort = lambda t, telemetry=None, **kw: cafs_sort_sharded(t, telemetry=telemetry)
    else:
        sort = cafs.cafs_sort
    cfg = datagen.CONFIGS[name]
    pristine = datagen.generate(cfg, rows, 0)
    x = torch.empty_like(pristine)
    st = torch.cuda.current_stream()
    for _ in range(4):
        x.copy_(pristine)
        sort(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        x.copy_(pristine)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        sort(x)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ok = bool((x[1:] >= x[:-1]).all().item())
    tels = []
    for _ in range(12):
        x.copy_(pristine)
        t = cafs.SortTelemetry()
        sort(x, telemetry=t, exact_telemetry=False)
        tels.append(t)
    tels = tels[2:]
    km = {k: statistics.median(t.kernel_ms[k] for t in tels if k in t.kernel_ms)
          for k in (tels[0].kernel_ms or {})}
    sm = {k: statistics.median(t.stage_ms[k] for t in tels if k in t.stage_ms)
          for k in (tels[0].stage_ms or {})}
    ideal = 16 * rows / 7.14e12 * 1e3
    path = getattr(tels[0], "sharded_path", None)
    print(f"{name} rows={rows} route={tels[0].route.value}/{tels[0].count_path or path} ok={ok} "
          f"call median={statistics.median(ts)*1e3:.1f} us min={min(ts)*1e3:.1f} us "
          f"(16 B/key at 7.14 TB/s: {ideal*1e3:.1f} us) "
          f"kernels_us={ {k: round(v*1e3, 1) for k, v in km.items()} } "
          f"stages_us={ {k: round(v*1e3, 1) for k, v in sm.items()} }")
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
