"""HBM write/read ceilings on this B200 (scratch): memset, torch fill, torch sum
over 8 GiB, CUDA events, best of 10."""
import torch
n = 1 << 30
x = torch.empty(n, dtype=torch.int64, device="cuda")
def t(fn, reps=10):
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best
B = n * 8
for name, fn in [("memset (zero_)", lambda: x.zero_()), ("fill_(7)", lambda: x.fill_(7)),
                 ("sum (read)", lambda: x.sum()), ("copy half->half", lambda: x[: n // 2].copy_(x[n // 2:]))]:
    s = t(fn)
    print(f"{name:18s} {s*1e3:8.3f} ms  {B / s / 1e12:6.3f} TB/s (of 8 GiB touched once)", flush=True)
