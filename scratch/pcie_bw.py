"""PCIe ceilings (scratch): pinned H2D and D2H of 8 GiB, alone and concurrently
(two streams), CUDA events, best of 3."""
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.int64, pin_memory=True)
d = torch.empty(n, dtype=torch.int64, device="cuda")
d2 = torch.empty(n, dtype=torch.int64, device="cuda")
B = n * 8
def t(fn):
    best = 1e9
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print("H2D", round(B / t(lambda: d.copy_(h, non_blocking=True)) / 1e9, 1), "GB/s")
print("D2H", round(B / t(lambda: h.copy_(d, non_blocking=True)) / 1e9, 1), "GB/s")
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
print("H2D+D2H concurrent", round(2 * B / t(both) / 1e9, 1), "GB/s total")
