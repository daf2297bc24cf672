"""Host memcpy bandwidth with threads (scratch)."""
import os, time, threading
import numpy as np, torch
n = 1 << 27  # 1 GB of int64
src = np.random.default_rng(0).integers(0, 1 << 62, n)
dst = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
print("cpus", os.cpu_count(), flush=True)
for T in (1, 2, 4, 8, 16):
    parts = np.array_split(np.arange(n), T)
    def work(a, b):
        np.copyto(dst[a:b], src[a:b])
    best = 1e9
    for rep in range(3):
        ths = [threading.Thread(target=work, args=(p[0], p[-1] + 1)) for p in parts]
        t = time.perf_counter()
        for th in ths: th.start()
        for th in ths: th.join()
        best = min(best, time.perf_counter() - t)
    print(f"T={T}: {n*8/best/1e9:.1f} GB/s pageable->pinned", flush=True)
