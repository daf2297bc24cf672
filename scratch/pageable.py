"""numpy (pageable) vs pinned vs registered host sort timings (scratch)."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
x = (np.random.default_rng(0).integers(0, 4096, n)).astype(np.int64)
y = x.copy()
cafs.cafs_sort(y)  # warm
for it in range(2):
    y = x.copy()
    t = time.perf_counter(); cafs.cafs_sort(y); t1 = time.perf_counter()
    print(f"pageable numpy: {(t1-t)*1e3:.1f} ms  {n/(t1-t)/1e9:.2f} Gkeys/s", flush=True)
cudart = torch.cuda.cudart()
for it in range(2):
    y = x.copy()
    t = time.perf_counter()
    r = cudart.cudaHostRegister(y.ctypes.data, y.nbytes, 0)
    t1 = time.perf_counter()
    cafs.cafs_sort(y)
    t2 = time.perf_counter()
    cudart.cudaHostUnregister(y.ctypes.data)
    t3 = time.perf_counter()
    print(f"registered: register {(t1-t)*1e3:.1f} ms sort {(t2-t1)*1e3:.1f} ms unregister {(t3-t2)*1e3:.1f} ms total {(t3-t)*1e3:.1f} ms {n/(t3-t)/1e9:.2f} Gkeys/s rc={r}", flush=True)
p = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
p[:] = x
t = time.perf_counter(); cafs.cafs_sort(p); t1 = time.perf_counter()
print(f"pinned: {(t1-t)*1e3:.1f} ms {n/(t1-t)/1e9:.2f} Gkeys/s")
