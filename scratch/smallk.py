"""Time the single-CTA kernels through the ABI (scratch experiment)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_25040_b200 import _lib
lib = _lib.load(); ctx = _lib.context(0); st = torch.cuda.current_stream()
def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); b.synchronize()
    return a.elapsed_time(b) / reps * 1e3
one = torch.empty(1, dtype=torch.int64, device="cuda")
print("gen_mix(1) us", timeit(lambda: lib.cafs_gen_mix(one.data_ptr(), 1, 1, 0, st.cuda_stream)))
for n in (16, 256, 4096, 8192):
    k = torch.from_numpy(np.random.default_rng(n).integers(0, 1 << 62, n)).cuda()
    c = torch.ones(n, dtype=torch.int64, device="cuda")
    def f():
        kk = k.clone(); cc = c.clone()
        assert lib.cafs_pair_sort(ctx, kk.data_ptr(), cc.data_ptr(), n, st.cuda_stream) == 0
    print("pair_sort n=%d us (incl 2 clones + D2D copies + sync)" % n, timeit(f))
for n in (4096, 1 << 20, 1 << 26):
    x = torch.randint(0, 1000, (n,), device="cuda")
    e = _lib.Estimate()
    print("estimate n=%d us (incl sync+D2H)" % n, timeit(lambda: lib.cafs_estimate_i64(ctx, x.data_ptr(), n, 1, ctypes.byref(e), st.cuda_stream)))
