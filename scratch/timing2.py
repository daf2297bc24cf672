"""Where does per-call overhead go? (scratch)"""
import ctypes, sys, time
import torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import _lib, datagen
cfg = datagen.CONFIGS[sys.argv[1]]
pristine = datagen.generate(cfg)
x = torch.empty_like(pristine)
lib = _lib.load(); ctx = _lib.context(0); st = torch.cuda.current_stream()
def c_call(flags):
    t = _lib.Telemetry()
    assert lib.cafs_sort_i64(ctx, x.data_ptr(), x.shape[0], 1, cafs.HASH_MULT, flags, ctypes.byref(t), st.cuda_stream) == 0
variants = {
    "C flags=0": lambda: c_call(0),
    "C timing": lambda: c_call(1),
    "py no-tel": lambda: cafs.cafs_sort(x),
    "py tel": lambda: cafs.cafs_sort(x, telemetry=cafs.SortTelemetry()),
}
for name, fn in variants.items():
    ts = []
    for i in range(30):
        x.copy_(pristine); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter(); a.record(st); fn(); b.record(st); b.synchronize(); h1 = time.perf_counter()
        ts.append((a.elapsed_time(b), (h1 - h0) * 1e3))
    ts = ts[10:]
    print(f"{name:12s} gpu-event {sum(t[0] for t in ts)/len(ts):.4f} ms  host {sum(t[1] for t in ts)/len(ts):.4f} ms")
import cProfile, pstats
x.copy_(pristine); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for i in range(50):
    cafs.cafs_sort(x, telemetry=cafs.SortTelemetry())
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
