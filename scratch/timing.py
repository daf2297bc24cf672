"""Host-overhead experiment: python wrapper vs raw C call vs kernel sum (scratch)."""
import ctypes, sys, time
import torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import _lib, datagen

for name in sys.argv[1:]:
    cfg = datagen.CONFIGS[name]
    pristine = datagen.generate(cfg)
    x = torch.empty_like(pristine)
    lib = _lib.load(); ctx = _lib.context(0); st = torch.cuda.current_stream()
    def py_call():
        cafs.cafs_sort(x)
    def c_call(flags=0):
        t = _lib.Telemetry()
        rc = lib.cafs_sort_i64(ctx, x.data_ptr(), x.shape[0], 1, cafs.HASH_MULT, flags, ctypes.byref(t), st.cuda_stream)
        assert rc == 0
        return t
    for fn, label in ((py_call, "python"), (c_call, "C")):
        ts = []
        for i in range(15):
            x.copy_(pristine); torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st); h0 = time.perf_counter(); fn(); h1 = time.perf_counter(); b.record(st); b.synchronize()
            ts.append((a.elapsed_time(b), (h1 - h0) * 1e3))
        ts = ts[5:]
        print(name, label, "gpu-event ms %.4f host ms %.4f" % (sum(t[0] for t in ts)/len(ts), sum(t[1] for t in ts)/len(ts)))
    x.copy_(pristine); torch.cuda.synchronize()
    t = c_call(1)
    print(name, "stage_ms", list(t.stage_ms), "kernel_ms", list(t.kernel_ms), "launches", t.kernels_launched)
