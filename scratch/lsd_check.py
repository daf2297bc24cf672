import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from oracle import gen as ogen
which = sys.argv[1]
if which == "fallback":
    x = ogen.mix_outputs(3, 20_000_000).view(np.int64).copy()
    t = torch.from_numpy(x).cuda()
    cafs.fallback_sort(t); torch.cuda.synchronize()
    print("fallback ok", np.array_equal(t.cpu().numpy(), np.sort(x)), flush=True)
elif which == "guard":
    n = 20_000_000
    x = ogen.mix_outputs(77, n).view(np.int64).copy()
    x[::n // 1024][:1024] = np.arange(1024, dtype=np.int64) % 100
    t = torch.from_numpy(x).cuda()
    tel = cafs.SortTelemetry()
    cafs.cafs_sort(t, telemetry=tel); torch.cuda.synchronize()
    print("guard ok", tel.guard_fired, np.array_equal(t.cpu().numpy(), np.sort(x)), flush=True)
elif which == "main17":
    n = 40_000_000
    x = ogen.mix_outputs(5, 17_000_000).view(np.int64)[np.random.default_rng(1).integers(0, 17_000_000, n)]
    t = torch.from_numpy(x).cuda()
    tel = cafs.SortTelemetry()
    cafs.cafs_sort(t, telemetry=tel); torch.cuda.synchronize()
    print("main17", tel.route, tel.guard_fired, np.array_equal(t.cpu().numpy(), np.sort(x)), flush=True)
