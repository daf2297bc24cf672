import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_25040_b200 as cafs
from oracle import gen as ogen
x = ogen.CONFIGS["cfg4"].generate(3_000_000)
want = np.sort(x)
for seq in ([False], [True], [False, True], [True, False], [False, False], [True, True]):
    for d in seq:
        t = torch.from_numpy(x.copy()).cuda()
        tel = cafs.SortTelemetry()
        try:
            cafs.cafs_sort(t, telemetry=tel, direct_range=d)
            ok = np.array_equal(t.cpu().numpy(), want)
            print(seq, d, "ok" if ok else "WRONG", tel.pairs, tel.route, flush=True)
        except Exception as e:
            print(seq, d, "EXC", e, flush=True)
