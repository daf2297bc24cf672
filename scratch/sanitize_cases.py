"""Small inputs through every route, for compute-sanitizer (scratch)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from oracle import gen as ogen
rng = np.random.default_rng(1)
cases = {
    "tiny": np.array([-5, 3, 1 << 40], np.int64)[rng.integers(0, 3, 70_001)],
    "main_dense": (np.minimum(rng.zipf(1.3, 90_003), 3000)).astype(np.int64),
    "main_hash": ogen.CONFIGS["cfg3"].generate(150_001),
    "main_hash_big": ogen.CONFIGS["cfg3"].generate(4_500_001),
    "fallback": ogen.mix_outputs(3, 60_001).view(np.int64).copy(),
    "small": rng.integers(-9, 9, 1_500).astype(np.int64),
    "i32": (np.minimum(rng.zipf(1.3, 80_001), 3000) - 7).astype(np.int32),
    "i32_hash": rng.integers(-2**31, 2**31 - 1, 20_000, dtype=np.int32)[rng.integers(0, 20_000, 100_003)],
}
for name, x in cases.items():
    for off in (0, 1):
        full = torch.from_numpy(np.concatenate([x[:1], x])).cuda()
        t = full[off:off + x.shape[0]] if off else full[1:]
        t = full[1:] if off else torch.from_numpy(x.copy()).cuda()
        tel = cafs.SortTelemetry()
        cafs.cafs_sort(t, telemetry=tel, exact_telemetry=(off == 0))
        assert np.array_equal(t.cpu().numpy(), np.sort(x)), (name, off)
    print(name, "ok", tel.route.value, flush=True)
