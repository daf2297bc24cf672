"""Device-side synthetic inputs for the BASELINE.json configs (bench and tests).

Generated in HBM by the ``cafs_gen_*`` kernels (csrc/gen.cu).  The streams are
the reference's counter-based SplitMix form (datagen.py:26-53), so row i of a
config depends only on i: every GPU of a sharded run generates its own rows,
and ``oracle/gen.py`` reproduces any row on the CPU bit-for-bit.

There is no public dataset behind BASELINE.json; seeded synthetic inputs with
the stated shapes and distributions stand in for it ("Inputs").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    k: int
    dist: str                 # "uniform" | "zipf"
    s: float = 0.0
    palette: str = "random"   # "random" | "codes"
    seed: int = 0
    desc: str = ""


CONFIGS = {
    "cfg1": Config("cfg1", 1_000_000, 200, "uniform", seed=1,
                   desc="N=1e6 int64, K=200 uniform-random keys, i.i.d. uniform"),
    "cfg2": Config("cfg2", 30_000_000, 8, "uniform", seed=2,
                   desc="N=3e7 int64, K=8 uniform-random keys, i.i.d. uniform (tiny route)"),
    "cfg3": Config("cfg3", 30_000_000, 130_000, "zipf", s=1.1, seed=3,
                   desc="N=3e7 int64, K=130000 random keys, Zipf s=1.1 in seeded rank order"),
    "cfg4": Config("cfg4", 1 << 30, 4096, "zipf", s=0.8, palette="codes", seed=4,
                   desc="N=2^30 int64 dictionary codes 0..4095, Zipf s=0.8"),
    "cfg5": Config("cfg5", 10_000_000, 6_000_000, "uniform", seed=5,
                   desc="N=1e7 int64, K=6e6 random keys, i.i.d. uniform (fallback route)"),
    # cfg4's shape over random int64 keys: no dense window (the hash paths)
    "cfg4r": Config("cfg4r", 1 << 30, 4096, "zipf", s=0.8, seed=6,
                    desc="N=2^30 int64, K=4096 random keys, Zipf s=0.8 (no dense window)"),
}


def zipf_cdf(k: int, s: float) -> np.ndarray:
    p = np.arange(1, k + 1, dtype=np.float64) ** (-float(s))
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    cdf[-1] = 1.0
    return cdf


def generate(cfg: Config | str, n: int | None = None, start: int = 0, device=None):
    """Rows [start, start + n) of a config as an int64 CUDA tensor."""
    import torch

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n = cfg.n - start if n is None else n
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    lib = _lib.load()
    stream = torch.cuda.current_stream(device).cuda_stream
    out = torch.empty(n, dtype=torch.int64, device=device)
    pal = None
    if cfg.palette == "random":
        pal = torch.empty(cfg.k, dtype=torch.int64, device=device)
        _lib.check(lib.cafs_gen_mix(pal.data_ptr(), cfg.k, cfg.seed, 0, stream), None, "gen_mix")
    cdf = None
    if cfg.dist == "zipf":
        cdf = torch.from_numpy(zipf_cdf(cfg.k, cfg.s)).to(device)
    rc = lib.cafs_gen_draw(out.data_ptr(), n, start, cfg.seed,
                           0 if pal is None else pal.data_ptr(), cfg.k,
                           0 if cdf is None else cdf.data_ptr(), stream)
    _lib.check(rc, None, "gen_draw")
    return out
