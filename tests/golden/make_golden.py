"""Generate the golden parity fixtures by running the REAL reference.

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It writes small JSON/NPZ fixtures next to this file.  The GPU box has no
/root/reference; tests there read only these committed fixtures.  Inputs are
either generator specs (restated bit-for-bit in oracle/gen.py, checked by
tests/test_oracle_golden.py) or, for hand-built adversarial cases, the raw
arrays in special_inputs.npz.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from cafs import buckets, cardinality, datagen, selftest, sorter  # noqa: E402  (the reference)
from cafs.sorter import Route, SortTelemetry, cafs_sort  # noqa: E402

from oracle import gen as ogen  # noqa: E402

ALT_MULT = 0xC2B2AE3D27D4EB4F


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def tel_record(tel: SortTelemetry, x_sorted: np.ndarray) -> dict:
    d = tel.decision
    est = d.estimate
    rec = {
        "route": tel.route.value,
        "k_hat": None if est is None else est.k_hat,
        "u": None if est is None else est.u,
        "f1": None if est is None else est.f1,
        "f2": None if est is None else est.f2,
        "saturated": None if est is None else bool(est.saturated),
        "spill_len": int(tel.spill_len),
        "guard_fired": bool(tel.guard_fired),
        "counted_total": int(tel.counted_total),
        "updates": int(tel.updates),
        "tiny_count_failed": bool(tel.tiny_count_failed),
        "stage_keys": sorted(tel.stage_ms),
        "sha256": sha(x_sorted),
    }
    if tel.table is not None:
        rec["table_buckets"] = int(tel.table.n_buckets)
        rec["hits"] = int(tel.table.stats.hits)
        rec["claims"] = int(tel.table.stats.claims)
        rec["spill_pushes"] = int(tel.table.stats.spill_pushes)
    return rec


def run_ref(x: np.ndarray, mult=None) -> dict:
    y = x.copy()
    tel = SortTelemetry()
    cafs_sort(y, telemetry=tel, hash_mult=mult)
    assert np.array_equal(y, np.sort(x))
    dec = sorter.dispatch(sorter.to_unsigned(x), hash_mult=mult) if x.shape[0] > 1 else None
    rec = tel_record(tel, y)
    if dec is not None and dec.route is Route.TINY_COUNT:
        rec["tiny_keys"] = [int(v) for v in dec.keys.tolist()]
    rec["dispatch_route"] = dec.route.value if dec is not None else "already_sorted"
    return rec


def known_answers() -> dict:
    rng = np.random.default_rng(2024)
    hashes = []
    for m in (1, 3, 7, 9, 12, 13, 16, 33, 63):
        for v in [0, 1, 2, (1 << 63), (1 << 64) - 1] + rng.integers(0, 1 << 63, 6).tolist():
            hashes.append([int(v), m, int(buckets.fast_hash(int(v), m))])
            hashes.append([int(v), m, int(buckets.fast_hash(int(v), m, ALT_MULT)), ALT_MULT])
    sizes = []
    for k_hat, n, cap in [(200, 10**7, 4), (4000, 10**7, 4), (10**4, 10**7, 4), (1, 10**7, 4),
                          (10**6, 1024, 4), (1, 4, 4), (200.3, 10**7, 4), (197.3, 10**6, 4),
                          (2088.8, 1 << 30, 4), (8.5, 30_000_000, 4), (262144.0, 10**7, 4),
                          (3.5, 2048, 8), (1e7, 1e7, 4)]:
        sizes.append([k_hat, int(n), cap, int(buckets.table_size_for(k_hat, int(n), cap))])
    for _ in range(60):
        k_hat = float(rng.uniform(1, 1e6))
        n = int(rng.integers(1, 10**9))
        sizes.append([k_hat, n, 4, int(buckets.table_size_for(k_hat, n, 4))])
    chao = []
    for u, f1, f2, n, sat in [(1, 0, 0, 10**6, False), (3, 2, 1, 10**6, False),
                              (1024, 300, 100, 5 * 10**5, True), (500, 499, 0, 520, False),
                              (17, 0, 5, 10**6, False), (8, 1, 0, 10**6, False),
                              (1023, 1022, 1, 10**7, False), (656, 519, 93, 1 << 30, False)]:
        chao.append([u, f1, f2, n, sat, cardinality.chao1(u, f1, f2, n, sat)])
    for _ in range(100):
        u = int(rng.integers(1, 1024))
        f1 = int(rng.integers(0, u + 1))
        f2 = int(rng.integers(0, u - f1 + 1))
        n = int(rng.integers(2048, 1 << 31))
        chao.append([u, f1, f2, n, False, cardinality.chao1(u, f1, f2, n, False)])
    mix = {"seed": 42, "outputs": [int(v) for v in datagen.mix_outputs(42, 8).tolist()]}
    return {"fast_hash": hashes, "table_size_for": sizes, "chao1": chao, "mix_outputs": mix}


def sweep_cases() -> list[dict]:
    out = []
    for i, (kind, n, k) in enumerate(selftest._sweep_points(42, selftest.ORACLE_POINTS)):
        seed = 42 + i
        if kind == "sorted_ramp":
            x = np.sort(datagen.gen_input(datagen.GenSpec(n, k, seed)))
        elif kind == "distinct":
            x = selftest._distinct_values(n, seed)
        else:
            x = datagen.gen_input(datagen.GenSpec(n, k, seed))
        # the restated generator must reproduce the reference's input bits
        if kind == "distinct":
            assert np.array_equal(ogen.distinct_values(n, seed), x)
        else:
            y = ogen.gen_input(n, k, seed)
            assert np.array_equal(np.sort(y) if kind == "sorted_ramp" else y, x)
        rec = run_ref(x)
        rec.update({"kind": kind, "n": n, "k": k, "seed": seed, "dtype": "uint64"})
        out.append(rec)
        # the same multiset as int64 exercises the sign-flip path
        if i % 4 == 0:
            xi = x.view(np.int64)
            rec = run_ref(xi)
            rec.update({"kind": kind, "n": n, "k": k, "seed": seed, "dtype": "int64"})
            out.append(rec)
    return out


def special_cases() -> tuple[list[dict], dict]:
    arrays = {}
    recs = []

    def add(name, x, mult=None):
        if name in ogen.GENERATED_SPECIAL:
            assert np.array_equal(ogen.GENERATED_SPECIAL[name](), x)
        else:
            arrays[name] = x
        rec = run_ref(x, mult)
        rec["name"] = name
        rec["dtype"] = str(x.dtype)
        if mult is not None:
            rec["hash_mult"] = mult
        recs.append(rec)

    info = np.iinfo(np.int64)
    rng = np.random.default_rng(44)
    pal = np.array([info.min, info.min + 1, -3, -1, 0, 1, 7, info.max - 1, info.max]
                   + list(range(100, 191)), np.int64)
    add("signed_extremes_main", pal[rng.integers(0, pal.shape[0], 50_000)])
    rng = np.random.default_rng(23)
    pal = np.array([-900, -5, 0, 17, 2**40], np.int64)
    add("tiny_signed", pal[rng.integers(0, 5, 10_000)])
    keys = (np.arange(8, dtype=np.uint64) + 3) * np.uint64(1_000_003)
    rng = np.random.default_rng(10)
    x = keys[rng.integers(0, 8, 100_000)]
    x[1] = 999
    add("tiny_failure", x)
    cand = np.arange(1, 1 + (64 << (7 + 4)), dtype=np.uint64)
    colliders = cand[buckets.fast_hash(cand, 7) == 0][:64]
    rng = np.random.default_rng(11)
    add("guard_colliders", colliders[rng.integers(0, 64, 20_000)])
    # acceptance c06: adversarial guard input, 1e6 keys colliding in M=256
    n = 1_000_000
    palette = selftest.collide_keys_exact(100, 8)
    data = selftest.collide_keys_exact(n, 8, offset=4096)
    stride = n // 1024
    idx = np.arange(0, min(n, 1024 * stride), stride)
    data[idx] = palette[np.arange(idx.shape[0]) % 100]
    add("guard_adversarial_c06", data)
    add("sorted_ramp_i64", np.arange(-50_000, 150_000, dtype=np.int64))
    x = np.arange(3 * 16384, dtype=np.int64)
    x[16384], x[16385] = x[16385], x[16384]
    add("inversion_at_chunk_boundary", x)
    x = np.arange(200_000, dtype=np.int64)
    x[-1] = -1
    add("inversion_at_end", x)
    add("small_n_1000", datagen.gen_input(datagen.GenSpec(1000, 50)))
    add("n2_unsorted", np.array([5, -3], np.int64))
    add("n2047", datagen.gen_input(datagen.GenSpec(2047, 100)).view(np.int64))
    add("n2048", datagen.gen_input(datagen.GenSpec(2048, 100)).view(np.int64))
    add("constant_after_first", np.concatenate([[7], np.full(9999, 3)]).astype(np.int64))
    add("all_equal_but_last", np.concatenate([np.full(99_999, 3), [1]]).astype(np.int64))
    add("two_keys_u64", np.array([3, 9], np.uint64)[np.random.default_rng(0).integers(0, 2, 50_000)])
    add("zero_and_max_u64", np.array([0, (1 << 64) - 1, 5], np.uint64)[
        np.random.default_rng(3).integers(0, 3, 30_000)])
    add("max_key_main", np.array([info.max, info.min] + list(range(40)), np.int64)[
        np.random.default_rng(4).integers(0, 42, 60_000)])
    add("alt_mult_main", datagen.gen_input(datagen.GenSpec(200_000, 300, 5)), ALT_MULT)
    add("alt_mult_guard", colliders[np.random.default_rng(12).integers(0, 64, 20_000)], ALT_MULT)
    # k_hat = 8.5 (u = 8, f1 = 1, f2 = 0) must route MAIN, not TINY
    n = 8192
    keys7 = np.arange(1, 8, dtype=np.int64) * -11
    x = keys7[np.random.default_rng(5).integers(0, 7, n)]
    x[::n // 1024] = keys7[np.arange(1024) % 7]
    x[0] = 999  # the one sampled singleton
    add("khat_8_5_routes_main", x)
    x = keys7[np.random.default_rng(6).integers(0, 7, n)]
    x[::n // 1024] = keys7[np.arange(1024) % 7]
    x[0] = 999
    x[8] = 999  # sampled twice: u=8, f1=0, f2=1 -> k_hat = 8 -> tiny
    add("khat_8_routes_tiny", x)
    add("distinct_1e4", selftest._distinct_values(10_000, 5))
    return recs, arrays


def dtype32_cases() -> tuple[list[dict], dict]:
    """int32 / uint32 columns through the reference (SUPPORTED_DTYPES, sorter.py:34):
    every route, and bucket-table spills in the 32-bit unsigned domain."""
    arrays, recs = {}, []

    def add(name, x, mult=None):
        arrays[name] = x
        rec = run_ref(x, mult)
        rec["name"] = name
        rec["dtype"] = str(x.dtype)
        if mult is not None:
            rec["hash_mult"] = mult
        recs.append(rec)

    i32 = np.iinfo(np.int32)
    rng = np.random.default_rng(320)
    add("i32_tiny", np.array([-7, -1, 0, 5, i32.max, i32.min], np.int32)[rng.integers(0, 6, 100_000)])
    z = np.minimum(rng.zipf(1.3, 500_000), 3000).astype(np.int32) - 1
    add("i32_main_codes", z)
    pal = rng.integers(i32.min, i32.max, 30_000, dtype=np.int32)
    add("i32_main_hash", pal[np.minimum(rng.zipf(1.1, 400_000), 30_000) - 1])
    pal = np.array([i32.min, i32.min + 1, -2, -1, 0, 1, i32.max - 1, i32.max]
                   + list(range(1000, 1100)), np.int32)
    add("i32_extremes_main", pal[rng.integers(0, pal.shape[0], 80_000)])
    add("i32_distinct", rng.permutation(np.arange(-100_000, 100_000, dtype=np.int32) * 7919))
    add("i32_small_n", rng.integers(-50, 50, 1500).astype(np.int32))
    add("i32_sorted", np.arange(-30_000, 30_000, dtype=np.int32))
    u32 = np.iinfo(np.uint32)
    pal = np.array([0, 1, 77, u32.max - 1, u32.max] + list(range(5000, 5300)), np.uint32)
    add("u32_main", pal[rng.integers(0, pal.shape[0], 300_000)])
    add("u32_tiny", np.array([3, 9, u32.max], np.uint32)[rng.integers(0, 3, 50_000)])
    cand = np.arange(1, 1 + (64 << (7 + 4)), dtype=np.uint32)
    colliders = cand[buckets.fast_hash(cand, 7) == 0][:64]
    add("u32_colliders", colliders[rng.integers(0, 64, 20_000)])
    add("i32_alt_mult", pal[rng.integers(0, pal.shape[0], 100_000)].astype(np.int32) - 2000,
        ALT_MULT)
    return recs, arrays


def config_cases() -> list[dict]:
    out = []
    for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
        c = ogen.CONFIGS[name]
        x = c.generate()
        rec = run_ref(x)
        rec["name"] = name
        out.append(rec)
        print(name, rec["route"], rec["k_hat"], rec["u"], rec["f1"], rec["f2"], rec["spill_len"],
              flush=True)
    # cfg4 (2^30 rows): dispatch depends only on the first monotone chunk and
    # the 1024 strided samples, so materialise just those rows.
    c = ogen.CONFIGS["cfg4"]
    n = c.n
    x = np.zeros(n, np.int64)  # lazily mapped; only touched rows matter
    x[:65536] = c.generate(65536, 0)
    stride = n // 1024
    for i in range(1024):
        x[i * stride] = c.generate(1, i * stride)[0]
    dec = sorter.dispatch(sorter.to_unsigned(x))
    est = dec.estimate
    m = buckets.table_size_for(max(1.0, est.k_hat), n, 4)
    out.append({"name": "cfg4", "dispatch_only": True, "route": dec.route.value,
                "dispatch_route": dec.route.value, "k_hat": est.k_hat, "u": est.u,
                "f1": est.f1, "f2": est.f2, "saturated": bool(est.saturated),
                "table_buckets": int(m)})
    print("cfg4", dec.route.value, est.k_hat, est.u, est.f1, est.f2, flush=True)
    return out


def write_dtype32() -> None:
    recs, arrays = dtype32_cases()
    np.savez_compressed(os.path.join(HERE, "dtype32_inputs.npz"), **arrays)
    with open(os.path.join(HERE, "dtype32_cases.json"), "w") as f:
        json.dump(recs, f, indent=0)


def main():
    os.makedirs(HERE, exist_ok=True)
    if "--only-dtype32" in sys.argv:
        write_dtype32()
        return
    write_dtype32()
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(known_answers(), f)
    recs, arrays = special_cases()
    np.savez_compressed(os.path.join(HERE, "special_inputs.npz"), **arrays)
    with open(os.path.join(HERE, "special_cases.json"), "w") as f:
        json.dump(recs, f, indent=0)
    with open(os.path.join(HERE, "sweep_cases.json"), "w") as f:
        json.dump(sweep_cases(), f, indent=0)
    with open(os.path.join(HERE, "config_cases.json"), "w") as f:
        json.dump(config_cases(), f, indent=1)


if __name__ == "__main__":
    main()
