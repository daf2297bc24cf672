#!/usr/bin/env python3
"""Benchmark: int64 keys sorted/sec on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl b200|reference]

N > 1 runs under torchrun (one process per GPU, NCCL); the column of the config
is sharded by rows and sorted with ``cafs_sort_sharded`` (strong scaling: the
total N is fixed).  A "step" is one full ``cafs_sort`` of the config's column
with the input resident in HBM; between steps the unsorted input is restored
by a device-to-device copy that is NOT timed (each sort is bracketed by CUDA
events on the launching stream; the step times are summed, max over ranks).
The input (8 GiB for cfg4) is far larger than the 126 MB L2.

``e2e`` is the same metric through the C ABI host entry point
(``cafs_sort_i64_host``: pinned host buffer -> H2D -> device pipeline -> D2H).
``--impl reference`` times the reference algorithm's CPU restatement
(oracle/, single-threaded like the reference) on a bounded sample.
"""

from __future__ import annotations

import argparse
import gc
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "int64 keys sorted/sec (Gkeys/s) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gkeys/s"


def measured_peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy r+w)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None
        self.path = None

    def start(self):
        # nvidia-smi writes straight to a file: no reader thread in this process,
        # so the timed host loop never waits on the GIL (a reader thread cost a
        # 5-10 ms switch-interval stall inside a step)
        import tempfile
        fd, self.path = tempfile.mkstemp(prefix="cafs_clocks_", suffix=".csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("CAFS_BENCH_SMI_MS", "100")],
                stdout=fd, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        finally:
            os.close(fd)
        t0 = time.time()  # nvidia-smi can take a second to print its first row
        while self.proc is not None and os.path.getsize(self.path) == 0 and time.time() - t0 < 5.0:
            time.sleep(0.05)

    def _parse(self):
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        self.rows.append(parts)
        finally:
            os.unlink(self.path)

    def stop(self) -> dict:
        if self.proc is None:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self._parse()
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        loaded = [r for r in self.rows if (num(r[4]) or 0) > 0] or self.rows
        sm = [num(r[1]) for r in loaded if num(r[1]) is not None]
        mx = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "samples_under_load": len(loaded)}


def ncu_traffic(config: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the
    committed `ncu --set full` capture of this config (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)[config]
        if kernel.startswith("fallback sort stage"):  # the stage's kernels together
            return sum(v["dram_bytes_per_launch"] for k, v in t.items()
                       if k.startswith(("msd_", "bucket_")))
        # "a + b + c": the kernels of one count stage together
        return sum(t[k.strip()]["dram_bytes_per_launch"] for k in kernel.split("+"))
    except Exception:
        return None


def cpu_baseline(config: str, column=None) -> dict:
    """The C oracle (a restatement of the reference algorithm; 1 thread, like the
    reference) timed on the config's whole column: `column` is the device
    column copied to host (same bits as the GPU sorted), else it is generated
    on the host."""
    from oracle import cafs_oracle as orc
    from oracle import gen as ogen

    c = ogen.CONFIGS[config]
    x = column if column is not None else orc.generate(c)
    rows = x.shape[0]
    best = float("inf")
    y = np.empty_like(x)
    for _ in range(2):
        np.copyto(y, x)
        t0 = time.perf_counter()
        orc.cafs_sort(y)
        best = min(best, time.perf_counter() - t0)
    return {"value": rows / best / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
            "same_config": rows == c.n,
            "sample": f"all {rows} rows of {config} (C restatement of the reference, "
                      f"single-threaded like the reference; min of 2, {best * 1e3:.1f} ms; "
                      f"nproc={os.cpu_count()})"}


def run_reference(args) -> None:
    """The reference algorithm on the host (the C restatement in oracle/,
    single-threaded like the reference): every step sorts the
    config's whole column (2^30 rows for cfg4, ~3-4 s per step)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cafs_oracle as orc
    from oracle import gen as ogen

    c = ogen.CONFIGS[args.config]
    rows = min(args.cpu_rows, c.n) if args.cpu_rows else c.n
    x = orc.generate(c, rows)
    y = np.empty_like(x)
    for _ in range(args.warmup):
        np.copyto(y, x)
        orc.cafs_sort(y)
    times = []
    for _ in range(args.steps):
        np.copyto(y, x)  # restore the unsorted column (untimed)
        t0 = time.perf_counter()
        orc.cafs_sort(y)
        times.append(time.perf_counter() - t0)
    assert bool((y[1:] >= y[:-1]).all())
    tot = sum(times)
    value = rows * args.steps / tot / 1e9
    # for scale, the box's aggregate: one invocation per host core on disjoint
    # slices of the column (ctypes releases the GIL) -- not one column's sort
    nthr = os.cpu_count() or 1
    np.copyto(y, x)
    per = rows // nthr
    t0 = time.perf_counter()
    ths = [threading.Thread(target=orc.cafs_sort, args=(y[i * per:(i + 1) * per],))
           for i in range(nthr)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    agg = per * nthr / (time.perf_counter() - t0) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (host-generated, same bits as "
        "the device generator)",
        "config": {"workload": args.config, "n": rows, "k": c.k, "same_config": rows == c.n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"all {rows} rows of {args.config} per step; C restatement of "
                                   "the reference (single-threaded by design, SPEC.md:284); "
                                   f"nproc={os.cpu_count()}",
                         "all_cores": {"value": agg, "cores": nthr,
                                       "sample": f"{nthr} concurrent invocations on disjoint "
                                                 f"{per}-row slices (not one column)"}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _relaunch(n: int) -> None:
    """Re-execute this command under torch.distributed.run with N local ranks."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc:
        raise SystemExit(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-rows", type=int, default=0,
                    help="reference arm: rows per step (0 = the whole config column)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-direct", action="store_true", help="disable the dense-range count path")
    ap.add_argument("--dtype", default="int64", choices=["int64", "int32"],
                    help="int32: the 4-byte-key path (cfg values truncated to 32 bits)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU code path (NCCL) even at one rank")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `bench.py --gpus N` outside torchrun: start the N ranks ourselves (one
        # process per GPU, the same launch the driver uses) and pass their exit
        # code through; rank 0 prints the line
        _relaunch(args.gpus)
        return
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}; "
                         "launch N ranks with torchrun --nproc-per-node N (or drop WORLD_SIZE)")
    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    import paper_2605_25040_b200 as cafs
    from paper_2605_25040_b200 import _lib, datagen
    from paper_2605_25040_b200.sharded import cafs_sort_sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    sharded = world > 1 or args.sharded
    if sharded:
        import torch.distributed as dist
        # NCCL_DEBUG=VERSION makes NCCL print its version on stdout: keep stdout
        # to the one JSON line
        if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
            del os.environ["NCCL_DEBUG"]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = datagen.CONFIGS[args.config]
    N = cfg.n
    per = N // world
    start = rank * per
    n_local = per if rank < world - 1 else N - per * (world - 1)
    pristine = datagen.generate(cfg, n_local, start)
    if args.dtype == "int32":
        pristine = pristine.to(torch.int32)
    kb = pristine.element_size()  # bytes per key
    x = torch.empty_like(pristine)
    stream = torch.cuda.current_stream()

    def barrier():
        if dist is not None:
            dist.barrier()

    def one_step(tel):
        if not sharded:
            cafs.cafs_sort(x, telemetry=tel, direct_range=not args.no_direct,
                           exact_telemetry=False)
        else:
            cafs_sort_sharded(x, telemetry=tel)

    # warm-up with the timed region's own call (no telemetry): the library
    # captures a CUDA graph per (buffer, shape, flags) on its second sighting,
    # so the timed steps replay it rather than paying the capture
    # (the native sharded path settles later: its communicator predicts the
    # column's route class after two calls and then captures that class's graph)
    for _ in range(max(args.warmup, 6) if sharded else args.warmup):
        x.copy_(pristine)
        one_step(None)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)

    def timed_loop(steps: int, with_tel: bool):
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        tels = []
        # no garbage-collector pause inside a step (a full collection in this
        # process takes ~10 ms; timeit does the same)
        gc.collect()
        gc.disable()
        # the GPU sat idle while nvidia-smi started (up to a second) and may have
        # dropped its clocks: two more untimed steps right before the timed ones
        # (a first timed step of 3.5-4 ms against 2.38 ms showed in 3 of ~8 runs)
        for _ in range(2):
            x.copy_(pristine)
            one_step(cafs.SortTelemetry() if with_tel else None)
        barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        for i in range(steps):
            x.copy_(pristine)  # restore the unsorted input (untimed)
            tel = cafs.SortTelemetry() if with_tel else None
            ev0[i].record(stream)
            one_step(tel)
            ev1[i].record(stream)
            tels.append(tel)
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - wall0
        gc.enable()
        return [a.elapsed_time(b) for a, b in zip(ev0, ev1)], tels, wall

    # the timed region: plain API calls (no per-call instrumentation)
    step_ms, _, wall = timed_loop(args.steps, False)
    tot_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([tot_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    # the same steps again with per-kernel CUDA events (telemetry); kernel
    # durations for the roofline come from these calls
    for _ in range(2):  # the telemetry calls' own graph, captured before they are timed
        x.copy_(pristine)
        one_step(cafs.SortTelemetry())
    torch.cuda.synchronize()
    prof_ms, tels, _ = timed_loop(args.steps, True)
    clk = clocks.stop()

    # correctness of the last step (cheap property checks at full size)
    ok = bool((x[1:] >= x[:-1]).all().item())
    if cfg.palette == "codes":
        ok &= bool(torch.equal(torch.bincount(x, minlength=cfg.k),
                               torch.bincount(pristine, minlength=cfg.k)))

    value = N * args.steps / (tot_ms / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    t0 = tels[-1]
    route = t0.route.value if t0.route else None
    # dominant kernel of the step: the count pass (reads 8 B/key) or the emit (writes 8 B/key)
    k_count = [t.kernel_ms.get("count_kernel") for t in tels if "count_kernel" in t.kernel_ms]
    k_emit = [t.kernel_ms.get("emit_kernel") for t in tels if "emit_kernel" in t.kernel_ms]
    roof = None
    kernels = {}
    count_name = {"tiny": "tiny_count_kernel", "dense": "hash_count_kernel",
                  "table": "hash_count_big_kernel",
                  "partitioned": "hp_count_kernel + hp_reduce_kernel + hp_place_kernel"}.get(
                      t0.count_path, "hash_count_kernel")
    for name, vals, kname in (("count", k_count, count_name), ("emit", k_emit, "emit_kernel")):
        if vals:
            avg = sum(vals) / len(vals)
            gbs = n_local * kb / (avg / 1e3) / 1e9
            kernels[name] = {"kernel": kname, "avg_ms": avg, "GB/s": gbs,
                             "share_of_step": avg / (tot_ms / args.steps)}
    k_est = [t.kernel_ms.get("estimate_kernel") for t in tels if "estimate_kernel" in t.kernel_ms]
    if k_est:
        kernels["estimate"] = {"kernel": "estimate_kernel", "avg_ms": sum(k_est) / len(k_est),
                               "share_of_step": sum(k_est) / len(k_est) / (tot_ms / args.steps)}
    if route and route.startswith("fallback"):
        # the fallback sort is a sequence of kernels (span, chunk histogram,
        # scatter, bucket sorts); its stage time against one read + one write
        k_sort = [t.stage_ms.get("sort_k") for t in tels if "sort_k" in t.stage_ms]
        if k_sort:
            avg = sum(k_sort) / len(k_sort)
            kernels["sort"] = {"kernel": "fallback sort stage (msd_* + bucket_*)", "avg_ms": avg,
                               "GB/s": n_local * 2 * kb / (avg / 1e3) / 1e9,
                               "share_of_step": avg / (tot_ms / args.steps)}
    if any("GB/s" in v for v in kernels.values()):
        dom = max((k for k in kernels if "GB/s" in kernels[k]), key=lambda k: kernels[k]["avg_ms"])
        d = kernels[dom]
        roof = {"bound": "hbm", "kernel": d["kernel"], "achieved": d["GB/s"], "peak": peak,
                "unit": "GB/s", "frac": d["GB/s"] / peak, "traffic": ncu_traffic(args.config + ("" if kb == 8 else "_int32"), d["kernel"]),
                "algorithmic_bytes_per_launch": n_local * kb * (2 if dom == "sort" else 1),
                "peak_source": peak_src,
                "step_frac": (2 * kb * N / (tot_ms / args.steps / 1e3) / 1e9) / world / peak,
                "kernels": kernels}

    if roof is None:  # sharded path: no per-kernel events; the whole step per rank
        step_s = tot_ms / args.steps / 1e3
        ach = 2 * kb * n_local / step_s / 1e9
        roof = {"bound": "hbm", "kernel": "whole step per rank (count + emit passes; the sharded "
                "path records no per-kernel events)", "achieved": ach, "peak": peak,
                "unit": "GB/s", "frac": ach / peak, "traffic": None,
                "algorithmic_bytes_per_launch": 2 * kb * n_local, "peak_source": peak_src,
                "step_frac": ach / peak, "kernels": kernels}

    # ---- e2e through the C ABI host entry point (pinned host buffers) ----
    e2e = None
    if not sharded and args.e2e_steps > 0:
        h_in = torch.empty(N, dtype=pristine.dtype, pin_memory=True)
        h_out = torch.empty(N, dtype=pristine.dtype, pin_memory=True)
        h_in.copy_(pristine)
        lib = _lib.load()
        ctx = _lib.context(local)
        tel_c = _lib.Telemetry()
        host_sort = lib.cafs_sort_i32_host if kb == 4 else lib.cafs_sort_i64_host
        host_name = "cafs_sort_i32_host" if kb == 4 else "cafs_sort_i64_host"
        host_sort(ctx, h_in.data_ptr(), h_out.data_ptr(), N, 1, cafs.HASH_MULT, 0,
                  ctypes.byref(tel_c), stream.cuda_stream)  # warm
        torch.cuda.synchronize()
        e_t = []
        for _ in range(args.e2e_steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            rc = host_sort(ctx, h_in.data_ptr(), h_out.data_ptr(), N, 1,
                           cafs.HASH_MULT, 0, ctypes.byref(tel_c), stream.cuda_stream)
            b.record(stream)
            b.synchronize()
            _lib.check(rc, ctx, host_name)
            e_t.append(a.elapsed_time(b))
        ok &= bool((h_out[1:] >= h_out[:-1]).all().item())
        e2e = {"value": N * len(e_t) / (sum(e_t) / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": N * kb, "d2h_bytes_per_step": N * kb,
               "ms_per_step": sum(e_t) / len(e_t),
               "path": f"{host_name} (C ABI), pinned host in/out buffers"}
        del h_in, h_out
    elif sharded and args.e2e_steps > 0:
        # every rank: its pinned host shard -> device -> cafs_sort_sharded -> its
        # rows of the sorted column back to pinned host memory; max over ranks
        h_in = torch.empty(n_local, dtype=pristine.dtype, pin_memory=True)
        h_out = torch.empty(n_local, dtype=pristine.dtype, pin_memory=True)
        h_in.copy_(pristine)
        e_t = []
        for i in range(args.e2e_steps + 1):  # the first call is a warm-up
            barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            x.copy_(h_in, non_blocking=True)
            cafs_sort_sharded(x)
            h_out.copy_(x, non_blocking=True)
            b.record(stream)
            b.synchronize()
            if i:
                e_t.append(a.elapsed_time(b))
        ok &= bool((h_out[1:] >= h_out[:-1]).all().item())
        tot_e = sum(e_t)
        if dist is not None:
            t = torch.tensor([tot_e], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot_e = float(t.item())
        e2e = {"value": N * len(e_t) / (tot_e / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": N * kb, "d2h_bytes_per_step": N * kb,
               "ms_per_step": tot_e / len(e_t),
               "path": "cafs_sort_sharded per rank (public API), pinned host shards in/out; "
                       "max over ranks"}
        del h_in, h_out

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        col = pristine if kb == 8 else pristine.to(torch.int64)
        cpu = cpu_baseline(args.config, col.cpu().numpy())

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
            "data": f"synthetic, device-generated ({cfg.desc}; seed {cfg.seed})"
                    + ("; values truncated to int32" if kb == 4 else ""),
            "config": {"workload": args.config, "n": N, "k": cfg.k, "dist": cfg.dist, "s": cfg.s,
                       "route": route, "count_path": t0.count_path, "parallelism": f"rows sharded x{world}" + (" (sharded path)" if sharded else ""),
                       "l2": "input 8 B x N >> 126 MB L2; unsorted input restored by an untimed "
                             "D2D copy before each step",
                       "direct_range": not args.no_direct},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(sum(t.kernels_launched for t in tels)),
            "profiled_steps": {"n": len(prof_ms), "ms_per_step": sum(prof_ms) / len(prof_ms),
                               "note": "kernel durations in `roofline` come from these steps, "
                                       "run right after the timed region with per-kernel "
                                       "CUDA events (telemetry on); the timed region has none"},
            "clocks": clk, "correct": ok, "wall_s_timed_region": wall,
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms),
                        "max": max(step_ms), "argmax": step_ms.index(max(step_ms))},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
