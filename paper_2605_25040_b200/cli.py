"""``sortfile``: sort a file of 64-bit integers on the GPU.

Mirrors the reference's ``cafs sortfile`` (cli.py:142-170, parser :209-214):
``--in PATH --out PATH [--binary]``, decimal lines (blank lines skipped) or raw
little-endian int64, telemetry on stderr as ``n=.. route=.. spill=.. guard=..``,
exit codes 0 success / 1 operational failure / 2 usage error.  The reference's
other subcommands (bench grid, analyze, selftest) are its harness, not the sort
path, and stay with the reference.

The binary path reads the file straight into pinned host memory, so the sort is
one H2D copy, the device pipeline and one D2H copy (cafs_sort_i64_host).

    python -m paper_2605_25040_b200.cli sortfile --in x.bin --out y.bin --binary
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

from .sorter import SortTelemetry, cafs_sort

_LO, _HI = -(1 << 63), (1 << 63) - 1


def read_text_ints(path) -> np.ndarray:
    """Decimal integers, one per line; errors name the 1-based line (cli.py:123-138)."""
    vals = []
    with open(path, "r", encoding="utf-8") as f:
        for ln, line in enumerate(f, start=1):
            s = line.strip()
            if not s:
                continue
            try:
                v = int(s)
            except ValueError:
                raise ValueError(f"{path}:{ln}: not an integer: {s!r}")
            if not _LO <= v <= _HI:
                raise ValueError(f"{path}:{ln}: {v} outside 64-bit signed range")
            vals.append(v)
    return np.array(vals, dtype=np.int64) if vals else np.empty(0, np.int64)


def read_binary_int64(path) -> np.ndarray:
    """Raw int64 rows (a trailing partial row is ignored, as np.fromfile does),
    read into pinned host memory when CUDA is available."""
    try:
        n = os.path.getsize(path) // 8
        buf = _host_buffer(n)
        with open(path, "rb") as f:
            if n:
                f.readinto(memoryview(buf).cast("B"))
    except OSError as e:
        raise OSError(f"cannot read {path}: {e}")
    return buf


def _host_buffer(n: int) -> np.ndarray:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.empty(n, np.int64)


def cmd_sortfile(args) -> int:
    src = getattr(args, "in")
    try:
        x = read_binary_int64(src) if args.binary else read_text_ints(src)
    except (OSError, ValueError) as e:
        print(f"cafs sortfile: {e}", file=sys.stderr)
        return 1
    tel = SortTelemetry()
    try:
        cafs_sort(x, telemetry=tel)
    except RuntimeError as e:  # no device / library: an operational failure
        print(f"cafs sortfile: {e}", file=sys.stderr)
        return 1
    route = tel.route.value if tel.route else "none"
    print(f"cafs sortfile: n={x.shape[0]} route={route} "
          f"spill={tel.spill_len} guard={'yes' if tel.guard_fired else 'no'}", file=sys.stderr)
    try:
        if args.binary:
            x.tofile(args.out)
        else:
            with open(args.out, "w", encoding="utf-8", newline="\n") as f:
                f.writelines(f"{v}\n" for v in x.tolist())
    except OSError as e:
        print(f"cafs sortfile: cannot write {args.out}: {e}", file=sys.stderr)
        return 1
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="cafs-b200",
                                description="GPU adaptive low-cardinality integer sort.")
    sub = p.add_subparsers(dest="command", required=True)
    f = sub.add_parser("sortfile", help="sort a file of 64-bit integers")
    f.add_argument("--in", required=True, help="input path")
    f.add_argument("--out", required=True, help="output path")
    f.add_argument("--binary", action="store_true",
                   help="raw little-endian int64 instead of decimal lines")
    f.set_defaults(fn=cmd_sortfile)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
