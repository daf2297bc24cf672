"""``sortfile`` CLI, mirroring the reference's tests/test_cli.py:155-220 cases.

Input errors and usage errors are decided before any device work (CPU tests);
the sorting cases run the device pipeline (gpu-marked).
"""

import numpy as np
import pytest

from paper_2605_25040_b200.cli import main as run


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except ImportError:  # pragma: no cover
        return False


gpu = pytest.mark.gpu
needs_gpu = pytest.mark.skipif(not _has_gpu(), reason="needs a CUDA device")


def test_non_numeric_line_names_line(tmp_path, capsys):
    src = tmp_path / "in.txt"
    src.write_text("1\nbanana\n3\n")
    assert run(["sortfile", "--in", str(src), "--out", str(tmp_path / "o")]) == 1
    assert ":2:" in capsys.readouterr().err


def test_out_of_range_value(tmp_path, capsys):
    src = tmp_path / "in.txt"
    src.write_text(f"{1 << 63}\n")
    assert run(["sortfile", "--in", str(src), "--out", str(tmp_path / "o")]) == 1
    assert ":1:" in capsys.readouterr().err


def test_missing_input(tmp_path):
    for extra in ([], ["--binary"]):
        assert run(["sortfile", "--in", str(tmp_path / "nope"), "--out",
                    str(tmp_path / "o")] + extra) == 1


def test_usage_errors_exit_2():
    with pytest.raises(SystemExit) as e:
        run([])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        run(["sortfile", "--in", "x"])
    assert e.value.code == 2


@gpu
@needs_gpu
def test_text_sort(tmp_path):
    src, dst = tmp_path / "in.txt", tmp_path / "out.txt"
    src.write_text("3\n1\n2\n")
    assert run(["sortfile", "--in", str(src), "--out", str(dst)]) == 0
    assert dst.read_text() == "1\n2\n3\n"
    src.write_text("5\n\n-12\n0\n")
    assert run(["sortfile", "--in", str(src), "--out", str(dst)]) == 0
    assert dst.read_text() == "-12\n0\n5\n"
    src.write_text("")
    assert run(["sortfile", "--in", str(src), "--out", str(dst)]) == 0
    assert dst.read_text() == ""


@gpu
@needs_gpu
def test_binary_round_trip_and_telemetry(tmp_path, capsys):
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    data = np.array([5, -3, 5, 0, 2**62, -(2**62)], np.int64)
    data.tofile(src)
    assert run(["sortfile", "--in", str(src), "--out", str(dst), "--binary"]) == 0
    assert np.array_equal(np.fromfile(dst, np.int64), np.sort(data))
    rng = np.random.default_rng(5)
    big = rng.integers(-1000, 1000, 3_000_000).astype(np.int64)  # the main route
    big.tofile(src)
    capsys.readouterr()
    assert run(["sortfile", "--in", str(src), "--out", str(dst), "--binary"]) == 0
    assert np.array_equal(np.fromfile(dst, np.int64), np.sort(big))
    err = capsys.readouterr().err
    assert "n=3000000" in err and "route=main" in err and "guard=no" in err
