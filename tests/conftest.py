"""Shared pytest setup: the ``gpu`` marker and fixture loaders."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU cases (still run by default)")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


_special_arrays = None


def special_input(name):
    """Input array of a golden special case (stored raw or regenerated)."""
    global _special_arrays
    from oracle import gen as ogen

    if name in ogen.GENERATED_SPECIAL:
        return ogen.GENERATED_SPECIAL[name]()
    if _special_arrays is None:
        _special_arrays = dict(np.load(os.path.join(GOLDEN, "special_inputs.npz")))
    return _special_arrays[name].copy()


def sweep_input(case):
    from oracle import gen as ogen

    if case["kind"] == "distinct":
        x = ogen.distinct_values(case["n"], case["seed"])
    else:
        x = ogen.gen_input(case["n"], case["k"], case["seed"])
        if case["kind"] == "sorted_ramp":
            x = np.sort(x)
    return x.view(np.int64) if case["dtype"] == "int64" else x


@pytest.fixture(scope="session")
def known_answers():
    return load_json("known_answers.json")


_dtype32_arrays = None


def dtype32_input(name):
    """Input array (int32 / uint32) of a golden 32-bit case."""
    global _dtype32_arrays
    if _dtype32_arrays is None:
        _dtype32_arrays = dict(np.load(os.path.join(GOLDEN, "dtype32_inputs.npz")))
    return _dtype32_arrays[name].copy()
