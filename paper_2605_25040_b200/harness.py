"""Adjacency to the reference's benchmark harness.

The reference's grid (``cafs/bench.py:94-136``) times any in-place sorter
registered in ``ALGORITHMS`` (name -> callable(x) on a numpy array) and checks
its output against ``np.sort``.  :func:`register` adds this package's sort to
such a registry, so ``run_point(n, k, ["cafs_b200"], registry=...)``, the CSV
export and the entropy-bin analysis run unchanged against the B200 path:

    from cafs import bench
    from paper_2605_25040_b200.harness import register
    bench.run_point(1_000_000, 200, ["cafs", "cafs_b200"],
                    registry=register(dict(bench.ALGORITHMS)))
"""

from __future__ import annotations

from .sorter import cafs_sort

NAME = "cafs_b200"


def cafs_b200(x) -> None:
    """In-place sort of a numpy array through the device pipeline (host entry point)."""
    cafs_sort(x)


def register(registry: dict, name: str = NAME) -> dict:
    """Add the B200 sort to a reference-style registry; returns it."""
    registry[name] = cafs_b200
    return registry


ALGORITHMS = {NAME: cafs_b200}
