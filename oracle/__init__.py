"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle for the B200 CAFS sort.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline
and ``--impl reference`` legs) may import this package.  The product package
``paper_2605_25040_b200`` never imports it: there is no CPU fallback.

* :mod:`oracle.cafs_oracle` -- ctypes binding of ``cafs_oracle.c``, a C
  restatement of the reference algorithm (``/root/reference/pkg/src/cafs``).
* :mod:`oracle.gen` -- numpy restatement of the synthetic input generators
  (bit-identical to the device generator in the product's ``gen.cu``).
"""
