"""CPU checkers for the SA scheduler hot path -- TEST INFRASTRUCTURE ONLY.

* ``oracle.ref``  -- ctypes face of the UNMODIFIED reference C++ library,
  compiled from /root/reference/proj/src by ``oracle/Makefile`` into
  ``oracle/_ref/libslosched_ref.so``.
* ``oracle.port`` -- ctypes face of ``slo_oracle.c``, the plain-C restatement
  (each function cites the reference file:line it follows).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs import this package, always as the checker or the timed CPU
baseline. The product package (``paper_2504_14966_b200``) never imports it.
"""
from .flat import FlatWorkload, TABLE_COEFFS  # noqa: F401
