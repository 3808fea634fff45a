"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the AsyncHZP hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2510_20111_b200``) never imports it and fails loudly if its CUDA
library is missing.

Two checkers live here:

* ``restated`` — our own CPU restatement: ``hzp_oracle.c`` (numerics, via
  ctypes) and ``sched_oracle.py`` (layout + task graph + ring-slot simulation
  in pure Python).  Each function cites the reference file:line it follows.
* ``ref`` — the reference itself, compiled from /root/reference/proj/src by
  ``oracle/Makefile`` into ``oracle/_ref/libhzpref.so`` (pinning the
  restatement; also the CPU baseline timed by bench.py).
"""
from .numerics import Oracle, RefLib, load_oracle, load_ref  # noqa: F401
