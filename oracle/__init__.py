"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package.  See oracle/erato_oracle.c (our plain-C
restatement) and oracle/ref_shim.cpp (ctypes shim over the unmodified reference
library built into oracle/_ref by oracle/Makefile).
"""
