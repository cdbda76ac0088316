"""Sweep of small geometries with large primes (few tiles per wave, empty ML or far classes) against
the reference run_sieve, tables and counts, with the invariant checks on (run on the GPU box)."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1111_3297_b200 as E
from oracle.oracle import Reference
R = Reference()
ctx = E.Context(0)
bad = 0
cases = []
for l in (10, 12, 13, 14):
    for n in (1, 2, 3, 4, 5, 7, 8, 9, 16, 17, 33):
        for f in ((1 << 30) + 12345, (1 << 40) + 999, 987654321):
            cases.append((l, f, n))
for (l, f, n) in cases:
    try:
        p = E.validate_params(l, f, n)
    except E.Error:
        continue
    t, st = ctx.table(p)
    rt, rc, _ = R.run_sieve(l, f, n, table=True)
    ok = st.prime_count == rc and np.array_equal(np.asarray(t).view(np.uint8).ravel(), np.asarray(rt).view(np.uint8).ravel())
    st2 = ctx.count(p, check_invariants=True)
    if not ok or st2.prime_count != rc:
        bad += 1
        print("MISMATCH", l, f, n, st.prime_count, rc, st.ml_primes, st.far_primes)
print("cases", len(cases), "bad", bad)
