#!/usr/bin/env python3
"""Small runs that launch every kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) on the GPU box:

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: base sieve + compaction, medium-only tiles, ML + far scatter (mod-30
and mod-210 entries), the k_gen/k_bin fallback, the invariant checkers, the
streaming output ring, extract_primes, f = 0 overlap runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1111_3297_b200 as E  # noqa: E402

CASES = [
    (10, 2048, 4, False), (17, 0, 64, True), (20, 523776, 48, False),   # small, overlap, medium + few large
    (21, (1 << 26) - 2048, 300, False),                                  # ML primes
    (22, (1 << 37) - 4096, 160, False),                                  # ML + far (ring of buckets)
]


def main():
    ctx = E.Context(0)
    total = 0
    small = os.environ.get("SANITIZE_SMALL") == "1"  # racecheck: skip the base sieve of 2^30
    for l, f, n, ovl in (CASES[:4] if small else CASES):
        p = E.validate_params(l, f, n, allow_overlap=ovl)
        t, st = ctx.table(p)
        c = ctx.count(p, check_invariants=not ovl)
        assert c.prime_count == st.prime_count
        total += st.prime_count
    p = E.validate_params(21, (1 << 26) - 2048, 40) if small else E.validate_params(22, (1 << 37) - 4096, 40)
    os.environ["ERATO_GPU_SCATTER"] = "genbin"
    g = ctx.count(p).prime_count
    del os.environ["ERATO_GPU_SCATTER"]
    assert g == ctx.count(p).prime_count
    pr = ctx.extract_primes(E.validate_params(16, 1 << 20, 8))
    assert len(pr) > 0 and np.all(np.diff(pr.astype(np.int64)) > 0)
    ctx.close()
    print("sanitize cases ok", total)


if __name__ == "__main__":
    main()
