#!/usr/bin/env python3
"""Exact algorithmic work of a run under the REFERENCE's class rules — the
roofline denominators of BASELINE.md / SURVEY.md §8(d), re-derived here.

  B = table bytes + 16 B per large-prime hit      (8 B pair read + 8 B write,
      PrimeOffsetPair /root/reference/proj/include/erato/base.hpp:25-28)
  A = shared-memory marks = wheel-medium marks + dense-medium marks + large hits
      (masks for p <= 61 are word ORs, not atomics)

Classes (classify_prime, src/base.cpp:11-17): small p <= 61; wheel-medium
64 <= p <= 2^l/16 (only cofactors coprime to 15, src/kernels.cpp:19-36);
dense-medium 2^l/16 < p < 2^l; large p > 2^l.  Marks are counted over
[u, v] from the first odd multiple >= u (the reference does not start at
p^2), except f = 0 runs, which follow the SURVEY.md §8c convention (p^2).

Also reports what THIS implementation does (wheel mod 30 for every p > 61,
tiles of 2^log_tile bits): its atomics and its large-prime record count.

    python tools/roofline_counts.py --config 5
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from oracle.oracle import Restated  # noqa: E402

# number of c in [1, x] coprime to 30, via a 30-periodic table
_T30 = np.array([sum(1 for c in range(1, r + 1) if np.gcd(c, 30) == 1) for r in range(30)], dtype=np.int64)


def coprime30_upto(x: np.ndarray) -> np.ndarray:
    x = np.maximum(x, 0)
    return 8 * (x // 30) + _T30[x % 30]


def coprime210_upto(x: np.ndarray) -> np.ndarray:
    """#{1 <= c <= x : gcd(c, 210) = 1}: coprime to 30, minus the multiples 7c' with c' coprime to 30."""
    x = np.maximum(x, 0)
    return coprime30_upto(x) - coprime30_upto(x // 7)


def odd_upto(x: np.ndarray) -> np.ndarray:
    return (np.maximum(x, 0) + 1) // 2


def counts(l: int, f: int, n: int, log_tile: int = 20, wave_tiles: int = 148):
    R = Restated()
    u = (f << (l + 1)) + 1
    v = (f + n) << (l + 1)
    T = n << l
    primes = R.simple_sieve(R.isqrt(v)).astype(np.int64)
    primes = primes[primes > 2]
    seg = 1 << l
    lo = np.maximum((u + primes - 1) // primes, 1)  # first cofactor c with c*p >= u
    if f == 0:
        lo = np.maximum(lo, primes)  # p^2 convention
    hi = v // primes
    n_odd = odd_upto(hi) - odd_upto(lo - 1)
    n_wheel = coprime30_upto(hi) - coprime30_upto(lo - 1)
    small = primes <= 61
    wheel = (~small) & (primes * 16 <= seg) & (primes <= seg)
    large = primes > seg
    dense = (~small) & (~wheel) & (~large)
    A_wheel = int(n_wheel[wheel].sum())
    A_dense = int(n_odd[dense].sum())
    H_large = int(n_odd[large].sum())
    B = T // 8 + 16 * H_large
    A = A_wheel + A_dense + H_large
    # this implementation: every p > 61 with the mod-30 wheel, from p^2 in overlap runs
    S = 1 << log_tile
    ours_med = (~small) & (primes <= S)
    ours_large = primes > S
    lo2 = lo.copy()
    if (u * u) <= v:
        lo2 = np.maximum(lo2, np.where(primes <= S, primes, 2))
    ours_marks = coprime30_upto(hi) - coprime30_upto(lo2 - 1)
    # large primes skipping cofactors divisible by 7 (mod-210 far entries / ML states)
    ours_marks210 = coprime210_upto(hi) - coprime210_upto(lo2 - 1)
    WSb = wave_tiles * S
    ml = (primes > S) & (primes <= WSb)
    far = primes > WSb
    return {
        "l": l, "f": f, "n": n, "table_bits": T, "base_primes": int(len(primes)),
        "ref_wheel_marks": A_wheel, "ref_dense_marks": A_dense, "ref_large_hits": H_large,
        "B_bytes": B, "A_atomics": A,
        "ours_medium_marks": int(ours_marks[ours_med].sum()),
        "ours_large_records": int(ours_marks[ours_large].sum()),
        # far primes (p > WS = wave_tiles * 2^log_tile) reach the wave through the bucket ring
        "ours_far_records": int(ours_marks[primes > wave_tiles * S].sum()),
        "ours_ml_records_mod30": int(ours_marks[ml].sum()),
        "ours_ml_records_mod210": int(ours_marks210[ml].sum()),
        "ours_far_records_mod210": int(ours_marks210[far].sum()),
        "ours_log_tile": log_tile,
        "ours_wave_tiles": wave_tiles,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, nargs="*", default=[1, 2, 3, 4, 5])
    args = ap.parse_args()
    out = {}
    for c in args.config:
        l, f, n, _ = CONFIGS[c]
        out[c] = counts(l, f, n)
        print(json.dumps({"config": c, **out[c]}), flush=True)


if __name__ == "__main__":
    main()
