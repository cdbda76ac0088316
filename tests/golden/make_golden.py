"""Generate tests/golden/ fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the container that has /root/reference (it builds oracle/_ref first):
    python tests/golden/make_golden.py [--skip-cfg5]

Outputs
  pins.json      count + sha256 of the bit table for BASELINE configs 1-5 and
                 the CLI smoke geometry, and for seeded random instances
                 (reference run_sieve + TableSink; configs 1-2 via the f = 0
                 assembly of SURVEY.md §8c: simple_sieve segment 0 +
                 run_sieve(l, 1, n-1));
  small_tables.npz  raw tables of a few tiny instances (byte-exact fixtures).
  known_answers.json  values the reference's own unit tests pin
                 (tests/test_params.cpp, test_wheel.cpp, test_kernels.cpp,
                 test_base.cpp, test_oracle.cpp), re-evaluated here through
                 the reference library so the fixture is checked, not typed.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference, build  # noqa: E402

CONFIGS = {
    "cfg1": (17, 0, 64, True),
    "cfg2": (20, 0, 4096, True),
    "cfg3": (20, (1 << 19) - 512, 1024, False),
    "cfg4": (21, (1 << 26) - 2048, 4096, False),
    "cfg5": (22, (1 << 37) - 4096, 8192, False),
    "smoke": (10, 2048, 4, False),
}


def sha(t: np.ndarray) -> str:
    return hashlib.sha256(t.tobytes()).hexdigest()


def random_instances(seed: int, count: int):
    """Seeded desk-scale instances in the spirit of testsup::random_instance
    (/root/reference/proj/tests/support.hpp:58-88): l in [4,16] test mode, v <= 2^36,
    plus instances guaranteed to have large primes (sqrt(v) > 2^l)."""
    rng = random.Random(seed)
    R = Reference()
    out = []
    while len(out) < count:
        l = rng.randint(4, 16)
        n = rng.randint(1, 64)
        if rng.random() < 0.5:
            fmax = max(1, ((1 << 36) >> (l + 1)) - n)
            f = rng.randint(1, fmax)
        else:  # with circles: v > 2^(2l)
            fmin = (1 << (2 * l)) >> (l + 1)
            f = fmin + 1 + rng.randrange(3 * fmin + 1)
        try:
            R.validate(l, f, n, test_mode=True)
        except Exception:
            continue
        out.append((l, f, n))
    return out


def main():
    build(reference=True)
    R = Reference()
    pins = {"configs": {}, "random": []}
    skip5 = "--skip-cfg5" in sys.argv
    for name, (l, f, n, ovl) in CONFIGS.items():
        if name == "cfg5" and skip5:
            continue
        t0 = time.time()
        if ovl:
            table, count = R.f0_table(l, n)
            prov = "assembled f=0: oracle simple_sieve segment 0 + reference run_sieve(l,1,n-1)"
        else:
            table, count, _ = R.run_sieve(l, f, n)
            prov = "reference run_sieve + TableSink"
        pins["configs"][name] = {"l": l, "f": f, "n": n, "allow_overlap": ovl, "count": count,
                                 "sha256": sha(table), "bytes": int(table.nbytes), "provenance": prov}
        print(name, count, f"{time.time() - t0:.1f}s", flush=True)
        del table
    small = {}
    for (l, f, n) in random_instances(1001, 48):
        table, count, _ = R.run_sieve(l, f, n, test_mode=True)
        pins["random"].append({"l": l, "f": f, "n": n, "test_mode": True, "count": count, "sha256": sha(table)})
        if table.nbytes <= 4096 and len(small) < 12:
            small[f"l{l}_f{f}_n{n}"] = table
    for (l, n) in [(12, 50), (4, 3), (10, 1), (16, 40)]:
        table, count = R.f0_table(l, n, test_mode=True)
        pins["random"].append({"l": l, "f": 0, "n": n, "test_mode": True, "allow_overlap": True, "count": count,
                               "sha256": sha(table)})
    np.savez_compressed(os.path.join(HERE, "small_tables.npz"), **small)

    # known answers pinned by the reference's own unit tests, evaluated via the reference
    ka = {
        "validate": [[10, 2048, 4, *R.validate(10, 2048, 4)]],  # test_params.cpp:21-27
        "first_offset": [[p, l, f, R.first_offset(p, l, f)] for (p, l, f) in
                         [(3, 4, 1), (7, 10, 3), (3, 4, 0), (1073741839, 22, (1 << 37) - 4096),
                          (1048583, 21, (1 << 26) - 2048)]],  # test_wheel.cpp:38-42, SURVEY §8c
        "params_from_midpoint": [[12, 21, 512, R.params_from_midpoint(12, 21, 512)],
                                 [12, 20, 1024, R.params_from_midpoint(12, 20, 1024)]],  # test_params.cpp:128-138
        "isqrt": [[4202496, R.isqrt(4202496)], [(1 << 64) - 1, R.isqrt((1 << 64) - 1)]],  # test_params.cpp:140-154
        "wheel_align": [[67, 14, 10, 1, *R.wheel_align(67, 14, 10, 1)]],  # test_wheel.cpp:87-96
        "pi_1e6": int(len(R.simple_sieve(10 ** 6))),  # test_oracle.cpp:35-38
        "rejects": [],
    }
    for (l, f, n, tm) in [(9, 1, 1, False), (31, 1, 1, False), (10, 0, 1, False), (10, 1, 0, False),
                          (10, 1, 2049, False), (10, 1, 2050, False), (4, 2048, 4, False), (3, 2048, 4, True),
                          (30, (1 << 33), 1, False)]:
        try:
            R.validate(l, f, n, test_mode=tm)
            ka["rejects"].append([l, f, n, tm, "OK"])
        except Exception as e:
            ka["rejects"].append([l, f, n, tm, e.name])
    with open(os.path.join(HERE, "known_answers.json"), "w") as fh:
        json.dump(ka, fh, indent=1)
    path = os.path.join(HERE, "pins.json")
    if skip5 and os.path.exists(path):  # keep a previously generated cfg5 pin
        old = json.load(open(path))
        if "cfg5" in old.get("configs", {}):
            pins["configs"]["cfg5"] = old["configs"]["cfg5"]
    with open(path, "w") as fh:
        json.dump(pins, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
