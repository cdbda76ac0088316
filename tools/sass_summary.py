#!/usr/bin/env python3
"""Static SASS summary of the hot kernels in liberato_gpu.so (cuobjdump -sass):
instruction count, the opcodes that matter for this path (ATOMS = shared
atomics, LDGSTS = cp.async, STG/LDG, BAR, SHFL, VOTE, MATCH) and a check that no
kernel calls a subroutine (CALL: e.g. a 64-bit division by a runtime value).

    python tools/sass_summary.py [paper_1111_3297_b200/liberato_gpu.so]
"""
import collections
import re
import subprocess
import sys

SO = sys.argv[1] if len(sys.argv) > 1 else "paper_1111_3297_b200/liberato_gpu.so"
HOT = ("k_tile", "k_ml_walk", "k_far_walk", "k_wave_sort", "k_scatter_ml", "k_scatter_far", "k_setup_large")
KEY = ("ATOMS", "RED", "ATOMG", "LDGSTS", "LDG", "STG", "LDS", "STS", "BAR", "SHFL", "VOTE", "MATCH", "CALL", "MUFU",
       "DMUL", "I2F", "F2I")


def main():
    out = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if cur and m:
            funcs[cur][m.group(1).split(".")[0]] += 1
    calls = 0
    print(f"# static SASS of {SO} (cuobjdump -sass), hot kernels")
    print("kernel".ljust(58), "instr", " ".join(k.rjust(6) for k in KEY))
    for f, c in funcs.items():
        if not any(h in f for h in HOT):
            continue
        if "k_setup_large" not in f:  # the wave kernels; setup runs once per run (fp64 reciprocal slow path)
            calls += c["CALL"]
        print(f[:58].ljust(58), str(sum(c.values())).rjust(5), " ".join(str(c[k]).rjust(6) for k in KEY))
    print(f"# CALL instructions in the wave kernels (k_tile, k_ml_walk, k_far_walk, k_wave_sort, legacy k_scatter_*): {calls} (must be 0)")
    return 1 if calls else 0


if __name__ == "__main__":
    sys.exit(main())
