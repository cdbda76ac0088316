#!/usr/bin/env python3
"""Paper-comparable Table-1 curve (the reference's `erato bench`,
src/bench.cpp:20-59): 2^30-bit intervals (l = 21, n = 2^9) centred on 10^e,
NullSink run_sieve, one warm-up then the median of `reps` timed runs.

GPU: the `erato-gpu bench` subcommand (C ABI erato_gpu_count, wall clock per run,
base primes and all setup included).  CPU: the unmodified reference run_sieve
(oracle/_ref) on one core, the reference's own protocol.

    python tools/table1.py --exps 12,13,14,15,16,17,18 --out profiles/r02_table1
"""
import argparse
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gpu_curve(exps, l, reps):
    cli = os.path.join(ROOT, "paper_1111_3297_b200", "erato-gpu")
    csv = "/tmp/erato_gpu_table1.csv"
    subprocess.run([cli, "bench", "--exps", ",".join(map(str, exps)), "--log-seg", str(l), "--csv", csv,
                    "--reps", str(reps), "--machine", "B200"], check=True, capture_output=True)
    rows = {}
    for line in open(csv).read().splitlines()[1:]:
        e, sec, _ = line.split(",")
        rows[int(e)] = float(sec)
    return rows


def cpu_curve(exps, l, reps):
    from oracle.oracle import Reference
    R = Reference()
    n = 1 << (30 - l)
    rows = {}
    for e in exps:
        f = R.params_from_midpoint(e, l, n)
        R.run_sieve(l, f, n, table=False)  # warm-up
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            R.run_sieve(l, f, n, table=False)
            ts.append(time.perf_counter() - t0)
        rows[e] = statistics.median(ts)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exps", default="12,13,14,15,16,17,18")
    ap.add_argument("--log-seg", type=int, default=21)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="profiles/table1")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    exps = [int(x) for x in a.exps.split(",")]
    g = gpu_curve(exps, a.log_seg, a.reps)
    c = {} if a.no_cpu else cpu_curve(exps, a.log_seg, a.reps)
    numbers = 1 << 31  # 2^30 bits = 2^31 numbers
    with open(a.out + ".csv", "w") as fh:
        fh.write("e,gpu_seconds,cpu_1thread_seconds,l\n")
        for e in exps:
            fh.write(f"{e},{g.get(e, float('nan')):.6f},{c.get(e, float('nan')):.6f},{a.log_seg}\n")
    with open(a.out + ".md", "w") as fh:
        fh.write("# Table-1 curve: 2^30-bit intervals (l = 21, n = 512) at 10^e, NullSink, warm-up + median of "
                 f"{a.reps}\n\n| e | B200 s | B200 numbers/s | reference 1 core s | reference numbers/s | speed-up |\n"
                 "|---|---|---|---|---|---|\n")
        for e in exps:
            gs, cs = g.get(e), c.get(e)
            fh.write(f"| {e} | {gs:.6f} | {numbers / gs:.3e} | " +
                     (f"{cs:.3f} | {numbers / cs:.3e} | {cs / gs:.0f}x |\n" if cs else "- | - | - |\n"))
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
