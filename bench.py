#!/usr/bin/env python3
"""bench.py — sieved numbers/s of the B200 segmented sieve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A step = one full run_sieve of the configuration on the device (base primes
to sqrt(v), first offsets, buckets, every tile), the bit table written to a
resident HBM buffer, the prime count left on the device.  N > 1: launched by
torchrun, one rank per GPU; rank g sieves the contiguous shard
erato_gpu_shard(f, n, g, N) and the counts are all-reduced over NCCL (the
only collective).  Between timed steps the L2 is flushed
(256 MiB write, untimed); every step is bracketed by CUDA events on the
launching stream; the reported time is the max over ranks.

--impl reference times the reference CPU implementation (oracle/_ref, the
unmodified erato library) on this host's cores over a bounded sample of the
same configuration.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# (l, f, n, allow_overlap) — BASELINE.json configs
CONFIGS = {
    1: (17, 0, 64, True),
    2: (20, 0, 4096, True),
    3: (20, (1 << 19) - 512, 1024, False),
    4: (21, (1 << 26) - 2048, 4096, False),
    5: (22, (1 << 37) - 4096, 8192, False),
}
CONFIG_NAMES = {
    1: "cfg1 odd sieve 1..2^24 (l=17,f=0,n=64)",
    2: "cfg2 odd sieve 1..2^33 (l=20,f=0,n=4096)",
    3: "cfg3 2^31 numbers @ midpoint 2^40 (l=20,f=2^19-512,n=1024)",
    4: "cfg4 2^34 numbers @ midpoint 2^48 (l=21,f=2^26-2048,n=4096)",
    5: "cfg5 2^36 numbers @ midpoint 2^60 (l=22,f=2^37-4096,n=8192)",
}
# Algorithmic roofline work per config (re-derived exactly by
# tools/roofline_counts.py): B = table bytes + 16 B per large-prime hit of the
# reference's class split; A = shared-atomic marks (wheel + dense + large).
ROOF = {
    1: (1_048_576, 2_704_493),
    2: (536_870_912, 2_168_312_711),
    3: (134_823_344, 785_728_312),
    4: (19_421_366_720, 7_608_331_782),
    5: (174_787_646_624, 37_185_502_020),
}
# Hit records of large primes in this implementation (mod-30 wheel, 2^20-bit
# tiles), tools/roofline_counts.py `ours_large_records`: k_bin moves 8 B per record.
# (cfg3's 37 primes just above the tile size are sieved as medium primes: no records)
LARGE_RECORDS = {1: 0, 2: 0, 3: 0, 4: 835_065_655, 5: 7_429_219_143}
# ... of which come from far primes (p > WS = 148 tiles), `ours_far_records`
FAR_RECORDS = {1: 0, 2: 0, 3: 0, 4: 0, 5: 1_789_110_090}
# Medium-prime marks (smem atomics in k_tile) of this implementation, `ours_medium_marks`
# (cfg3: + its 37 primes just above the tile size, sieved as medium primes)
MEDIUM_MARKS = {1: 2_704_493, 2: 2_151_023_657, 3: 673_995_484, 4: 5_391_802_774, 5: 21_567_210_790}
# dram__bytes_read.sum + dram__bytes_write.sum per launch from `ncu --set full`
# (profiles/r01_ncu_summary.txt, cfg5 wave 100)
NCU_TRAFFIC = {5: {"k_tile": 135.7e6 + 3.7e6, "k_scatter_ml": 69.5e6 + 113.5e6, "k_scatter_far": 65.1e6 + 42.7e6}}
METRIC = "sieved numbers/sec at 2^48 & 2^60 midpoints, 1/2/4/8 GPU; % of HBM roofline"
R_ATOM_MEASURED = 3.47e12  # smem atomicOr/s per B200, microbench/mb_atomics.cu (profiles/r01_microbench_atomics.log)


def peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (getattr(self, "out", "") or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(r[0] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1111_3297_b200 as E
    from paper_1111_3297_b200 import _lib

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    l, f, n, overlap = CONFIGS[args.config]
    fg, ng = E.shard(f, n, rank, world)
    params = E.validate_params(l, fg, ng, allow_overlap=overlap)
    ctx = E.Context(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    table = torch.empty((params.table_bytes() + 15) // 16 * 16, dtype=torch.uint8, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(flags_extra=0):
        st = _lib.Stats()
        import ctypes as C
        rc = _lib.load().erato_gpu_run(ctx.handle, params.l, params.f, params.n, params.flags | flags_extra,
                                       C.c_void_p(table.data_ptr()), C.c_void_p(count.data_ptr()),
                                       C.c_void_p(stream.cuda_stream), 1, C.byref(st))
        if rc:
            E.erato._check(rc)
        if world > 1:
            dist.all_reduce(count, op=dist.ReduceOp.SUM)
        return st

    st = None
    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()
    launches_per_step = st.kernel_launches if st is not None else 0
    # ---- timed region: K steps, L2 flushed between steps (untimed) ----
    times = []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st_t = step()
            e1.record(stream)
            launches_per_step = launches_per_step or st_t.kernel_launches
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    t_local = sum(times)
    total_count = int(count.item())
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    else:
        t_max = t_local
    numbers = n << (l + 1)  # whole job: v - u + 1 over all ranks
    value = numbers * args.steps / t_max

    # ---- per-kernel phase split (one extra untimed-for-value pass) ----
    flush.fill_(1)
    ph = step(flags_extra=0x100)
    # ---- e2e through the public C-ABI (host call, count back to host) ----
    e2e_times = []
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st_e = ctx.count(params)  # erato_gpu_count: everything incl. init, count D2H
        if world > 1:
            c = torch.tensor([st_e.prime_count], dtype=torch.int64, device=dev)
            dist.all_reduce(c)
        e2e_times.append(time.perf_counter() - t0)
    t_e2e = sum(e2e_times)
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e_value = numbers * args.steps / t_e2e
    # e2e with the whole table copied to pinned host memory every step
    e2e_table = None
    if not args.no_table_e2e:
        import ctypes as C
        host = torch.empty(params.table_bytes(), dtype=torch.uint8, pin_memory=True)
        tt_times = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st_t = _lib.Stats()
            rc = _lib.load().erato_gpu_sieve_to_host(ctx.handle, params.l, params.f, params.n, params.flags,
                                                     C.cast(C.c_void_p(host.data_ptr()), _lib.u8p),
                                                     host.numel(), C.byref(st_t))
            if rc:
                E.erato._check(rc)
            tt_times.append(time.perf_counter() - t0)
        t_tab = sum(tt_times) / len(tt_times)
        if world > 1:
            tt = torch.tensor([t_tab], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_tab = float(tt.item())
        e2e_table = {"value": numbers / t_tab, "unit": "numbers/s", "h2d_bytes_per_step": 32 * world,
                     "d2h_bytes_per_step": params.table_bytes() * world + 116 * world,
                     "api": "erato_gpu_sieve_to_host (TableSink semantics: whole bit table to pinned host memory)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm, hbm_src = peaks()
    B, A = ROOF[args.config]
    ms = t_max / args.steps * 1e3
    t_hbm = B / (hbm * 1e9)
    t_atom = A / R_ATOM_MEASURED
    bound = "hbm" if t_hbm >= t_atom else "atomic"
    achieved_gbs = B / (ms / 1e3) / 1e9 / world  # per GPU, each GPU does 1/world of B
    # dominant kernel (largest device time in the phase-timed pass).  Default
    # large-prime path: k_scatter_ml (time in gen_s) + k_scatter_far (bin_s);
    # ERATO_GPU_SCATTER=genbin: k_gen + k_bin
    mode = os.environ.get("ERATO_GPU_SCATTER", "split")
    if mode == "genbin":
        split = {"k_tile": ph.small_s, "k_gen": ph.gen_s, "k_bin": ph.bin_s}
    else:
        split = {"k_tile": ph.small_s, "k_scatter_ml": ph.gen_s, "k_scatter_far": ph.bin_s}
    dom = max(split, key=split.get)
    waves = max(ph.waves, 1)
    recs = LARGE_RECORDS[args.config] / world
    alg = {  # algorithmic bytes per launch
        "k_bin": 8.0 * recs / waves,                                   # read + write each record
        "k_gen": (4.0 * recs + 8.0 * ph.base_primes) / waves,          # records out + prime state
        # ML: records out + prime state read/write; far: record out + entry in + entry out
        "k_scatter_ml": (4.0 * (recs - FAR_RECORDS[args.config] / world) + 8.0 * ph.base_primes) / waves,
        "k_scatter_far": 20.0 * FAR_RECORDS[args.config] / world / waves,
        "k_tile": (params.table_bytes() + 4.0 * recs) / waves,         # table out + records in
    }
    launch_s = split[dom] / waves
    dom_gbs = alg[dom] / launch_s / 1e9 if launch_s > 0 else 0.0
    # the tile kernel's other bound: its shared-memory atomics (medium marks + hit records)
    tile_launch_s = split["k_tile"] / waves
    tile_atoms = (MEDIUM_MARKS[args.config] + LARGE_RECORDS[args.config]) / world / waves
    tile_atomic = {"kernel": "k_tile", "achieved": round(tile_atoms / tile_launch_s, 1) if tile_launch_s > 0 else 0.0,
                   "peak": R_ATOM_MEASURED, "unit": "smem atomics/s",
                   "frac": round(tile_atoms / tile_launch_s / R_ATOM_MEASURED, 4) if tile_launch_s > 0 else 0.0}
    roof = {
        "bound": "hbm",
        "kernel": dom,
        "achieved": round(dom_gbs, 1),
        "peak": hbm,
        "unit": "GB/s",
        "frac": round(dom_gbs / hbm, 4),
        "traffic": NCU_TRAFFIC.get(args.config, {}).get(dom),
        "alg_bytes_per_launch": alg[dom],
        "launch_us": round(launch_s * 1e6, 2),
        "peak_source": hbm_src,
        "tile_atomic": tile_atomic,
    }
    run_roof = {
        "bound": bound,
        "definition": "north star: t_roof = max(B/BW_HBM, A/R_atom) for the whole run (SURVEY.md 8d)",
        "achieved_gbs": round(achieved_gbs, 1),
        "frac_hbm": round(achieved_gbs / hbm, 4),
        "algorithmic_bytes_per_step": B,
        "shared_atomics_per_step": A,
        "atomic_rate_achieved": round(A / (ms / 1e3) / world, 1),
        "atomic_rate_peak": R_ATOM_MEASURED,
        "t_roof_ms": round(max(t_hbm, t_atom) * 1e3 / world, 3),
        "binding_term": bound,
        "frac_of_roofline": round(max(t_hbm, t_atom) / world / (ms / 1e3), 4),
        "kernel_split_ms": {**{k: round(v * 1e3, 3) for k, v in split.items()}, "init": round(ph.init_s * 1e3, 3)},
    }
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "numbers/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "deterministic (l,f,n) interval; no dataset",
        "config": {"workload": CONFIG_NAMES[args.config], "l": l, "f": f, "n": n,
                   "numbers": numbers, "count": total_count,
                   "l2": "flushed between steps (256 MiB write); working set > L2",
                   "parallelism": f"range-shard x{world}"},
        "e2e": {"value": e2e_value, "unit": "numbers/s", "h2d_bytes_per_step": 32 * world,
                "d2h_bytes_per_step": 116 * world,
                "api": "erato_gpu_count (C ABI, NullSink semantics as the reference bench; includes base primes + init)"},
        "e2e_table": e2e_table,
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roof,
        "roofline_run": run_roof,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def _ref_worker(job):
    l, f, n = job
    from oracle.oracle import Reference
    R = Reference()
    t0 = time.perf_counter()
    _, cnt, ph = R.run_sieve(l, f, n, table=False)
    return cnt, time.perf_counter() - t0, ph


def reference_sample(cfg: int, procs: int, nseg: int):
    """The unmodified reference run_sieve (NullSink) over the first nseg segments
    of the config, split into `procs` contiguous ranges run in parallel processes."""
    import multiprocessing as mp
    l, f, n, overlap = CONFIGS[cfg]
    nseg = max(1, min(nseg, n))
    jobs = []
    for g in range(procs):
        b, e = nseg * g // procs, nseg * (g + 1) // procs
        if e > b:
            fb = f + b
            if overlap and fb == 0:
                fb = 1  # the reference rejects f = 0; time its f >= 1 remainder
                if e - b - 1 <= 0:
                    continue
                jobs.append((l, fb, e - b - 1))
            else:
                jobs.append((l, fb, e - b))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        res = pool.map(_ref_worker, jobs)
    wall = time.perf_counter() - t0
    numbers = sum(j[2] << (l + 1) for j in jobs)
    init = max(r[2][0] for r in res)
    return numbers, wall, init, len(jobs)


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def sample_segments(cfg: int, procs: int, budget_s: float) -> int:
    """Segments per sample so the reference's per-process segment work is
    about budget_s (rates from SURVEY.md §6, 1 core), at least procs."""
    l, f, n, _ = CONFIGS[cfg]
    per_seg = {1: 0.008 / 64, 2: 5.4 / 4096, 3: 1.7 / 1024, 4: 25.0 / 4096, 5: 160.0 / 8192}[cfg]
    return int(min(n, max(procs, procs * budget_s / per_seg)))


def cpu_baseline(cfg: int, budget_s: float = 8.0):
    procs = cpu_threads()
    nseg = sample_segments(cfg, procs, budget_s)
    numbers, wall, init, used = reference_sample(cfg, procs, nseg)
    l = CONFIGS[cfg][0]
    return {"value": numbers / wall, "unit": "numbers/s", "cores": used, "kind": "reference",
            "sample": f"reference run_sieve (oracle/_ref, NullSink) on {nseg} of {CONFIGS[cfg][2]} segments "
                      f"(l={l}), {used} processes x 1 thread over contiguous range splits; wall {wall:.2f}s "
                      f"incl. per-process init (max {init:.2f}s); CPU: {cpu_model()}"}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    ref_so = os.path.join(HERE, "oracle", "_ref", "liberato_ref.so")
    if not os.path.exists(ref_so):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liberato_ref.so not built"}))
        return
    procs = cpu_threads()
    nseg = sample_segments(args.config, procs, args.cpu_budget)
    l, f, n, _ = CONFIGS[args.config]
    for _ in range(min(args.warmup, 1)):
        reference_sample(args.config, procs, min(nseg, procs))
    tot_numbers, tot_wall, used = 0, 0.0, procs
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        numbers, wall, init, used = reference_sample(args.config, procs, nseg)
        tot_numbers += numbers
        tot_wall += wall
    value = tot_numbers / tot_wall
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "numbers/s", "n_gpus": world,
        "steps": steps, "warmup": min(args.warmup, 1), "ms_per_step": tot_wall / steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "deterministic (l,f,n) interval; no dataset",
        "config": {"workload": CONFIG_NAMES[args.config], "l": l, "f": f, "n": n},
        "cpu_baseline": {"value": value, "unit": "numbers/s", "cores": used, "kind": "reference",
                         "sample": f"{nseg} of {n} segments per step, {used} processes x 1 thread, "
                                   f"unmodified reference run_sieve (NullSink); CPU: {cpu_model()}"},
        "e2e": {"value": value, "unit": "numbers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=8.0, help="seconds of reference segment work per process")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-table-e2e", action="store_true", help="skip the table-to-host e2e measurement")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
