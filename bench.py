#!/usr/bin/env python3
"""bench.py — sieved numbers/s of the B200 segmented sieve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A step = one full run_sieve of the configuration on the device (base primes
to sqrt(v), first offsets, buckets, every tile), the bit table written to a
resident HBM buffer, the prime count left on the device.  N > 1: one rank per
GPU (torchrun; `--gpus N` without torchrun re-launches itself under it);
rank g sieves the contiguous shard erato_gpu_shard(f, n, g, N) and the counts
are all-reduced over NCCL (the only collective).  Between
timed steps the L2 is flushed (256 MiB write, untimed); every step is
bracketed by CUDA events on the launching stream; the reported time is the
max over ranks.  The headline config is cfg5 (midpoint 2^60); the metric's
other midpoint, cfg4 (2^48), is measured the same way in the same run and
reported in the "cfg4" sub-object.

--impl reference times the reference CPU implementation (oracle/_ref, the
unmodified erato library) on this host's cores.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
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
# tools/roofline_counts.py, profiles/r01_roofline_counts.jsonl): B = table bytes
# + 16 B per large-prime hit of the reference's class split; A = shared-atomic
# marks (wheel + dense + large).
ROOF = {
    1: (1_048_576, 2_704_493),
    2: (536_870_912, 2_168_312_711),
    3: (134_823_344, 785_728_312),
    4: (19_421_366_720, 7_608_331_782),
    5: (174_787_646_624, 37_185_502_020),
}
# This implementation's own medium-prime marks (tools/roofline_counts.py `ours_*`, 2^20-bit tiles);
# the large-prime hit records are counted on the device by the run itself (stats.large_records /
# far_records with ERATO_GPU_CHECK_INVARIANTS) — they depend on the wheel modulus and the ML/far split.
# (cfg3's 37 primes just above the tile size are sieved as medium primes: no records)
MEDIUM_MARKS = {1: 2_704_493, 2: 2_151_023_657, 3: 673_975_296, 4: 5_391_802_774, 5: 21_567_210_790}
METRIC = "sieved numbers/sec at 2^48 & 2^60 midpoints, 1/2/4/8 GPU; % of HBM roofline"
# smem atomicOr/s per B200 at random word addresses (the sieve's bank-conflict
# mix), 1024-thread CTAs over a 128 KiB tile: microbench/mb_atomics.cu
# k_smem_atom_pure (16 unrolled ATOMS per loop, addresses in registers),
# profiles/r02_microbench_atomics.log
R_ATOM_MEASURED = 4.06e12
NCU_TRAFFIC_FILE = os.path.join(HERE, "profiles", "ncu_traffic.json")
# the device code of the wave kernels (a capture of other device code is not used)
KERNEL_SOURCES = [os.path.join(HERE, "paper_1111_3297_b200", "csrc", "sieve_kernels.cuh")]


def peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_src_sha() -> str:
    h = hashlib.sha256()
    for p in KERNEL_SOURCES:
        with open(p, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_traffic(cfg: int):
    """dram bytes read+written per launch from the ncu --set full capture of
    THESE kernel sources (profiles/ncu_traffic.json carries the sources' hash;
    a capture of other sources is not used)."""
    try:
        with open(NCU_TRAFFIC_FILE) as fh:
            d = json.load(fh)
    except Exception:
        return None, "no capture"
    if d.get("kernel_src_sha") != kernel_src_sha() or int(d.get("config", 0)) != cfg:
        return None, "capture is of other kernel sources / config"
    return d.get("per_launch_bytes", {}), d.get("source", "")


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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


def relaunch_under_torchrun(args) -> None:
    """`bench.py --gpus N` (N > 1) outside torchrun: one rank per GPU via
    torch.distributed.run on 127.0.0.1; fails loudly if N GPUs are not there."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested, {have} CUDA devices visible"}), flush=True)
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


# ---------------------------------------------------------------------------
class Rank:
    """This process's GPU, context and (N > 1) process group."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        import paper_1111_3297_b200 as E
        self.torch, self.dist, self.E = torch, dist, E
        self.rank, self.world, self.local = dist_env()
        # BENCH_TEST_SAME_DEVICE=1 (tests only): every rank on cuda:0 over gloo, to
        # exercise the multi-rank path on a 1-GPU box (NCCL refuses two ranks per GPU);
        # such a line is marked "test_topology" and is not a scaling measurement
        self.test_topology = os.environ.get("BENCH_TEST_SAME_DEVICE") == "1" and self.world > 1
        if self.test_topology:
            self.local = 0
        torch.cuda.set_device(self.local)
        if self.world > 1:
            if self.test_topology:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.dev = torch.device("cuda", self.local)
        self.ctx = E.Context(self.local)
        self.stream = torch.cuda.current_stream(self.dev)
        self.flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def allreduce(self, x: float, op: str = "max", dtype=None):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=dtype or self.torch.float64,
                              device="cpu" if self.test_topology else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return t.item()

    def params(self, cfg: int):
        l, f, n, overlap = CONFIGS[cfg]
        fg, ng = self.E.shard(f, n, self.rank, self.world)
        return self.E.validate_params(l, fg, ng, allow_overlap=overlap)


def measure(R: Rank, cfg: int, steps: int, warmup: int):
    """Device-timed steps of one config (count left on the device, NCCL
    all-reduce of the count inside the step for N > 1)."""
    import ctypes as C
    from paper_1111_3297_b200 import _lib
    torch, E = R.torch, R.E
    params = R.params(cfg)
    table = torch.empty((params.table_bytes() + 15) // 16 * 16, dtype=torch.uint8, device=R.dev)
    count = torch.zeros(1, dtype=torch.int64, device=R.dev)

    def step(flags_extra=0):
        st = _lib.Stats()
        rc = _lib.load().erato_gpu_run(R.ctx.handle, params.l, params.f, params.n, params.flags | flags_extra,
                                       C.c_void_p(table.data_ptr()), C.c_void_p(count.data_ptr()),
                                       C.c_void_p(R.stream.cuda_stream), 1, C.byref(st))
        E.erato._check(rc)
        if R.world > 1:
            if R.test_topology:  # gloo: through the host
                c = count.cpu()
                R.dist.all_reduce(c, op=R.dist.ReduceOp.SUM)
                count.copy_(c)
            else:
                R.dist.all_reduce(count, op=R.dist.ReduceOp.SUM)
        return st

    st = None
    for _ in range(warmup):
        st = step()
    torch.cuda.synchronize()
    launches = st.kernel_launches if st is not None else 0
    times = []
    with ClockSampler(R.local) as clk:
        R.barrier()
        torch.cuda.synchronize()
        for _ in range(steps):
            R.flush_buf.fill_(1)  # L2 flush between steps (untimed)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(R.stream)
            st_t = step()
            e1.record(R.stream)
            launches = launches or st_t.kernel_launches
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        torch.cuda.synchronize()
        # short configs (cfg1-3: a millisecond per step): keep the same load running, untimed, until the
        # clock sampler (one nvidia-smi line per 50 ms) has seen it
        t_load = time.perf_counter()
        while sum(times) < 0.5 and time.perf_counter() - t_load < 0.6:
            step()
        torch.cuda.synchronize()
        R.barrier()
    t_max = R.allreduce(sum(times), "max")
    total_count = int(count.item())
    l, f, n, _ = CONFIGS[cfg]
    numbers = n << (l + 1)  # whole job: v - u + 1 over all ranks
    # per-kernel phase split: one extra pass with CUDA events around every launch
    R.flush_buf.fill_(1)
    ph = step(flags_extra=0x100)
    # the run's own record counts: one pass with the device invariant checks on (untimed)
    inv = step(flags_extra=0x200)
    del table
    return {"cfg": cfg, "params": params, "times": times, "t_max": t_max, "count": total_count, "numbers": numbers,
            "value": numbers * steps / t_max, "ms": t_max / steps * 1e3, "launches": launches, "phase": ph,
            "records": (inv.large_records, inv.far_records), "clocks": clk.summary()}


def roofline(m, world: int):
    """The north-star run roofline and the per-kernel rooflines."""
    cfg, ph = m["cfg"], m["phase"]
    hbm, hbm_src = peaks()
    B, A = ROOF[cfg]
    secs = m["ms"] / 1e3
    t_hbm = B / (hbm * 1e9)
    t_atom = A / R_ATOM_MEASURED
    bound = "hbm" if t_hbm >= t_atom else "atomic"
    run = {
        "definition": "north star: t_roof = max(B/BW_HBM, A/R_atom) for the whole run (SURVEY.md 8d); "
                      "B and A from the reference's class split, divided over the ranks",
        "bound": bound,
        "algorithmic_bytes_per_step": B,
        "shared_atomics_per_step": A,
        "achieved_gbs": round(B / secs / 1e9 / world, 1),
        "frac_hbm": round(B / secs / 1e9 / world / hbm, 4),
        "atomic_rate_achieved": round(A / secs / world, 1),
        "atomic_rate_peak": R_ATOM_MEASURED,
        "t_roof_ms": round(max(t_hbm, t_atom) * 1e3 / world, 3),
        "frac_of_roofline": round(max(t_hbm, t_atom) / world / secs, 4),
        "kernel_split_ms": {"k_tile": round(ph.small_s * 1e3, 3), "k_ml_walk": round(ph.gen_s * 1e3, 3),
                            "k_far_walk": round(ph.walk_s * 1e3, 3),
                            "k_wave_sort": round((ph.bin_s - ph.walk_s) * 1e3, 3), "init": round(ph.init_s * 1e3, 3),
                            "masks_phase_cta0": round(ph.masks_s * 1e3, 3)},
        "kernel_split_note": "from one extra pass with CUDA events around every launch; there k_wave_sort runs after "
                             "k_ml_walk, in the timed steps beside it on a side stream (the sum exceeds ms_per_step)",
        "large_prime_wheel": ph.wheel,
    }
    # ---- per-kernel: algorithmic bytes per launch / average launch time ----
    # record counts of THIS run (device-counted with ERATO_GPU_CHECK_INVARIANTS
    # in an untimed pass): all large-prime hit records, and the far primes' share
    waves = max(ph.waves, 1)
    recs, far = m["records"]
    ml = recs - far
    nwin = max(ph.far_windows, 1)
    table_bytes = m["params"].table_bytes()
    alg = {
        # table written once + every hit record read once
        "k_tile": (table_bytes + 4.0 * recs) / waves,
        # per wave: ML records written + every ML prime read (4 B) and its state read and rewritten (8 B + 8 B)
        "k_ml_walk": 4.0 * ml / waves + 20.0 * ph.ml_primes,
        # per window of waves: far records written + every far prime read (4 B), state read and rewritten (8 B + 8 B)
        "k_far_walk": 4.0 * far / nwin + 20.0 * ph.far_primes,
        # per wave: the wave's far records read and written once
        "k_wave_sort": 8.0 * far / waves,
    }
    launch_s = {"k_tile": ph.small_s / waves, "k_ml_walk": ph.gen_s / waves, "k_far_walk": ph.walk_s / nwin,
                "k_wave_sort": (ph.bin_s - ph.walk_s) / waves}
    step_s = {"k_tile": ph.small_s, "k_ml_walk": ph.gen_s, "k_far_walk": ph.walk_s, "k_wave_sort": ph.bin_s - ph.walk_s}
    traffic, tsrc = ncu_traffic(cfg)
    kernels = {}
    for k in alg:
        if launch_s[k] <= 0:
            continue
        ach = alg[k] / launch_s[k] / 1e9
        kernels[k] = {"alg_bytes_per_launch": round(alg[k]), "launch_us": round(launch_s[k] * 1e6, 2),
                      "achieved": round(ach, 1), "frac": round(ach / hbm, 4),
                      "traffic": (traffic or {}).get(k)}
    tile_atoms = MEDIUM_MARKS[cfg] / world / waves + recs / waves
    run["large_prime_records"] = {"all": recs, "far": far}
    if launch_s["k_tile"] > 0:
        kernels["k_tile"]["smem_atomics_per_launch"] = round(tile_atoms)
        kernels["k_tile"]["atomic_rate"] = round(tile_atoms / launch_s["k_tile"], 1)
        kernels["k_tile"]["atomic_frac"] = round(tile_atoms / launch_s["k_tile"] / R_ATOM_MEASURED, 4)
    dom = max(step_s, key=step_s.get)  # the kernel with the largest share of the step
    d = kernels.get(dom, {})
    roof = {"bound": "hbm", "kernel": dom, "achieved": d.get("achieved", 0.0), "peak": hbm, "unit": "GB/s",
            "frac": d.get("frac", 0.0), "traffic": d.get("traffic"),
            "alg_bytes_per_launch": d.get("alg_bytes_per_launch"), "launch_us": d.get("launch_us"),
            "peak_source": hbm_src, "traffic_source": tsrc, "kernels": kernels}
    return roof, run


def e2e_count(R: Rank, cfg: int, steps: int):
    """The user's call: erato_gpu_count through the C ABI (scalars in, count
    back to the host), wall clock around it, max over ranks."""
    params = R.params(cfg)
    ts = []
    R.barrier()
    for _ in range(steps):
        R.flush_buf.fill_(1)
        R.torch.cuda.synchronize()
        t0 = time.perf_counter()
        c = R.ctx.count(params).prime_count
        if R.world > 1:
            c = int(R.allreduce(c, "sum", dtype=R.torch.int64))
        ts.append(time.perf_counter() - t0)
    return R.allreduce(sum(ts), "max") / steps


def e2e_table(R: Rank, cfg: int, steps: int):
    """erato_gpu_sieve_to_host into pinned memory (TableSink semantics): every
    wave's slice is copied D2H while the next waves sieve."""
    import ctypes as C
    from paper_1111_3297_b200 import _lib
    params = R.params(cfg)
    host = R.torch.empty(params.table_bytes(), dtype=R.torch.uint8, pin_memory=True)
    ts = []
    for _ in range(steps):
        R.flush_buf.fill_(1)
        R.torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = _lib.Stats()
        R.E.erato._check(_lib.load().erato_gpu_sieve_to_host(
            R.ctx.handle, params.l, params.f, params.n, params.flags,
            C.cast(C.c_void_p(host.data_ptr()), _lib.u8p), host.numel(), C.byref(st)))
        ts.append(time.perf_counter() - t0)
    del host
    return R.allreduce(sum(ts), "max") / steps, params.table_bytes()


def e2e_file(R: Rank, cfg: int, steps: int, out_dir: str):
    """write_table (FileSink semantics) to out_dir: streamed wave slices,
    pwrite at the shard's offset of the one reference-named file."""
    l, f, n, overlap = CONFIGS[cfg]
    whole = R.E.validate_params(l, f, n, allow_overlap=overlap)
    params = R.params(cfg)
    ts = []
    path = None
    for _ in range(steps):
        R.barrier()
        t0 = time.perf_counter()
        path, _ = R.ctx.write_table(out_dir, whole, params.f, params.n)
        R.barrier()
        ts.append(time.perf_counter() - t0)
    t = R.allreduce(sum(ts), "max") / steps
    size = os.path.getsize(path) if path else 0
    R.barrier()
    if R.rank == 0 and path:
        os.unlink(path)
    return t, path, size


def run_ours(args):
    R = Rank()
    head = measure(R, args.config, args.steps, args.warmup)
    secondary = None
    if args.config == 5 and not args.no_cfg4:
        secondary = measure(R, 4, args.steps, args.warmup)
    e2e_steps = max(1, min(args.steps, 5))
    t_e2e = e2e_count(R, args.config, e2e_steps)
    tab = None if args.no_table_e2e else e2e_table(R, args.config, max(1, min(args.steps, 3)))
    fil = None if args.no_file_e2e else e2e_file(R, args.config, max(1, min(args.steps, 2)), args.out_dir)
    if R.rank != 0:
        if R.world > 1:
            R.dist.destroy_process_group()
        return
    world = R.world
    roof, run_roof = roofline(head, world)
    line = {
        "metric": METRIC,
        "value": head["value"],
        "unit": "numbers/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms"],
        "step_ms": [round(t * 1e3, 3) for t in head["times"]],  # this rank's timed steps, one by one
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "deterministic (l,f,n) interval; no dataset",
        "config": {"workload": CONFIG_NAMES[args.config], "l": CONFIGS[args.config][0], "f": CONFIGS[args.config][1],
                   "n": CONFIGS[args.config][2], "numbers": head["numbers"]},
        "count": head["count"],
        "parallelism": f"range-shard x{world} (one rank per GPU, NCCL all-reduce of the count)"
                       + (" [TEST TOPOLOGY: all ranks on cuda:0 over gloo]" if R.test_topology else ""),
        "l2": "flushed between steps (256 MiB write, untimed); working set > L2",
        "e2e": {"value": head["numbers"] / t_e2e, "unit": "numbers/s", "h2d_bytes_per_step": 32 * world,
                "d2h_bytes_per_step": 8 * world,
                "api": "erato_gpu_count (C ABI, NullSink semantics as the reference bench; base primes + init "
                       "included; the count comes back to the host)"},
        "gpu_launches": head["launches"] * args.steps,
        "roofline": roof,
        "roofline_run": run_roof,
        "clocks": head["clocks"],
    }
    if tab is not None:
        line["e2e_table"] = {"value": head["numbers"] / tab[0], "unit": "numbers/s",
                             "h2d_bytes_per_step": 32 * world, "d2h_bytes_per_step": tab[1] * world + 8 * world,
                             "api": "erato_gpu_sieve_to_host (TableSink semantics: the whole table to pinned host "
                                    "memory, each wave's slice copied while the next waves sieve)"}
    if fil is not None:
        line["e2e_file"] = {"value": head["numbers"] / fil[0], "unit": "numbers/s", "seconds": round(fil[0], 3),
                            "file": fil[1], "bytes": fil[2],
                            "api": "erato_gpu_write_table (FileSink semantics: wave slices streamed through "
                                   "pinned slots and pwrite()n; neither HBM nor host memory holds the whole table)"}
    if secondary is not None:
        r4, run4 = roofline(secondary, world)
        line["cfg4"] = {"workload": CONFIG_NAMES[4], "value": secondary["value"], "unit": "numbers/s",
                        "ms_per_step": secondary["ms"], "steps": args.steps, "count": secondary["count"],
                        "roofline_run": run4, "roofline": {k: r4[k] for k in ("kernel", "achieved", "frac", "kernels")},
                        "clocks": secondary["clocks"]}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)
    if world > 1:
        R.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# The reference CPU implementation (oracle/_ref: the unmodified erato library).
def _ref_worker(job):
    l, f, n = job
    from oracle.oracle import Reference
    R = Reference()
    t0 = time.perf_counter()
    _, cnt, ph = R.run_sieve(l, f, n, table=False)
    return cnt, time.perf_counter() - t0, ph


def reference_sample(cfg: int, procs: int, nseg: int):
    """The unmodified reference run_sieve (NullSink, the protocol of
    src/bench.cpp:11-16) over the first nseg segments of the config, split
    into `procs` contiguous ranges run as parallel single-threaded processes.
    Returns (numbers, wall seconds, max per-process init seconds, processes,
    count)."""
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
    if len(jobs) == 1:
        res = [_ref_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(len(jobs)) as pool:
            res = pool.map(_ref_worker, jobs)
    wall = time.perf_counter() - t0
    numbers = sum(j[2] << (l + 1) for j in jobs)
    init = max(r[2][0] for r in res)
    return numbers, wall, init, len(jobs), sum(r[0] for r in res)


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


def one_thread_segments(cfg: int, budget_s: float) -> int:
    """Segments whose single-core reference segment work is about budget_s
    (rates from SURVEY.md §6)."""
    l, f, n, _ = CONFIGS[cfg]
    per_seg = {1: 0.008 / 64, 2: 5.4 / 4096, 3: 1.7 / 1024, 4: 25.0 / 4096, 5: 160.0 / 8192}[cfg]
    return int(min(n, max(1, budget_s / per_seg)))


def one_thread_figure(cfg: int, budget_s: float, reps: int):
    """1 process x 1 thread (the reference is single-threaded by design,
    /root/reference/SPEC.md:481) on a bounded sample; median of reps runs."""
    nseg = one_thread_segments(cfg, budget_s)
    runs = [reference_sample(cfg, 1, nseg) for _ in range(reps)]
    walls = sorted(r[1] for r in runs)
    med = walls[len(walls) // 2]
    numbers, _, init, _, _ = runs[0]
    seg_s = med - init
    return {"value": numbers / med, "unit": "numbers/s", "cores": 1, "kind": "reference",
            "segments_only_value": numbers / seg_s if seg_s > 0 else None,
            "init_s": round(init, 2), "wall_s": round(med, 2), "init_share": round(init / med, 3),
            "runs": reps, "sample": f"{nseg} of {CONFIGS[cfg][2]} segments, 1 process x 1 thread, median of {reps}"}


def all_cores_figure(cfg: int, reps: int):
    """P = all host threads as P single-threaded processes over contiguous
    range splits of the WHOLE config (exact: every sub-range keeps u^2 > v);
    median of reps runs."""
    procs = cpu_threads()
    l, f, n, _ = CONFIGS[cfg]
    runs = [reference_sample(cfg, procs, n) for _ in range(reps)]
    walls = sorted(r[1] for r in runs)
    med = walls[len(walls) // 2]
    numbers, _, init, used, cnt = runs[0]
    return {"value": numbers / med, "unit": "numbers/s", "cores": used, "kind": "reference",
            "init_s": round(init, 2), "wall_s": round(med, 2), "init_share": round(init / med, 3), "count": cnt,
            "runs": reps, "sample": f"all {n} segments, {used} processes x 1 thread over contiguous range splits, "
                                    f"median of {reps}"}


def cpu_baseline(cfg: int, budget_s: float = 5.0, reps: int = 1):
    allp = all_cores_figure(cfg, reps)
    one = one_thread_figure(cfg, budget_s, reps)
    return {"value": allp["value"], "unit": "numbers/s", "cores": allp["cores"], "kind": "reference",
            "sample": allp["sample"] + f"; unmodified reference run_sieve (oracle/_ref, NullSink); each process "
                                       f"pays the reference's own init (max {allp['init_s']} s of {allp['wall_s']} s "
                                       f"wall); CPU: {cpu_model()}",
            "all_cores": allp, "one_thread": one}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    ref_so = os.path.join(HERE, "oracle", "_ref", "liberato_ref.so")
    if not os.path.exists(ref_so):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liberato_ref.so not built"}))
        return
    l, f, n, _ = CONFIGS[args.config]
    if args.warmup > 0:  # warm-up (bench.cpp:37-42): page the library and the CPU in on a small config
        reference_sample(3, cpu_threads(), 64)
    reps = max(1, min(args.steps, 3))
    allp = all_cores_figure(args.config, reps)
    one = one_thread_figure(args.config, args.cpu_budget, reps)
    value = allp["value"]
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "numbers/s", "n_gpus": world,
        "steps": reps, "warmup": 1 if args.warmup > 0 else 0, "ms_per_step": allp["wall_s"] * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "deterministic (l,f,n) interval; no dataset",
        "config": {"workload": CONFIG_NAMES[args.config], "l": l, "f": f, "n": n, "numbers": n << (l + 1)},
        "count": allp["count"],
        "protocol": "reference bench protocol (src/bench.cpp:37-42): one warm-up, then the median of "
                    f"{reps} runs; NullSink run_sieve; value = the whole config on all host threads",
        "cpu_baseline": {"value": value, "unit": "numbers/s", "cores": allp["cores"], "kind": "reference",
                         "sample": allp["sample"] + f"; unmodified reference run_sieve; CPU: {cpu_model()}",
                         "all_cores": allp, "one_thread": one},
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
    ap.add_argument("--cpu-budget", type=float, default=5.0, help="seconds of 1-thread reference segment work")
    ap.add_argument("--out-dir", default="/tmp", help="directory of the file-output e2e run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-table-e2e", action="store_true", help="skip the table-to-host e2e measurement")
    ap.add_argument("--no-file-e2e", action="store_true", help="skip the write_table e2e measurement")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the cfg4 (2^48 midpoint) measurement")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    rank, world, local = dist_env()
    if world != args.gpus and "WORLD_SIZE" in os.environ and args.gpus != 1:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    run_ours(args)


if __name__ == "__main__":
    main()
