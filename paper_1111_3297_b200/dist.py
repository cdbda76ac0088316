"""Multi-process driver: contiguous segment-range sharding.

One process per GPU (torchrun); rank g sieves the segments
erato_gpu_shard(f, n, g, world) on its own device — base primes and offsets
are recomputed per rank, there is no data-path collective — and the only
collective is a sum all-reduce of the zero-bit counts (NCCL over NVLink on
the B200 box, gloo in the CPU tests).  Shard tables are disjoint byte ranges
of the one output file (erato_gpu_write_table part mode, pwrite at offset).
bench.py's multi-GPU path and tests/test_multiproc.py go through here; the
single-process multi-GPU entry (one thread per device, NCCL inside
liberato_gpu.so) is erato.MultiGPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

from .erato import Context, SieveParams, shard, validate_params


@dataclass
class ShardResult:
    rank: int
    world: int
    params: Optional[SieveParams]  # this rank's (l, f_g, n_g); None for an empty shard
    count: int                     # this rank's zero bits
    total: int                     # all-reduced over the ranks


def shard_params(l: int, f: int, n: int, rank: int, world: int, test_mode: bool = False,
                 allow_overlap: bool = False) -> Optional[SieveParams]:
    """This rank's sub-range, or None when the rank has no segments (world > n).
    The whole range is validated like the reference does; shards of a valid
    range are valid (u_g >= u, v_g <= v keeps u_g^2 > v_g)."""
    validate_params(l, f, n, test_mode=test_mode, allow_overlap=allow_overlap)
    fg, ng = shard(f, n, rank, world)
    if ng == 0:
        return None
    return validate_params(l, fg, ng, test_mode=test_mode, allow_overlap=allow_overlap)


def run_sharded(l: int, f: int, n: int, sieve_count: Callable[[SieveParams], int], rank: int, world: int,
                allreduce: Optional[Callable[[int], int]] = None, test_mode: bool = False,
                allow_overlap: bool = False) -> ShardResult:
    """Sieve this rank's shard with `sieve_count` (returns its zero-bit count)
    and all-reduce the counts with `allreduce` (identity when world == 1).
    A rank with an empty shard contributes 0 and still joins the reduction."""
    p = shard_params(l, f, n, rank, world, test_mode, allow_overlap)
    c = int(sieve_count(p)) if p is not None else 0
    total = allreduce(c) if (allreduce and world > 1) else c
    return ShardResult(rank, world, p, c, int(total))


def gpu_count(ctx: Context) -> Callable[[SieveParams], int]:
    """sieve_count for run_sharded on the CUDA path (NullSink run)."""
    return lambda p: ctx.count(p).prime_count


def torch_allreduce_sum(device=None) -> Callable[[int], int]:
    """Sum all-reduce of one integer through torch.distributed (NCCL or gloo)."""
    import torch
    import torch.distributed as dist

    def red(x: int) -> int:
        t = torch.tensor([x], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return int(t.item())

    return red
