"""World-size-2 and -4 gloo tests of the N>1 path on CPU: contiguous shards,
one count all-reduce, shard tables concatenating to the full table, and a
rank with an empty shard (world > n) that still joins the reduction.  The
per-rank sieve is the CPU oracle here (test infrastructure); on the B200 box
it is the CUDA path (tests/test_gpu_output_multi.py, bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [(12, 4096, 37, False, False), (17, 0, 64, False, True), (20, (1 << 19) - 512, 16, False, False),
         (10, 6, 3, False, False), (12, 4096, 3, False, False)]  # the last: world 4 > n = 3 (an empty shard)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Restated
    from paper_1111_3297_b200.dist import run_sharded, torch_allreduce_sum
    R = Restated()
    out = []
    for (l, f, n, tm, ovl) in CASES:
        tables = {}

        def sieve_count(p):
            t, c = R.bit_table(p.l, p.f, p.n, test_mode=tm, allow_overlap=ovl)
            tables["t"] = t
            return c

        res = run_sharded(l, f, n, sieve_count, rank, world, torch_allreduce_sum(), test_mode=tm,
                          allow_overlap=ovl)
        gathered = [None] * world
        fg, ng = (res.params.f, res.params.n) if res.params is not None else (f + n, 0)
        dist.all_gather_object(gathered, (fg, ng, tables.get("t", np.zeros(0, np.uint8))))
        out.append((res.total, gathered))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_shards_concatenate_and_counts_sum(world, restated):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, (l, f, n, tm, ovl) in enumerate(CASES):
        full, cfull = restated.bit_table(l, f, n, test_mode=tm, allow_overlap=ovl)
        totals = {results[r][k][0] for r in range(world)}
        assert totals == {cfull}
        parts = [x for x in results[0][k][1] if x[1]]
        assert parts[0][0] == f and sum(x[1] for x in parts) == n
        assert np.array_equal(np.concatenate([x[2] for x in parts]), full)
