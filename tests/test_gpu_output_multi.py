"""GPU tests of the output pipeline, the multi-GPU paths, the asynchronous
run's overflow signal and prime extraction, all through the C ABI.

* streaming (erato_gpu_run_to_sink / write_table / sieve_to_host): the table
  leaves the device as ordered wave slices; FileSink output equals the
  reference file (src/driver.cpp:29-51) up to the full cfg5 table;
* capacity overflows (forced with ERATO_GPU_TEST_CAP_SCALE) are retried
  without a sink ever seeing a byte twice, and a sync = 0 run reports them on
  the device (ERATO_GPU_COUNT_OVERFLOW);
* extract_primes equals the reference PrimeCollectSink element for element
  (src/driver.cpp:53-57, :65-81) on full cfg3 and a cfg5 sub-range;
* multi-GPU: the single-process C-ABI entry (erato_gpu_multi_*, NCCL when
  the devices are distinct) and the one-process-per-shard path (two ranks on
  cuda:0 over gloo, each running the CUDA path on its shard).
"""
import hashlib
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha_file(path):
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        while True:
            b = fh.read(64 << 20)
            if not b:
                break
            h.update(b)
    return h.hexdigest()


# ---------------------------------------------------------------- streaming
@pytest.mark.parametrize("l,f,n", [(22, (1 << 37) - 4096, 300), (12, 4096, 8), (20, 523776, 333),
                                   (17, 0, 64)])
def test_stream_slices_in_order_exactly_once(gpu_ctx, reference, restated, l, f, n):
    import paper_1111_3297_b200 as E
    ovl = f == 0
    p = E.validate_params(l, f, n, allow_overlap=ovl)
    got = np.zeros(p.table_bytes(), np.uint8)
    seen = []

    def on_slice(view, offset):
        seen.append((offset, view.nbytes))
        got[offset:offset + view.nbytes] = view

    st = gpu_ctx.stream(p, on_slice)
    assert seen[0][0] == 0
    for (o0, n0), (o1, _) in zip(seen, seen[1:]):
        assert o1 == o0 + n0  # contiguous, in order, no repeats
    assert seen[-1][0] + seen[-1][1] == p.table_bytes()
    if ovl:
        ref, cnt = restated.bit_table(l, f, n, allow_overlap=True)
    else:
        ref, cnt, _ = reference.run_sieve(l, f, n)
    assert st.prime_count == cnt and np.array_equal(got, ref)


def test_stream_sink_error_aborts(gpu_ctx):
    import paper_1111_3297_b200 as E
    p = E.validate_params(22, (1 << 37) - 4096, 300)
    calls = []

    def bad(view, offset):
        calls.append(offset)
        if len(calls) == 2:
            raise ValueError("disk full")

    with pytest.raises(ValueError):
        gpu_ctx.stream(p, bad)
    assert len(calls) == 2  # nothing delivered after the failing slice
    assert gpu_ctx.count(p).prime_count > 0  # the context stays usable


def test_write_table_cfg5_streams_to_reference_file(gpu_ctx, pins):
    """The full cfg5 table (4 GiB) through the streaming FileSink: never held
    whole in HBM or host memory, byte-identical to the reference file pin."""
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg5"]
    p = E.validate_params(rec["l"], rec["f"], rec["n"])
    with tempfile.TemporaryDirectory() as d:
        path, st = gpu_ctx.write_table(d, p)
        assert os.path.basename(path) == "erato_l22_f137438949376_n8192.bits"
        assert os.path.getsize(path) == rec["bytes"]
        assert st.prime_count == rec["count"]
        assert sha_file(path) == rec["sha256"]
        assert os.listdir(d) == [os.path.basename(path)]  # no temporary left behind


def test_write_table_failure_leaves_no_file(gpu_ctx):
    import paper_1111_3297_b200 as E
    l = 30
    f = (((1 << 64) - 1) >> (l + 1)) - 1
    p = E.validate_params(l, f, 1)  # 2^32 base primes: ALLOC_LIMIT under the default cap
    with tempfile.TemporaryDirectory() as d:
        with pytest.raises(E.Error) as ei:
            gpu_ctx.write_table(d, p)
        assert ei.value.code == E.errc.alloc_limit
        assert os.listdir(d) == []


# ---------------------------------------------------------------- overflow
def _fresh_ctx_with_cap_scale(scale):
    import paper_1111_3297_b200 as E
    os.environ["ERATO_GPU_TEST_CAP_SCALE"] = str(scale)
    try:
        return E.Context(0)
    finally:
        del os.environ["ERATO_GPU_TEST_CAP_SCALE"]


@pytest.mark.parametrize("l,f,n", [(22, (1 << 37) - 4096, 300), (21, (1 << 26) - 2048, 256)])
def test_overflow_retry_streams_each_byte_once(reference, l, f, n):
    import paper_1111_3297_b200 as E
    p = E.validate_params(l, f, n)
    ctx = _fresh_ctx_with_cap_scale(0.25)
    try:
        got = np.zeros(p.table_bytes(), np.uint8)
        seen = []

        def on_slice(view, offset):
            seen.append((offset, view.nbytes))
            got[offset:offset + view.nbytes] = view

        st = ctx.stream(p, on_slice)
    finally:
        ctx.close()
    assert st.retries >= 1
    offs = [o for o, _ in seen]
    assert offs == sorted(set(offs)) and sum(nb for _, nb in seen) == p.table_bytes()
    ref, cnt, _ = reference.run_sieve(l, f, n)
    assert st.prime_count == cnt and np.array_equal(got, ref)


def test_async_run_reports_overflow_on_device():
    """sync = 0 cannot retry; a capacity overflow must not hand back a wrong
    count silently: the caller's device count word reads ERATO_GPU_COUNT_OVERFLOW."""
    import torch
    import paper_1111_3297_b200 as E
    from paper_1111_3297_b200 import _lib
    p = E.validate_params(22, (1 << 37) - 4096, 300)
    ctx = _fresh_ctx_with_cap_scale(0.25)
    try:
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda:0")
        ctx.run_device(p, dev_count=cnt.data_ptr(), sync=False)
        torch.cuda.synchronize()
        assert int(cnt.item()) & ((1 << 64) - 1) == _lib.COUNT_OVERFLOW
        good = ctx.count(p)  # sync = 1 retries to an exact count
        ctx.run_device(p, dev_count=cnt.data_ptr(), sync=False)
        torch.cuda.synchronize()
        assert int(cnt.item()) == good.prime_count
        with pytest.raises(E.Error) as ei:  # invariant checks are read on the host
            _lib.load()
            st = _lib.Stats()
            import ctypes as C
            E.erato._check(_lib.load().erato_gpu_run(ctx.handle, p.l, p.f, p.n, p.flags | E.erato.CHECK_INVARIANTS,
                                                     None, C.c_void_p(cnt.data_ptr()), None, 0, C.byref(st)))
        assert ei.value.code == E.errc.invalid_argument
    finally:
        ctx.close()


# ---------------------------------------------------------------- extract_primes
def test_extract_primes_cfg3_equals_reference_collect_sink(gpu_ctx, reference, pins):
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg3"]
    p = E.validate_params(rec["l"], rec["f"], rec["n"])
    got = gpu_ctx.extract_primes(p)
    assert len(got) == rec["count"] == 77_449_842
    ref = reference.extract_primes(rec["l"], rec["f"], rec["n"])
    assert np.array_equal(got, ref)


def test_extract_primes_cfg5_subrange_equals_reference(gpu_ctx, reference, pins):
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg5"]
    l, f, n = rec["l"], rec["f"] + 1000, 24
    got = gpu_ctx.extract_primes(E.validate_params(l, f, n))
    ref = reference.extract_primes(l, f, n)
    assert len(got) == len(ref) > 0 and np.array_equal(got, ref)


def test_extract_primes_single_pass_cache(gpu_ctx):
    import paper_1111_3297_b200 as E
    p = E.validate_params(20, 523776, 64)
    a = gpu_ctx.extract_primes(p)  # count, then copy (one sieve)
    b = gpu_ctx.extract_primes(p, cap=len(a))
    assert np.array_equal(a, b)
    c = gpu_ctx.extract_primes(E.validate_params(20, 523776 + 64, 64))
    assert c[0] > a[-1]


# ---------------------------------------------------------------- multi-GPU, one process
def test_multi_c_abi_single_device_nccl(pins):
    """One shard, NCCL communicator over one device: the all-reduce path runs."""
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg3"]
    m = E.MultiGPU([0])
    try:
        assert m.uses_nccl
        st = m.count(E.validate_params(rec["l"], rec["f"], rec["n"]))
        assert st.prime_count == rec["count"]
    finally:
        m.close()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_c_abi_shards_on_one_device(pins, world):
    """The shard threads (test topology: every shard on cuda:0, counts summed
    on the host) reproduce the cfg3 count and, writing concurrently into one
    file, the cfg3 table."""
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg3"]
    p = E.validate_params(rec["l"], rec["f"], rec["n"])
    m = E.MultiGPU([0] * world)
    try:
        assert not m.uses_nccl
        assert m.count(p).prime_count == rec["count"]
        with tempfile.TemporaryDirectory() as d:
            path, st = m.write_table(d, p)
            assert st.prime_count == rec["count"]
            assert sha_file(path) == rec["sha256"]
    finally:
        m.close()


def test_multi_c_abi_more_shards_than_segments(reference):
    import paper_1111_3297_b200 as E
    m = E.MultiGPU([0, 0, 0, 0])
    try:
        st = m.count(E.validate_params(12, 4096, 3))
    finally:
        m.close()
    assert st.prime_count == reference.run_sieve(12, 4096, 3, table=False)[1]


def test_multi_c_abi_cfg5_count(pins):
    import paper_1111_3297_b200 as E
    rec = pins["configs"]["cfg5"]
    m = E.MultiGPU([0, 0])
    try:
        assert m.count(E.validate_params(rec["l"], rec["f"], rec["n"])).prime_count == rec["count"]
    finally:
        m.close()


# ---------------------------------------------------------------- one process per shard
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


WORKER = r'''
import os, sys, json
sys.path.insert(0, os.environ["ROOT"])
import torch.distributed as dist
import paper_1111_3297_b200 as E
from paper_1111_3297_b200.dist import gpu_count, run_sharded, shard_params, torch_allreduce_sum
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
ctx = E.Context(0)
out = {}
for name, (l, f, n) in json.loads(os.environ["CASES"]).items():
    res = run_sharded(l, f, n, gpu_count(ctx), rank, world, torch_allreduce_sum())
    out[name] = res.total
    p = E.validate_params(l, f, n)
    sp = shard_params(l, f, n, rank, world)
    if name == "cfg3":  # every rank streams its shard into the one file
        ctx.write_table(os.environ["OUTDIR"], p, sp.f, sp.n)
    dist.barrier()
if rank == 0:
    print("RESULT " + json.dumps(out), flush=True)
ctx.close()
dist.destroy_process_group()
'''


def test_two_ranks_on_cuda0_over_gloo(pins):
    """The bench/torchrun decomposition on hardware: 2 processes, each running
    the CUDA path on its contiguous shard, one all-reduce of the counts; the
    shards' pwrite()s into one file give the cfg3 table."""
    import json
    rec3, rec5 = pins["configs"]["cfg3"], pins["configs"]["cfg5"]
    cases = {"cfg3": [rec3["l"], rec3["f"], rec3["n"]], "cfg5": [rec5["l"], rec5["f"], rec5["n"]]}
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        procs = []
        for r in range(2):
            env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                       ROOT=ROOT, CASES=json.dumps(cases), OUTDIR=d)
            procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, stdout=subprocess.PIPE,
                                          stderr=subprocess.STDOUT, text=True))
        outs = [pr.communicate(timeout=600)[0] for pr in procs]
        assert all(pr.returncode == 0 for pr in procs), outs
        line = [x for x in outs[0].splitlines() if x.startswith("RESULT ")][0]
        res = json.loads(line[7:])
        assert res["cfg3"] == rec3["count"] and res["cfg5"] == rec5["count"]
        path = os.path.join(d, f"erato_l{rec3['l']}_f{rec3['f']}_n{rec3['n']}.bits")
        assert sha_file(path) == rec3["sha256"]
