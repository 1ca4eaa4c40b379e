"""The multi-GPU path's host logic on CPU with world_size 2 (gloo).

Each rank takes its share of the index space with me_partition (the same
function the library's comm sweep uses), computes its survivors (here with the
oracle: there is no GPU), exchanges the per-rank stats rows like the NCCL
allgather does, and turns them into global offsets with me_join_counts.  The
concatenation in rank order must equal the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import me_inputs as mi


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, space_name, q):
    import ctypes

    import oracle
    from paper_2411_06465_b200 import _abi
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = mi.config(space_name) if space_name != "rand" else mi.Space(
            models=mi.random_models(3, seed=4, small=True), world=[6, 12], caps_gb=[1, 2], mbs=[1, 2],
            seq=[8, 12], gbs=24, uneven=1)
        total = oracle.space_size(sp)
        L = _abi.lib()
        for (b, e) in ((0, total), (17, total - 5), (3, 3)):
            lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
            _abi.check(L.me_partition(b, e, rank, world, ctypes.byref(lo), ctypes.byref(hi)), "me_partition")
            idx, rows, n, caps = oracle.sweep(sp, lo.value, hi.value) if hi.value > lo.value else (
                np.zeros(0, np.uint64), None, 0, [0] * len(sp.caps_gb))
            stats = torch.tensor([n] + list(caps) + [0] * (8 - len(caps)), dtype=torch.int64)
            gathered = [torch.zeros(9, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(gathered, stats)
            flat = (ctypes.c_uint64 * (9 * world))(*[int(x) for g in gathered for x in g.tolist()])
            off, glob = ctypes.c_uint64(), ctypes.c_uint64()
            capg = (ctypes.c_uint64 * 8)()
            _abi.check(L.me_join_counts(flat, world, 9, len(caps), rank, ctypes.byref(off), ctypes.byref(glob),
                                        capg), "me_join_counts")
            parts = [None] * world
            dist.all_gather_object(parts, (lo.value, hi.value, off.value, idx.tolist()))
            if rank == 0:
                ref_idx, _, ref_n, ref_caps = oracle.sweep(sp, b, e) if e > b else (np.zeros(0), None, 0,
                                                                                    [0] * len(caps))
                cat = [x for p in parts for x in p[3]]
                ok = (cat == [int(x) for x in ref_idx] and glob.value == ref_n
                      and [capg[i] for i in range(len(caps))] == list(ref_caps)
                      and parts[0][0] == b and parts[-1][1] == e
                      and all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))
                      and all(parts[r + 1][2] == parts[r][2] + len(parts[r][3]) for r in range(world - 1)))
                q.put((b, e, ok))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("space_name", ["C1", "rand"])
def test_two_rank_partition_and_join(space_name):
    from paper_2411_06465_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, space_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    results = [q.get(timeout=5) for _ in range(3)]
    assert all(ok for _, _, ok in results), results


def test_bench_units_partition_space():
    import bench
    total = 84_165_588_480
    ranges = [bench.unit_range(total, u) for u in range(bench.UNITS)]
    assert ranges[0][0] == 0 and ranges[-1][1] == total
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(bench.UNITS - 1))


def cyclic_worker(rank, world, port, space_name, chunk, q):
    """bench.py's default N>1 partition: rank r sweeps blocks r, r+N, ... of
    the libme cyclic deal (me_cyclic_block) alone -- here with the oracle --
    and the per-block counts are allgathered (gloo here; libme's
    me_result_join does it with NCCL and a device scan on the GPU)."""
    import oracle
    import paper_2411_06465_b200 as me
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = mi.config(space_name)
        total = oracle.space_size(sp)
        for (b, e) in ((0, total), (5, total - 3)):
            mine, nq = me.cyclic_blocks(b, e, chunk, rank, world)
            idx = [oracle.sweep(sp, cb, ce)[0].tolist() for cb, ce in mine]
            parts = [None] * world
            dist.all_gather_object(parts, (mine, idx))
            if rank == 0:
                ref_idx, _, ref_n, _ = oracle.sweep(sp, b, e)
                calls = [parts[x % world][0][x // world] for x in range(nq)]
                got = [parts[x % world][1][x // world] for x in range(nq)]
                cat = [x for g in got for x in g]
                ok = (cat == [int(x) for x in ref_idx] and len(cat) == ref_n
                      and calls[0][0] == b and calls[-1][1] == e
                      and all(calls[i][1] == calls[i + 1][0] for i in range(nq - 1)))
                q.put((b, e, ok))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunk", [7, 64])
def test_two_rank_cyclic_partition_and_join(chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=cyclic_worker, args=(r, 2, port, "C1", chunk, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    results = [q.get(timeout=5) for _ in range(2)]
    assert all(ok for _, _, ok in results), results


def test_cyclic_blocks_cover_range():
    import paper_2411_06465_b200 as me
    for b, e, chunk, world in ((0, 100, 7, 3), (5, 6, 4, 4), (3, 3, 2, 2), (0, 1 << 36, 1 << 28, 8), (0, 10, 3, 8)):
        per = [me.cyclic_blocks(b, e, chunk, r, world) for r in range(world)]
        nq = per[0][1]
        assert nq == (-(-(e - b) // chunk) if e > b else 0)
        calls = sorted(c for blocks, _ in per for c in blocks)
        assert len(calls) == nq
        for r, (blocks, _) in enumerate(per):
            assert blocks == sorted(blocks)
            assert all((lo - b) // chunk % world == r for lo, _ in blocks)
        if calls:
            assert calls[0][0] == b and calls[-1][1] == e
            assert all(calls[i][1] == calls[i + 1][0] for i in range(len(calls) - 1))
    with pytest.raises(me.MEError):
        me.cyclic_blocks(0, 10, 0, 0, 1)
