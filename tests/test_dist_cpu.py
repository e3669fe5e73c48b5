"""Host-side plumbing of the multi-GPU path on CPU (gloo, world size 2):
shard layout and the NCCL unique-id exchange that bench.py / users run before
bl_load_design (BASELINE north star: column-sharded features over NCCL)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1701_05936_b200 import bl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        j0, j1 = bl.shard_range(p, world, rank, block=1000)
        d = bl.make_dist(rank, world, (j0, j1), p)
        import ctypes
        uid = ctypes.string_at(d.nccl_unique_id, 128)
        got = [None] * world
        dist.all_gather_object(got, (rank, j0, j1, uid, d.col_offset, d.p_global, d.backend))
        q.put(got if rank == 0 else None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [100_000, 1_339_511])
def test_shards_and_id_exchange_world2(p):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = None
    for _ in range(world):
        v = q.get(timeout=120)
        got = got or v
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    got = sorted(got)
    assert got[0][1] == 0 and got[-1][2] == p                      # shards cover [0, p)
    assert all(got[r][2] == got[r + 1][1] for r in range(world - 1))   # contiguous, rank order
    assert all(g[1] % 1000 == 0 for g in got)                         # whole 1000-column blocks
    assert got[0][3] == got[1][3] and len(got[0][3]) == 128           # one NCCL id for the job
    assert all(g[4] == g[1] and g[5] == p and g[6] == 0 for g in got)


def test_shard_range_small():
    for p in (1, 7, 64, 1001):
        for world in (1, 2, 3, 8):
            rs = [bl.shard_range(p, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == p
            assert all(rs[r][1] == rs[r + 1][0] for r in range(world - 1))


def _coll_worker(rank, world, port, q):
    """Drive the host-collective adapters of bl.host_coll_dist (bl_dist.backend = 2) exactly as
    libbl calls them (C function pointers, host buffers), over gloo between processes."""
    import ctypes
    import numpy as np
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def allgather(send):
            t = torch.tensor(np.frombuffer(send, dtype=np.uint8).copy())
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return b"".join(o.numpy().tobytes() for o in out)

        def bcast(buf, root):
            t = torch.tensor(np.frombuffer(bytes(buf), dtype=np.uint8).copy())
            dist.broadcast(t, src=root)
            buf[:] = t.numpy().tobytes()

        def allreduce_sum(v):
            dist.all_reduce(torch.from_numpy(v))

        d = bl.host_coll_dist(rank, world, (rank * 10, rank * 10 + 10), 10 * world, allgather, bcast, allreduce_sum)
        hc = d.host_coll.contents
        assert d.backend == 2 and d.p_global == 10 * world
        send = (ctypes.c_int32 * 3)(rank, 100 + rank, -rank)
        recv = (ctypes.c_int32 * (3 * world))()
        rc1 = hc.allgather(None, ctypes.cast(send, ctypes.c_void_p), ctypes.cast(recv, ctypes.c_void_p), 12)
        buf = (ctypes.c_double * 4)(*([rank + 0.5] * 4))
        rc2 = hc.bcast(None, ctypes.cast(buf, ctypes.c_void_p), 32, 1)
        acc = (ctypes.c_double * 3)(1.0, rank, 2.0 * rank)
        rc3 = hc.allreduce_sum_f64(None, ctypes.cast(acc, ctypes.c_void_p), 3)
        q.put((rank, (rc1, rc2, rc3), list(recv), list(buf), list(acc)))
    finally:
        dist.destroy_process_group()


def test_host_collective_adapters_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coll_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, rcs, recv, buf, acc in got:
        assert rcs == (0, 0, 0)
        assert recv == [0, 100, 0, 1, 101, -1]               # rank order
        assert buf == [1.5] * 4                              # root 1's payload
        assert acc == [2.0, 1.0, 2.0]                        # sums over the ranks
