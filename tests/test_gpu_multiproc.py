"""Sharded fits across PROCESSES (the workers are processes
sharing one X).  Each rank is its own process with its own CUDA context; the library's
collectives go through caller-supplied host collectives (bl_dist.backend = 2) implemented
with torch.distributed over gloo -- marshalling only.  Both ranks share the one GPU of this
box; the collectives are host-side, so no kernel of one rank waits on a kernel of the
other.  The column-sharded path, lockstep CV included, must be bitwise the single-GPU path."""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

bl = pytest.importorskip("paper_1701_05936_b200.bl")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _instance(dtype):
    kind = "geno" if dtype == np.int8 else "corr"
    return synth.random_instance(140, 900, dtype=dtype, seed=71, kind=kind, n_true=10, const_cols=2)


def _gloo_colls(world):
    import torch
    import torch.distributed as dist

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
        t = torch.from_numpy(v)
        dist.all_reduce(t)

    return allgather, bcast, allreduce_sum


def _worker(rank, world, port, dtype_name, lams, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        inst = _instance(np.dtype(dtype_name).type)
        j0, j1 = bl.shard_range(inst.p, world, rank)
        ag, bc, ar = _gloo_colls(world)
        dd = bl.host_coll_dist(rank, world, (j0, j1), inst.p, ag, bc, ar)
        d = bl.Design(np.ascontiguousarray(inst.host_X()[j0:j1]), inst.n, dist=dd)
        lm = d.lambda_max(inst.y, 0.5)
        p = d.fit_path(inst.y, lams, alpha=0.5, tol=1e-9)
        c = d.cv(inst.y, lams, K=4, alpha=0.5, tol=1e-9, seed=9)
        q.put((rank, lm, p.col_ptr, p.feat, p.beta_std, p.kkt_rounds, c.cve, c.cvse, c.full.beta_std, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, None, None, None, None, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype", [np.float32, np.int8])
def test_sharded_fit_across_processes_is_bitwise_single_gpu(dtype):
    import torch.multiprocessing as mp
    inst = _instance(dtype)
    d1 = bl.Design(inst.host_X(), inst.n)
    lm = d1.lambda_max(inst.y, 0.5)
    lams = synth.lambda_grid(lm, 25, 0.1)
    ref = d1.fit_path(inst.y, lams, alpha=0.5, tol=1e-9)
    rcv = d1.cv(inst.y, lams, K=4, alpha=0.5, tol=1e-9, seed=9)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, np.dtype(dtype).name, lams, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for rank, glm, col_ptr, feat, beta, kkt, cve, cvse, cvb, err in got:
        assert err is None, (rank, err)
        assert glm == lm
        assert np.array_equal(col_ptr, ref.col_ptr) and np.array_equal(feat, ref.feat)
        assert np.array_equal(beta, ref.beta_std) and np.array_equal(kkt, ref.kkt_rounds)
        assert np.array_equal(cve, rcv.cve) and np.array_equal(cvse, rcv.cvse)
        assert np.array_equal(cvb, rcv.full.beta_std)
