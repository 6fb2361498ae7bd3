"""GPU: the library's own sharded step (phm_instantiate_apply_sharded /
phm_apply_sharded), SURVEY.md §8(e).

* NCCL communicator at world size 1 (one GPU): the sharded entry points,
  with their graph capture and the (local) all-reduce, equal the unsharded
  step.
* Two processes sharing the one GPU, each holding its row shard, exchanging
  through a gloo-backed callback communicator: the library runs the split
  forward pass, the x-hat all-reduce, the partial near / far products and the
  y all-reduce; every rank's y equals the unsharded GPU result. (Ranks on one
  GPU never wait on each other's kernels: the callback synchronises and
  exchanges on the host.)"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _case(ph, fmt, sym, rank=0, world=1):
    pts = ph.generate_points(4000, 3, 12)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT, symmetric_near=sym, shard_rank=rank, shard_count=world)
    return pts, (ph.offline_h2 if fmt == "h2" else ph.offline_h)(pts, cfg)


def test_nccl_world1_sharded_step_equals_unsharded(ph):
    import torch

    pts, pm = _case(ph, "h2", True)
    comm = ph.Comm.nccl(pm.ctx, ph.Comm.unique_id(), 0, 1)
    assert comm.info() == {"rank": 0, "world": 1, "nccl": True}
    inst = ph.instantiate(pm, [0.3])
    x = ph.generate_normal(4000, 3)
    X = np.stack([x, ph.generate_normal(4000, 4)], axis=1)
    xd = torch.from_numpy(x).cuda()
    yd = torch.zeros(4000, dtype=torch.float64, device="cuda")
    for th in ([0.11], [0.27], [0.11], [0.44]):  # repeated steps replay the captured graph
        inst.instantiate_apply_sharded_device(comm, th, xd.data_ptr(), yd.data_ptr(), 1)
        pm.ctx.sync()
        ref = ph.instantiate(pm, th)
        assert rel(yd.cpu().numpy(), ref.apply(x)) <= 1e-13
        assert rel(inst.instantiate_apply_sharded(comm, th, X), ref.apply(X)) <= 1e-13
    inst.apply_sharded_device(comm, xd.data_ptr(), yd.data_ptr(), 1)
    pm.ctx.sync()
    assert rel(yd.cpu().numpy(), ph.instantiate(pm, [0.44]).apply(x)) <= 1e-13
    bad = ph.Comm.nccl(pm.ctx, ph.Comm.unique_id(), 0, 1)
    pts2, shard = _case(ph, "h2", True, 0, 2)
    with pytest.raises(ph.LogicError):  # communicator does not match the shard
        ph.instantiate(shard, [0.3]).instantiate_apply_sharded(bad, [0.3], x)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fmt, sym, q):
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_03109_b200 as ph
        from paper_2511_03109_b200.dist import host_allreduce_comm

        torch.cuda.set_device(0)
        pts, full = _case(ph, fmt, sym)
        _, shard = _case(ph, fmt, sym, rank, world)
        comm = host_allreduce_comm()
        x = ph.generate_normal(4000, 5)
        X = np.stack([x, ph.generate_normal(4000, 6), ph.generate_normal(4000, 7), x, x], axis=1)
        inst = ph.instantiate(shard, [0.3])
        errs = []
        for th in ([0.08], [0.3], [0.47]):
            ref = ph.instantiate(full, th)
            errs.append(rel(inst.instantiate_apply_sharded(comm, th, x), ref.apply(x)))
            errs.append(rel(inst.instantiate_apply_sharded(comm, th, X), ref.apply(X)))
        # above 32 RHS a symmetric shard runs the one-sided K9 for its own
        # rows plus Z-only products for partner rows on the other rank
        X40 = np.stack([ph.generate_normal(4000, 10 + j) for j in range(40)], axis=1)
        ref = ph.instantiate(full, [0.47])  # same theta as the last step: apply_sharded below reuses it
        errs.append(rel(inst.instantiate_apply_sharded(comm, [0.47], X40), ref.apply(X40)))
        xd = torch.from_numpy(x).cuda()
        yd = torch.zeros(4000, dtype=torch.float64, device="cuda")
        inst.apply_sharded_device(comm, xd.data_ptr(), yd.data_ptr(), 1)
        shard.ctx.sync()
        errs.append(rel(yd.cpu().numpy(), ph.instantiate(full, [0.47]).apply(x)))
        q.put((rank, max(errs), shard.info()["row_begin"], shard.info()["row_end"]))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e), -1, -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fmt,sym", [("h2", True), ("h2", False), ("h", True)])
def test_two_ranks_on_one_gpu_library_exchange(fmt, sym):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fmt, sym, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for rank, err, b, e in res:
        assert isinstance(err, float), err
        assert err <= 1e-13, (rank, err)
    assert res[0][2] == 0 and res[0][3] == res[1][2] and res[1][3] == 4000
