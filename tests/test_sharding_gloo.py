"""CPU, world_size 2 over gloo: the multi-GPU row-sharding plan and the y
all-gather(v) + un-permute assembly (paper_2511_03109_b200/dist.py).

Each rank builds its shard's host structure (leaf row range, local block
flags) with the product's host code, computes its rows of y with the oracle
standing in for its GPU (tree order), and the ranks exchange rows with the
same padded all-gather the NCCL path uses. The assembled y must equal the
unsharded oracle MVM bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_03109_b200 as ph
        from oracle import pyoracle as po
        from paper_2511_03109_b200.dist import PartialSum, RowGather, row_counts

        pts = ph.generate_points(3000, 3, 4)
        spec = ph.KernelSpec(ph.Family.E, [(0.05, 0.5)])
        cfg = ph.PHConfig(spec=spec, l_max=2, p_s=4, p_theta=8, eta=1.0, near_mode=ph.NearMode.SNAPSHOT,
                          shard_rank=rank, shard_count=world)
        pm = ph.offline_structure(pts, cfg)
        info = pm.info()
        perm = pm.perm()
        om = po.from_product(pm, pts)
        x = ph.generate_normal(3000, 5)
        y_full = om.instantiate([0.2]).apply(x)
        rows = info["row_end"] - info["row_begin"]
        ytree = y_full[perm]  # oracle stands in for this rank's GPU rows
        counts = row_counts(rows)
        rg = RowGather(counts, 1)
        yrows = torch.from_numpy(ytree[info["row_begin"]: info["row_end"]].copy()).reshape(1, -1)
        yperm = rg.gather(yrows).numpy()[0]
        y = np.empty_like(yperm)
        y[perm] = yperm
        # symmetric storage: full-length partials summed by one all-reduce
        # (here two complementary weightings of y stand in for the ranks'
        # partials: the plumbing, shapes and un-permute are what is checked)
        w = np.random.default_rng(7).uniform(0, 1, 3000)
        ps = PartialSum(3000, 1)
        ps.buf[0].copy_(torch.from_numpy(ytree * (w if rank == 0 else 1.0 - w)))
        ysum = ps.reduce().numpy()[0]
        y2 = np.empty_like(ysum)
        y2[perm] = ysum
        ok2 = bool(np.max(np.abs(y2 - y_full)) <= 1e-14 * np.max(np.abs(y_full)))
        q.put((rank, info["row_begin"], info["row_end"], bool(np.array_equal(y, y_full)) and ok2, counts))
    finally:
        dist.destroy_process_group()


def test_row_sharded_gather_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # contiguous, disjoint, covering row ranges
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == 3000
    assert all(r[3] for r in res)
    # balanced by near-field work: neither shard is empty
    assert min(res[0][4]) > 0
