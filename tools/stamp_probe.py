"""Schedule probe for the fused C3 step: runs instantiate_apply_device a few
times with PHM_STAMPS=1 (device-clock stamps at fixed points, printed to
stderr by the library). Stamps: 0 step start (main), 1 side start, 2 class
stage done, 3 near pass start, 4 near pass end, 5 coupling start, 6 coupling
end, 7 side chain end, 8 step end; microseconds after stamp 0.

    PHM_STAMPS=1 python tools/stamp_probe.py [--config c3] [--steps 6]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--shards", type=int, default=0, help="time row shard --rank of N through the sharded step")
    ap.add_argument("--rank", type=int, default=0)
    a = ap.parse_args()
    import torch

    import bench
    import paper_2511_03109_b200 as ph

    c = bench.CONFIGS[a.config]
    pts = bench.make_points(ph, c, 0)
    thetas = bench.theta_vectors(c, 32, 0)
    x = torch.from_numpy(ph.generate_normal(c["n"], 1)).cuda()
    y = torch.empty_like(x)
    ctx = ph.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    if a.shards:
        pm = ph.offline_h2(pts, bench.make_cfg(ph, c, a.rank, a.shards), ctx)
        comm = ph.Comm.probe(a.rank, a.shards)
    else:
        pm = ph.offline_h2(pts, bench.make_cfg(ph, c), ctx)
    inst = ph.instantiate(pm, thetas[0])
    for s in range(a.steps):
        print("step", s, file=sys.stderr, flush=True)
        if a.shards:
            inst.instantiate_apply_sharded_device(comm, thetas[s % 32], x.data_ptr(), y.data_ptr(), 1)
        else:
            inst.instantiate_apply_device(thetas[s % 32], x.data_ptr(), y.data_ptr(), 1)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
