"""Per-rank cost of the row-sharded step (C3, or C4 with --config c4), measured on ONE GPU: builds shard
r of N (the rank's own near pairs, far blocks, the classes they use, its
share of the forward pass) and times the library's sharded step
(phm_instantiate_apply_sharded) with a probe communicator whose two
all-reduces are no-ops, as CUDA graphs, with CUDA events. Predicts the N-GPU
step (max over ranks + the x-hat and y all-reduces); not a multi-GPU
measurement.

    python tools/shard_probe.py --n-shards 2 4 8 --ranks 0 -1
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-shards", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--ranks", type=int, nargs="+", default=[0, -1])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rhs", type=int, default=0)
    ap.add_argument("--legacy", action="store_true",
                    help="time the round-1 partial step (replicated forward pass and class stage) instead")
    a = ap.parse_args()
    import torch

    import bench
    import paper_2511_03109_b200 as ph

    c = bench.CONFIGS[a.config]
    m = a.rhs or c.get("rhs", 1)
    pts = bench.make_points(ph, c, 0)
    thetas = bench.theta_vectors(c, 32, 0)
    x = torch.from_numpy(np.stack([ph.generate_normal(c["n"], 1 + j) for j in range(m)])).cuda()
    part = torch.zeros((m, c["n"]), dtype=torch.float64, device="cuda")
    ctx = ph.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    for N in a.n_shards:
        for r in a.ranks:
            rank = r % N
            import time
            t0 = time.time()
            pm = ph.offline_h2(pts, bench.make_cfg(ph, c, rank, N), ctx)
            build_s = time.time() - t0
            info = pm.info()
            inst = ph.instantiate(pm, thetas[0])
            comm = ph.Comm.probe(rank, N)

            def step(s):
                if a.legacy:
                    inst.instantiate_apply_partial_device(thetas[s % 32], x.data_ptr(), part.data_ptr(), m)
                else:
                    inst.instantiate_apply_sharded_device(comm, thetas[s % 32], x.data_ptr(), part.data_ptr(), m)

            for s in range(3):
                step(s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for s in range(a.steps):
                step(s)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            # per-kernel split (separate loop: timers add events)
            ctx.enable_timing(True)
            ctx.reset_timers()
            for s in range(a.steps):
                step(s)
            torch.cuda.synchronize()
            kern = {}
            for name in ("near_inst_mvm", "near_inst", "near_mrhs", "class_inst", "near_w", "near_gather", "coupling",
                         "coupling_reduce", "leaf_fwd", "up", "down", "leaf_bwd", "gather"):
                t, cnt = ctx.timer(name)
                if cnt:
                    kern[name] = round(t / a.steps, 4)
            ctx.enable_timing(False)
            print(json.dumps({"config": a.config, "rhs": m, "shards": N, "rank": rank, "ms_per_step": ms,
                              "path": "legacy partial" if a.legacy else "library sharded (probe comm)",
                              "rows": info["row_end"] - info["row_begin"], "near_stored": info["near_stored"],
                              "device_bytes": info["device_bytes"], "build_s": build_s,
                              "kernels_ms_per_step": kern}), flush=True)
            del inst, pm
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
