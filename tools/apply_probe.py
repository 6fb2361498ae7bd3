"""Times (and, under ncu, exposes) the standalone H^2 MVM of BASELINE config 3
(`phm_apply_device`, one vector or --rhs m) on one GPU: CUDA events over
--steps applies after warm-up, per-kernel event times in a second pass.

    python tools/apply_probe.py [--config c3] [--rhs 1] [--steps 20]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rhs", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--save", default=None, help="np.save y (tree of the last apply) here")
    ap.add_argument("--pre-steps", type=int, default=0,
                    help="run this many fused instantiate+apply steps (and reinstantiates) first, as bench.py does")
    ap.add_argument("--pre-fused", type=int, default=None, help="fused steps first (default: --pre-steps)")
    ap.add_argument("--pre-inst", type=int, default=None, help="reinstantiates first (default: --pre-steps)")
    ap.add_argument("--idle", type=float, default=0.0, help="seconds of idle GPU between the pre-steps and the timing")
    a = ap.parse_args()
    import torch

    import bench
    import paper_2511_03109_b200 as ph

    c = bench.CONFIGS[a.config]
    m = a.rhs
    ctx = ph.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    pts = bench.make_points(ph, c, 0)
    pm = ph.offline_h2(pts, bench.make_cfg(ph, c), ctx)
    inst = ph.instantiate(pm, bench.theta_vectors(c, 1, 0)[0])
    x = torch.from_numpy(np.stack([ph.generate_normal(c["n"], 1 + j) for j in range(m)])).cuda()
    y = torch.empty_like(x)
    thetas = bench.theta_vectors(c, 32, 0)
    for s in range(a.pre_steps if a.pre_fused is None else a.pre_fused):
        inst.instantiate_apply_device(thetas[s % 32], x.data_ptr(), y.data_ptr(), m)
    for s in range(a.pre_steps if a.pre_inst is None else a.pre_inst):
        inst.reinstantiate(thetas[s % 32])
    torch.cuda.synchronize()
    if a.idle > 0:
        import time
        time.sleep(a.idle)
    for _ in range(5):
        inst.apply_device(x.data_ptr(), y.data_ptr(), m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.steps):
        inst.apply_device(x.data_ptr(), y.data_ptr(), m)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    ctx.enable_timing(True)
    ctx.reset_timers()
    for _ in range(a.steps):
        inst.apply_device(x.data_ptr(), y.data_ptr(), m)
    torch.cuda.synchronize()
    kern = {}
    for name in ("near_mvm", "near_gather", "near_mrhs", "coupling", "coupling_reduce", "leaf_fwd", "up", "down",
                 "leaf_bwd", "gather", "scatter", "zero"):
        t, cnt = ctx.timer(name)
        if cnt:
            kern[name] = round(t / a.steps, 4)
    if a.save:
        np.save(a.save, y.cpu().numpy())
    info = pm.info()
    print(json.dumps({"config": a.config, "rhs": m, "pre_fused": a.pre_steps if a.pre_fused is None else a.pre_fused,
                      "pre_inst": a.pre_steps if a.pre_inst is None else a.pre_inst, "idle_s": a.idle, "apply_ms": ms, "near_stored": info["near_stored"],
                      "kernels_ms_per_apply": kern}))


if __name__ == "__main__":
    main()
