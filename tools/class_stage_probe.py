"""Class stage (K2) probe: times k_class_inst / k_class_inst_pf alone at a
BASELINE config (CUDA events around the launch, per-kernel timers) and
writes a digest of every H_k / C_k so that two runs (PHM_CLASS_PF=0 / 1) can
be compared bitwise.

    python tools/class_stage_probe.py [--config c3] [--digest out.npy]
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--shards", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    a = ap.parse_args()
    import torch

    import bench
    import paper_2511_03109_b200 as ph

    c = bench.CONFIGS[a.config]
    ctx = ph.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    pts = bench.make_points(ph, c, 0)
    pm = ph.offline_h2(pts, bench.make_cfg(ph, c, a.rank, a.shards), ctx)
    thetas = bench.theta_vectors(c, 32, 0)
    inst = ph.instantiate(pm, thetas[0])
    ctx.enable_timing(True)
    ctx.reset_timers()
    for s in range(a.steps):
        inst.reinstantiate(thetas[s % 32])
    torch.cuda.synchronize()
    t, cnt = ctx.timer("class_inst")
    ctx.enable_timing(False)
    inst.reinstantiate(thetas[3])
    info = pm.info()
    h = hashlib.sha256()
    ncls = info["n_classes"]
    for k in range(ncls):
        h.update(inst.class_c(k).tobytes())
    print(json.dumps({"config": a.config, "shards": a.shards, "rank": a.rank, "class_inst_ms": t / max(cnt, 1),
                      "launches": cnt, "n_classes": ncls, "pf": os.environ.get("PHM_CLASS_PF", "1"),
                      "c_digest": h.hexdigest()[:16]}), flush=True)


if __name__ == "__main__":
    main()
