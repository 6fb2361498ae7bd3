"""Small workload touching every online kernel, run against the build with
device-side invariant checks (tools/check_build.sh; compute-sanitizer is not
available on this pool). Checks results against the oracle so a silent
corruption also fails."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def main():
    import paper_2511_03109_b200 as ph
    from oracle import pyoracle as po

    worst = 0.0
    # H^2, snapshot, symmetric: fused pass, TMA GEMV, K9 two-sided / one-sided,
    # coupling DMMA, basis passes, theta batch
    pts = ph.generate_points(1500, 3, 1)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_h2(pts, cfg)
    om = po.from_product(pm, pts)
    inst = ph.instantiate(pm, [0.2])
    x = ph.generate_normal(1500, 2)
    X = np.stack([ph.generate_normal(1500, s) for s in range(5)], axis=1)
    worst = max(worst, rel(inst.apply(x), om.instantiate([0.2]).apply(x)))
    worst = max(worst, rel(inst.instantiate_apply([0.3], x), om.instantiate([0.3]).apply(x)))
    worst = max(worst, rel(inst.apply(X), om.instantiate([0.3]).apply(X)))
    X40 = np.random.default_rng(0).standard_normal((1500, 40))
    worst = max(worst, rel(inst.apply(X40), om.instantiate([0.3]).apply(X40)))
    b = ph.instantiate_batch(pm, [[0.1], [0.4]])
    worst = max(worst, rel(b[1].apply(x), om.instantiate([0.4]).apply(x)))
    # TT near mode, H form
    cfg2 = ph.PHConfig(spec=ph.KernelSpec(ph.Family.SE, [(0.25, 1.0)]), l_max=2, p_s=4, p_theta=6, eps=1e-4,
                       near_mode=ph.NearMode.TT)
    pts2 = ph.generate_points(600, 2, 4)
    pm2 = ph.offline_h(pts2, cfg2)
    om2 = po.from_product(pm2, pts2)
    x2 = ph.generate_normal(600, 3)
    worst = max(worst, rel(ph.instantiate(pm2, [0.5]).apply(x2), om2.instantiate([0.5]).apply(x2)))
    print(f"sanitize workload ok: worst rel err {worst:.3e}")
    if not worst <= 1e-11:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
