"""Generates tests/golden/*.npz: small seeded cases of the parametric path
with the reference's outputs (instantiated near blocks D_b, class tensors
H_k / C_k, and y = K(theta) x), so the GPU parity tests can check the CUDA
path against committed vectors with no checker in the loop, and the CPU
tests can detect any drift of the oracle or of the reference build.

Provenance: the REFERENCE ITSELF -- the unmodified proj/src compiled by
oracle/ref_build.sh against oracle/eigen_shim into oracle/_ref/libphmat_ref.so
(pyref). The reference rebuilds tree, blocks, classes, grids and basis from
the points, evaluates every snapshot-mode near tensor with its own
near_oracle (nearfield.cpp:7-48), and runs its own instantiate / apply /
pttk_online / assemble_L_R. The offline TT data both sides share (the TT
cores of the classes and of TT-mode near blocks) is the product's host build
(phm_matrix_build_host), the same code on every machine.

    python tests/golden/make_golden.py      # rewrites the .npz files
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def cases(ph):
    """name -> (points, PHConfig, format, thetas, n_rhs)."""
    return {
        "h2_snapshot_3d_e": (ph.generate_points(1500, 3, 5),
                             ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8,
                                         eta=1.0, near_mode=ph.NearMode.SNAPSHOT, seed=0),
                             ph.Format.H2, [[0.05], [0.173]], 2),
        "h_tt_2d_gauss": (ph.generate_points(1024, 2, 0),
                          ph.PHConfig(spec=ph.KernelSpec(ph.Family.GAUSS, [(0.1, 1.0)]), l_max=2, p_s=6, p_theta=8,
                                      eta=1.0, near_mode=ph.NearMode.TT, seed=0),
                          ph.Format.H, [[0.1], [0.3456]], 1),
        "h2_snapshot_3d_m52_amplitude": (ph.generate_mixture_points(1200, 3, 8, 0.05, 1),
                                         ph.PHConfig(spec=ph.KernelSpec(ph.Family.MATERN52, [(0.05, 0.5), (0.5, 2.0)],
                                                                        amplitude=True),
                                                     l_max=2, p_s=4, p_theta=[8, 6], eta=1.0,
                                                     near_mode=ph.NearMode.SNAPSHOT, seed=0),
                                         ph.Format.H2, [[0.11, 0.7], [0.4, 1.9]], 1),
    }


def sample_ids(count, k):
    return np.unique(np.linspace(0, count - 1, min(k, count)).astype(np.int64))


def generate(ph, pr, name, spec):
    pts, cfg, fmt, thetas, m = spec
    pm = ph.offline_structure(pts, cfg, fmt)
    R = pr.RefMatrix.from_product(pm, pts, near="tt" if cfg.near_mode == ph.NearMode.TT else "snapshot")
    near, far, key = pm.blocks()
    info = pm.info()
    nb = sample_ids(len(near), 8)
    ks = sample_ids(info["n_classes"], 4)
    X = np.stack([ph.generate_normal(pts.shape[0], 7 + j) for j in range(m)], axis=1)
    out = {"points": pts, "x": X, "thetas": np.array(thetas, dtype=np.float64), "near_ids": nb, "class_ids": ks}
    for i, th in enumerate(thetas):
        ri = R.instantiate(th)
        out[f"y{i}"] = ri.apply(X)
        for b in nb:
            out[f"d{i}_{b}"] = ri.near_d(int(b))
        for k in ks:
            out[f"h{i}_{k}"] = R.class_h(int(k), th)
            if fmt == ph.Format.H2:
                out[f"c{i}_{k}"] = R.class_c(int(k), th, info["P"])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    return out


def main():
    import paper_2511_03109_b200 as ph
    from oracle import pyref as pr

    for name, spec in cases(ph).items():
        out = generate(ph, pr, name, spec)
        print(name, sum(v.nbytes for v in out.values()), "bytes")


if __name__ == "__main__":
    main()
