"""GPU parity against the COMPILED REFERENCE (oracle/_ref/libphmat_ref.so: the
unmodified proj/src built against oracle/eigen_shim), at every BASELINE
config's own size that fits one GPU.

The reference rebuilds tree / blocks / classes / grids / basis from the same
points, evaluates every snapshot-mode near tensor itself (near_oracle,
nearfield.cpp:7-48) and runs its own instantiate / apply / pttk_online /
assemble_L_R / coupling_apply / nearfield_online. It is handed only the
offline coupling TT cores (the data both sides share).

Tolerances are the north_star's (fp64): D_b, H_k, C_k within 1e-12 relative
Frobenius; y within 1e-11 relative 2-norm.

* C1 (BASELINE configs[0]) at full size: n = 4096, 2D, param-H, Gaussian,
  all 16 evenly spaced l; every D_b, every far H_b, S_b/T_b, and y.
* C2 (configs[1]) at full size: n = 65,536, 2D, H^2, Matern-3/2, p_s = 8,
  p_theta = 10; 3 harness theta draws; every D_b, H_k and C_k, and y.
* C3 (configs[2], the headline) at full size: n = 2^18; 2,000 sampled D_b,
  every H_k, 300 sampled C_k, and y (plain apply and the fused step) on
  probe rows, composed by the reference from the blocks that reach them.
* C4 form (configs[3]) at the largest n one GPU holds with the config's
  leaf size: n = 2^17 mixture, leaf 32, Matern-5/2 x sigma^2 on 8 x 6,
  64 RHS: sampled D_b / C_k and probe rows of 4 RHS columns.
"""
import os
import sys

import numpy as np
import pytest

from helpers import node_rows

pytestmark = pytest.mark.gpu

TOL_BLOCK = 1e-12
TOL_Y = 1e-11
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = os.cpu_count() or 1


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _bench():
    sys.path.insert(0, ROOT)
    import bench

    return bench


def _sizes(pm):
    return pm.nodes()[0][:, 3]


def _first_far_of_class(pm):
    _, _, key = pm.blocks()
    first = np.full(pm.info()["n_classes"], -1, dtype=np.int64)
    for i in range(len(key) - 1, -1, -1):
        first[key[i]] = i
    return first


def _check_blocks(ph, pm, inst, R, theta, near_ids, class_ids, ri=None, log=None):
    sizes = _sizes(pm)
    near, _, _ = pm.blocks()
    first = _first_far_of_class(pm)
    wd = 0.0
    for b in near_ids:
        s, t = near[b]
        g = inst.near_d(int(b), (int(sizes[s]), int(sizes[t])))
        r = ri.near_d(int(b)) if ri is not None else R.near_online(int(b), theta)
        wd = max(wd, rel(g, r))
    assert wd <= TOL_BLOCK, f"D_b rel err {wd:.3e}"
    info = pm.info()
    wh = wc = 0.0
    for k in class_ids:
        wh = max(wh, rel(inst.far_h(int(first[k])), R.class_h(int(k), theta)))
        if pm.format == ph.Format.H2:
            wc = max(wc, rel(inst.class_c(int(k)), R.class_c(int(k), theta, info["P"])))
    assert wh <= TOL_BLOCK, f"H_k rel err {wh:.3e}"
    assert wc <= TOL_BLOCK, f"C_k rel err {wc:.3e}"
    if log:
        log("D_b", wd)
        log("H_k", wh)
        if pm.format == ph.Format.H2:
            log("C_k", wc)
    return wd, wh, wc


def test_c1_full_size_vs_reference(ph, pr, parity_log):
    log = lambda k, v: parity_log("c1_full_size", k, v)  # noqa: E731
    b = _bench()
    c = b.CONFIGS["c1"]
    pts = b.make_points(ph, c, 0)
    assert np.array_equal(pts, pr.generate_points(c["n"], c["d"], 0))
    pm = ph.offline_h(pts, b.make_cfg(ph, c))
    R = pr.RefMatrix.from_product(pm, pts, near="snapshot", threads=THREADS)
    near, far, key = pm.blocks()
    # S_b, T_b: the reference's own pttk_offline (rows in the reference's
    # ascending index order)
    rows = node_rows(pm)
    for i in range(len(far)):
        S, T = pm.far_st(i)
        Sr, Tr = R.far_st(i)
        S, T = S[np.argsort(rows(far[i, 0]))], T[np.argsort(rows(far[i, 1]))]
        assert rel(S, Sr) <= TOL_BLOCK and rel(T, Tr) <= TOL_BLOCK
        log("S_b_T_b", max(rel(S, Sr), rel(T, Tr)))
    x = ph.generate_normal(c["n"], 1)
    for j in range(16):
        theta = [0.1 + 0.9 * j / 15]
        inst, ri = ph.instantiate(pm, theta), R.instantiate(theta)
        _check_blocks(ph, pm, inst, R, theta, range(len(near)), range(pm.info()["n_classes"]), ri=ri, log=log)
        wf = max(rel(inst.far_h(i), ri.far_h(i)) for i in range(len(far)))
        assert wf <= TOL_BLOCK
        log("far_h", wf)
        y = ri.apply(x)
        e1, e2 = rel(inst.apply(x), y), rel(inst.instantiate_apply(theta, x), y)
        assert e1 <= TOL_Y and e2 <= TOL_Y
        log("y_apply", e1)
        log("y_fused", e2)


def test_c2_full_size_vs_reference(ph, pr, parity_log):
    log = lambda k, v: parity_log("c2_full_size", k, v)  # noqa: E731
    b = _bench()
    c = b.CONFIGS["c2"]
    pts = b.make_points(ph, c, 0)
    pm = ph.offline_h2(pts, b.make_cfg(ph, c))
    R = pr.RefMatrix.from_product(pm, pts, near="snapshot", threads=THREADS)
    near, _, _ = pm.blocks()
    x = ph.generate_normal(c["n"], 1)
    for theta in b.theta_vectors(c, 3, 0):
        theta = list(theta)
        inst, ri = ph.instantiate(pm, theta), R.instantiate(theta)
        _check_blocks(ph, pm, inst, R, theta, range(len(near)), range(pm.info()["n_classes"]), ri=ri, log=log)
        y = ri.apply(x)
        e1, e2 = rel(inst.apply(x), y), rel(inst.instantiate_apply(theta, x), y)
        assert e1 <= TOL_Y and e2 <= TOL_Y
        log("y_apply", e1)
        log("y_fused", e2)


@pytest.fixture(scope="module")
def c3(ph, pr):
    b = _bench()
    c = b.CONFIGS["c3"]
    pts = b.make_points(ph, c, 0)
    pm = ph.offline_h2(pts, b.make_cfg(ph, c))
    R = pr.RefMatrix.from_product(pm, pts, near="none", finalize=False)
    return pm, R, c, pts


def test_c3_full_size_blocks_vs_reference(ph, c3, parity_log):
    log = lambda k, v: parity_log("c3_full_size_sampled", k, v)  # noqa: E731
    pm, R, c, pts = c3
    b = _bench()
    info = pm.info()
    rng = np.random.default_rng(3)
    near_ids = np.sort(rng.choice(info["n_near"], 2000, replace=False))
    cls = np.sort(rng.choice(info["n_classes"], 300, replace=False))
    for theta in b.theta_vectors(c, 2, 0):
        theta = list(theta)
        inst = ph.instantiate(pm, theta)
        _check_blocks(ph, pm, inst, R, theta, near_ids, cls, log=log)
        # every class's H_k
        first = _first_far_of_class(pm)
        wh = max(rel(inst.far_h(int(first[k])), R.class_h(k, theta)) for k in range(info["n_classes"]))
        assert wh <= TOL_BLOCK


def test_c3_full_size_y_rows_vs_reference(ph, c3, parity_log):
    log = lambda k, v: parity_log("c3_full_size_sampled", k, v)  # noqa: E731
    pm, R, c, pts = c3
    b = _bench()
    x = ph.generate_normal(c["n"], 1)
    rows = np.sort(np.random.default_rng(5).choice(c["n"], 48, replace=False))
    inst = ph.instantiate(pm, [0.3])
    for theta in b.theta_vectors(c, 2, 1):
        theta = list(theta)
        yr = R.apply_rows(theta, x, rows, threads=THREADS)
        inst.reinstantiate(theta)
        e1, e2 = rel(inst.apply(x)[rows], yr), rel(inst.instantiate_apply(theta, x)[rows], yr)
        assert e1 <= TOL_Y and e2 <= TOL_Y
        log("y_rows_apply", e1)
        log("y_rows_fused", e2)


def test_c4_form_largest_single_gpu_vs_reference(ph, pr, parity_log):
    log = lambda k, v: parity_log("c4_form_n2^17_64rhs", k, v)  # noqa: E731
    """BASELINE configs[3] form with its leaf size (32) at n = 2^17 (l_max 4):
    mixture of 16 Gaussians, Matern-5/2 x sigma^2 on an 8 x 6 grid, 64 RHS
    through the block (DMMA) path. 1.26e9 near entries, 45 GB on device."""
    b = _bench()
    c = dict(b.CONFIGS["c4"], n=1 << 17, l_max=4)
    pts = b.make_points(ph, c, 0)
    pm = ph.offline_h2(pts, b.make_cfg(ph, c))
    R = pr.RefMatrix.from_product(pm, pts, near="none", finalize=False)
    info = pm.info()
    rng = np.random.default_rng(8)
    near_ids = np.sort(rng.choice(info["n_near"], 150, replace=False))
    cls = np.sort(rng.choice(info["n_classes"], 200, replace=False))
    X = np.stack([ph.generate_normal(c["n"], 100 + j) for j in range(64)], axis=1)
    rows = np.sort(rng.choice(c["n"], 6, replace=False))
    for theta in ([0.083, 1.37], [0.41, 0.62]):
        inst = ph.instantiate(pm, theta)
        _check_blocks(ph, pm, inst, R, theta, near_ids, cls, log=log)
        Y = inst.apply(X)
        Yf = inst.instantiate_apply(theta, X)
        cols = [0, 21, 42, 63]
        yr = R.apply_rows(theta, X[:, cols], rows, threads=THREADS)
        for q, j in enumerate(cols):
            e1, e2 = rel(Y[rows, j], yr[:, q]), rel(Yf[rows, j], yr[:, q])
            assert e1 <= TOL_Y and e2 <= TOL_Y
            log("Y_rows_apply", e1)
            log("Y_rows_fused", e2)


@pytest.mark.parametrize("h2,near_tt,family", [(True, True, "se"), (False, True, "se"), (True, False, "e"),
                                               (False, False, "mc")])
def test_reference_artifact_on_gpu(ph, pr, tmp_path, parity_log, h2, near_tt, family):
    """The drop-in path `phmat build --artifact` -> GPU instantiate
    (tools/phmat.cpp:155-204): the reference builds and saves its own
    parametric matrix (its TT-cross; TT or Direct near mode), the product
    loads the file onto the GPU (phm_matrix_load), and instantiate + apply
    there equal the reference's instantiate + apply of the same file."""
    log = lambda k, v: parity_log(f"reference_artifact_{'h2' if h2 else 'h'}_{'tt' if near_tt else 'direct'}", k, v)  # noqa: E731,E501
    fam = {"se": pr.REF_SE, "e": pr.REF_E, "mc": pr.REF_MC}[family]
    path = str(tmp_path / "ref.hmat")
    pr.build_save(path, 2000, 3, 8, h2, fam, [(0.25, 1.0)], 2, 4, 6, eps=1e-6, eta=1.0, near_tt=near_tt,
                  threads=THREADS)
    R = pr.load(path)
    pm = ph.load_parametric(path)
    near, far, key = pm.blocks()
    sizes = _sizes(pm)
    x = pr.generate_normal(2000, 2)
    for th in ([0.25], [0.61], [1.0]):
        inst, ri = ph.instantiate(pm, th), R.instantiate(th)
        wd = max(rel(inst.near_d(b, (sizes[near[b, 0]], sizes[near[b, 1]])), ri.near_d(b)) for b in range(len(near)))
        wf = max(rel(inst.far_h(i), ri.far_h(i)) for i in range(0, len(far), 5))
        y = ri.apply(x)
        ey, ef = rel(inst.apply(x), y), rel(inst.instantiate_apply(th, x), y)
        assert wd <= TOL_BLOCK and wf <= TOL_BLOCK and ey <= TOL_Y and ef <= TOL_Y
        log("D_b", wd)
        log("far_h", wf)
        log("y_apply", ey)
        log("y_fused", ef)


def test_cpp_facade_drop_in_against_reference(tmp_path):
    """tests/cpp/dropin_check.cpp (built by oracle/ref_build.sh): the same C++
    program text against the reference's API (namespace phmat, CPU) and the
    product's facade (namespace phmat_b200, include/phmat_b200.hpp, GPU),
    both on Eigen types: the reference builds + saves, the facade loads onto
    the GPU, instantiate / apply / far_h / near_d / to_dense agree, the
    facade's own offline_h2 has the reference's structure, and the exception
    types match."""
    import json
    import subprocess

    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_check")
    assert os.path.exists(exe), "oracle/_ref/dropin_check not built (oracle/ref_build.sh)"
    res = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert res.returncode == 0 and out["ok"], res.stdout + res.stderr


def test_c5_sweep_batch_and_10_rhs_vs_reference(ph, c3, parity_log):
    """C5 (BASELINE configs[4]) = the C3 matrix, thetas instantiated 8 per
    snapshot pass (phm_instantiate_batch) and applied to 10 RHS each (K9 +
    multi-RHS coupling): probe rows of every RHS column against the
    reference's rows, for every theta of one batch."""
    log = lambda k, v: parity_log("c5_full_size_batch8_10rhs", k, v)  # noqa: E731
    pm, R, c, pts = c3
    b = _bench()
    thetas = b.theta_vectors(b.CONFIGS["c5"], 8, 3)
    insts = ph.instantiate_batch(pm, thetas)
    X = np.stack([ph.generate_normal(c["n"], 40 + j) for j in range(10)], axis=1)
    rows = np.sort(np.random.default_rng(9).choice(c["n"], 12, replace=False))
    info = pm.info()
    near_ids = np.sort(np.random.default_rng(4).choice(info["n_near"], 200, replace=False))
    for q, (th, inst) in enumerate(zip(thetas, insts)):
        th = list(th)
        if q in (0, 7):
            _check_blocks(ph, pm, inst, R, th, near_ids, range(0, info["n_classes"], 25), log=log)
        Y = inst.apply(X)
        yr = R.apply_rows(th, X, rows, threads=THREADS)
        e = max(rel(Y[rows, j], yr[:, j]) for j in range(10))
        assert e <= TOL_Y
        log("Y_rows_10rhs", e)
