"""Baselines (proj/src/baselines.cpp): H-ACA and H^2-HCA at one fixed theta,
factorised on the host, applied through the GPU engine. The relations are
the reference's own (proj/tests/test_baselines.cpp)."""
import numpy as np
import pytest


def test_aca_partial_rank_one_recovered_exactly(ph):
    """test_baselines.cpp:33-43."""
    rng = np.random.default_rng(3)
    u, v = rng.uniform(-1, 1, 40), rng.uniform(-1, 1, 33)
    V, Y, capped = ph.aca_partial(np.outer(u, v), 1e-10, 20, 7)
    assert V.shape[1] == 1
    assert np.max(np.abs(V @ Y.T - np.outer(u, v))) <= 1e-13


def test_aca_partial_zero_matrix_gives_rank_zero(ph):
    """test_baselines.cpp:45-49."""
    V, Y, capped = ph.aca_partial(np.zeros((15, 18)), 1e-8, 10, 3)
    assert V.shape[1] == 0 and not capped


def test_aca_partial_admissible_se_block(ph, po):
    """test_baselines.cpp:51-69: an admissible SE block to 1e-5 max-relative."""
    pts = ph.generate_points(512, 3, 42)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=3, p_theta=3, eta=np.sqrt(3.0))
    pm = ph.offline_structure(pts, cfg)
    ints, _ = pm.nodes()
    _, far, _ = pm.blocks()
    perm = pm.perm()
    # tree-order ranges: a node's points are perm[start : start + count];
    # children are consecutive ids after their parent
    starts = np.zeros(len(ints), dtype=np.int64)
    for i in range(len(ints)):
        if ints[i, 2] >= 0:
            off = starts[i]
            for c in range(ints[i, 2], ints[i, 2] + 8):
                starts[c] = off
                off += ints[c, 3]
    blk = next(b for b in far if ints[b[0], 3] >= 6 and ints[b[1], 3] >= 6)
    rows = perm[starts[blk[0]]: starts[blk[0]] + ints[blk[0], 3]]
    cols = perm[starts[blk[1]]: starts[blk[1]] + ints[blk[1], 3]]
    exact = po.dense_kernel(pts, ph.Family.SE, [0.4])[np.ix_(rows, cols)]
    V, Y, _ = ph.aca_partial(exact, 1e-6, 64, 11)
    assert np.max(np.abs(V @ Y.T - exact)) <= 1e-5 * np.max(np.abs(exact))
    assert V.shape[1] <= 30


def _exact(po, ph, pts, fam, theta):
    return po.dense_kernel(pts, fam, theta)


@pytest.mark.gpu
def test_h_aca_mvm_error_eval_accounting_mean_rank(ph, po):
    """test_baselines.cpp:71-98."""
    n = 512
    pts = ph.generate_points(n, 3, 8)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, eta=np.sqrt(3.0), threads=2)
    eps = 1e-6
    ha = ph.h_aca(pts, cfg, [0.6], eps=eps, r_max=120)
    info = ha.info()
    pm = ph.offline_structure(pts, ph.PHConfig(spec=cfg.spec, l_max=2, p_s=3, p_theta=3, eta=np.sqrt(3.0)),
                              ph.Format.H)
    near, _, _ = pm.blocks()
    ints, _ = pm.nodes()
    near_entries = int(sum(ints[s, 3] * ints[t, 3] for s, t in near))
    assert info["near_evals"] + info["far_evals"] >= near_entries
    exact = _exact(po, ph, pts, ph.Family.SE, [0.6])
    x = np.random.default_rng(4).uniform(-1, 1, n)
    want = exact @ x
    assert np.linalg.norm(ha.apply(x) - want) <= 10 * eps * np.linalg.norm(want)
    assert np.linalg.norm(ha.to_dense() - exact) <= 10 * eps * np.linalg.norm(exact)
    assert 0.0 < ha.mean_far_rank() <= 40.0
    with pytest.raises(ph.LogicError):
        ha.reinstantiate([0.5])


@pytest.mark.gpu
def test_h2_hca_mvm_error_and_coupling_ratio(ph, po):
    """test_baselines.cpp:100-128."""
    n = 480
    pts = ph.generate_points(n, 3, 9)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=7, eta=np.sqrt(3.0), threads=2)
    eps = 1e-6
    hc = ph.h2_hca(pts, cfg, [0.8], eps=eps, r_max=200)
    info = hc.info()
    assert info["far_evals"] > 0
    exact = _exact(po, ph, pts, ph.Family.SE, [0.8])
    x = np.random.default_rng(5).uniform(0, 1, n)
    want = exact @ x
    assert np.linalg.norm(hc.apply(x) - want) <= 10 * eps * np.linalg.norm(want)
    assert np.linalg.norm(hc.to_dense() - exact) <= 100 * eps * np.linalg.norm(exact)
    expect = 2.0 * info["n_far"] * 343.0 * hc.mean_far_rank() / (n * n)
    assert hc.coupling_ratio() == pytest.approx(expect, rel=1e-12)
    # the apply is the dense operator it reconstructs (to rounding)
    X = np.random.default_rng(6).standard_normal((n, 3))
    assert np.linalg.norm(hc.apply(X) - hc.to_dense() @ X) <= 1e-12 * np.linalg.norm(hc.to_dense() @ X)


@pytest.mark.gpu
def test_baselines_share_the_mvm_interface(ph, po):
    """test_baselines.cpp:130-149."""
    pts = ph.generate_points(200, 2, 3)
    base = dict(spec=ph.KernelSpec.default(ph.Family.E), l_max=2, eta=np.sqrt(2.0), threads=1)
    ops = [ph.h_aca(pts, ph.PHConfig(**base), [0.5], eps=1e-5, r_max=60),
           ph.h2_hca(pts, ph.PHConfig(**base, p_s=5), [0.5], eps=1e-5, r_max=60)]
    exact = _exact(po, ph, pts, ph.Family.E, [0.5])
    x = np.ones(200)
    for op in ops:
        assert op.rows() == 200
        assert np.linalg.norm(op.apply(x) - exact @ x) <= 1e-3 * np.linalg.norm(exact @ x)
