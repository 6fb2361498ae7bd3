"""GPU: the reference's own relations (proj/tests/*.cpp) restated on the CUDA
path, through the C ABI.

* exact at theta grid nodes, zero online evaluations (test_nearfield.cpp:95-128)
* two-node midpoint averages the slices (test_nearfield.cpp:181-200)
* pttk_online at a grid node is the middle-core slice (test_farfield.cpp:242-258)
* H-form and H^2-form far blocks agree (test_farfield.cpp:287-308)
* translated blocks share bitwise-identical cores (test_farfield.cpp:335-380)
* instantiate + MVMs perform zero kernel evaluations (test_phmatrix.cpp:150-171)
* translation cache off: bitwise-equal instantiated matrices (test_phmatrix.cpp:325-353)
"""
import numpy as np
import pytest

from helpers import node_rows

pytestmark = pytest.mark.gpu


def _sizes(pm):
    return pm.nodes()[0][:, 3]


def _exact_block(po, pts, rows_s, rows_t, family, theta):
    K = po.dense_kernel(pts[np.concatenate([rows_s, rows_t])], family, theta)
    return K[: len(rows_s), len(rows_s):]


@pytest.mark.parametrize("mode", ["tt", "snapshot"])
def test_near_exact_at_grid_nodes_and_zero_online_evals(ph, po, mode):
    """test_nearfield.cpp:95-128 (3D, 512 points, 10 theta nodes, se): at grid
    thetas only the TT error remains (10 eps of max|K|); off the grid the
    theta interpolation joins in (1e-4 + 10 eps); online: zero evaluations."""
    pts = ph.generate_points(512, 3, 10)
    eps = 1e-5
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=4, p_theta=10, eps=eps, seed=4,
                      near_mode=ph.NearMode.TT if mode == "tt" else ph.NearMode.SNAPSHOT)
    pm = ph.offline_h2(pts, cfg)
    near, _, _ = pm.blocks()
    rows = node_rows(pm)
    sizes = _sizes(pm)
    nodes = pm.theta_grid(0)
    before = pm.info()["evals_online"]
    blocks = [b for b in range(len(near)) if near[b, 0] == near[b, 1]][:3] + [0, len(near) // 2]
    for k in range(10):
        inst = ph.instantiate(pm, [nodes[k]])
        for b in blocks:
            s, t = near[b]
            d = inst.near_d(b, (sizes[s], sizes[t]))
            ex = _exact_block(po, pts, rows(s), rows(t), ph.Family.SE, [nodes[k]])
            assert np.max(np.abs(d - ex)) <= 10 * eps * np.max(np.abs(ex))
    rng = np.random.default_rng(3)
    for _ in range(5):
        th = [rng.uniform(0.25, 1.0)]
        inst = ph.instantiate(pm, th)
        inst.apply(ph.generate_normal(512, 1))
        for b in blocks:
            s, t = near[b]
            d = inst.near_d(b, (sizes[s], sizes[t]))
            ex = _exact_block(po, pts, rows(s), rows(t), ph.Family.SE, th)
            assert np.max(np.abs(d - ex)) <= 1e-4 + 10 * eps
    assert pm.info()["evals_online"] == before


@pytest.mark.parametrize("mode", ["tt", "snapshot"])
def test_two_theta_nodes_midpoint_averages_slices(ph, mode):
    """test_nearfield.cpp:181-200: p_theta = 2 on [0.4, 0.8], D(0.6) =
    (D(x0) + D(x1)) / 2 within 1e-12."""
    pts = ph.generate_points(128, 2, 30)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.SE, [(0.4, 0.8)]), l_max=1, p_s=4, p_theta=2, eps=1e-12,
                      r_max_near=4, near_mode=ph.NearMode.TT if mode == "tt" else ph.NearMode.SNAPSHOT)
    pm = ph.offline_h2(pts, cfg)
    near, _, _ = pm.blocks()
    sizes = _sizes(pm)
    x0, x1 = pm.theta_grid(0)
    i_mid, i0, i1 = ph.instantiate(pm, [0.6]), ph.instantiate(pm, [x0]), ph.instantiate(pm, [x1])
    for b in range(len(near)):
        sh = (sizes[near[b, 0]], sizes[near[b, 1]])
        d = i_mid.near_d(b, sh)
        assert np.max(np.abs(d - 0.5 * (i0.near_d(b, sh) + i1.near_d(b, sh)))) <= 1e-12


def test_pttk_online_at_grid_node_is_the_core_slice(ph):
    """test_farfield.cpp:242-258 (2D, p_s 4, 6 theta nodes): H(node k) equals
    slice k of the middle core within 1e-13 of max(1, |slice|)."""
    pts = ph.generate_points(256, 2, 3)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=4, p_theta=6, eps=1e-8)
    pm = ph.offline_h(pts, cfg)
    _, far, key = pm.blocks()
    nodes = pm.theta_grid(0)
    before = pm.info()["evals_online"]
    for k in range(6):
        inst = ph.instantiate(pm, [nodes[k]])
        for i in range(0, len(far), max(1, len(far) // 10)):
            core = pm.coupling_cores(int(key[i]))[2]  # d = 2: the middle core
            sl = core[:, k, :]
            h = inst.far_h(i)
            assert np.max(np.abs(h - sl)) <= 1e-13 * max(1.0, np.max(np.abs(sl)))
    assert pm.info()["evals_online"] == before


def test_h_and_h2_far_blocks_agree(ph):
    """test_farfield.cpp:287-308 (2D, multiquadric, p_s 5, 6 theta nodes): the
    H form S H T^T and the H^2 form U_s L H R^T U_t^T of every far block
    agree within 1e-11 (compared through to_dense; near blocks are shared)."""
    pts = ph.generate_points(300, 2, 19)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.MC), l_max=2, p_s=5, p_theta=6, eps=1e-7)
    a, b = ph.offline_h(pts, cfg), ph.offline_h2(pts, cfg)
    rng = np.random.default_rng(4)
    for _ in range(3):
        th = [rng.uniform(0.25, 1.0)]
        da, db = ph.instantiate(a, th).to_dense(), ph.instantiate(b, th).to_dense()
        assert np.max(np.abs(da - db)) <= 1e-11


def test_translated_blocks_share_bitwise_cores(ph):
    """test_farfield.cpp:335-380: with the translation cache off every far
    block gets its own TT-cross, seeded by its translation key, so blocks of
    one class carry bitwise-identical cores; per-level offsets stay within
    +-3 (at most 7^d classes per level)."""
    pts = ph.generate_points(1024, 3, 70)
    base = dict(spec=ph.KernelSpec(ph.Family.E, [(0.25, 1.0)]), l_max=2, p_s=4, p_theta=4, eps=1e-5, seed=123)
    on = ph.offline_structure(pts, ph.PHConfig(**base), ph.Format.H)
    off = ph.offline_structure(pts, ph.PHConfig(**base, translation_cache=False), ph.Format.H)
    _, far, key = on.blocks()
    assert on.info()["n_classes"] < len(far)
    keys = on.class_keys()
    assert np.all(np.abs(keys[:, 1:4]) <= 3)
    for lvl in np.unique(keys[:, 0]):
        assert (keys[:, 0] == lvl).sum() <= 343
    seen = {}
    checked = 0
    for i in range(len(far)):
        k = int(key[i])
        if k in seen:
            ca, cb = off.coupling_cores(seen[k]), off.coupling_cores(i)
            assert all(np.array_equal(x, y) for x, y in zip(ca, cb))
            checked += 1
        else:
            seen[k] = i
        if checked >= 20:
            break
    assert checked > 0


def test_translation_cache_off_gives_bitwise_equal_instances(ph):
    """test_phmatrix.cpp:325-353: cache off, same instantiated far_h / near_d
    and S / T bitwise, more offline kernel work."""
    pts = ph.generate_points(400, 2, 15)
    base = dict(spec=ph.KernelSpec.default(ph.Family.E), l_max=2, p_s=4, p_theta=5, eps=1e-4, seed=1,
                near_mode=ph.NearMode.TT)
    on = ph.offline_h(pts, ph.PHConfig(**base))
    off = ph.offline_h(pts, ph.PHConfig(**base, translation_cache=False))
    assert off.info()["evals_offline"] > on.info()["evals_offline"]
    ia, ib = ph.instantiate(on, [0.5]), ph.instantiate(off, [0.5])
    near, far, _ = on.blocks()
    sizes = _sizes(on)
    for i in range(len(far)):
        assert np.array_equal(ia.far_h(i), ib.far_h(i))
        sa, ta = on.far_st(i)
        sb, tb = off.far_st(i)
        assert np.array_equal(sa, sb) and np.array_equal(ta, tb)
    for b in range(len(near)):
        sh = (sizes[near[b, 0]], sizes[near[b, 1]])
        assert np.array_equal(ia.near_d(b, sh), ib.near_d(b, sh))
    x = ph.generate_normal(400, 2)
    assert np.array_equal(ia.apply(x), ib.apply(x))


def test_online_stage_zero_kernel_evaluations(ph):
    """test_phmatrix.cpp:150-171: H and H^2 instantiate + MVM charge nothing
    to the online counter in TT and snapshot modes."""
    pts = ph.generate_points(420, 2, 3)
    for mode in (ph.NearMode.TT, ph.NearMode.SNAPSHOT):
        cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=5, p_theta=6, eps=1e-4, seed=1,
                          near_mode=mode)
        ph_, ph2 = ph.offline_h(pts, cfg), ph.offline_h2(pts, cfg)
        off = ph_.info()["evals_offline"]
        assert off > 0
        x = np.random.default_rng(5).uniform(-1, 1, 420)
        rng = np.random.default_rng(6)
        for _ in range(3):
            th = [rng.uniform(0.25, 1.0)]
            ph.instantiate(ph_, th).apply(x)
            ph.instantiate(ph2, th).apply(x)
            ph.instantiate(ph2, th).instantiate_apply(th, x)
        assert ph_.info()["evals_online"] == 0 and ph2.info()["evals_online"] == 0
        assert ph_.info()["evals_offline"] == off
