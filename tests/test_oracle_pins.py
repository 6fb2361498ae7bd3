"""CPU: pin the oracle (oracle/oracle.cpp) against the reference's own
known-answer tests. The reference C++ cannot be built here (Eigen3 absent),
so these relations ARE the pins: every case below restates a doctest of
proj/tests/*.cpp (file:line in each docstring)."""
import math

import numpy as np
import pytest

E, TPS, SE, MC, MN, GAUSS, M32, M52 = range(8)


# ------------------------------------------------------------------ kernels
def bessel_k_quad(nu, z):
    """K_nu(z) = int_0^inf exp(-z cosh t) cosh(nu t) dt (test_kernels.cpp:13-37)."""
    x, w = np.polynomial.legendre.leggauss(16)
    t_max = math.acosh(max(2.0, 740.0 / z))
    panels = 256
    h = t_max / panels
    total = 0.0
    for p in range(panels):
        t = (p + 0.5) * h + 0.5 * h * x
        total += 0.5 * h * np.sum(w * np.exp(-z * np.cosh(t)) * np.cosh(nu * t))
    return total


def test_pointwise_values(po):
    """test_kernels.cpp:64-80."""
    lam = 0.62
    assert po.kernel_value(SE, 0.0, [lam]) == 1.0
    assert po.kernel_value(E, lam, [lam]) == pytest.approx(math.exp(-1.0), rel=1e-15)
    assert po.kernel_value(TPS, lam, [lam]) == 0.0
    assert po.kernel_value(TPS, 0.0, [lam]) == 0.0
    assert po.kernel_value(MC, lam, [lam]) == pytest.approx(math.sqrt(2.0), rel=1e-15)
    assert po.kernel_value(MN, lam, [lam, 0.5]) == pytest.approx(math.exp(-1.0), rel=1e-12)


def test_matern_half_is_exponential(po):
    """test_kernels.cpp:82-93."""
    for lam in (0.25, 0.5, 0.77, 1.0):
        for r in (1e-8, 1e-3, 0.05, 0.3, 0.9, 1.7):
            assert po.kernel_value(MN, r, [lam, 0.5]) == pytest.approx(po.kernel_value(E, r, [lam]), rel=1e-10)


def test_matern_against_quadrature(po):
    """test_kernels.cpp:111-122 (std::cyl_bessel_k vs the integral)."""
    for nu in (0.5, 1.0, 1.5, 2.2, 3.0):
        for lam in (0.25, 0.6, 1.0):
            for r in (0.0, 1e-5, 0.04, 0.33, 1.2, 1.7320508075688772):
                if r == 0.0:
                    ref = 1.0
                else:
                    z = math.sqrt(2 * nu) * r / lam
                    ref = 2 ** (1 - nu) / math.gamma(nu) * z ** nu * bessel_k_quad(nu, z)
                assert po.kernel_value(MN, r, [lam, nu]) == pytest.approx(ref, rel=1e-11)


def test_single_parameter_families_closed_forms(po):
    """Gauss / Matern-3/2 / Matern-5/2 (BASELINE configs) vs closed forms, and
    Matern-3/2 / -5/2 equal the generic Matern at nu = 3/2, 5/2."""
    for lam in (0.05, 0.2, 0.5, 1.0):
        for r in (0.0, 1e-4, 0.03, 0.2, 0.7):
            assert po.kernel_value(GAUSS, r, [lam]) == pytest.approx(math.exp(-r * r / (2 * lam * lam)), rel=1e-14)
            s3 = math.sqrt(3) * r / lam
            assert po.kernel_value(M32, r, [lam]) == pytest.approx((1 + s3) * math.exp(-s3), rel=1e-14)
            s5 = math.sqrt(5) * r / lam
            assert po.kernel_value(M52, r, [lam]) == pytest.approx((1 + s5 + s5 * s5 / 3) * math.exp(-s5), rel=1e-14)
            if r > 0:
                assert po.kernel_value(M32, r, [lam]) == pytest.approx(po.kernel_value(MN, r, [lam, 1.5]), rel=1e-10)
                assert po.kernel_value(M52, r, [lam]) == pytest.approx(po.kernel_value(MN, r, [lam, 2.5]), rel=1e-10)
            # amplitude multiplies (theta = (l, sigma^2))
            assert po.kernel_value(M52, r, [lam, 1.7], amp=True) == pytest.approx(
                1.7 * po.kernel_value(M52, r, [lam]), rel=1e-15)


# ----------------------------------------------------------------- geometry
def test_diam_dist_admissibility(po):
    """test_geometry.cpp:36-63."""
    adm, diam, dist = po.box_admissible([0], [1], [2], [3], 1.0)
    assert dist == pytest.approx(1.0) and adm
    _, diam, dist = po.box_admissible([0, 0], [1, 1], [0, 0], [1, 1], 1.0)
    assert dist == 0.0 and diam == pytest.approx(math.sqrt(2))
    _, _, dist = po.box_admissible([0, 0], [1, 1], [2, 2], [3, 3], 1.0)
    assert dist == pytest.approx(math.sqrt(2))
    _, _, dist = po.box_admissible([0], [2], [1], [3], 1.0)
    assert dist == 0.0
    eta = math.sqrt(3)
    assert po.box_admissible([0, 0, 0], [1, 1, 1], [2, 0, 0], [3, 1, 1], eta)[0]       # one-box separation
    assert not po.box_admissible([0, 0, 0], [1, 1, 1], [1, 0, 0], [2, 1, 1], eta)[0]   # touching
    # equality case at eta = 1: offset (2,2,2) at side 1 is admissible exactly
    assert po.box_admissible([0, 0, 0], [1, 1, 1], [2, 2, 2], [3, 3, 3], 1.0)[0]


def test_single_point_lmax0(po):
    """test_geometry.cpp:65-77."""
    m = po.OracleMatrix(np.array([[0.5]]), 0, 1.0, 2, SE, [(0.25, 1.0)], 2)
    c = m.counts()
    assert c["nodes"] == 1 and c["n_far"] == 0 and c["n_near"] == 1 and c["c_sp"] == 1
    assert list(m.perm()) == [0]


def test_quadtree_tiles(po):
    """test_geometry.cpp:79-102: d=2, l_max=2 gives 16 quarter-side leaves."""
    pts = po.generate_points(200, 2, 3)
    m = po.OracleMatrix(pts, 2, math.sqrt(2), 2, SE, [(0.25, 1.0)], 2)
    ints, boxes = m.nodes()
    leaves = np.where(ints[:, 2] < 0)[0]
    assert len(leaves) == 16
    assert np.allclose(boxes[leaves, 3:5] - boxes[leaves, 0:2], 0.25, atol=1e-15)
    assert len({(ints[i, 4], ints[i, 5]) for i in leaves}) == 16
    assert ints[leaves, 3].sum() == 200


def test_midpoint_goes_to_lower_child(po):
    """test_geometry.cpp:117-124."""
    m = po.OracleMatrix(np.array([[0.5], [0.75]]), 1, 1.0, 2, SE, [(0.25, 1.0)], 2)
    ints, _ = m.nodes()
    assert list(ints[1:3, 3]) == [1, 1]
    assert list(m.perm()) == [0, 1]


def test_point_outside_root_rejected(po):
    """test_geometry.cpp:126-131."""
    with pytest.raises(ValueError):
        po.OracleMatrix(np.array([[1.5, 0.5]]), 1, 1.0, 2, SE, [(0.25, 1.0)], 2)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_block_tree_coverage_and_sparsity(po, d):
    """test_geometry.cpp:143-165: coverage = n^2, far blocks same level and
    admissible, near blocks are leaf pairs, c_sp <= 2^d 3^d."""
    n = 2048 if d == 3 else 512
    pts = po.generate_points(n, d, 17 + d)
    eta = math.sqrt(d)
    m = po.OracleMatrix(pts, 3, eta, 2, SE, [(0.25, 1.0)], 2)
    ints, boxes = m.nodes()
    near, far, _ = m.blocks()
    sizes = ints[:, 3].astype(np.int64)
    cover = (sizes[near[:, 0]] * sizes[near[:, 1]]).sum() + (sizes[far[:, 0]] * sizes[far[:, 1]]).sum()
    assert cover == n * n
    assert np.all(ints[far[:, 0], 0] == ints[far[:, 1], 0])
    for s, t in far[:: max(1, len(far) // 300)]:
        assert po.box_admissible(boxes[s, :d], boxes[s, 3:3 + d], boxes[t, :d], boxes[t, 3:3 + d], eta)[0]
    assert np.all(ints[near[:, 0], 2] < 0) and np.all(ints[near[:, 1], 2] < 0)
    assert m.counts()["c_sp"] <= (1 << d) * 3 ** d


def test_empty_boxes_never_reach_block_lists(po):
    """test_geometry.cpp:196-216."""
    from oracle.pyoracle import lib, _DP

    u = np.empty(64)
    lib().orc_rng_uniform(9, 64, u.ctypes.data_as(_DP))
    pts = 0.05 * u.reshape(32, 2)
    m = po.OracleMatrix(pts, 2, math.sqrt(2), 2, SE, [(0.25, 1.0)], 2)
    ints, _ = m.nodes()
    near, far, _ = m.blocks()
    assert (ints[:, 2] < 0).sum() == 16
    for blk in (near, far):
        assert np.all(ints[blk[:, 0], 3] > 0) and np.all(ints[blk[:, 1], 3] > 0)
    sizes = ints[:, 3].astype(np.int64)
    cover = (sizes[near[:, 0]] * sizes[near[:, 1]]).sum() + (sizes[far[:, 0]] * sizes[far[:, 1]]).sum()
    assert cover == 32 * 32


# ---------------------------------------------------------------- chebyshev
def test_grid_nodes(po):
    """test_chebyshev.cpp:11-23."""
    x, _, _ = po.cheb_grid(0.0, 2.0, 1)
    assert x[0] == pytest.approx(1.0)
    x, _, _ = po.cheb_grid(-1.0, 1.0, 2)
    assert x[0] == pytest.approx(-math.sqrt(2) / 2) and x[1] == pytest.approx(math.sqrt(2) / 2)
    x, _, _ = po.cheb_grid(0.25, 0.5, 8)
    assert np.all(np.diff(x) > 0)


def test_cardinal_and_partition_of_unity(po):
    """test_chebyshev.cpp:25-43."""
    x, _, _ = po.cheb_grid(0.3, 1.7, 9)
    for j in range(9):
        v = po.lagrange_all(0.3, 1.7, 9, x[j])
        assert np.array_equal(v, np.eye(9)[j])
    from oracle.pyoracle import lib, _DP

    u = np.empty(100)  # the reference's own draws: Rng(5).uniform(-0.5, 2.5)
    lib().orc_rng_uniform(5, 100, u.ctypes.data_as(_DP))
    for t in -0.5 + 3.0 * u:
        assert po.lagrange_all(0.3, 1.7, 9, t).sum() == pytest.approx(1.0, rel=1e-12)


def test_two_node_symmetry(po):
    """test_chebyshev.cpp:45-49 and test_farfield.cpp:84-89."""
    v = po.lagrange_all(-1.0, 1.0, 2, 0.0)
    assert v == pytest.approx([0.5, 0.5])
    v = po.lagrange_all(0.5, 1.5, 2, 1.0)
    assert v[0] == pytest.approx(0.5, rel=1e-14) and v[1] == pytest.approx(0.5, rel=1e-14)


def test_polynomial_reproduction(po):
    """test_chebyshev.cpp:51-71."""
    rng = np.random.default_rng(12)
    for p in (3, 6, 11):
        x, _, _ = po.cheb_grid(-0.4, 0.9, p)
        coef = rng.uniform(-1, 1, p)
        poly = np.polynomial.polynomial.Polynomial(coef)
        for t in rng.uniform(-0.4, 0.9, 40):
            assert po.lagrange_all(-0.4, 0.9, p, t) @ poly(x) == pytest.approx(poly(t), rel=1e-12, abs=1e-13)


def test_degenerate_interval_finite(po):
    """test_chebyshev.cpp:73-81."""
    _, w, _ = po.cheb_grid(0.5, 0.5, 4)
    assert np.all(np.isfinite(w))
    assert np.isfinite(po.lagrange_all(0.5, 0.5, 4, 0.5 + 1e-3).sum())


def test_fast_kron_vs_dense(po):
    """test_chebyshev.cpp:177-227: (A_d x ... x A_1) x, transposed too."""
    rng = np.random.default_rng(3)
    for d in (1, 2, 3):
        for p in (2, 4, 5):
            fs = [rng.uniform(-1, 1, (p, p)) for _ in range(d)]
            x = rng.uniform(-1, 1, p ** d)
            dense = fs[0]
            for f in fs[1:]:
                dense = np.kron(f, dense)
            assert np.max(np.abs(po.fast_kron(fs, x) - dense @ x)) <= 1e-13
            assert np.max(np.abs(po.fast_kron(fs, x, True) - dense.T @ x)) <= 1e-13


def test_h2_mvm_equals_dense_assembly(po):
    """Forward/backward (chebyshev.cpp:223-298) vs the dense basis assembly
    used by to_dense (test_chebyshev.cpp:256-294, test_phmatrix.cpp:100-132):
    the oracle's H^2 apply equals its own induced dense matrix times x, given
    synthetic coupling cores."""
    pts = po.generate_points(300, 2, 77)
    m = po.OracleMatrix(pts, 2, math.sqrt(2), 4, SE, [(0.25, 1.0)], 3, h2=True)
    rng = np.random.default_rng(0)
    cnt = m.counts()
    for k in range(cnt["n_classes"]):
        ranks = [1, 3, 5, 4, 3, 1]
        dims = [4, 4, 3, 4, 4]
        m.set_coupling(k, [rng.uniform(-1, 1, (ranks[i], dims[i], ranks[i + 1])) for i in range(5)])
    m.make_near_snapshots()
    m.finalize()
    inst = m.instantiate([0.5])
    x = rng.uniform(-1, 1, 300)
    assert np.max(np.abs(inst.apply(x) - inst.to_dense() @ x)) <= 1e-12 * max(1.0, np.max(np.abs(inst.to_dense())))


def test_generate_points_is_the_reference_stream(po):
    """harness.cpp:174-181: Rng(mix_seed(seed, 'poin')), uniform = (g >> 11) 2^-53,
    row-major fill; first value pinned against a direct mt19937_64 transcription."""
    from oracle.pyoracle import lib

    seed = lib().orc_mix_seed(0, 0x706F696E)
    # std::mt19937_64 reference implementation (the standard's algorithm)
    mt = [0] * 312
    mt[0] = seed
    for i in range(1, 312):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & (2 ** 64 - 1)
    y = 0
    upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
    i = 0
    yv = (mt[i] & upper) | (mt[i + 1] & lower)
    mt[i] = mt[i + 156] ^ (yv >> 1) ^ (0xB5026F5AA96619E9 if yv & 1 else 0)  # n = 312, m = 156
    y = mt[0]
    y ^= (y >> 29) & 0x5555555555555555
    y ^= (y << 17) & 0x71D67FFFEDA60000
    y ^= (y << 37) & 0xFFF7EEE000000000
    y ^= y >> 43
    first = (y >> 11) * 2.0 ** -53
    assert po.generate_points(1, 1, 0)[0, 0] == first
