"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs and the same offline data.

Tolerances are the north_star's (fp64): instantiated blocks D_b, H_k, C_k
within 1e-12 relative Frobenius; MVM output within 1e-11 relative 2-norm.
Relations follow the reference's tests (proj/tests/test_phmatrix.cpp,
test_nearfield.cpp, test_farfield.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_BLOCK = 1e-12
TOL_Y = 1e-11


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _node_sizes(pm):
    ints, _ = pm.nodes()
    return ints[:, 3]


def _build(ph, po, pts, cfg, fmt, mask=None):
    pm = ph.offline_h2(pts, cfg) if fmt == ph.Format.H2 else ph.offline_h(pts, cfg)
    om = po.from_product(pm, pts, snapshot_mask=mask)
    return pm, om


def _check_instance(ph, pm, om, theta, block_stride=1):
    inst = ph.instantiate(pm, theta)
    oi = om.instantiate(theta)
    sizes = _node_sizes(pm)
    near, far, key = pm.blocks()
    worst = 0.0
    for b in range(0, len(near), block_stride):
        s, t = near[b]
        shape = (sizes[s], sizes[t])
        worst = max(worst, rel(inst.near_d(b, shape), oi.near(b, shape)))
    assert worst <= TOL_BLOCK, f"near D_b rel err {worst:.3e}"
    ncls = pm.info()["n_classes"]
    wh = 0.0
    for i in range(0, len(far), max(1, len(far) // 200)):
        wh = max(wh, rel(inst.far_h(i), oi.class_h(key[i])))
    assert wh <= TOL_BLOCK, f"far H rel err {wh:.3e}"
    if pm.format == ph.Format.H2:
        P = pm.info()["P"]
        wc = 0.0
        for k in range(0, ncls, max(1, ncls // 50)):
            wc = max(wc, rel(inst.class_c(k), oi.class_c(k, P)))
        assert wc <= TOL_BLOCK, f"C_k rel err {wc:.3e}"
    return inst, oi


@pytest.mark.parametrize("fam,sym", [("e", True), ("e", False), ("m32", True), ("gauss", False)])
def test_h2_snapshot_3d_matches_oracle(ph, po, fam, sym):
    pts = ph.generate_points(3000, 3, 0)
    box = {"e": (0.05, 0.5), "m32": (0.05, 0.5), "gauss": (0.1, 1.0)}[fam]
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.from_id(fam), [box]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT, seed=0, symmetric_near=sym)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    for theta in ([box[0]], [0.5 * (box[0] + box[1]) + 0.0123], [box[1]]):
        inst, oi = _check_instance(ph, pm, om, theta, block_stride=7)
        x = ph.generate_normal(pts.shape[0], 11)
        assert rel(inst.apply(x), oi.apply(x)) <= TOL_Y


def test_snapshot_generation_matches_oracle(ph, po):
    """K11 entries equal the reference's near_oracle (nearfield.cpp:35-46)."""
    pts = ph.generate_points(1500, 3, 3)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    info = pm.info()
    # symmetric storage keeps only sigma <= tau blocks (about half)
    assert info["near_stored"] < 0.6 * info["near_entries"]
    sizes = _node_sizes(pm)
    near, _, _ = pm.blocks()
    worst = 0.0
    for b in range(0, len(near), 5):
        s, t = near[b]
        shape = (sizes[s], sizes[t])
        assert pm.near_rank(b) == 8
        for kap in (0, 3, 7):
            g = pm.near_column(b, kap, shape).ravel(order="F")
            o = om.near_snapshot_column(b, kap, shape[0] * shape[1])
            worst = max(worst, np.max(np.abs(g - o) / np.maximum(np.abs(o), 1e-300)))
    assert worst <= 1e-15, f"snapshot max rel err {worst:.3e}"


def test_h_tt_mode_2d_c1_like(ph, po):
    """BASELINE config 1 shape (param-H, Gaussian, p_s = 6, p_theta = 8), reduced n."""
    pts = ph.generate_points(1024, 2, 0)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.GAUSS, [(0.1, 1.0)]), l_max=2, p_s=6, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.TT, seed=0)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H)
    for theta in ([0.1], [0.3456], [1.0]):
        inst, oi = _check_instance(ph, pm, om, theta)
        x = ph.generate_normal(pts.shape[0], 2)
        assert rel(inst.apply(x), oi.apply(x)) <= TOL_Y


def test_h2_tt_mode_and_accuracy_vs_exact(ph, po):
    """test_phmatrix.cpp:54-82: induced dense vs exact <= 10 eps ||K||_F."""
    pts = ph.generate_points(512, 3, 42)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=6, p_theta=8, eps=1e-4, seed=1)
    for fmt in (ph.Format.H, ph.Format.H2):
        pm, om = _build(ph, po, pts, cfg, fmt)
        rng = np.random.default_rng(9)
        for _ in range(3):
            theta = [rng.uniform(0.25, 1.0)]
            inst, oi = _check_instance(ph, pm, om, theta)
            exact = po.dense_kernel(pts, ph.Family.SE, theta)
            dense = inst.to_dense()
            assert np.linalg.norm(dense - exact) <= 10 * cfg.eps * np.linalg.norm(exact)
            assert rel(dense, oi.to_dense()) <= TOL_Y


def test_direct_near_mode(ph, po):
    """test_phmatrix.cpp:173-192: direct mode charges one online eval per near entry."""
    pts = ph.generate_points(256, 3, 23)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=1, p_s=4, p_theta=6, eps=1e-4, seed=1,
                      near_mode=ph.NearMode.DIRECT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H)
    before = pm.info()["evals_online"]
    inst, oi = _check_instance(ph, pm, om, [0.5])
    near, _, _ = pm.blocks()
    sizes = _node_sizes(pm)
    entries = int(sum(sizes[s] * sizes[t] for s, t in near))
    assert pm.info()["evals_online"] - before == entries
    exact = po.dense_kernel(pts, ph.Family.SE, [0.5])
    assert np.linalg.norm(inst.to_dense() - exact) <= 10 * cfg.eps * np.linalg.norm(exact)


def test_mvm_relations(ph, po):
    """Linearity, zero-in-zero-out, e_j extracts a column, determinism
    (test_phmatrix.cpp:100-148, 194-216)."""
    pts = ph.generate_points(2000, 3, 5)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_h2(pts, cfg)
    inst = ph.instantiate(pm, [0.21])
    n = pts.shape[0]
    rng = np.random.default_rng(4)
    x, z = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    assert np.all(inst.apply(np.zeros(n)) == 0.0)
    lhs = inst.apply(2 * x - 3 * z)
    rhs = 2 * inst.apply(x) - 3 * inst.apply(z)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs)) + 1e-14
    y1, y2 = inst.apply(x), inst.apply(x)
    assert np.array_equal(y1, y2)  # bitwise deterministic
    inst2 = ph.instantiate(pm, [0.21])
    assert np.array_equal(inst2.apply(x), y1)
    Y = inst.apply(np.eye(n)[:, [0, 100, n - 1]])
    for c, j in enumerate([0, 100, n - 1]):
        e = np.zeros(n)
        e[j] = 1.0
        assert np.max(np.abs(inst.apply(e) - Y[:, c])) <= 1e-13


def test_multi_rhs_matches_column_loop(ph, po):
    pts = ph.generate_points(2500, 3, 8)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.MATERN52, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    inst = ph.instantiate(pm, [0.3])
    X = np.stack([ph.generate_normal(pts.shape[0], s) for s in range(5)], axis=1)
    Y = inst.apply(X)
    Yo = om.instantiate([0.3]).apply(X)
    for c in range(X.shape[1]):
        assert rel(Y[:, c], Yo[:, c]) <= TOL_Y
        # the block path (K9 DMMA near field) vs the single-vector path (K6)
        assert rel(Y[:, c], inst.apply(X[:, c])) <= 1e-14
    assert np.array_equal(inst.apply(X), Y)  # deterministic


@pytest.mark.parametrize("sym,m", [(True, 64), (False, 70), (True, 7)])
def test_block_rhs_dmma_near_field(ph, po, sym, m):
    """K9 (multi-RHS near field on mma.sync f64) over symmetric and full
    storage, column counts across the 64-wide column tiles."""
    pts = ph.generate_points(2200, 3, 21)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT, symmetric_near=sym)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    inst = ph.instantiate(pm, [0.27])
    rng = np.random.default_rng(m)
    X = rng.standard_normal((2200, m))
    Y = inst.apply(X)
    Yo = om.instantiate([0.27]).apply(X)
    assert rel(Y, Yo) <= TOL_Y


@pytest.mark.parametrize("sym,m", [(True, 10), (True, 17), (False, 10), (True, 18)])
def test_block_rhs_tail_columns_on_gemv(ph, po, sym, m):
    """H^2 with m = 8k + (1 or 2) right-hand sides (BASELINE config 5: m =
    10): K9 takes the first 8k columns, the tail columns run on the HBM GEMV
    (K6). Every column against the oracle; the tail columns are the
    single-vector path bit for bit."""
    pts = ph.generate_points(2300, 3, 33)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT, symmetric_near=sym)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    inst = ph.instantiate(pm, [0.19])
    rng = np.random.default_rng(100 + m)
    X = rng.standard_normal((2300, m))
    Y = inst.apply(X)
    Yo = om.instantiate([0.19]).apply(X)
    for c in range(m):
        assert rel(Y[:, c], Yo[:, c]) <= TOL_Y
        assert rel(Y[:, c], inst.apply(X[:, c])) <= 1e-14
    assert np.array_equal(inst.apply(X), Y)  # deterministic


def test_two_parameter_amplitude_kernel(ph, po):
    """theta = (l, sigma^2) with an 8 x 6 tensor grid (BASELINE config 4 form)."""
    pts = ph.generate_mixture_points(3000, 3, 16, 0.05, 0)
    spec = ph.KernelSpec(ph.Family.MATERN52, [(0.05, 0.5), (0.5, 2.0)], amplitude=True)
    cfg = ph.PHConfig(spec=spec, l_max=2, p_s=4, p_theta=[8, 6], eta=1.0, near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    assert pm.near_rank(0) == 8  # sigma^2 enters linearly: rank-1 amplitude core
    for theta in ([0.05, 0.5], [0.17, 1.3], [0.5, 2.0]):
        inst, oi = _check_instance(ph, pm, om, theta, block_stride=11)
        x = ph.generate_normal(pts.shape[0], 3)
        assert rel(inst.apply(x), oi.apply(x)) <= TOL_Y


def test_errors_map_to_reference_exceptions(ph):
    pts = ph.generate_points(128, 2, 8)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=1, p_s=4, p_theta=5, eps=1e-4)
    pm = ph.offline_h(pts, cfg)
    with pytest.raises(ph.DomainError):
        ph.instantiate(pm, [3.0])
    inst = ph.instantiate(pm, [0.5])
    with pytest.raises(ph.InvalidArgument):
        inst.apply(np.zeros(129))


def test_symmetric_storage_is_exact(ph):
    """D_{tau,sigma} = D_{sigma,tau}^T bitwise, and the symmetric two-sided
    near GEMV agrees with the full-storage one to rounding."""
    pts = ph.generate_points(3000, 3, 6)
    base = dict(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                near_mode=ph.NearMode.SNAPSHOT)
    a = ph.offline_h2(pts, ph.PHConfig(**base, symmetric_near=True))
    b = ph.offline_h2(pts, ph.PHConfig(**base, symmetric_near=False))
    ia, ib = ph.instantiate(a, [0.123]), ph.instantiate(b, [0.123])
    sizes = _node_sizes(a)
    near, _, _ = a.blocks()
    for k in range(0, len(near), 13):
        s, t = near[k]
        assert np.array_equal(ia.near_d(k, (sizes[s], sizes[t])), ib.near_d(k, (sizes[s], sizes[t])))
    x = ph.generate_normal(3000, 1)
    assert rel(ia.apply(x), ib.apply(x)) <= 1e-14


@pytest.mark.parametrize("fmt,sym", [("h2", True), ("h2", False), ("h", True), ("h", False)])
def test_row_sharded_apply_on_one_gpu(ph, fmt, sym):
    """The multi-GPU row-sharded path with the shards built one after another
    on one GPU. Symmetric near storage: every shard's full-length partial y
    (phm_apply_partial_device / phm_instantiate_apply_partial_device), summed
    over shards, equals the unsharded MVM. Full storage: the shards' rows
    (phm_apply_rows_device) concatenated in rank order equal it too."""
    import torch

    pts = ph.generate_points(4000, 3, 12)
    base = dict(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                near_mode=ph.NearMode.SNAPSHOT, symmetric_near=sym)
    build = ph.offline_h2 if fmt == "h2" else ph.offline_h
    full = build(pts, ph.PHConfig(**base))
    x = ph.generate_normal(4000, 2)
    y_ref = ph.instantiate(full, [0.3]).apply(x)
    y_ref2 = ph.instantiate(full, [0.41]).apply(x)
    world = 3
    xd = torch.from_numpy(x).cuda()
    rows, perm = [], None
    ysum = np.zeros(4000)
    ysum2 = np.zeros(4000)
    stored = 0
    for r in range(world):
        pm = build(pts, ph.PHConfig(**base, shard_rank=r, shard_count=world))
        info = pm.info()
        stored += info["near_stored"]
        inst = ph.instantiate(pm, [0.3])
        part = torch.zeros(4000, dtype=torch.float64, device="cuda")
        inst.apply_partial_device(xd.data_ptr(), part.data_ptr(), 1)
        pm.ctx.sync()
        ysum += part.cpu().numpy()
        inst.instantiate_apply_partial_device([0.41], xd.data_ptr(), part.data_ptr(), 1)
        pm.ctx.sync()
        ysum2 += part.cpu().numpy()
        if sym:
            yr = torch.zeros(max(1, info["row_end"] - info["row_begin"]), dtype=torch.float64, device="cuda")
            with pytest.raises(ph.LogicError):
                inst.apply_rows_device(xd.data_ptr(), yr.data_ptr(), 1)
        else:
            yr = torch.zeros(max(1, info["row_end"] - info["row_begin"]), dtype=torch.float64, device="cuda")
            inst.apply_rows_device(xd.data_ptr(), yr.data_ptr(), 1)
            pm.ctx.sync()
            rows.append((info["row_begin"], yr[: info["row_end"] - info["row_begin"]].cpu().numpy()))
        perm = pm.perm()
    # the shards together store the unsharded near data exactly once
    assert stored == full.info()["near_stored"]
    y = np.empty(4000)
    y[perm] = ysum
    assert rel(y, y_ref) <= 1e-13
    y[perm] = ysum2
    assert rel(y, y_ref2) <= 1e-13
    if not sym:
        rows.sort(key=lambda t: t[0])
        yperm = np.concatenate([r for _, r in rows])
        assert yperm.size == 4000
        y[perm] = yperm
        assert rel(y, y_ref2) <= 1e-13  # the instances now hold theta = 0.41


@pytest.mark.parametrize("fmt,mode", [("h2", "snapshot"), ("h2", "tt"), ("h", "snapshot")])
def test_fused_instantiate_apply_equals_separate_calls(ph, po, fmt, mode):
    pts = ph.generate_points(2000, 3, 14)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT if mode == "snapshot" else ph.NearMode.TT)
    pm = ph.offline_h2(pts, cfg) if fmt == "h2" else ph.offline_h(pts, cfg)
    inst = ph.instantiate(pm, [0.4])
    x = ph.generate_normal(2000, 4)
    X = np.stack([x, 2 * x, ph.generate_normal(2000, 5), x, x], axis=1)
    for theta in ([0.11], [0.37]):
        # the snapshot path fuses K1 with the near GEMV (one TMA pass): D is
        # bit-identical to a separate instantiate, y agrees to rounding
        # (near row sums are accumulated in a different order)
        y_fused = inst.instantiate_apply(theta, x)
        ref = ph.instantiate(pm, theta)
        near, _, _ = pm.blocks()
        sizes = _node_sizes(pm)
        for k in range(0, len(near), 7):
            sh = (sizes[near[k][0]], sizes[near[k][1]])
            assert np.array_equal(inst.near_d(k, sh), ref.near_d(k, sh))
        assert rel(y_fused, ref.apply(x)) <= 1e-14
        assert np.array_equal(inst.instantiate_apply(theta, X), ref.apply(X))
    om = po.from_product(pm, pts)
    assert rel(inst.instantiate_apply([0.2], x), om.instantiate([0.2]).apply(x)) <= TOL_Y
    with pytest.raises(ph.DomainError):
        inst.instantiate_apply([0.9], x)


def test_artifact_round_trip_on_device(ph, tmp_path):
    """test_phmatrix.cpp:289-323: save -> load preserves the instantiated
    matrices (bitwise for TT mode; snapshot mode is written as full-rank TTs
    and reloads into the TT path with identical D_b)."""
    pts = ph.generate_points(1500, 3, 77)
    for mode in (ph.NearMode.TT, ph.NearMode.SNAPSHOT):
        cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.MC), l_max=2, p_s=4, p_theta=5, eps=1e-4,
                          near_mode=mode)
        pm = ph.offline_h2(pts, cfg)
        path = str(tmp_path / f"a{mode}.phm")
        ph.save_parametric(pm, path)
        lm = ph.load_parametric(path)
        x = ph.generate_normal(1500, 2)
        a, b = ph.instantiate(pm, [0.63]), ph.instantiate(lm, [0.63])
        near, _, _ = pm.blocks()
        sizes = _node_sizes(pm)
        for k in range(0, len(near), 9):
            s, t = near[k]
            assert np.array_equal(a.near_d(k, (sizes[s], sizes[t])), b.near_d(k, (sizes[s], sizes[t])))
        if mode == ph.NearMode.TT:
            assert np.array_equal(a.apply(x), b.apply(x))
        else:
            assert rel(a.apply(x), b.apply(x)) <= 1e-14


def test_estimate_error_matches_oracle_rows(ph, po):
    """harness.cpp:183-236 on the GPU: exact probe rows equal the oracle's
    dense kernel rows, approx rows equal the oracle MVM, and the error of a
    well-resolved matrix is small."""
    pts = ph.generate_points(1200, 3, 9)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT, seed=0)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    inst = ph.instantiate(pm, [0.21])
    err, det = inst.estimate_error(200, seed=3, details=True)
    rows = det["rows"]
    assert len(set(rows.tolist())) == 200  # without replacement
    K = po.dense_kernel(pts, ph.Family.E, [0.21])
    exact = K[rows] @ det["x"]
    assert np.max(np.abs(det["exact"] - exact)) <= 1e-12 * np.max(np.abs(exact))
    approx = om.instantiate([0.21]).apply(det["x"])[rows]
    assert rel(det["approx"], approx) <= TOL_Y
    assert err == pytest.approx(np.linalg.norm(exact - approx) / np.linalg.norm(exact), rel=1e-9)
    assert err < 1e-2


def test_reinstantiate_in_place(ph, po):
    pts = ph.generate_points(2000, 3, 1)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_h2(pts, cfg)
    a = ph.instantiate(pm, [0.4])
    x = ph.generate_normal(2000, 9)
    ya = a.apply(x)
    b = ph.instantiate(pm, [0.1])
    b.reinstantiate([0.4])
    assert np.array_equal(b.apply(x), ya)


@pytest.mark.parametrize("n,l_max", [(2999, 2), (2001, 1)])
def test_near_gemv_paths_odd_n_and_large_leaves(ph, po, n, l_max):
    """The TMA near passes take whole leaves of <= 128 rows (l_max 2 here);
    larger leaves (l_max 1: ~250 rows) fall back to the row-sliced kernel.
    Odd n puts the x panels of RHS columns > 0 on odd elements."""
    pts = ph.generate_points(n, 3, 31)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=l_max, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    sizes = _node_sizes(pm)
    ints, _ = pm.nodes()
    leaf_max = max(int(sizes[i]) for i in range(len(sizes)) if ints[i, 0] == l_max)
    assert (leaf_max <= 128) == (l_max == 2)
    inst = ph.instantiate(pm, [0.19])
    oi = om.instantiate([0.19])
    rng = np.random.default_rng(n)
    for m in (1, 2, 3, 5, 40):  # 5: two-sided K9 over 128-row slices; 40: one-sided K9
        X = rng.standard_normal((n, m)) if m > 1 else rng.standard_normal(n)
        assert rel(inst.apply(X), oi.apply(X)) <= TOL_Y
    x = rng.standard_normal(n)
    y = inst.instantiate_apply([0.44], x)
    assert rel(y, om.instantiate([0.44]).apply(x)) <= TOL_Y


@pytest.mark.parametrize("p_theta", [3, 5, 10, 13, 20])
def test_fused_near_pass_across_snapshot_ranks(ph, po, p_theta):
    """Each snapshot rank R <= 16 has its own k_near_tma instantiation (stage
    geometry depends on R); R > 16 takes the separate K1 + K6 kernels."""
    pts = ph.generate_points(2400, 3, 17)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.MATERN32, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=p_theta, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    inst = ph.instantiate(pm, [0.3])
    x = ph.generate_normal(2400, 6)
    near, _, _ = pm.blocks()
    sizes = _node_sizes(pm)
    for theta in ([0.06], [0.377]):
        y = inst.instantiate_apply(theta, x)
        assert rel(y, om.instantiate(theta).apply(x)) <= TOL_Y
        ref = ph.instantiate(pm, theta)
        for k in range(0, len(near), 11):
            sh = (sizes[near[k][0]], sizes[near[k][1]])
            assert np.array_equal(inst.near_d(k, sh), ref.near_d(k, sh))


@pytest.mark.parametrize("mode", ["snapshot", "tt"])
def test_theta_batched_instantiate(ph, po, mode):
    """instantiate_batch (one snapshot pass for the whole batch) equals a loop
    of single instantiates bit for bit; batches above 16 thetas are split;
    a theta outside the box fails the whole call before any launch."""
    pts = ph.generate_points(2000, 3, 27)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT if mode == "snapshot" else ph.NearMode.TT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    thetas = np.linspace(0.05, 0.5, 18).reshape(-1, 1)
    insts = ph.instantiate_batch(pm, thetas)
    assert len(insts) == 18
    near, _, _ = pm.blocks()
    sizes = _node_sizes(pm)
    x = ph.generate_normal(2000, 3)
    for b in (0, 7, 15, 16, 17):
        ref = ph.instantiate(pm, thetas[b])
        for k in range(0, len(near), 13):
            sh = (sizes[near[k][0]], sizes[near[k][1]])
            assert np.array_equal(insts[b].near_d(k, sh), ref.near_d(k, sh))
        assert np.array_equal(insts[b].apply(x), ref.apply(x))
    assert rel(insts[5].apply(x), om.instantiate(thetas[5]).apply(x)) <= TOL_Y
    ph.reinstantiate_batch(insts[:3], [[0.3], [0.2], [0.1]])
    assert np.array_equal(insts[1].apply(x), ph.instantiate(pm, [0.2]).apply(x))
    with pytest.raises(ph.DomainError):
        ph.instantiate_batch(pm, [[0.2], [0.9]])


def test_h_form_far_blocks_beyond_48kb_shared(ph, po):
    """H form whose coarsest far blocks have > 6,000 rows: k_far_h stages the
    sigma rows in more than 48 KB of shared memory (opt-in attribute)."""
    pts = ph.generate_points(24000, 1, 5)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=5, p_s=8, p_theta=6, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H)
    ints, _ = pm.nodes()
    _, far, _ = pm.blocks()
    assert max(int(ints[s, 3]) for s, _ in far) > 6000
    x = ph.generate_normal(24000, 9)
    assert rel(ph.instantiate(pm, [0.2]).apply(x), om.instantiate([0.2]).apply(x)) <= TOL_Y


def test_concurrent_host_threads_share_one_matrix(ph, po):
    """Two host threads applying instances of one matrix at the same time (the
    C ABI releases the GIL): the matrix serialises its launch sequences, so
    both get their own exact result."""
    import threading

    pts = ph.generate_points(2000, 3, 41)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_h2(pts, cfg)
    a, b = ph.instantiate(pm, [0.1]), ph.instantiate(pm, [0.4])
    xs = [ph.generate_normal(2000, s) for s in (1, 2)]
    want = [a.apply(xs[0]), b.apply(xs[1])]
    got = [[], []]

    def run(k, inst):
        for _ in range(20):
            got[k].append(inst.apply(xs[k]))

    ts = [threading.Thread(target=run, args=(0, a)), threading.Thread(target=run, args=(1, b))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k in (0, 1):
        assert all(np.array_equal(y, want[k]) for y in got[k])


def test_clustered_points_large_leaves(ph, po):
    """Mixture points (the C4 generator) leave some leaves with hundreds of
    rows: row-sliced near items, the shared-memory leaf gather, and the
    two-sided block-RHS kernel over slices, against the oracle."""
    n = 12000
    pts = ph.generate_mixture_points(n, 3, 16, 0.05, 3)
    spec = ph.KernelSpec(ph.Family.MATERN52, [(0.05, 0.5), (0.5, 2.0)], amplitude=True)
    cfg = ph.PHConfig(spec=spec, l_max=2, p_s=4, p_theta=[6, 4], eta=1.0, near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    ints, _ = pm.nodes()
    assert ints[ints[:, 0] == 2, 3].max() > 300
    theta = [0.21, 1.3]
    inst, oi = ph.instantiate(pm, theta), om.instantiate(theta)
    rng = np.random.default_rng(12)
    for m in (1, 5, 40):
        X = rng.standard_normal((n, m)) if m > 1 else rng.standard_normal(n)
        assert rel(inst.apply(X), oi.apply(X)) <= TOL_Y
    x = rng.standard_normal(n)
    assert rel(inst.instantiate_apply([0.33, 0.7], x), om.instantiate([0.33, 0.7]).apply(x)) <= TOL_Y


@pytest.mark.parametrize("n,d,l_max", [(1, 3, 2), (7, 2, 2), (33, 1, 3), (200, 3, 0)])
def test_tiny_and_degenerate_sizes(ph, po, n, d, l_max):
    """Edge cases: a single point, fewer points than leaves (empty leaves),
    1D, and l_max = 0 (one leaf, no far field) through every entry point."""
    pts = ph.generate_points(n, d, 5)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=l_max, p_s=3, p_theta=5, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    for fmt in (ph.Format.H2, ph.Format.H):
        pm, om = _build(ph, po, pts, cfg, fmt)
        inst = ph.instantiate(pm, [0.2])
        oi = om.instantiate([0.2])
        x = ph.generate_normal(n, 1)
        assert rel(inst.apply(x), oi.apply(x)) <= TOL_Y
        X = np.stack([x, 2 * x, ph.generate_normal(n, 2), x, x], axis=1)
        assert rel(inst.apply(X), oi.apply(X)) <= TOL_Y
        assert rel(inst.instantiate_apply([0.4], x), om.instantiate([0.4]).apply(x)) <= TOL_Y
        assert rel(inst.to_dense(), om.instantiate([0.4]).to_dense()) <= TOL_Y


_SCHEDULE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2511_03109_b200 as ph
pts = ph.generate_points(12000, 3, 21)
cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=3, p_s=4, p_theta=8, eta=1.0,
                  near_mode=ph.NearMode.SNAPSHOT)
pm = ph.offline_h2(pts, cfg)
inst = ph.instantiate(pm, [0.3])
x = ph.generate_normal(12000, 2)
ys = [inst.instantiate_apply(t, x) for t in ([0.12], [0.29], [0.12], [0.29])]
np.save(sys.argv[2], np.stack(ys))
"""


def test_coupling_schedule_does_not_change_results(ph, tmp_path):
    """The fused step's coupling runs as a capped grid resident beside the
    near pass, items in class-major order. Per-item
    partials and their reduction order are fixed, so y is bitwise the same
    with the full grid (PHM_COUPLING_RESIDENT=0) and the item order
    (PHM_COUPLING_ORDER=0), with and without CUDA graphs (the first call per
    key runs directly, the second captures, later ones replay)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "sched.py"
    script.write_text(_SCHEDULE_SCRIPT)
    outs = {}
    capped = {"PHM_COUPLING_RESIDENT": "1"}  # forced: this matrix's near pass is short
    for tag, env in (("default", capped), ("full", {"PHM_COUPLING_RESIDENT": "0"}),
                     ("unordered", {**capped, "PHM_COUPLING_ORDER": "0"}), ("nographs", {**capped, "PHM_GRAPHS": "0"})):
        out = tmp_path / f"{tag}.npy"
        subprocess.run([sys.executable, str(script), root, str(out)], check=True, timeout=600,
                       env={**os.environ, **env})
        outs[tag] = np.load(out)
    ref = outs["default"]
    assert np.array_equal(ref[0], ref[2]) and np.array_equal(ref[1], ref[3])  # direct vs captured vs replayed
    for tag in ("full", "unordered", "nographs"):
        assert np.array_equal(outs[tag], ref), tag


_K9_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2511_03109_b200 as ph
pts = ph.generate_points(9000, 3, 8)
cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=3, p_s=4, p_theta=8, eta=1.0,
                  near_mode=ph.NearMode.SNAPSHOT)
pm = ph.offline_h2(pts, cfg)
inst = ph.instantiate(pm, [0.21])
X = np.stack([ph.generate_normal(9000, 30 + j) for j in range(int(sys.argv[3]))], axis=1)
np.save(sys.argv[2], inst.apply(X))
"""


@pytest.mark.parametrize("m", [10, 24])
def test_k9_ring_depth_does_not_change_results(ph, po, tmp_path, m):
    """The two-sided K9 picks its ring depth from the tallest leaf
    (PHM_K9_STAGES overrides it); every depth gives bitwise the same y, and
    y matches the oracle."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "k9.py"
    script.write_text(_K9_SCRIPT)
    outs = {}
    for st in ("0", "2", "3"):
        out = tmp_path / f"y{st}.npy"
        subprocess.run([sys.executable, str(script), root, str(out), str(m)], check=True, timeout=600,
                       env={**os.environ, "PHM_K9_STAGES": st})
        outs[st] = np.load(out)
    assert np.array_equal(outs["0"], outs["2"]) and np.array_equal(outs["0"], outs["3"])
    pts = ph.generate_points(9000, 3, 8)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=3, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    om = po.from_product(ph.offline_structure(pts, cfg), pts).instantiate([0.21])
    X = np.stack([ph.generate_normal(9000, 30 + j) for j in range(m)], axis=1)
    ref = np.stack([om.apply(X[:, j]) for j in range(m)], axis=1)
    assert rel(outs["0"], ref) <= TOL_Y


def test_graph_replay_after_workspace_growth(ph, po):
    """the lazily grown two-sided K9 partials must not be
    left dangling in a captured graph. Sequence m = 64, 8, 8 (captured), 16
    (grows the partials), 8 (replay) against the oracle, plus more distinct
    x pointers than the graph cache holds (LRU eviction)."""
    import torch

    pts = ph.generate_points(2500, 3, 19)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm, om = _build(ph, po, pts, cfg, ph.Format.H2)
    inst = ph.instantiate(pm, [0.25])
    oi = om.instantiate([0.25])
    rng = np.random.default_rng(2)
    X = rng.standard_normal((2500, 64))
    Yo = oi.apply(X)
    for m in (64, 8, 8, 16, 8, 8, 32, 8):
        assert rel(inst.apply(X[:, :m]), Yo[:, :m]) <= TOL_Y, m
    xs = [torch.from_numpy(X[:, j].copy()).cuda() for j in range(20)]
    y = torch.zeros(2500, dtype=torch.float64, device="cuda")
    oi2 = om.instantiate([0.37])
    for rep in range(2):
        for j, xd in enumerate(xs):
            inst.instantiate_apply_device([0.37], xd.data_ptr(), y.data_ptr(), 1)
            pm.ctx.sync()
            if j % 7 == 0:
                assert rel(y.cpu().numpy(), oi2.apply(X[:, j])) <= TOL_Y


def test_two_matrices_on_one_context_from_two_threads(ph, po):
    """matrices sharing a Context serialise on the
    Context's lock (its stream, events and timers are shared)."""
    import threading

    pts = ph.generate_points(1800, 3, 23)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    a, oa = _build(ph, po, pts, cfg, ph.Format.H2)
    b, ob = _build(ph, po, pts, cfg, ph.Format.H2)
    assert a.ctx is b.ctx
    x = ph.generate_normal(1800, 4)
    ya, yb = oa.instantiate([0.2]).apply(x), ob.instantiate([0.4]).apply(x)
    errs = []

    def run(pm, th, yref):
        inst = ph.instantiate(pm, th)
        for _ in range(30):
            e = rel(inst.instantiate_apply(th, x), yref)
            if e > TOL_Y:
                errs.append(e)

    ts = [threading.Thread(target=run, args=(a, [0.2], ya)), threading.Thread(target=run, args=(b, [0.4], yb))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs


_NEAR_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2511_03109_b200 as ph
from oracle import pyoracle as po
pts = ph.generate_points(12000, 3, 23)
cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=3, p_s=4, p_theta=8, eta=1.0,
                  near_mode=ph.NearMode.SNAPSHOT)
pm = ph.offline_h2(pts, cfg)
inst = ph.instantiate(pm, [0.21])
x = ph.generate_normal(12000, 3)
ys = [inst.apply(x) for _ in range(3)] + [inst.instantiate_apply([0.21], x)]
ref = po.from_product(pm, pts).instantiate([0.21]).apply(x)
np.save(sys.argv[2], np.stack(ys + [ref]))
"""


@pytest.mark.gpu
def test_near_gemv_kernels_and_item_order(ph, tmp_path):
    """apply's near GEMV: the lean kernel (default; 4 consumer warps, two
    CTAs per SM beside the coupling) and the 8-warp kernel
    (PHM_NEAR_GEMV=0) both match the oracle to 1e-13 and each other to
    rounding; the longest-first item order (PHM_ITEM_ORDER=0 turns it off)
    changes no bit of y, since every item writes fixed partial segments;
    repeated applies (direct, captured, replayed) are bitwise equal."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "near.py"
    script.write_text(_NEAR_SCRIPT)
    outs = {}
    for tag, env in (("lean", {}), ("old", {"PHM_NEAR_GEMV": "0"}), ("unordered", {"PHM_ITEM_ORDER": "0"}),
                     ("lean1", {"PHM_NEAR_LEAN_PER_SM": "1", "PHM_NEAR_LEAN_NST": "3"})):
        out = tmp_path / f"{tag}.npy"
        subprocess.run([sys.executable, str(script), root, str(out)], check=True, timeout=600,
                       env={**os.environ, **env})
        outs[tag] = np.load(out)
    for tag, ys in outs.items():
        ref = ys[-1]
        assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2]), tag
        for y in ys[:4]:
            assert rel(y, ref) <= 1e-13, tag
    assert np.array_equal(outs["lean"][:4], outs["unordered"][:4])
    assert np.array_equal(outs["lean"][:3], outs["lean1"][:3])  # same kernel, one CTA per SM
    assert rel(outs["lean"][0], outs["old"][0]) <= 1e-14


@pytest.mark.gpu
def test_split_leaf_forward_big_clustered_leaves(ph, po):
    """Leaves of more than kLeafChunk (256) points -- clustered points at a
    shallow l_max -- run the leaf forward pass split into chunks with an
    ordered per-leaf sum (K3 for m >= 4); y of block right-hand sides matches
    the oracle and the column-by-column apply, and repeats bitwise."""
    pts = ph.generate_mixture_points(12000, 3, 16, 0.05, 3)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=4, p_theta=8, eta=1.0,
                      near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_h2(pts, cfg)
    sizes = _node_sizes(pm)
    ints, _ = pm.nodes()
    assert sizes[ints[:, 2] < 0].max() > 256  # the split path is exercised
    om = po.from_product(pm, pts)
    inst = ph.instantiate(pm, [0.19])
    for m in (6, 24):
        X = np.stack([ph.generate_normal(12000, 40 + j) for j in range(m)], axis=1)
        Y = inst.apply(X)
        assert np.array_equal(Y, inst.apply(X))
        assert rel(Y, om.instantiate([0.19]).apply(X)) <= 1e-12
        assert rel(Y[:, 1], inst.apply(X[:, 1])) <= 1e-13
