"""CPU: pins against the COMPILED REFERENCE (oracle/_ref/libphmat_ref.so, the
unmodified /root/reference/proj/src built against oracle/eigen_shim by
oracle/ref_build.sh).

1. The shimmed reference build passes the reference's own doctest suites
   (proj/tests/test_*.cpp, compiled unmodified against oracle/doctest_shim).
2. The product's host structure (tree, permutation, node boxes, near / far
   lists, translation classes) is bitwise the reference's, at the
   BASELINE configs' own sizes.
3. The oracle (oracle/oracle.cpp) equals the reference on the online path
   (D_b, H_k, C_k, y) on the same offline data.
4. The H form's S_b / T_b of the product's host build equal the reference's
   pttk_offline (farfield.cpp:126-147)."""
import os
import subprocess

import numpy as np
import pytest
from helpers import node_rows

from oracle import pyref as pr

# One reference case fails under the shim: the offline TT-cross of 4 of 316
# coupling tensors stalls at the rank cap (est. error 0.22), so the induced
# matrix misses 10*eps. It is offline data production (tt.cpp:269-480), not
# the online path, and does not depend on the SVD (checked with LAPACK
# dgesdd in place of the shim's Jacobi SVD); the product's restatement of the
# cross stalls on the same tensors. Every other case passes.
KNOWN_OFFLINE_FAILURES = {"induced dense matrix matches the kernel matrix (H and H2, d = 3)"}
SUITES = ["kernels", "geometry", "chebyshev", "tt", "farfield", "nearfield", "baselines", "phmatrix"]


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("suite", SUITES)
def test_reference_doctest_suite(suite):
    exe = os.path.join(pr.TEST_DIR, f"test_{suite}")
    if not os.path.exists(exe):
        pr.build()
    res = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    failed = [ln[7:].strip() for ln in res.stdout.splitlines() if ln.startswith("[FAIL]")]
    passed = [ln for ln in res.stdout.splitlines() if ln.startswith("[ ok ]")]
    assert passed, res.stdout + res.stderr
    assert set(failed) <= KNOWN_OFFLINE_FAILURES, res.stdout + res.stderr


STRUCT_CASES = [
    # (name, n, d, l_max, eta, points)
    ("c1", 4096, 2, 3, 1.0, "uniform0"),
    ("c2", 65536, 2, 5, 1.0, "uniform0"),
    ("c3", 262144, 3, 4, 1.0, "uniform0"),
    ("small3d", 2000, 3, 3, 1.0, "uniform"),
    ("default_eta", 1500, 3, 2, 0.0, "uniform"),
    ("d1", 700, 1, 4, 0.0, "uniform"),
    ("mixture", 3000, 3, 3, 1.0, "mixture"),
    ("grid_ties", 257, 2, 4, 2.0, "grid"),
]


def _points(ph, n, d, kind):
    if kind == "uniform0":
        return ph.generate_points(n, d, 0)
    if kind == "uniform":
        return ph.generate_points(n, d, 7)
    if kind == "mixture":
        return ph.generate_mixture_points(n, d, 16, 0.05, 3)
    g = np.linspace(0.0, 1.0, 17)
    rng = np.random.default_rng(1)
    return g[rng.integers(0, 17, (n, d))]


def _compare_structure(ph, pts, l_max, eta):
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=l_max, p_s=2, p_theta=2, eta=eta,
                      eps=1e-2, near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_structure(pts, cfg)
    R = pr.RefMatrix(pts, l_max, eta)
    assert np.array_equal(pm.perm(), R.perm())
    ints, _ = pm.nodes()
    rn = R.nodes()
    # product node ints: level, parent, first child, size, ...
    assert np.array_equal(ints[:, 3].astype(np.int64), rn["size"])
    near, far, key = pm.blocks()
    rnear, rfar, rkey = R.blocks()
    assert np.array_equal(near, rnear)
    assert np.array_equal(far, rfar)
    assert np.array_equal(key, rkey)
    inf, cnt = pm.info(), R.counts()
    for k in ("nodes", "n_near", "n_far", "n_classes", "c_sp"):
        assert inf[k] == cnt[k], k
    assert cnt["coverage"] == pts.shape[0] ** 2
    return pm, R, cnt


@pytest.mark.parametrize("name,n,d,l_max,eta,kind", STRUCT_CASES)
def test_structure_bitwise_vs_reference(ph, name, n, d, l_max, eta, kind):
    pts = _points(ph, n, d, kind)
    if kind.startswith("uniform"):  # the product's point stream is the reference's generate_points
        assert np.array_equal(pts, pr.generate_points(n, d, 0 if kind == "uniform0" else 7))
    _, R, cnt = _compare_structure(ph, pts, l_max, eta)
    expected = {  # SURVEY.md §8(d) structure table
        "c1": (1012, 1944, 112, 60),
        "c2": (20116, 68400, 280, 84),
        "c3": (383272, 2156952, 2526, 936),
    }
    if name in expected:
        assert (cnt["n_near"], cnt["n_far"], cnt["n_classes"], cnt["c_sp"]) == expected[name]


def test_c4_structure_vs_reference(ph):
    """BASELINE config 4: n = 2^20 mixture of 16 Gaussians, leaf 32 (l_max 5)."""
    pts = ph.generate_mixture_points(1 << 20, 3, 16, 0.05, 0)
    R = pr.RefMatrix(pts, 5, 1.0)
    cnt = R.counts()
    near, _, _ = R.blocks()
    sizes = R.nodes()["size"]
    sigma_d = int((sizes[near[:, 0]] * sizes[near[:, 1]]).sum())
    # SURVEY.md §8(d) estimated 0.92-0.99M near blocks, <= 3,676 classes,
    # c_sp 936, Sigma_D 3.2-3.5e10 and about 5.7M far blocks from a
    # throwaway mixture generator; the seeded generator here (harness-style
    # Rng stream) lands at Sigma_D = 2.89e10, counted here by
    # the reference itself.
    assert (cnt["n_near"], cnt["n_far"], cnt["n_classes"], cnt["c_sp"]) == (976918, 5315886, 3658, 936)
    assert sigma_d == 28915924608
    pm = ph.offline_structure(pts, ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=5, p_s=2,
                                               p_theta=2, eta=1.0, eps=1e-2, near_mode=ph.NearMode.SNAPSHOT))
    assert np.array_equal(pm.perm(), R.perm())
    pn, pf, pk = pm.blocks()
    rn, rf, rk = R.blocks()
    assert np.array_equal(pn, rn) and np.array_equal(pf, rf) and np.array_equal(pk, rk)


ONLINE_CASES = {
    "h2_e_3d": dict(n=1500, d=3, seed=5, fam="e", boxes=[(0.05, 0.5)], l_max=2, p_s=4, p_theta=8, fmt="h2",
                    near="snapshot", thetas=[[0.05], [0.173], [0.5]]),
    "h_gauss_2d_tt": dict(n=1024, d=2, seed=0, fam="gauss", boxes=[(0.1, 1.0)], l_max=2, p_s=6, p_theta=8,
                          fmt="h", near="tt", thetas=[[0.1], [0.3456]]),
    "h2_m32_2d": dict(n=2048, d=2, seed=1, fam="m32", boxes=[(0.05, 0.5)], l_max=3, p_s=6, p_theta=10, fmt="h2",
                      near="snapshot", thetas=[[0.077], [0.31]]),
    "h2_m52_amp_mix": dict(n=1200, d=3, seed=1, fam="m52", boxes=[(0.05, 0.5), (0.5, 2.0)], l_max=2, p_s=4,
                           p_theta=[8, 6], fmt="h2", near="snapshot", thetas=[[0.11, 0.7], [0.4, 1.9]],
                           amplitude=True, mixture=True),
}


def _product_case(ph, c):
    if c.get("mixture"):
        pts = ph.generate_mixture_points(c["n"], c["d"], 8, 0.05, c["seed"])
    else:
        pts = ph.generate_points(c["n"], c["d"], c["seed"])
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.from_id(c["fam"]), c["boxes"], amplitude=c.get("amplitude", False)),
                      l_max=c["l_max"], p_s=c["p_s"], p_theta=c["p_theta"], eta=1.0, seed=0,
                      near_mode=ph.NearMode.SNAPSHOT if c["near"] == "snapshot" else ph.NearMode.TT)
    fmt = ph.Format.H2 if c["fmt"] == "h2" else ph.Format.H
    return pts, cfg, fmt


@pytest.mark.parametrize("name", sorted(ONLINE_CASES))
def test_oracle_equals_reference_online(ph, po, name):
    """The restated oracle vs the reference itself on identical offline data."""
    c = ONLINE_CASES[name]
    pts, cfg, fmt = _product_case(ph, c)
    pm = ph.offline_structure(pts, cfg, fmt)
    R = pr.RefMatrix.from_product(pm, pts, near=c["near"])
    om = po.from_product(pm, pts)
    near, far, key = pm.blocks()
    sizes = pm.nodes()[0][:, 3]
    info = pm.info()
    X = np.stack([ph.generate_normal(pts.shape[0], 3 + j) for j in range(2)], axis=1)
    for th in c["thetas"]:
        ri, oi = R.instantiate(th), om.instantiate(th)
        for b in range(0, len(near), max(1, len(near) // 60)):
            shape = (int(sizes[near[b, 0]]), int(sizes[near[b, 1]]))
            assert rel(oi.near(b, shape), ri.near_d(b)) <= 1e-12
        for k in range(info["n_classes"]):
            assert rel(oi.class_h(k), R.class_h(k, th)) <= 1e-12
        if fmt == ph.Format.H2:
            for k in range(0, info["n_classes"], max(1, info["n_classes"] // 20)):
                assert rel(oi.class_c(k, info["P"]), R.class_c(k, th, info["P"])) <= 1e-12
        for i in range(0, len(far), max(1, len(far) // 40)):
            assert rel(ri.far_h(i), R.class_h(key[i], th)) == 0.0  # far_h copies the class H
        Y = ri.apply(X)
        Yo = np.stack([oi.apply(X[:, j]) for j in range(X.shape[1])], axis=1)
        assert rel(Yo, Y) <= 1e-12


def test_reference_apply_rows_equals_full_apply(ph):
    """rfd_apply_rows (the full-size probe used on the GPU) equals rows of the
    reference's own InstantiatedH2Matrix::apply."""
    c = ONLINE_CASES["h2_e_3d"]
    pts, cfg, fmt = _product_case(ph, c)
    pm = ph.offline_structure(pts, cfg, fmt)
    R = pr.RefMatrix.from_product(pm, pts, near="snapshot")
    x = ph.generate_normal(pts.shape[0], 9)
    rows = np.array([0, 17, 500, 999, 1499])
    for th in ([0.06], [0.33]):
        y = R.instantiate(th).apply(x)
        assert rel(R.apply_rows(th, x, rows), y[rows]) <= 1e-14
    Rn = pr.RefMatrix.from_product(pm, pts, near="none", finalize=False)  # snapshots on the fly
    assert rel(Rn.apply_rows([0.33], x, rows), y[rows]) <= 1e-14


def test_h_form_far_factors_vs_reference_pttk_offline(ph):
    """S_b, T_b of the product's host build = the reference's pttk_offline,
    at BASELINE config 1's structure (far blocks at internal levels too; the
    product's rows are in tree order, the reference's ascending)."""
    pts = ph.generate_points(4096, 2, 0)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.GAUSS, [(0.1, 1.0)]), l_max=3, p_s=6, p_theta=8, eta=1.0,
                      seed=0, near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_structure(pts, cfg, ph.Format.H)
    R = pr.RefMatrix.from_product(pm, pts, near="none", finalize=False)
    R.make_near_snapshots()
    R.finalize()
    _, far, _ = pm.blocks()
    rows = node_rows(pm)
    ints, _ = pm.nodes()
    levels = set()
    for i in range(0, len(far), 7):
        S, T = pm.far_st(i)
        Sr, Tr = R.far_st(i)
        S, T = S[np.argsort(rows(far[i, 0]))], T[np.argsort(rows(far[i, 1]))]
        assert rel(S, Sr) <= 1e-13 and rel(T, Tr) <= 1e-13
        levels.add(int(ints[far[i, 0], 0]))
    assert len(levels) >= 2


def test_reference_domain_error_and_grid(ph):
    """farfield.cpp:23-24: theta outside the box -> domain_error, through the
    compiled reference; grids equal the product's theta grids bitwise."""
    c = ONLINE_CASES["h2_e_3d"]
    pts, cfg, fmt = _product_case(ph, c)
    pm = ph.offline_structure(pts, cfg, fmt)
    R = pr.RefMatrix.from_product(pm, pts, near="snapshot")
    with pytest.raises(pr.RefDomainError):
        R.instantiate([0.6])
    nodes, _ = R.theta_grid(0)
    assert np.array_equal(nodes, pm.theta_grid(0))


@pytest.mark.parametrize("h2,near_tt", [(True, True), (False, True), (True, False)])
def test_reference_written_artifact_loads_into_product(ph, po, tmp_path, h2, near_tt):
    """the reference's own `phmat build --artifact` path
    (offline_h / offline_h2 with its TT-cross for couplings and near blocks,
    then save_parametric; tools/phmat.cpp:155-171) read by the product's
    loader (phm_matrix_load_host). The loaded structure is the reference's,
    and the oracle fed the loaded TT data reproduces the reference's own
    instantiate + apply of the same file (load_parametric_h/_h2)."""
    path = str(tmp_path / "ref.hmat")
    pr.build_save(path, 900, 2, 3, h2, pr.REF_SE, [(0.25, 1.0)], 2, 5, 6, eps=1e-6, eta=1.0, near_tt=near_tt)
    assert ph.artifact_is_h2(path) == h2
    R = pr.load(path)
    pm = ph.load_parametric_structure(path)
    pts = pr.generate_points(900, 2, 3)
    near, far, key = pm.blocks()
    rn, rf, rk = R.blocks()
    assert np.array_equal(near, rn) and np.array_equal(far, rf) and np.array_equal(key, rk)
    assert np.array_equal(pm.perm(), R.perm())
    if not near_tt:
        return  # Direct mode: the near field is evaluated online (checked on the GPU)
    om = po.from_product(pm, pts)
    x = pr.generate_normal(900, 4)
    for th in ([0.3], [0.77]):
        ri, oi = R.instantiate(th), om.instantiate(th)
        assert rel(oi.apply(x), ri.apply(x)) <= 1e-12
        sizes = pm.nodes()[0][:, 3]
        for b in range(0, len(near), 17):
            assert rel(oi.near(b, (int(sizes[near[b, 0]]), int(sizes[near[b, 1]]))), ri.near_d(b)) <= 1e-12
