"""CPU: the product's offline TT machinery (host C++ restatement of
proj/src/tt.cpp and aca_impl.hpp) against the reference's relations in
proj/tests/test_tt.cpp (inputs drawn from the reference's own Rng stream)."""
import numpy as np
import pytest


def rng_uniform(seed, count, a=0.0, b=1.0):
    from oracle.pyoracle import lib, _DP

    u = np.empty(count)
    lib().orc_rng_uniform(seed, count, u.ctypes.data_as(_DP))
    return a + (b - a) * u


def random_tt(modes, ranks, seed):
    """test_tt.cpp:11-22: cores filled from Rng(seed).uniform(-1, 1) in core order."""
    total = sum(ranks[k] * modes[k] * ranks[k + 1] for k in range(len(modes)))
    vals = rng_uniform(seed, total, -1.0, 1.0)
    cores, off = [], 0
    for k in range(len(modes)):
        sz = ranks[k] * modes[k] * ranks[k + 1]
        cores.append(vals[off: off + sz].reshape((ranks[k], modes[k], ranks[k + 1]), order="F"))
        off += sz
    return cores


def test_separable_rank_one(ph):
    """test_tt.cpp:154-178."""
    v = rng_uniform(6, 21)
    a, b, c = 0.2 + v[:6], 0.2 + v[6:13], 0.2 + v[13:]
    full = np.einsum("i,j,k->ijk", a, b, c)
    cores, info = ph.tt_cross(full, eps=1e-12, seed=99)
    assert max(max(cc.shape[0], cc.shape[2]) for cc in cores) == 1
    assert not info["rank_capped"]
    assert np.max(np.abs(ph.tt_full(cores) - full)) <= 1e-13


@pytest.mark.parametrize("t", range(5))
def test_round_trip_random_tt(ph, t):
    """test_tt.cpp:180-207: recovered ranks <= true + 1, max error <= 10 eps."""
    modes = [[5, 6, 7], [12, 9, 4, 6], [4, 4, 4, 4, 4], [3, 5, 3, 5, 3, 5], [2, 3, 4, 3, 2, 3, 2]][t]
    ranks = [[1, 3, 2, 1], [1, 4, 5, 3, 1], [1, 2, 4, 3, 2, 1], [1, 3, 3, 3, 3, 2, 1], [1, 2, 2, 5, 2, 2, 2, 1]][t]
    full = ph.tt_full(random_tt(modes, ranks, 100 + t))
    cores, info = ph.tt_cross(full, eps=1e-10, seed=1234 + t)
    got = [1] + [c.shape[2] for c in cores]
    assert all(g <= r + 1 for g, r in zip(got, ranks)), (got, ranks)
    assert np.max(np.abs(ph.tt_full(cores) - full)) <= 10 * 1e-10 * np.max(np.abs(full))


def test_eval_budget(ph):
    """test_tt.cpp:209-233: fresh evaluations within 4x of the cross budget."""
    g = np.arange(10) / 9.0
    x, y, z, w = np.meshgrid(g, g, g, g, indexing="ij")
    full = np.exp(-(x * x + 0.5 * x * y + y * z + 0.3 * z * w))
    cores, info = ph.tt_cross(full, eps=1e-8, seed=7)
    assert info["est_rel_error"] <= 1e-7
    r = max(c.shape[2] for c in cores)
    budget = r * (10 + 10) + r * r * (10 + 10)
    assert info["evals"] <= 4 * budget


def test_stopping_metadata(ph):
    """test_tt.cpp:235-248."""
    full = ph.tt_full(random_tt([8, 8, 8], [1, 4, 4, 1], 55))
    _, info = ph.tt_cross(full, eps=1e-9, seed=2)
    assert info["converged"] and info["est_rel_error"] <= 1e-8


def test_rank_cap_flag(ph):
    """test_tt.cpp:250-264."""
    dense = rng_uniform(31, 400, -1, 1).reshape(20, 20)  # row-major fill like the reference
    cores, info = ph.tt_cross(dense, eps=1e-12, r_max=5, seed=3)
    assert info["rank_capped"] and not info["converged"]
    assert cores[0].shape[2] <= 5


def test_one_mode_copies_vector(ph):
    """test_tt.cpp:266-275."""
    v = np.sin(0.3 * np.arange(9))
    cores, info = ph.tt_cross(v)
    assert len(cores) == 1 and np.array_equal(cores[0].ravel(), v) and info["evals"] == 9


def test_rounding_pad_then_round(ph):
    """test_tt.cpp:277-301."""
    v = rng_uniform(8, 18, -1, 1)
    a, b, c = v[:5], v[5:11], v[11:]
    c0 = np.zeros((1, 5, 3)); c0[0, :, 0] = a
    c1 = np.zeros((3, 6, 3)); c1[0, :, 0] = b
    c2 = np.zeros((3, 7, 1)); c2[0, :, 0] = c
    before = ph.tt_full([c0, c1, c2])
    rounded = ph.tt_round([c0, c1, c2], eps=1e-13)
    assert rounded[0].shape[2] == 1 and rounded[1].shape[2] == 1
    assert np.max(np.abs(ph.tt_full(rounded) - before)) <= 1e-12 * max(1.0, np.max(np.abs(before)))


def test_rounding_bound_and_idempotence(ph):
    """test_tt.cpp:303-317."""
    tt = random_tt([6, 7, 6, 5], [1, 4, 6, 3, 1], 77)
    full = ph.tt_full(tt)
    for eps in (1e-2, 1e-6):
        r1 = ph.tt_round(tt, eps=eps)
        approx = ph.tt_full(r1)
        assert np.linalg.norm(approx - full) <= eps * np.linalg.norm(full) * 1.0000001
        assert all(r1[k].shape[0] <= tt[k].shape[0] for k in range(4))
        r2 = ph.tt_round(r1, eps=eps)
        assert [c.shape for c in r2] == [c.shape for c in r1]
        assert np.max(np.abs(ph.tt_full(r2) - approx)) <= 1e-14 * max(1.0, np.max(np.abs(approx)))


def test_zero_tensor(ph):
    """test_tt.cpp:334-342."""
    cores, _ = ph.tt_cross(np.zeros((5, 5, 5)), eps=1e-10)
    assert max(max(c.shape[0], c.shape[2]) for c in cores) == 1
    assert np.max(np.abs(ph.tt_full(cores))) == 0.0


def test_tt_svd_fallback_accuracy_on_coupling_tensors(ph, po):
    """Offline far field: every class's TT reproduces the coupling tensor to
    within eps of its max entry (the robustness fallback guarantees this
    even where the reference's cross stalls)."""
    pts = ph.generate_points(512, 3, 42)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=6, p_theta=8, eps=1e-4, seed=1)
    pm = ph.offline_structure(pts, cfg, ph.Format.H2)
    om = po.OracleMatrix(pts, 2, np.sqrt(3), 6, ph.Family.SE, [(0.25, 1.0)], 8)
    _, far, key = pm.blocks()
    first = {}
    for i, k in enumerate(key):
        first.setdefault(int(k), i)
    rng = np.random.default_rng(0)
    for k in list(first)[::17]:
        F = ph.tt_full(pm.coupling_cores(k))
        errs, mx = 0.0, 0.0
        for _ in range(200):
            idx = [int(rng.integers(0, m)) for m in F.shape]
            e = om.coupling_entry(first[k], idx)
            errs = max(errs, abs(F[tuple(idx)] - e))
            mx = max(mx, abs(e))
        assert errs <= 2 * cfg.eps * mx, (k, errs, mx)
