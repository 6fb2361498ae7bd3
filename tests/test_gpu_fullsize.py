"""BASELINE config 3 at full size (n = 2^18, 3D, H^2, snapshot near field)
through size-independent properties (the oracle is too slow at this size):
accuracy against exact kernel rows (the reference harness's
estimate_error), linearity, fused == separate instantiate+apply, theta-batched
== single instantiate, block RHS == column loop, and determinism."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3(ph):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    c = bench.CONFIGS["c3"]
    pts = bench.make_points(ph, c, 0)
    pm = ph.offline_h2(pts, bench.make_cfg(ph, c))
    return pm, c


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _rows_oracle(ph, pm, c, pts, theta, x, rows):
    """The oracle's y at `rows`, exactly: it instantiates and applies only the
    near blocks whose sigma is a leaf holding a probe row and the far blocks
    whose sigma is such a leaf or one of its ancestors (every block that
    reaches those rows), plus the full basis passes."""
    from oracle import pyoracle as po

    po.lib().orc_set_threads(os.cpu_count() or 1)
    om = po.OracleMatrix(pts, c["l_max"], c["eta"], c["p_s"], ph.Family.from_id(c["family"]), [c["box"]],
                         c["p_theta"], h2=True)
    cnt = om.counts()
    for k in range(cnt["n_classes"]):
        om.set_coupling(k, pm.coupling_cores(k))
    ints, _ = pm.nodes()
    starts = np.zeros(len(ints), dtype=np.int64)
    nch = 2 ** c["d"]
    for i in range(len(ints)):
        if ints[i, 2] >= 0:
            off = starts[i]
            for ch in range(ints[i, 2], ints[i, 2] + nch):
                starts[ch] = off
                off += ints[ch, 3]
    pos = np.empty(c["n"], dtype=np.int64)
    pos[pm.perm()] = np.arange(c["n"])
    leaves = np.where(ints[:, 2] < 0)[0]
    lstart = starts[leaves]
    order = np.argsort(lstart)
    keep = set()
    for r in rows:
        li = leaves[order[np.searchsorted(lstart[order], pos[r], side="right") - 1]]
        node = li
        while node >= 0:
            keep.add(int(node))
            node = int(ints[node, 1])
    near, far, _ = pm.blocks()
    near_mask = np.array([s in keep for s, _ in near], dtype=np.uint8)
    far_mask = np.array([s in keep for s, _ in far], dtype=np.uint8)
    om.make_near_snapshots(near_mask)
    om.finalize()
    oi, _ = om.instantiate_timed(theta, near_mask)
    y, _ = oi.apply_sample(x, near_mask, far_mask)
    return y[rows]


def test_c3_full_size_parity_on_probe_rows(ph, c3):
    """Rows of the full-size GPU MVM (plain apply and the fused
    instantiate+apply step) against the oracle's exact rows."""
    pm, c = c3
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    pts = bench.make_points(ph, c, 0)
    n = c["n"]
    x = ph.generate_normal(n, 1)
    rows = np.random.default_rng(11).choice(n, 24, replace=False)
    theta = [0.17]
    want = _rows_oracle(ph, pm, c, pts, theta, x, rows)
    inst = ph.instantiate(pm, theta)
    assert rel(inst.apply(x)[rows], want) <= 1e-11
    assert rel(inst.instantiate_apply(theta, x)[rows], want) <= 1e-11


def test_c3_accuracy_against_exact_rows(ph, c3):
    """The harness's estimate_error at the config (p_s = 4 is a coarse far
    field: the error grows as l shrinks toward the box edge)."""
    pm, c = c3
    errs = [ph.instantiate(pm, th).estimate_error(probe_rows=200, seed=1) for th in ([0.05], [0.17], [0.5])]
    assert all(np.isfinite(e) for e in errs)
    assert errs[2] <= errs[1] <= errs[0] <= 0.05, errs


def test_c3_linearity_determinism_and_fused_path(ph, c3):
    pm, c = c3
    n = c["n"]
    rng = np.random.default_rng(3)
    x, z = rng.standard_normal(n), rng.standard_normal(n)
    inst = ph.instantiate(pm, [0.23])
    y = inst.apply(x)
    assert np.array_equal(y, inst.apply(x))
    assert rel(inst.apply(2 * x - 3 * z), 2 * y - 3 * inst.apply(z)) <= 1e-13
    # the benchmarked step (fused near pass) against instantiate + apply
    y_fused = inst.instantiate_apply([0.31], x)
    ref = ph.instantiate(pm, [0.31])
    assert rel(y_fused, ref.apply(x)) <= 1e-14
    near, _, _ = pm.blocks()
    ints, _ = pm.nodes()
    for k in range(0, len(near), 9973):
        sh = (int(ints[near[k][0], 3]), int(ints[near[k][1], 3]))
        assert np.array_equal(inst.near_d(k, sh), ref.near_d(k, sh))


def test_c3_theta_batch_and_block_rhs(ph, c3):
    pm, c = c3
    n = c["n"]
    thetas = [[0.07], [0.2], [0.33], [0.46]]
    batch = ph.instantiate_batch(pm, thetas)
    near, _, _ = pm.blocks()
    ints, _ = pm.nodes()
    rng = np.random.default_rng(5)
    X = rng.standard_normal((n, 10))
    for b, th in enumerate(thetas):
        single = ph.instantiate(pm, th)
        for k in range(b, len(near), 19997):
            sh = (int(ints[near[k][0], 3]), int(ints[near[k][1], 3]))
            assert np.array_equal(batch[b].near_d(k, sh), single.near_d(k, sh))
        if b == 0:
            Y = single.apply(X)
            for col in (0, 9):
                assert rel(Y[:, col], single.apply(X[:, col])) <= 1e-14
