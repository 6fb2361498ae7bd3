"""CPU: the product's host structure (paper_2511_03109_b200/csrc/host/core.cpp:
Morton-routing tree build + DFS block recursion) is bit-exact with the
oracle's transliteration of the reference (geometry.cpp:46-157,
phmatrix.cpp:29-41): permutation, node boxes and coordinates, near / far
lists in DFS order, translation classes in first-seen order, c_sp."""
import math

import numpy as np
import pytest

CASES = [
    # (n, d, l_max, eta, points)
    (4096, 2, 3, 1.0, "uniform"),       # BASELINE config 1 structure
    (2000, 3, 3, 1.0, "uniform"),
    (1500, 3, 2, 0.0, "uniform"),       # reference default eta = sqrt(d)
    (700, 1, 4, 0.0, "uniform"),
    (3000, 3, 3, 1.0, "mixture"),       # clustered, empty boxes, skewed leaves
    (257, 2, 4, 2.0, "grid"),           # points exactly on split midpoints
]


def make_points(ph, n, d, kind):
    if kind == "uniform":
        return ph.generate_points(n, d, 7)
    if kind == "mixture":
        return ph.generate_mixture_points(n, d, 16, 0.05, 3)
    g = np.linspace(0.0, 1.0, 17)  # dyadic coordinates incl. 0, 1 and all midpoints
    rng = np.random.default_rng(1)
    return g[rng.integers(0, 17, (n, d))]


@pytest.mark.parametrize("n,d,l_max,eta,kind", CASES)
def test_structure_bit_exact(ph, po, n, d, l_max, eta, kind):
    pts = make_points(ph, n, d, kind)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=l_max, p_s=2, p_theta=2, eta=eta,
                      eps=1e-2, near_mode=ph.NearMode.SNAPSHOT)
    pm = ph.offline_structure(pts, cfg)
    om = po.OracleMatrix(pts, l_max, eta if eta > 0 else math.sqrt(d), 2, ph.Family.E, [(0.05, 0.5)], 2)
    assert np.array_equal(pm.perm(), om.perm())
    pi, pb = pm.nodes()
    oi, ob = om.nodes()
    assert np.array_equal(pi, oi)
    assert np.array_equal(pb.view(np.uint64), ob.view(np.uint64))  # bitwise boxes
    for a, b in zip(pm.blocks(), om.blocks()):
        assert np.array_equal(a, b)
    assert np.array_equal(pm.class_keys(), om.class_keys())
    inf, cnt = pm.info(), om.counts()
    for k in ("nodes", "n_near", "n_far", "n_classes", "c_sp", "constructed"):
        assert inf[k] == cnt[k], k


def test_baseline_config_structure_counts(ph, po):
    """SURVEY.md §8(d) structure table for BASELINE configs 1 and 3."""
    pts = ph.generate_points(4096, 2, 0)
    om = po.OracleMatrix(pts, 3, 1.0, 6, ph.Family.GAUSS, [(0.1, 1.0)], 8, h2=False)
    c = om.counts()
    assert (c["n_near"], c["n_far"], c["n_classes"], c["c_sp"]) == (1012, 1944, 112, 60)
    pts = ph.generate_points(262144, 3, 0)
    om = po.OracleMatrix(pts, 4, 1.0, 4, ph.Family.E, [(0.05, 0.5)], 8)
    c = om.counts()
    assert (c["n_near"], c["n_far"], c["n_classes"], c["c_sp"]) == (383272, 2156952, 2526, 936)
    near, far, _ = om.blocks()
    ints, _ = om.nodes()
    sizes = ints[:, 3].astype(np.int64)
    assert (sizes[near[:, 0]] * sizes[near[:, 1]]).sum() == 1572470682  # Sigma_D at C3


def test_sorted_index_sets_and_partition(ph):
    """test_geometry.cpp:104-115: children partition the parent; within a
    node the original indices ascend (tree-order ranges of perm)."""
    pts = ph.generate_points(500, 3, 11)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=2, p_s=2, p_theta=2, eps=1e-2)
    pm = ph.offline_structure(pts, cfg)
    ints, _ = pm.nodes()
    perm = pm.perm()
    assert sorted(perm.tolist()) == list(range(500))
    begin = np.zeros(len(ints), dtype=np.int64)
    pos = 0
    for i in range(len(ints)):
        if ints[i, 2] < 0:
            begin[i] = pos
            pos += ints[i, 3]
    for i in range(len(ints) - 1, -1, -1):
        if ints[i, 2] >= 0:
            begin[i] = begin[ints[i, 2]]
            assert ints[i, 3] == ints[ints[i, 2]: ints[i, 2] + 8, 3].sum()
    for i in range(len(ints)):
        seg = perm[begin[i]: begin[i] + ints[i, 3]]
        if ints[i, 2] < 0:  # leaf: the reference's sorted index set, in order
            assert np.all(np.diff(seg) > 0)
        else:  # internal: same set; the tree order groups it by child
            assert len(np.unique(seg)) == len(seg)


def test_midpoint_tie_goes_lower(ph):
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=1, p_s=2, p_theta=2, eps=1e-2)
    pm = ph.offline_structure(np.array([[0.5], [0.75]]), cfg)
    ints, _ = pm.nodes()
    assert list(ints[1:3, 3]) == [1, 1]


def test_invalid_inputs_raise(ph):
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.05, 0.5)]), l_max=1, p_s=2, p_theta=2)
    with pytest.raises(ph.InvalidArgument):
        ph.offline_structure(np.array([[1.5, 0.5]]), cfg)
    bad = ph.PHConfig(spec=ph.KernelSpec(ph.Family.E, [(0.0, 0.5)]), l_max=1, p_s=2, p_theta=2)
    with pytest.raises(ph.InvalidArgument):
        ph.offline_structure(np.array([[0.5, 0.5]]), bad)
    mn = ph.PHConfig(spec=ph.KernelSpec(ph.Family.MN, [(0.25, 1.0), (0.25, 3.0)]), l_max=1, p_s=2, p_theta=2)
    with pytest.raises(ph.InvalidArgument):  # nu lower bound 1/2 (kernels.cpp:37-38)
        ph.offline_structure(np.array([[0.5, 0.5]]), mn)


def test_metrics_relations(ph, po):
    """test_phmatrix.cpp:218-254: nf_ratio, m_a, c_sp bound, storage_gb."""
    pts = ph.generate_points(512, 3, 31)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=4, p_theta=5, eps=1e-3, seed=1)
    mh = ph.metrics(ph.offline_structure(pts, cfg, ph.Format.H))
    pm2 = ph.offline_structure(pts, cfg, ph.Format.H2)
    mh2 = ph.metrics(pm2)
    near, far, key = pm2.blocks()
    ints, _ = pm2.nodes()
    s = ints[:, 3].astype(np.int64)
    assert mh["nf_ratio"] == pytest.approx((s[near[:, 0]] * s[near[:, 1]]).sum() / 512.0 ** 2)
    assert mh2["nf_ratio"] == mh["nf_ratio"]
    assert mh["m_a"] == mh2["m_a"] == len(set(key.tolist())) <= len(far)
    assert mh["c_sp"] <= 216 and mh["rank"] >= 1.0
    assert 0 < mh2["coupling_ratio"] < mh2["ff_ratio"]
    assert mh["storage_gb"] == pytest.approx(mh["storage_entries"] * 8.0 / 1e9)


@pytest.mark.parametrize("world", [4, 8])
def test_row_shards_balance_streamed_entries(ph, world):
    """Row shards are contiguous leaf ranges balanced by the near entries each
    rank streams: with symmetric snapshot storage a rank streams the pairs
    whose owner leaf it holds (owner of {a, b}, a < b: a when a + b is even,
    else b -- device.cu), each once. Every rank's share is within a few
    leaves' worth of the mean, and the ranges tile the rows."""
    pts = ph.generate_points(40000, 3, 2)
    spec = ph.KernelSpec(ph.Family.E, [(0.05, 0.5)])
    shares, ranges = [], []
    for r in range(world):
        cfg = ph.PHConfig(spec=spec, l_max=3, p_s=4, p_theta=8, eta=1.0, near_mode=ph.NearMode.SNAPSHOT,
                          shard_rank=r, shard_count=world)
        pm = ph.offline_structure(pts, cfg)
        info = pm.info()
        ints, _ = pm.nodes()
        near, _, _ = pm.blocks()
        lo, hi = info["row_begin"], info["row_end"]
        ranges.append((lo, hi))
        count = ints[:, 3]
        # leaves own contiguous row ranges in leaf-id order (perm)
        begin = np.full(len(ints), -1, dtype=np.int64)
        leaves = np.flatnonzero(ints[:, 2] < 0)
        begin[leaves] = np.concatenate([[0], np.cumsum(count[leaves])[:-1]])
        w = 0
        for s, t in near:
            if not (lo <= begin[s] < hi):
                continue
            if s != t and (s < t) != ((s + t) % 2 == 0):
                continue  # stored by the partner leaf
            w += int(count[s]) * int(count[t])
        shares.append(w)
    assert ranges[0][0] == 0 and ranges[-1][1] == 40000
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    mean = sum(shares) / world
    leaf_max = max(shares) / (512 // world)  # ~leaves per rank at l_max 3
    assert max(abs(s - mean) for s in shares) <= 2 * leaf_max, shares
