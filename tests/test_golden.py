"""Committed golden vectors (tests/golden/*.npz, made by
tests/golden/make_golden.py from the COMPILED REFERENCE, oracle/_ref).

CPU: the reference build reproduces every vector bit for bit, and the oracle
(the restatement) within 1e-13 (any drift of either checker, or of the host
offline build feeding them, fails here).
GPU: the CUDA path (through the C ABI) matches the vectors at the
north_star's tolerances, with no checker in the loop."""
import importlib.util
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
TOL_BLOCK = 1e-12
TOL_Y = 1e-11


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _mg():
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "golden", "make_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


NAMES = ["h2_snapshot_3d_e", "h_tt_2d_gauss", "h2_snapshot_3d_m52_amplitude"]


def _load(name):
    return dict(np.load(os.path.join(HERE, "golden", name + ".npz")))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(ph, po, name):
    mg = _mg()
    pts, cfg, fmt, thetas, m = mg.cases(ph)[name]
    g = _load(name)
    assert np.array_equal(pts, g["points"])  # the reference's point stream
    pm = ph.offline_structure(pts, cfg, fmt)
    om = po.from_product(pm, pts)
    sizes = pm.nodes()[0][:, 3]
    near, _, _ = pm.blocks()
    for i, th in enumerate(thetas):
        oi = om.instantiate(th)
        y = np.stack([oi.apply(g["x"][:, j]) for j in range(m)], axis=1)
        assert rel(y, g[f"y{i}"]) <= 1e-13
        for b in g["near_ids"]:
            s, t = near[b]
            assert rel(oi.near(int(b), (int(sizes[s]), int(sizes[t]))), g[f"d{i}_{b}"]) <= 1e-13
        for k in g["class_ids"]:
            assert rel(oi.class_h(int(k)), g[f"h{i}_{k}"]) <= 1e-13


@pytest.mark.parametrize("name", NAMES)
def test_reference_reproduces_golden(ph, name):
    from oracle import pyref as pr

    mg = _mg()
    pts, cfg, fmt, thetas, m = mg.cases(ph)[name]
    g = _load(name)
    pm = ph.offline_structure(pts, cfg, fmt)
    R = pr.RefMatrix.from_product(pm, pts, near="tt" if cfg.near_mode == ph.NearMode.TT else "snapshot")
    for i, th in enumerate(thetas):
        ri = R.instantiate(th)
        assert np.array_equal(ri.apply(g["x"]), g[f"y{i}"])
        for b in g["near_ids"]:
            assert np.array_equal(ri.near_d(int(b)), g[f"d{i}_{b}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_cuda_path_matches_golden(ph, name):
    mg = _mg()
    pts, cfg, fmt, thetas, m = mg.cases(ph)[name]
    g = _load(name)
    pm = ph.offline_h2(pts, cfg) if fmt == ph.Format.H2 else ph.offline_h(pts, cfg)
    sizes = pm.nodes()[0][:, 3]
    near, far, key = pm.blocks()
    far_of_class = {}
    for i, k in enumerate(key):
        far_of_class.setdefault(int(k), i)
    inst = ph.instantiate(pm, thetas[0])
    for i, th in enumerate(thetas):
        inst.reinstantiate(th)
        for b in g["near_ids"]:
            s, t = near[b]
            assert rel(inst.near_d(int(b), (int(sizes[s]), int(sizes[t]))), g[f"d{i}_{b}"]) <= TOL_BLOCK
        for k in g["class_ids"]:
            if int(k) in far_of_class:
                assert rel(inst.far_h(far_of_class[int(k)]), g[f"h{i}_{k}"]) <= TOL_BLOCK
            if fmt == ph.Format.H2:
                assert rel(inst.class_c(int(k)), g[f"c{i}_{k}"]) <= TOL_BLOCK
        assert rel(inst.apply(g["x"]), g[f"y{i}"]) <= TOL_Y
        # the benchmarked fused step on the same vectors
        assert rel(inst.instantiate_apply(th, g["x"]), g[f"y{i}"]) <= TOL_Y
