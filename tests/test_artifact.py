"""HMAT v1 artifacts (proj/src/serialize.cpp): the product's reader and
writer against an independent Python restatement of the byte format, plus
the reference's round-trip relations (test_phmatrix.cpp:289-323)."""
import os
import struct

import numpy as np
import pytest


def _make(ph, fmt):
    pts = ph.generate_points(300, 2, 5)
    cfg = ph.PHConfig(spec=ph.KernelSpec.default(ph.Family.SE), l_max=2, p_s=4, p_theta=5, eps=1e-4, seed=1,
                      near_mode=ph.NearMode.TT)
    return pts, cfg, ph.offline_structure(pts, cfg, fmt)


@pytest.mark.parametrize("fmt", [0, 1])
def test_round_trip_host(ph, tmp_path, fmt):
    """save -> load reproduces structure and every TT / S / T bitwise."""
    pts, cfg, pm = _make(ph, fmt)
    path = str(tmp_path / "a.phm")
    ph.save_parametric(pm, path)
    assert ph.artifact_is_h2(path) == (fmt == ph.Format.H2)
    lm = ph.load_parametric_structure(path)
    assert lm.format == fmt and lm.config.p_s == 4 and lm.config.l_max == 2
    assert np.array_equal(lm.perm(), pm.perm())
    for a, b in zip(lm.blocks(), pm.blocks()):
        assert np.array_equal(a, b)
    for k in range(pm.info()["n_classes"]):
        for a, b in zip(lm.coupling_cores(k), pm.coupling_cores(k)):
            assert np.array_equal(a, b)
    near, far, _ = pm.blocks()
    for b in range(len(near)):
        for a, c in zip(lm.near_tt_cores(b), pm.near_tt_cores(b)):
            assert np.array_equal(a, c)
    if fmt == ph.Format.H:
        for i in range(0, len(far), 7):
            for a, c in zip(lm.far_st(i), pm.far_st(i)):
                assert np.array_equal(a, c)
    else:
        for k in range(0, pm.info()["n_classes"], 5):
            for a, c in zip(lm.class_lr(k), pm.class_lr(k)):
                assert np.array_equal(a, c)


def test_reader_accepts_independently_written_bytes(ph, tmp_path):
    """A file produced by the Python restatement of serialize.cpp's writer is
    byte-identical to the product's writer output."""
    pts, cfg, pm = _make(ph, ph.Format.H2)
    ours = str(tmp_path / "ours.phm")
    ph.save_parametric(pm, ours)
    near, far, key = pm.blocks()
    cpl = [pm.coupling_cores(k) for k in range(pm.info()["n_classes"])]
    path = str(tmp_path / "py.phm")
    with open(path, "wb") as f:
        w = lambda fmt, *v: f.write(struct.pack("<" + fmt, *v))
        w("II", 0x54414D48, 1)
        w("B", 1)
        w("B", ph.Family.SE)
        w("i", 1)
        w("dd", 0.25, 1.0)
        w("iii", 2, 4, 5)
        w("dd", 1e-4, 0.0)
        w("qq", 120, 150)
        w("Q", 1)
        w("BB", 0, 1)
        w("i", 2)
        w("q", 300)
        w("dd", 0.0, 1.0)
        w("dd", 0.0, 1.0)
        f.write(np.asfortranarray(pts).tobytes(order="F"))
        for blocks in (far, near):
            w("q", len(blocks))
            for s, t in blocks:
                w("ii", int(s), int(t))
        w("q", len(key))
        for k in key:
            w("i", int(k))
        w("q", len(cpl))

        def tt(cores):
            w("B", len(cores))
            for c in cores:
                w("qqq", *c.shape)
                f.write(np.asarray(c, dtype=np.float64).tobytes(order="F"))

        for cores in cpl:
            w("ii", 2, 1)
            w("B", 0)
            w("d", 0.0)
            w("Q", 0)
            tt(cores)
        ints, _ = pm.nodes()
        w("q", len(near))
        for b, (s, t) in enumerate(near):
            w("qq", int(ints[s, 3]), int(ints[t, 3]))
            w("B", 0)
            w("d", 0.0)
            w("Q", 0)
            tt(pm.near_tt_cores(b))
    # coupling metadata (rank_capped / est / evals) differs; compare the rest
    lm = ph.load_parametric_structure(path)
    assert np.array_equal(lm.perm(), pm.perm())
    for k in range(len(cpl)):
        for a, b in zip(lm.coupling_cores(k), cpl[k]):
            assert np.array_equal(a, b)
    a, b = open(path, "rb").read(), open(ours, "rb").read()
    assert len(a) == len(b)


def test_reader_rejects_bad_files(ph, tmp_path):
    pts, cfg, pm = _make(ph, ph.Format.H2)
    path = str(tmp_path / "a.phm")
    ph.save_parametric(pm, path)
    raw = open(path, "rb").read()
    bad = str(tmp_path / "bad.phm")
    open(bad, "wb").write(b"XXXX" + raw[4:])
    with pytest.raises(ph.PhmatError):
        ph.load_parametric_structure(bad)
    open(bad, "wb").write(raw[: len(raw) // 2])
    with pytest.raises(ph.PhmatError):
        ph.load_parametric_structure(bad)
    # topology check: perturb one point so the rebuilt tree differs
    n_off = 4 + 4 + 1 + 1 + 4 + 16 + 12 + 16 + 16 + 8 + 2 + 4 + 8 + 32
    arr = bytearray(raw)
    pts2 = np.frombuffer(bytes(arr[n_off: n_off + 8 * 600]), dtype=np.float64).copy()
    pts2[:] = 1.0 - pts2  # mirrored points -> different leaf populations
    arr[n_off: n_off + 8 * 600] = pts2.tobytes()
    open(bad, "wb").write(bytes(arr))
    with pytest.raises(ph.PhmatError):
        ph.load_parametric_structure(bad)


def test_extensions_are_not_written_as_v1(ph, tmp_path):
    pts = ph.generate_points(200, 2, 1)
    cfg = ph.PHConfig(spec=ph.KernelSpec(ph.Family.MATERN32, [(0.05, 0.5)]), l_max=1, p_s=3, p_theta=4,
                      near_mode=ph.NearMode.TT)
    pm = ph.offline_structure(pts, cfg, ph.Format.H2)
    with pytest.raises(ph.InvalidArgument):
        ph.save_parametric(pm, str(tmp_path / "x.phm"))
