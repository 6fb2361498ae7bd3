"""ctypes wrapper of the CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs; never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

_DP = C.POINTER(C.c_double)
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_U8P = C.POINTER(C.c_uint8)
_P = C.c_void_p

_SIG = {
    "orc_last_error": ([], C.c_char_p),
    "orc_set_threads": ([C.c_int], None),
    "orc_generate_points": ([C.c_int64, C.c_int, C.c_uint64, _DP], None),
    "orc_mix_seed": ([C.c_uint64, C.c_uint64], C.c_uint64),
    "orc_rng_uniform": ([C.c_uint64, C.c_int64, _DP], None),
    "orc_kernel_value": ([C.c_int, C.c_int, C.c_double, _DP], C.c_double),
    "orc_cheb_grid": ([C.c_double, C.c_double, C.c_int, _DP, _DP, _DP], None),
    "orc_lagrange_all": ([C.c_double, C.c_double, C.c_int, C.c_double, _DP], C.c_int),
    "orc_box_admissible": ([C.c_int, _DP, _DP, _DP, _DP, C.c_double, _DP, _DP], C.c_int),
    "orc_fast_kron": ([C.c_int, C.c_int, _DP, _DP, C.c_int, _DP], None),
    "orc_matrix_create": ([_DP, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _DP,
                           _DP, _I32P, C.c_int, C.POINTER(_P)], C.c_int),
    "orc_matrix_destroy": ([_P], None),
    "orc_matrix_counts": ([_P, _I64P], None),
    "orc_matrix_nodes": ([_P, _I32P, _DP], None),
    "orc_matrix_perm": ([_P, _I32P], None),
    "orc_matrix_blocks": ([_P, _I32P, _I32P, _I32P], None),
    "orc_matrix_class_keys": ([_P, _I64P], None),
    "orc_matrix_theta_grid": ([_P, C.c_int, _DP], None),
    "orc_set_coupling": ([_P, C.c_int, C.c_int, _I64P, _DP], C.c_int),
    "orc_set_near_tt": ([_P, C.c_int64, C.c_int, _I64P, _DP], C.c_int),
    "orc_make_near_snapshots": ([_P, _U8P], C.c_int),
    "orc_near_snapshot_column": ([_P, C.c_int64, C.c_int64, _DP], C.c_int),
    "orc_finalize": ([_P], C.c_int),
    "orc_far_st": ([_P, C.c_int64, _DP, _DP], C.c_int),
    "orc_class_LR": ([_P, C.c_int, _DP, _DP, _I64P], C.c_int),
    "orc_instantiate": ([_P, _DP, C.POINTER(_P)], C.c_int),
    "orc_instantiate_timed": ([_P, _DP, _U8P, _DP, C.POINTER(_P)], C.c_int),
    "orc_inst_destroy": ([_P], None),
    "orc_inst_class_h": ([_P, C.c_int, _DP, _I64P], C.c_int),
    "orc_inst_near": ([_P, C.c_int64, _DP], C.c_int),
    "orc_inst_class_c": ([_P, C.c_int, _DP], C.c_int),
    "orc_apply": ([_P, _DP, _DP, C.c_int64], C.c_int),
    "orc_apply_sample": ([_P, _DP, _DP, _U8P, _U8P, _DP], C.c_int),
    "orc_to_dense": ([_P, _DP, C.c_int64], C.c_int),
    "orc_dense_kernel": ([_DP, C.c_int64, C.c_int, C.c_int, C.c_int, _DP, _DP], None),
    "orc_coupling_entry": ([_P, C.c_int64, _I64P, _DP], C.c_int),
}

_lib = None


class OracleError(RuntimeError):
    pass


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        for k, (a, r) in _SIG.items():
            f = getattr(L, k)
            f.argtypes = a
            f.restype = r
        _lib = L
    return _lib


_EXC = {2: ValueError, 3: ValueError, 4: RuntimeError, 1: RuntimeError}


def _ck(code):
    if code:
        raise _EXC.get(code, OracleError)(lib().orc_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(_DP)


def generate_points(n, d, seed):
    out = np.empty((n, d))
    lib().orc_generate_points(n, d, seed, _dp(out))
    return out


def kernel_value(fam, r, theta, amp=False):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    return lib().orc_kernel_value(fam, 1 if amp else 0, r, _dp(th))


def cheb_grid(lo, hi, p):
    x, w, lh = np.empty(p), np.empty(p), np.empty(2)
    lib().orc_cheb_grid(lo, hi, p, _dp(x), _dp(w), _dp(lh))
    return x, w, lh


def lagrange_all(lo, hi, p, x):
    out = np.empty(p)
    _ck(lib().orc_lagrange_all(lo, hi, p, x, _dp(out)))
    return out


def box_admissible(alo, ahi, blo, bhi, eta):
    a0, a1, b0, b1 = (np.ascontiguousarray(v, dtype=np.float64) for v in (alo, ahi, blo, bhi))
    diam, dist = C.c_double(), C.c_double()
    adm = lib().orc_box_admissible(len(a0), _dp(a0), _dp(a1), _dp(b0), _dp(b1), eta, C.byref(diam), C.byref(dist))
    return bool(adm), diam.value, dist.value


def fast_kron(factors, x, transposed=False):
    f = np.ascontiguousarray(np.stack(factors), dtype=np.float64)  # d x p x p, row-major entries
    d, p, _ = f.shape
    xv = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(p ** d)
    lib().orc_fast_kron(d, p, _dp(f), _dp(xv), 1 if transposed else 0, _dp(out))
    return out


def dense_kernel(points, fam, theta, amp=False):
    p = np.ascontiguousarray(points, dtype=np.float64)
    n, d = p.shape
    th = np.ascontiguousarray(theta, dtype=np.float64)
    out = np.empty((n, n), order="F")
    lib().orc_dense_kernel(_dp(p), n, d, fam, 1 if amp else 0, _dp(th), out.ctypes.data_as(_DP))
    return out


class OracleMatrix:
    """Reference-order CPU restatement of a parametric H / H^2 matrix."""

    def __init__(self, points, l_max, eta, p_s, family, theta_box, p_theta, h2=True, amplitude=False):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        self.n, self.d = pts.shape
        lo = np.array([b[0] for b in theta_box], dtype=np.float64)
        hi = np.array([b[1] for b in theta_box], dtype=np.float64)
        pt = [p_theta] * len(theta_box) if isinstance(p_theta, int) else list(p_theta)
        pt = np.array(pt, dtype=np.int32)
        self.p_theta = pt
        self.h2 = h2
        h = _P()
        _ck(lib().orc_matrix_create(_dp(pts), self.n, self.d, l_max, eta, p_s, family, 1 if amplitude else 0,
                                    len(theta_box), _dp(lo), _dp(hi), pt.ctypes.data_as(_I32P), 1 if h2 else 0,
                                    C.byref(h)))
        self._h = h
        self._keep = []

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_matrix_destroy(self._h)
            self._h = None

    def counts(self):
        c = np.empty(8, dtype=np.int64)
        lib().orc_matrix_counts(self._h, c.ctypes.data_as(_I64P))
        keys = ("n", "d", "nodes", "n_near", "n_far", "n_classes", "c_sp", "constructed")
        return dict(zip(keys, (int(v) for v in c)))

    def nodes(self):
        nn = self.counts()["nodes"]
        ints = np.empty((nn, 7), dtype=np.int32)
        boxes = np.empty((nn, 6))
        lib().orc_matrix_nodes(self._h, ints.ctypes.data_as(_I32P), _dp(boxes))
        return ints, boxes

    def perm(self):
        out = np.empty(self.n, dtype=np.int32)
        lib().orc_matrix_perm(self._h, out.ctypes.data_as(_I32P))
        return out

    def blocks(self):
        c = self.counts()
        near = np.empty((c["n_near"], 2), dtype=np.int32)
        far = np.empty((c["n_far"], 2), dtype=np.int32)
        key = np.empty(c["n_far"], dtype=np.int32)
        lib().orc_matrix_blocks(self._h, near.ctypes.data_as(_I32P), far.ctypes.data_as(_I32P),
                                key.ctypes.data_as(_I32P))
        return near, far, key

    def class_keys(self):
        k = self.counts()["n_classes"]
        out = np.empty((k, 4), dtype=np.int64)
        lib().orc_matrix_class_keys(self._h, out.ctypes.data_as(_I64P))
        return out

    def theta_grid(self, k):
        out = np.empty(int(self.p_theta[k]))
        lib().orc_matrix_theta_grid(self._h, k, _dp(out))
        return out

    @staticmethod
    def _pack(cores):
        dims = np.array([c.shape for c in cores], dtype=np.int64).ravel()
        data = np.concatenate([np.asfortranarray(c).ravel(order="F") for c in cores]).astype(np.float64)
        return dims, np.ascontiguousarray(data)

    def set_coupling(self, k, cores):
        dims, data = self._pack(cores)
        _ck(lib().orc_set_coupling(self._h, k, len(cores), dims.ctypes.data_as(_I64P), _dp(data)))

    def set_near_tt(self, b, cores):
        dims, data = self._pack(cores)
        _ck(lib().orc_set_near_tt(self._h, b, len(cores), dims.ctypes.data_as(_I64P), _dp(data)))

    def make_near_snapshots(self, mask=None):
        m = None
        if mask is not None:
            mk = np.ascontiguousarray(mask, dtype=np.uint8)
            self._keep.append(mk)
            m = mk.ctypes.data_as(_U8P)
        _ck(lib().orc_make_near_snapshots(self._h, m))

    def near_snapshot_column(self, b, kap, size):
        out = np.empty(size)
        _ck(lib().orc_near_snapshot_column(self._h, b, kap, _dp(out)))
        return out

    def finalize(self):
        _ck(lib().orc_finalize(self._h))

    def far_st(self, i, shape_s, shape_t):
        S = np.empty(shape_s, order="F")
        T = np.empty(shape_t, order="F")
        _ck(lib().orc_far_st(self._h, i, S.ctypes.data_as(_DP), T.ctypes.data_as(_DP)))
        return S, T

    def class_lr(self, k):
        dims = np.empty(4, dtype=np.int64)
        _ck(lib().orc_class_LR(self._h, k, None, None, dims.ctypes.data_as(_I64P)))
        L = np.empty((dims[0], dims[1]), order="F")
        R = np.empty((dims[2], dims[3]), order="F")
        _ck(lib().orc_class_LR(self._h, k, L.ctypes.data_as(_DP), R.ctypes.data_as(_DP), dims.ctypes.data_as(_I64P)))
        return L, R

    def coupling_entry(self, far_index, idx):
        i = np.ascontiguousarray(idx, dtype=np.int64)
        out = C.c_double()
        _ck(lib().orc_coupling_entry(self._h, far_index, i.ctypes.data_as(_I64P), C.byref(out)))
        return out.value

    def instantiate(self, theta):
        th = np.ascontiguousarray(theta, dtype=np.float64).ravel()
        h = _P()
        _ck(lib().orc_instantiate(self._h, _dp(th), C.byref(h)))
        return OracleInstance(self, h)

    def instantiate_timed(self, theta, mask=None):
        th = np.ascontiguousarray(theta, dtype=np.float64).ravel()
        secs = np.zeros(2)
        h = _P()
        mk = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        _ck(lib().orc_instantiate_timed(self._h, _dp(th), None if mk is None else mk.ctypes.data_as(_U8P), _dp(secs),
                                        C.byref(h)))
        return OracleInstance(self, h), secs


class OracleInstance:
    def __init__(self, m, h):
        self.m = m
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_inst_destroy(self._h)
            self._h = None

    def class_h(self, k):
        rc = np.empty(2, dtype=np.int64)
        _ck(lib().orc_inst_class_h(self._h, k, None, rc.ctypes.data_as(_I64P)))
        out = np.empty((rc[0], rc[1]), order="F")
        _ck(lib().orc_inst_class_h(self._h, k, out.ctypes.data_as(_DP), rc.ctypes.data_as(_I64P)))
        return out

    def near(self, b, shape):
        out = np.empty(shape[0] * shape[1])
        _ck(lib().orc_inst_near(self._h, b, _dp(out)))
        return out.reshape(shape, order="F")

    def class_c(self, k, P):
        out = np.empty(P * P)
        _ck(lib().orc_inst_class_c(self._h, k, _dp(out)))
        return out.reshape((P, P), order="F")

    def apply(self, x):
        xa = np.asarray(x, dtype=np.float64)
        vec = xa.ndim == 1
        m = 1 if vec else xa.shape[1]
        xf = np.asfortranarray(xa.reshape(self.m.n, m))
        y = np.empty((self.m.n, m), order="F")
        _ck(lib().orc_apply(self._h, xf.ctypes.data_as(_DP), y.ctypes.data_as(_DP), m))
        return y[:, 0].copy() if vec else y

    def apply_sample(self, x, near_mask=None, far_mask=None):
        xv = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.m.n)
        secs = np.zeros(3)
        nm = None if near_mask is None else np.ascontiguousarray(near_mask, dtype=np.uint8)
        fm = None if far_mask is None else np.ascontiguousarray(far_mask, dtype=np.uint8)
        _ck(lib().orc_apply_sample(self._h, _dp(xv), _dp(y), None if nm is None else nm.ctypes.data_as(_U8P),
                                   None if fm is None else fm.ctypes.data_as(_U8P), _dp(secs)))
        return y, secs

    def to_dense(self, guard=8192):
        n = self.m.n
        out = np.empty((n, n), order="F")
        _ck(lib().orc_to_dense(self._h, out.ctypes.data_as(_DP), guard))
        return out


def from_product(pm, points, snapshot_mask=None):
    """Oracle twin of a product ParametricMatrix on the same points, fed the
    product's offline TT data (far-field cores, TT near blocks). Snapshot-mode
    near tensors are recomputed by the oracle itself (checks K11 too)."""
    cfg = pm.config
    spec = cfg.spec
    import paper_2511_03109_b200 as ph

    eta = cfg.eta if cfg.eta > 0 else float(np.sqrt(points.shape[1]))
    om = OracleMatrix(points, cfg.l_max, eta, cfg.p_s, spec.family, spec.theta_box, cfg.p_theta,
                      h2=pm.format == ph.Format.H2, amplitude=spec.amplitude)
    ncls = om.counts()["n_classes"]
    for k in range(ncls):
        om.set_coupling(k, pm.coupling_cores(k))
    if cfg.near_mode == ph.NearMode.TT:
        for b in range(om.counts()["n_near"]):
            om.set_near_tt(b, pm.near_tt_cores(b))
    elif cfg.near_mode == ph.NearMode.SNAPSHOT:
        om.make_near_snapshots(snapshot_mask)
    om.finalize()
    return om
