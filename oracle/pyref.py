"""ctypes wrapper of the COMPILED REFERENCE (oracle/_ref/libphmat_ref.so).

TEST INFRASTRUCTURE ONLY. The library is the unmodified reference sources
(/root/reference/proj/src) built against oracle/eigen_shim by
oracle/ref_build.sh, plus oracle/ref_driver.cpp (a C driver over the
reference's public API). Imported by tests/, __graft_entry__.smoke() and
bench.py's reference arm; never by the product package.

`RefMatrix.from_product(pm)` mirrors a product ParametricMatrix into the
reference's own types: the reference rebuilds the tree, blocks, classes,
theta grids and nested basis from the same points and config; it takes the
offline coupling TT cores (the data both sides share) and, in snapshot mode,
evaluates every near tensor itself with near_oracle (nearfield.cpp:7-48), so
the GPU's K11 snapshots are pinned too.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libphmat_ref.so")
TEST_DIR = os.path.join(_HERE, "_ref", "tests")

_DP = C.POINTER(C.c_double)
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_P = C.c_void_p

# reference KernelFamily ids (kernels.hpp:21)
REF_E, REF_TPS, REF_SE, REF_MC, REF_MN = range(5)

_SIG = {
    "rfd_last_error": ([], C.c_char_p),
    "rfd_generate_points": ([C.c_int64, C.c_int, C.c_uint64, _DP], C.c_int),
    "rfd_generate_normal": ([C.c_int64, C.c_uint64, _DP], C.c_int),
    "rfd_theta_draws": ([C.c_double, C.c_double, C.c_int64, C.c_uint64, _DP], C.c_int),
    "rfd_kernel_value": ([C.c_int, C.c_double, _DP, C.c_int], C.c_double),
    "rfd_lagrange": ([C.c_double, C.c_double, C.c_int, C.c_double, _DP], C.c_int),
    "rfd_cheb_grid": ([C.c_double, C.c_double, C.c_int, _DP, _DP], C.c_int),
    "rfd_create": ([_DP, C.c_int64, C.c_int, C.c_int, C.c_double, C.POINTER(_P)], C.c_int),
    "rfd_destroy": ([_P], None),
    "rfd_counts": ([_P, _I64P], C.c_int),
    "rfd_perm": ([_P, _I32P], C.c_int),
    "rfd_nodes": ([_P, _I32P, _I32P, _I32P, _I64P, _I64P], C.c_int),
    "rfd_blocks": ([_P, _I32P, _I32P, _I32P, _I32P, _I32P], C.c_int),
    "rfd_setup": ([_P, C.c_int, C.c_int, C.c_int, _DP, _DP, C.c_int, C.c_int], C.c_int),
    "rfd_theta_grid": ([_P, C.c_int, _DP, _DP], C.c_int),
    "rfd_set_eval": ([_P, C.c_int, C.c_double, C.c_double, C.c_int], C.c_int),
    "rfd_set_coupling": ([_P, C.c_int, C.c_int, _I64P, _DP], C.c_int),
    "rfd_set_near_tt": ([_P, C.c_int64, C.c_int, _I64P, _DP], C.c_int),
    "rfd_make_near_snapshots": ([_P, C.c_int], C.c_int),
    "rfd_finalize": ([_P, C.c_int], C.c_int),
    "rfd_far_st": ([_P, C.c_int64, _DP, _DP, _I64P], C.c_int),
    "rfd_instantiate": ([_P, _DP, C.POINTER(_P), _DP], C.c_int),
    "rfd_inst_destroy": ([_P], None),
    "rfd_inst_near_d": ([_P, C.c_int64, _DP], C.c_int),
    "rfd_inst_far_h": ([_P, C.c_int64, _DP, _I64P], C.c_int),
    "rfd_inst_apply": ([_P, _DP, _DP, C.c_int64, C.c_int, _DP], C.c_int),
    "rfd_inst_to_dense": ([_P, _DP, C.c_int64], C.c_int),
    "rfd_class_h": ([_P, C.c_int, _DP, _DP, _I64P], C.c_int),
    "rfd_class_c": ([_P, C.c_int, _DP, _DP], C.c_int),
    "rfd_near_online": ([_P, C.c_int64, _DP, _DP], C.c_int),
    "rfd_apply_rows": ([_P, _DP, _DP, C.c_int, _I64P, C.c_int64, _DP, C.c_int], C.c_int),
    "rfd_bench_create": ([C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, _DP, _DP, C.c_int, C.c_int,
                          C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double, C.c_int64, C.c_int,
                          C.POINTER(_P)], C.c_int),
    "rfd_bench_destroy": ([_P], None),
    "rfd_build_save": ([C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, _DP, _DP, C.c_int, C.c_int,
                        C.c_int, C.c_double, C.c_double, C.c_int, C.c_char_p, C.c_int], C.c_int),
    "rfd_load": ([C.c_char_p, C.POINTER(_P)], C.c_int),
    "rfd_bench_info": ([_P, _DP], C.c_int),
    "rfd_bench_step": ([_P, C.c_int, _DP, _DP, C.c_int, _DP, _DP], C.c_int),
}

_lib = None


class RefError(RuntimeError):
    pass


class RefDomainError(RefError):
    pass


def available() -> bool:
    return os.path.exists(LIB_PATH)


def build() -> None:
    subprocess.run([os.path.join(_HERE, "ref_build.sh")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not available():
            build()
        L = C.CDLL(LIB_PATH)
        for k, (a, r) in _SIG.items():
            f = getattr(L, k)
            f.argtypes, f.restype = a, r
        _lib = L
    return _lib


def _chk(code):
    if code:
        msg = lib().rfd_last_error().decode()
        raise (RefDomainError if code == 1 else RefError)(msg)


def _dp(a):
    return a.ctypes.data_as(_DP)


def generate_points(n: int, d: int, seed: int) -> np.ndarray:
    out = np.empty((n, d), dtype=np.float64)
    _chk(lib().rfd_generate_points(n, d, seed, _dp(out)))
    return out


def generate_normal(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _chk(lib().rfd_generate_normal(n, seed, _dp(out)))
    return out


def theta_draws(lo: float, hi: float, count: int, seed: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _chk(lib().rfd_theta_draws(lo, hi, count, seed, _dp(out)))
    return out


def lagrange(lo: float, hi: float, p: int, x: float) -> np.ndarray:
    out = np.empty(p, dtype=np.float64)
    _chk(lib().rfd_lagrange(lo, hi, p, x, _dp(out)))
    return out


def _pack(cores):
    dims = np.array([c.shape for c in cores], dtype=np.int64).ravel()
    data = np.concatenate([np.asarray(c, dtype=np.float64).ravel(order="F") for c in cores])
    return dims, np.ascontiguousarray(data)


def resample_core(core: np.ndarray, lo: float, hi: float, p_new: int) -> np.ndarray:
    """Re-expresses a theta-core sampled on the p_old-node Chebyshev grid on
    the p_new >= p_old grid: slice j' = sum_j L_j^old(x'_j') slice j. A
    degree p_old-1 polynomial is reproduced exactly, so the reference's
    one-p_theta grid (PHConfig::p_theta, phmatrix.hpp:24) interpolates the
    same function as the product's per-dimension grid (up to rounding)."""
    r0, p_old, r1 = core.shape
    if p_old == p_new:
        return core
    xs, _ = cheb_grid(lo, hi, p_new)
    out = np.zeros((r0, p_new, r1))
    for jn, x in enumerate(xs):
        L = lagrange(lo, hi, p_old, x)
        out[:, jn, :] = np.tensordot(L, core, axes=([0], [1]))
    return out


def cheb_grid(lo: float, hi: float, p: int):
    """The reference's cheb_grid (chebyshev.cpp:10-43): nodes, weights."""
    nodes, w = np.empty(p), np.empty(p)
    _chk(lib().rfd_cheb_grid(lo, hi, p, _dp(nodes), _dp(w)))
    return nodes, w


def build_save(path, n, d, seed, h2, family, boxes, l_max, p_s, p_theta, eps=1e-5, eta=1.0, near_tt=True,
               threads=0):
    """The reference's own offline build (offline_h / offline_h2 on its
    generate_points) saved as an HMAT v1 artifact (save_parametric)."""
    lo = np.array([b[0] for b in boxes], dtype=np.float64)
    hi = np.array([b[1] for b in boxes], dtype=np.float64)
    _chk(lib().rfd_build_save(n, d, seed, 1 if h2 else 0, family, len(boxes), _dp(lo), _dp(hi), l_max, p_s, p_theta,
                              eps, eta, 1 if near_tt else 0, os.fsencode(path), threads))


def load(path) -> "RefMatrix":
    """load_parametric_h / _h2 of the reference into a RefMatrix."""
    h = _P()
    _chk(lib().rfd_load(os.fsencode(path), C.byref(h)))
    R = RefMatrix.__new__(RefMatrix)
    R._h = h
    R._near_shape = None
    R.n = int(R.nodes()["size"][0])  # the root holds every point
    return R


class RefInst:
    def __init__(self, parent: "RefMatrix", h, seconds):
        self.parent, self._h, self.seconds = parent, h, seconds

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.rfd_inst_destroy(self._h)
            self._h = None

    def near_d(self, b: int) -> np.ndarray:
        ns, nt = self.parent.near_shape(b)
        out = np.empty(ns * nt)
        _chk(lib().rfd_inst_near_d(self._h, b, _dp(out)))
        return out.reshape((ns, nt), order="F")

    def far_h(self, i: int) -> np.ndarray:
        shape = np.zeros(2, dtype=np.int64)
        _chk(lib().rfd_inst_far_h(self._h, i, None, shape.ctypes.data_as(_I64P)))
        out = np.empty(int(shape[0] * shape[1]))
        _chk(lib().rfd_inst_far_h(self._h, i, _dp(out), shape.ctypes.data_as(_I64P)))
        return out.reshape(tuple(shape), order="F")

    def apply(self, x) -> np.ndarray:
        """y = K(theta) x (x: n or n x m), the reference's apply per column."""
        X = np.asarray(x, dtype=np.float64)
        one = X.ndim == 1
        Xf = np.asfortranarray(X.reshape(X.shape[0], -1))
        Y = np.empty_like(Xf)
        sec = C.c_double()
        _chk(lib().rfd_inst_apply(self._h, _dp(Xf), _dp(Y), Xf.shape[0], Xf.shape[1], C.byref(sec)))
        self.apply_seconds = sec.value
        return Y[:, 0] if one else Y

    def to_dense(self, guard: int = 8192) -> np.ndarray:
        n = self.parent.n
        out = np.empty(n * n)
        _chk(lib().rfd_inst_to_dense(self._h, _dp(out), guard))
        return out.reshape((n, n), order="F")


class RefMatrix:
    """The reference's structure (+ optionally its parametric matrix)."""

    def __init__(self, points, l_max: int, eta: float):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        self.n, self.d = pts.shape
        self.points = pts
        h = _P()
        _chk(lib().rfd_create(_dp(pts), self.n, self.d, l_max, eta, C.byref(h)))
        self._h = h
        self._near_shape = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.rfd_destroy(self._h)
            self._h = None

    # structure
    def counts(self) -> dict:
        out = np.zeros(8, dtype=np.int64)
        _chk(lib().rfd_counts(self._h, out.ctypes.data_as(_I64P)))
        keys = ["nodes", "leaves", "n_near", "n_far", "n_classes", "c_sp", "block_count", "coverage"]
        return dict(zip(keys, (int(v) for v in out)))

    def perm(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int32)
        _chk(lib().rfd_perm(self._h, out.ctypes.data_as(_I32P)))
        return out

    def nodes(self) -> dict:
        nn = self.counts()["nodes"]
        lv, pa, fc = (np.empty(nn, dtype=np.int32) for _ in range(3))
        sz = np.empty(nn, dtype=np.int64)
        co = np.empty((nn, 3), dtype=np.int64)
        _chk(lib().rfd_nodes(self._h, lv.ctypes.data_as(_I32P), pa.ctypes.data_as(_I32P),
                             fc.ctypes.data_as(_I32P), sz.ctypes.data_as(_I64P), co.ctypes.data_as(_I64P)))
        return dict(level=lv, parent=pa, first_child=fc, size=sz, coords=co)

    def blocks(self):
        c = self.counts()
        near = np.empty((2, c["n_near"]), dtype=np.int32)
        far = np.empty((2, c["n_far"]), dtype=np.int32)
        key = np.empty(c["n_far"], dtype=np.int32)
        _chk(lib().rfd_blocks(self._h, near[0].ctypes.data_as(_I32P), near[1].ctypes.data_as(_I32P),
                              far[0].ctypes.data_as(_I32P), far[1].ctypes.data_as(_I32P),
                              key.ctypes.data_as(_I32P)))
        return near.T.copy(), far.T.copy(), key

    def near_shape(self, b: int):
        if self._near_shape is None:
            near, _, _ = self.blocks()
            sz = self.nodes()["size"]
            self._near_shape = np.stack([sz[near[:, 0]], sz[near[:, 1]]], axis=1)
        ns, nt = self._near_shape[b]
        return int(ns), int(nt)

    # parametric data
    def setup(self, h2: bool, family: int, boxes, p_theta: int, p_s: int) -> None:
        lo = np.array([b[0] for b in boxes], dtype=np.float64)
        hi = np.array([b[1] for b in boxes], dtype=np.float64)
        self.boxes = [(float(a), float(b)) for a, b in boxes]
        self.p_theta = p_theta
        self.h2 = h2
        _chk(lib().rfd_setup(self._h, 1 if h2 else 0, family, len(boxes), _dp(lo), _dp(hi), p_theta, p_s))

    def theta_grid(self, k: int):
        nodes, w = np.empty(self.p_theta), np.empty(self.p_theta)
        _chk(lib().rfd_theta_grid(self._h, k, _dp(nodes), _dp(w)))
        return nodes, w

    def set_eval(self, family: int, nu: float = 0.0, lam_scale: float = 1.0, amplitude: bool = False) -> None:
        _chk(lib().rfd_set_eval(self._h, family, nu, lam_scale, 1 if amplitude else 0))

    def set_coupling(self, k: int, cores) -> None:
        dims, data = _pack(cores)
        _chk(lib().rfd_set_coupling(self._h, k, len(cores), dims.ctypes.data_as(_I64P), _dp(data)))

    def set_near_tt(self, b: int, cores) -> None:
        dims, data = _pack(cores)
        _chk(lib().rfd_set_near_tt(self._h, b, len(cores), dims.ctypes.data_as(_I64P), _dp(data)))

    def make_near_snapshots(self, threads: int = 0) -> None:
        _chk(lib().rfd_make_near_snapshots(self._h, threads))

    def finalize(self, threads: int = 0) -> None:
        _chk(lib().rfd_finalize(self._h, threads))

    def far_st(self, i: int):
        shape = np.zeros(4, dtype=np.int64)
        _chk(lib().rfd_far_st(self._h, i, None, None, shape.ctypes.data_as(_I64P)))
        S = np.empty(int(shape[0] * shape[1]))
        T = np.empty(int(shape[2] * shape[3]))
        _chk(lib().rfd_far_st(self._h, i, _dp(S), _dp(T), shape.ctypes.data_as(_I64P)))
        return S.reshape((shape[0], shape[1]), order="F"), T.reshape((shape[2], shape[3]), order="F")

    def instantiate(self, theta) -> RefInst:
        th = np.ascontiguousarray(np.atleast_1d(theta), dtype=np.float64)
        h = _P()
        sec = C.c_double()
        _chk(lib().rfd_instantiate(self._h, _dp(th), C.byref(h), C.byref(sec)))
        return RefInst(self, h, sec.value)

    def class_h(self, k: int, theta) -> np.ndarray:
        th = np.ascontiguousarray(np.atleast_1d(theta), dtype=np.float64)
        shape = np.zeros(2, dtype=np.int64)
        _chk(lib().rfd_class_h(self._h, k, _dp(th), None, shape.ctypes.data_as(_I64P)))
        out = np.empty(int(shape[0] * shape[1]))
        _chk(lib().rfd_class_h(self._h, k, _dp(th), _dp(out), shape.ctypes.data_as(_I64P)))
        return out.reshape(tuple(shape), order="F")

    def class_c(self, k: int, theta, P: int) -> np.ndarray:
        th = np.ascontiguousarray(np.atleast_1d(theta), dtype=np.float64)
        out = np.empty(P * P)
        _chk(lib().rfd_class_c(self._h, k, _dp(th), _dp(out)))
        return out.reshape((P, P), order="F")

    def near_online(self, b: int, theta) -> np.ndarray:
        th = np.ascontiguousarray(np.atleast_1d(theta), dtype=np.float64)
        ns, nt = self.near_shape(b)
        out = np.empty(ns * nt)
        _chk(lib().rfd_near_online(self._h, b, _dp(th), _dp(out)))
        return out.reshape((ns, nt), order="F")

    def apply_rows(self, theta, x, rows, threads: int = 0) -> np.ndarray:
        """Rows of y = K(theta) x (x: n or n x m) from the reference's pieces
        restricted to the blocks that reach them (rfd_apply_rows)."""
        th = np.ascontiguousarray(np.atleast_1d(theta), dtype=np.float64)
        X = np.asarray(x, dtype=np.float64)
        one = X.ndim == 1
        Xf = np.asfortranarray(X.reshape(X.shape[0], -1))
        r = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((r.size, Xf.shape[1]), order="F")
        _chk(lib().rfd_apply_rows(self._h, _dp(th), _dp(Xf), Xf.shape[1], r.ctypes.data_as(_I64P), r.size,
                                  _dp(out), threads))
        return out[:, 0] if one else out

    # ---------------------------------------------------------------- mirror
    @classmethod
    def from_product(cls, pm, points, near: str = "snapshot", finalize: bool = True, threads: int = 0):
        """Mirror of a product ParametricMatrix in the reference's types.

        near = "snapshot": the reference evaluates every near tensor itself
        (near_oracle) -- snapshot mode; "tt": the product's near TT cores;
        "none": no near data (per-block / row-probe entry points only)."""
        cfg = pm.config
        spec = cfg.spec
        fam = int(spec.family)
        boxes = [tuple(b) for b in spec.theta_box]
        pt = cfg.p_theta
        pts = [pt] * len(boxes) if isinstance(pt, int) else list(pt)
        p_ref = max(pts)
        # grid family: any reference family with the same parameter count
        # (make_theta_grids validates it); only the box defines the grid.
        grid_family = REF_MN if len(boxes) == 2 else (fam if fam <= 3 else REF_E)
        if fam == 4 and len(boxes) == 2:
            grid_family = REF_MN
        R = cls(points, cfg.l_max, cfg.eta)
        R.setup(pm.format == 1, grid_family, boxes, p_ref, cfg.p_s)
        if fam <= 4:
            R.set_eval(fam)
        elif fam == 5:  # Gaussian exp(-r^2/(2 l^2)) = se at lambda = sqrt(2) l
            R.set_eval(REF_SE, lam_scale=float(np.sqrt(2.0)), amplitude=spec.amplitude)
        elif fam == 6:
            R.set_eval(REF_MN, nu=1.5, amplitude=spec.amplitude)
        elif fam == 7:
            R.set_eval(REF_MN, nu=2.5, amplitude=spec.amplitude)
        d = points.shape[1]
        for k in range(pm.info()["n_classes"]):
            cores = pm.coupling_cores(k)
            for i, (b, p) in enumerate(zip(boxes, pts)):
                if p != p_ref:
                    cores[d + i] = resample_core(cores[d + i], b[0], b[1], p_ref)
            R.set_coupling(k, cores)
        if near == "snapshot":
            R.make_near_snapshots(threads)
        elif near == "tt":
            for b in range(pm.info()["n_near"]):
                cores = pm.near_tt_cores(b)
                for i, (bx, p) in enumerate(zip(boxes, pts)):
                    if p != p_ref:
                        cores[1 + i] = resample_core(cores[1 + i], bx[0], bx[1], p_ref)
                R.set_near_tt(b, cores)
        if finalize and near != "none":
            R.finalize(threads)
        return R


class RefBench:
    """The reference's own CPU arm for bench.py (no product code involved):
    the reference builds its parametric matrix (offline_h / offline_h2,
    Direct near mode, then snapshot TTs of a 1/stride sample of near blocks)
    and times its own instantiate + apply on the sample and on a fixed-cost
    matrix (every class, one far block per sigma)."""

    # product family id -> (grid family, eval family, nu, lambda scale)
    FAMILIES = {"e": (REF_E, REF_E, 0.0, 1.0), "se": (REF_SE, REF_SE, 0.0, 1.0),
                "gauss": (REF_SE, REF_SE, 0.0, float(np.sqrt(2.0))),
                "m32": (REF_E, REF_MN, 1.5, 1.0), "m52": (REF_E, REF_MN, 2.5, 1.0)}

    def __init__(self, n, d, seed, h2, family, box, l_max, p_s, p_theta, eta, eps, stride, threads):
        gfam, efam, nu, lam = self.FAMILIES[family]
        lo = np.array([box[0]], dtype=np.float64)
        hi = np.array([box[1]], dtype=np.float64)
        h = _P()
        _chk(lib().rfd_bench_create(n, d, seed, 1 if h2 else 0, gfam, 1, _dp(lo), _dp(hi), l_max, p_s, p_theta, eta,
                                    eps, efam, nu, lam, stride, threads, C.byref(h)))
        self._h = h
        self.n = n
        self.stride = stride
        info = np.zeros(5)
        _chk(lib().rfd_bench_info(h, _dp(info)))
        self.near_frac, self.far_frac, self.build_s = float(info[0]), float(info[1]), float(info[2])
        self.near_blocks, self.far_blocks = int(info[3]), int(info[4])

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.rfd_bench_destroy(self._h)
            self._h = None

    def step(self, which: int, theta, x: np.ndarray):
        th = np.ascontiguousarray(np.atleast_1d(theta), dtype=np.float64)
        X = np.asfortranarray(x.reshape(self.n, -1))
        y = np.empty(self.n)
        t = np.zeros(2)
        _chk(lib().rfd_bench_step(self._h, which, _dp(th), _dp(X), X.shape[1], _dp(y), _dp(t)))
        return float(t[0]), float(t[1])
