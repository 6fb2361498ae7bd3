"""B200-native online stage of parametric H / H^2 matrices (arXiv 2511.03109).

Python mirror of the reference's C++ API (proj/include/phmat/phmatrix.hpp)
over the C ABI in include/phmat_b200.h. The names follow the reference:

    pm   = offline_h2(points, PHConfig(...))         # phmatrix.hpp:82-91
    inst = instantiate(pm, theta)                     # phmatrix.hpp:133-138
    y    = inst.apply(x)                              # phmatrix.hpp:95-128
    inst.far_h(i), inst.near_d(b), inst.to_dense()    # phmatrix.hpp:102-128
    metrics(pm)                                       # phmatrix.hpp:141-153

Every online computation runs in the CUDA kernels of libphmat_b200.so; there
is no CPU fallback. Importing works without a GPU (structure-only builds via
``offline_structure``); instantiate/apply raise if no sm_100 device exists.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "PHConfig", "KernelSpec", "Family", "Format", "NearMode",
    "Context", "ParametricMatrix", "InstantiatedMatrix",
    "offline_h", "offline_h2", "offline_structure", "instantiate", "metrics",
    "generate_points", "generate_mixture_points", "generate_normal", "instantiate_batch", "reinstantiate_batch",
    "h_aca", "h2_hca", "aca_partial", "Baseline", "BaselineMatrix",
    "PhmatError", "DomainError", "InvalidArgument", "LogicError", "CudaError",
    "library_path", "lib",
]

_HERE = os.path.dirname(os.path.abspath(__file__))


def library_path() -> str:
    # PHM_LIB selects another in-tree build (tools/check_build.sh builds
    # libphmat_b200_checked.so with device-side invariant checks)
    name = os.environ.get("PHM_LIB", "libphmat_b200.so")
    if os.path.basename(name) != name or not name.startswith("libphmat_b200"):
        raise ImportError("PHM_LIB must name an in-tree libphmat_b200*.so")
    return os.path.join(_HERE, name)


class PhmatError(RuntimeError):
    """std::runtime_error (size guards, artifacts)."""


class DomainError(ValueError):
    """std::domain_error: theta outside the parameter box (farfield.cpp:23-24)."""


class InvalidArgument(ValueError):
    """std::invalid_argument: length mismatch / malformed spec (phmatrix.cpp:228)."""


class LogicError(RuntimeError):
    """std::logic_error: PHMAT_CHECK failures (common.hpp:15-18)."""


class CudaError(RuntimeError):
    """CUDA runtime failure or no sm_100 device."""


_ERRORS = {1: PhmatError, 2: DomainError, 3: InvalidArgument, 4: LogicError, 5: CudaError, 6: IndexError}


class _Config(C.Structure):
    _fields_ = [
        ("family", C.c_int32), ("amplitude", C.c_int32), ("d_theta", C.c_int32),
        ("p_theta", C.c_int32 * 3), ("theta_lo", C.c_double * 3), ("theta_hi", C.c_double * 3),
        ("format", C.c_int32), ("l_max", C.c_int32), ("p_s", C.c_int32), ("near_mode", C.c_int32),
        ("eps", C.c_double), ("eta", C.c_double), ("r_max_far", C.c_int64), ("r_max_near", C.c_int64),
        ("seed", C.c_uint64), ("translation_cache", C.c_int32), ("threads", C.c_int32),
        ("shard_rank", C.c_int32), ("shard_count", C.c_int32), ("symmetric_near", C.c_int32),
        ("reserved", C.c_int32),
    ]


class _Info(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "n", "d", "nodes", "n_near", "n_far", "n_classes", "c_sp", "constructed", "P",
        "row_begin", "row_end", "near_entries", "near_stored", "near_stream_elems", "device_bytes", "storage_entries")] + [
        (k, C.c_double) for k in (
            "storage_gb", "nf_ratio", "ff_ratio", "coupling_ratio", "rank", "tree_s", "ff_s", "nf_s", "upload_s")] + [
        ("evals_offline", C.c_uint64), ("evals_online", C.c_uint64), ("evals_audit", C.c_uint64),
        ("any_rank_capped", C.c_int32), ("pad", C.c_int32)]


class _BaselineInfo(C.Structure):
    _fields_ = [("method", C.c_int32), ("any_capped", C.c_int32)] + [
        (k, C.c_double) for k in ("mean_far_rank", "coupling_ratio", "far_build_s", "near_build_s")] + [
        ("far_evals", C.c_uint64), ("near_evals", C.c_uint64)] + [
        (k, C.c_int64) for k in ("n_far", "n_near", "n_classes")]


_P = C.c_void_p
_DP = C.POINTER(C.c_double)
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_U64P = C.POINTER(C.c_uint64)

# Every symbol of include/phmat_b200.h with its argument types.
SIGNATURES = {
    "phm_last_error": ([], C.c_char_p),
    "phm_version": ([], C.c_int),
    "phm_config_default": ([C.POINTER(_Config)], None),
    "phm_context_create": ([C.c_int, C.POINTER(_P)], C.c_int),
    "phm_context_destroy": ([_P], C.c_int),
    "phm_context_set_stream": ([_P, _P], C.c_int),
    "phm_context_get_stream": ([_P, C.POINTER(_P)], C.c_int),
    "phm_context_sync": ([_P], C.c_int),
    "phm_context_enable_timing": ([_P, C.c_int], C.c_int),
    "phm_context_timer": ([_P, C.c_char_p, _DP, _I64P], C.c_int),
    "phm_context_reset_timers": ([_P], C.c_int),
    "phm_context_launches": ([_P, _I64P], C.c_int),
    "phm_matrix_build": ([_P, _DP, C.c_int64, C.c_int, C.POINTER(_Config), C.POINTER(_P)], C.c_int),
    "phm_matrix_build_host": ([_DP, C.c_int64, C.c_int, C.POINTER(_Config), C.POINTER(_P)], C.c_int),
    "phm_matrix_load": ([_P, C.c_char_p, C.c_int, C.POINTER(_P)], C.c_int),
    "phm_matrix_save": ([_P, C.c_char_p], C.c_int),
    "phm_matrix_load_host": ([C.c_char_p, C.c_int, C.POINTER(_P)], C.c_int),
    "phm_artifact_is_h2": ([C.c_char_p, C.POINTER(C.c_int)], C.c_int),
    "phm_matrix_config": ([_P, C.POINTER(_Config)], C.c_int),
    "phm_matrix_destroy": ([_P], C.c_int),
    "phm_matrix_info": ([_P, C.POINTER(_Info)], C.c_int),
    "phm_matrix_perm": ([_P, _I32P], C.c_int),
    "phm_matrix_nodes": ([_P, _I32P, _DP], C.c_int),
    "phm_matrix_blocks": ([_P, _I32P, _I32P, _I32P], C.c_int),
    "phm_matrix_class_keys": ([_P, _I64P], C.c_int),
    "phm_matrix_theta_grid": ([_P, C.c_int, _DP], C.c_int),
    "phm_matrix_coupling": ([_P, C.c_int64, _I32P, _I64P, _DP, _I64P], C.c_int),
    "phm_matrix_near_tt": ([_P, C.c_int64, _I32P, _I64P, _DP, _I64P], C.c_int),
    "phm_matrix_near_rank": ([_P, C.c_int64, _I64P], C.c_int),
    "phm_matrix_near_column": ([_P, C.c_int64, C.c_int64, _DP], C.c_int),
    "phm_matrix_far_st": ([_P, C.c_int64, _DP, _DP, _I64P], C.c_int),
    "phm_matrix_class_lr": ([_P, C.c_int64, _DP, _DP, _I64P], C.c_int),
    "phm_parametric_vectors": ([_P, _DP, C.c_int, _DP], C.c_int),
    "phm_instantiate": ([_P, _DP, C.c_int, C.POINTER(_P)], C.c_int),
    "phm_reinstantiate": ([_P, _DP, C.c_int], C.c_int),
    "phm_instantiate_batch": ([_P, _DP, C.c_int, C.c_int, _P], C.c_int),
    "phm_baseline_build": ([_P, _DP, C.c_int64, C.c_int, _P, C.c_int, _DP, C.c_int, C.c_double, C.c_int64, _P],
                           C.c_int),
    "phm_baseline_info_get": ([_P, _P], C.c_int),
    "phm_aca_partial_dense": ([_DP, C.c_int64, C.c_int64, C.c_double, C.c_int64, C.c_uint64, _I64P,
                               C.POINTER(C.c_int32), _DP, _DP], C.c_int),
    "phm_reinstantiate_batch": ([_P, C.c_int, _DP, C.c_int], C.c_int),
    "phm_instance_destroy": ([_P], C.c_int),
    "phm_instance_sync": ([_P], C.c_int),
    "phm_instance_far_h": ([_P, C.c_int64, _DP, _I64P, _I64P], C.c_int),
    "phm_instance_near_d": ([_P, C.c_int64, _DP], C.c_int),
    "phm_instance_class_c": ([_P, C.c_int64, _DP], C.c_int),
    "phm_apply": ([_P, _DP, C.c_int64, _DP, C.c_int64], C.c_int),
    "phm_apply_device": ([_P, _P, _P, C.c_int64], C.c_int),
    "phm_instantiate_apply": ([_P, _DP, C.c_int, _DP, C.c_int64, _DP, C.c_int64], C.c_int),
    "phm_instantiate_apply_device": ([_P, _DP, C.c_int, _P, _P, C.c_int64], C.c_int),
    "phm_apply_rows_device": ([_P, _P, _P, C.c_int64], C.c_int),
    "phm_apply_partial_device": ([_P, _P, _P, C.c_int64], C.c_int),
    "phm_instantiate_apply_partial_device": ([_P, _DP, C.c_int, _P, _P, C.c_int64], C.c_int),
    "phm_unpermute_device": ([_P, _P, _P, C.c_int64], C.c_int),
    "phm_comm_unique_id": ([C.c_char_p], C.c_int),
    "phm_comm_create_nccl": ([_P, C.c_char_p, C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "phm_comm_create_callback": ([_P, _P, C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "phm_comm_create_probe": ([C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "phm_comm_destroy": ([_P], C.c_int),
    "phm_comm_info": ([_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "phm_instantiate_apply_sharded": ([_P, _P, _DP, C.c_int, _P, _P, C.c_int64], C.c_int),
    "phm_instantiate_apply_sharded_host": ([_P, _P, _DP, C.c_int, _DP, C.c_int64, _DP, C.c_int64], C.c_int),
    "phm_apply_sharded": ([_P, _P, _P, _P, C.c_int64], C.c_int),
    "phm_to_dense": ([_P, _DP, C.c_int64], C.c_int),
    "phm_estimate_error": ([_P, C.c_int64, C.c_uint64, _DP, _I64P, _DP, _DP, _DP], C.c_int),
    "phm_generate_points": ([C.c_int64, C.c_int, C.c_uint64, _DP], C.c_int),
    "phm_generate_mixture_points": ([C.c_int64, C.c_int, C.c_int, C.c_double, C.c_uint64, _DP], C.c_int),
    "phm_generate_normal": ([C.c_int64, C.c_uint64, _DP], C.c_int),
    "phm_theta_draws": ([C.c_double, C.c_double, C.c_int64, C.c_uint64, _DP], C.c_int),
    "phm_tt_cross_dense": ([_DP, _I64P, C.c_int, C.c_double, C.c_int64, C.c_uint64, C.c_int, _I32P, _I64P, _DP,
                            C.c_int64, _I64P, _U64P, _I32P, _DP], C.c_int),
    "phm_tt_round": ([C.c_int, _I64P, _DP, C.c_double, C.c_double, _I32P, _I64P, _DP, C.c_int64, _I64P], C.c_int),
}

_lib = None


def lib():
    """Loads the in-tree libphmat_b200.so; fails loudly if it was not built."""
    global _lib
    if _lib is None:
        path = library_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(code: int) -> None:
    if code != 0:
        msg = lib().phm_last_error().decode(errors="replace")
        raise _ERRORS.get(code, PhmatError)(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def _f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        out = out.reshape(shape)
    return out


# ------------------------------------------------------------------- config
class Family:
    E, TPS, SE, MC, MN, GAUSS, MATERN32, MATERN52 = range(8)
    _IDS = {"e": 0, "tps": 1, "se": 2, "mc": 3, "mn": 4, "gauss": 5, "m32": 6, "m52": 7}

    @classmethod
    def from_id(cls, s: str) -> int:  # kernel_family_from_id, kernels.cpp:8-15
        if s not in cls._IDS:
            raise InvalidArgument(f"unknown kernel id: {s}")
        return cls._IDS[s]


class Format:
    H, H2 = 0, 1


class NearMode:
    TT, DIRECT, SNAPSHOT = 0, 1, 2


@dataclass
class KernelSpec:
    """KernelSpec (kernels.hpp:31-38) + optional trailing amplitude sigma^2."""
    family: int = Family.SE
    theta_box: List[Sequence[float]] = field(default_factory=lambda: [(0.25, 1.0)])
    amplitude: bool = False

    @staticmethod
    def default(family: int) -> "KernelSpec":  # default_kernel_spec, kernels.cpp:41-47
        box = [(0.25, 1.0)]
        if family == Family.MN:
            box.append((0.5, 3.0))
        return KernelSpec(family, box)


@dataclass
class PHConfig:
    """PHConfig (phmatrix.hpp:20-35); p_theta may be per parameter dimension."""
    spec: KernelSpec = field(default_factory=KernelSpec)
    l_max: int = 2
    p_s: int = 15
    p_theta: Sequence[int] | int = 27
    eps: float = 1e-5
    eta: float = 0.0
    r_max_far: int = 120
    r_max_near: int = 150
    seed: int = 0
    near_mode: int = NearMode.TT
    translation_cache: bool = True
    threads: int = 0
    shard_rank: int = 0
    shard_count: int = 1
    symmetric_near: bool = True

    def to_c(self, fmt: int) -> _Config:
        c = _Config()
        lib().phm_config_default(C.byref(c))
        box = list(self.spec.theta_box)
        c.family = self.spec.family
        c.amplitude = 1 if self.spec.amplitude else 0
        c.d_theta = len(box)
        pt = [self.p_theta] * len(box) if isinstance(self.p_theta, int) else list(self.p_theta)
        if len(pt) != len(box):
            raise InvalidArgument("p_theta needs one entry per parameter dimension")
        for k, (lo, hi) in enumerate(box):
            c.theta_lo[k] = lo
            c.theta_hi[k] = hi
            c.p_theta[k] = pt[k]
        c.format = fmt
        c.l_max, c.p_s, c.near_mode = self.l_max, self.p_s, self.near_mode
        c.eps, c.eta = self.eps, self.eta
        c.r_max_far, c.r_max_near, c.seed = self.r_max_far, self.r_max_near, self.seed
        c.translation_cache = 1 if self.translation_cache else 0
        c.threads, c.shard_rank, c.shard_count = self.threads, self.shard_rank, self.shard_count
        c.symmetric_near = 1 if self.symmetric_near else 0
        return c


# ------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream. Raises CudaError without an sm_100 device."""

    _default: Optional["Context"] = None

    def __init__(self, device: int = 0):
        h = _P()
        _check(lib().phm_context_create(device, C.byref(h)))
        self._h = h
        self.device = device

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(0)
        return cls._default

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.phm_context_destroy(self._h)
            self._h = None

    def set_stream(self, stream_ptr: int) -> None:
        _check(lib().phm_context_set_stream(self._h, _P(stream_ptr)))

    @property
    def stream(self) -> int:
        s = _P()
        _check(lib().phm_context_get_stream(self._h, C.byref(s)))
        return s.value or 0

    def sync(self) -> None:
        _check(lib().phm_context_sync(self._h))

    def enable_timing(self, on: bool = True) -> None:
        _check(lib().phm_context_enable_timing(self._h, 1 if on else 0))

    def timer(self, name: str):
        ms, cnt = C.c_double(), C.c_int64()
        _check(lib().phm_context_timer(self._h, name.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def reset_timers(self) -> None:
        _check(lib().phm_context_reset_timers(self._h))

    @property
    def launches(self) -> int:
        v = C.c_int64()
        _check(lib().phm_context_launches(self._h, C.byref(v)))
        return v.value


# ------------------------------------------------------------------- matrix
class ParametricMatrix:
    """ParametricHMatrix / ParametricH2Matrix (phmatrix.hpp:40-80), GPU resident."""

    def __init__(self, handle, ctx: Optional[Context], fmt: int, config: PHConfig, n: int, d: int):
        self._h = handle
        self.ctx = ctx
        self.format = fmt
        self.config = config
        self._n = n
        self._d = d
        self._info = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.phm_matrix_destroy(self._h)
            self._h = None

    # structure -------------------------------------------------------
    def info(self) -> dict:
        inf = _Info()
        _check(lib().phm_matrix_info(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in _Info._fields_ if k != "pad"}

    def n(self) -> int:
        return self._n

    def d(self) -> int:
        return self._d

    def perm(self) -> np.ndarray:
        out = np.empty(self._n, dtype=np.int32)
        _check(lib().phm_matrix_perm(self._h, out.ctypes.data_as(_I32P)))
        return out

    def nodes(self):
        nn = self.info()["nodes"]
        ints = np.empty((nn, 7), dtype=np.int32)
        boxes = np.empty((nn, 6), dtype=np.float64)
        _check(lib().phm_matrix_nodes(self._h, ints.ctypes.data_as(_I32P), _dp(boxes)))
        return ints, boxes

    def blocks(self):
        inf = self.info()
        near = np.empty((inf["n_near"], 2), dtype=np.int32)
        far = np.empty((inf["n_far"], 2), dtype=np.int32)
        key = np.empty(inf["n_far"], dtype=np.int32)
        _check(lib().phm_matrix_blocks(self._h, near.ctypes.data_as(_I32P), far.ctypes.data_as(_I32P),
                                       key.ctypes.data_as(_I32P)))
        return near, far, key

    def class_keys(self) -> np.ndarray:
        k = self.info()["n_classes"]
        out = np.empty((k, 4), dtype=np.int64)
        _check(lib().phm_matrix_class_keys(self._h, out.ctypes.data_as(_I64P)))
        return out

    def theta_grid(self, k: int) -> np.ndarray:
        pt = self.config.p_theta
        p = pt if isinstance(pt, int) else list(pt)[k]
        out = np.empty(p, dtype=np.float64)
        _check(lib().phm_matrix_theta_grid(self._h, k, _dp(out)))
        return out

    def _cores(self, fn, idx):
        nc = C.c_int32()
        dims = np.zeros(30, dtype=np.int64)
        ln = C.c_int64()
        _check(fn(self._h, idx, C.byref(nc), dims.ctypes.data_as(_I64P), None, C.byref(ln)))
        data = np.empty(ln.value, dtype=np.float64)
        _check(fn(self._h, idx, C.byref(nc), dims.ctypes.data_as(_I64P), _dp(data), C.byref(ln)))
        dims = dims[: 3 * nc.value].reshape(-1, 3)
        cores, off = [], 0
        for r0, m, r1 in dims:
            sz = int(r0 * m * r1)
            cores.append(data[off: off + sz].reshape((int(r0), int(m), int(r1)), order="F"))
            off += sz
        return cores

    def coupling_cores(self, cls: int):
        """TT cores (r0, m, r1) of translation class cls (CouplingTT::tt)."""
        return self._cores(lib().phm_matrix_coupling, cls)

    def near_tt_cores(self, b: int):
        return self._cores(lib().phm_matrix_near_tt, b)

    def near_rank(self, b: int) -> int:
        r = C.c_int64()
        _check(lib().phm_matrix_near_rank(self._h, b, C.byref(r)))
        return r.value

    def near_column(self, b: int, kap: int, shape) -> np.ndarray:
        out = np.empty(shape[0] * shape[1], dtype=np.float64)
        _check(lib().phm_matrix_near_column(self._h, b, kap, _dp(out)))
        return out.reshape(shape, order="F")

    def far_st(self, i: int):
        dims = np.zeros(4, dtype=np.int64)
        _check(lib().phm_matrix_far_st(self._h, i, None, None, dims.ctypes.data_as(_I64P)))
        S = np.empty((dims[0], dims[1]), order="F")
        T = np.empty((dims[2], dims[3]), order="F")
        _check(lib().phm_matrix_far_st(self._h, i, S.ctypes.data_as(_DP), T.ctypes.data_as(_DP), None))
        return S, T

    def class_lr(self, k: int):
        dims = np.zeros(4, dtype=np.int64)
        _check(lib().phm_matrix_class_lr(self._h, k, None, None, dims.ctypes.data_as(_I64P)))
        L = np.empty((dims[0], dims[1]), order="F")
        R = np.empty((dims[2], dims[3]), order="F")
        _check(lib().phm_matrix_class_lr(self._h, k, L.ctypes.data_as(_DP), R.ctypes.data_as(_DP), None))
        return L, R

    def parametric_vectors(self, theta) -> List[np.ndarray]:
        th = _f64(theta).ravel()
        pt = self.config.p_theta
        ps = [pt] * th.size if isinstance(pt, int) else list(pt)
        out = np.empty(sum(ps), dtype=np.float64)
        _check(lib().phm_parametric_vectors(self._h, _dp(th), th.size, _dp(out)))
        res, off = [], 0
        for p in ps:
            res.append(out[off: off + p].copy())
            off += p
        return res


class InstantiatedMatrix:
    """InstantiatedHMatrix / InstantiatedH2Matrix (phmatrix.hpp:102-128)."""

    def __init__(self, parent: ParametricMatrix, handle, theta):
        self.parent = parent
        self._h = handle
        self.theta = list(theta)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.phm_instance_destroy(self._h)
            self._h = None

    def rows(self) -> int:
        return self.parent.n()

    def reinstantiate(self, theta) -> None:
        th = _f64(theta).ravel()
        _check(lib().phm_reinstantiate(self._h, _dp(th), th.size))
        self.theta = list(th)

    def sync(self) -> None:
        _check(lib().phm_instance_sync(self._h))

    def apply(self, x) -> np.ndarray:
        """y = K~(theta) x; x is (n,) or (n, m) in the original point order."""
        xa = np.asarray(x, dtype=np.float64)
        vec = xa.ndim == 1
        n_rows = xa.shape[0]
        m = 1 if vec else xa.shape[1]
        xf = np.asfortranarray(xa.reshape(n_rows, m))
        y = np.empty((self.parent.n(), m), dtype=np.float64, order="F")
        _check(lib().phm_apply(self._h, xf.ctypes.data_as(_DP), n_rows, y.ctypes.data_as(_DP), m))
        return y[:, 0].copy() if vec else y

    def instantiate_apply(self, theta, x) -> np.ndarray:
        """reinstantiate(theta) then apply(x) as one overlapped schedule."""
        th = _f64(theta).ravel()
        xa = np.asarray(x, dtype=np.float64)
        vec = xa.ndim == 1
        n_rows = xa.shape[0]
        m = 1 if vec else xa.shape[1]
        xf = np.asfortranarray(xa.reshape(n_rows, m))
        y = np.empty((self.parent.n(), m), dtype=np.float64, order="F")
        _check(lib().phm_instantiate_apply(self._h, _dp(th), th.size, xf.ctypes.data_as(_DP), n_rows,
                                           y.ctypes.data_as(_DP), m))
        self.theta = list(th)
        return y[:, 0].copy() if vec else y

    def instantiate_apply_device(self, theta, x_ptr: int, y_ptr: int, m: int = 1) -> None:
        th = _f64(theta).ravel()
        _check(lib().phm_instantiate_apply_device(self._h, _dp(th), th.size, _P(x_ptr), _P(y_ptr), m))
        self.theta = list(th)

    def apply_device(self, x_ptr: int, y_ptr: int, m: int = 1) -> None:
        _check(lib().phm_apply_device(self._h, _P(x_ptr), _P(y_ptr), m))

    def instantiate_apply_sharded_device(self, comm: "Comm", theta, x_ptr: int, y_ptr: int, m: int = 1) -> None:
        """This rank's shard of instantiate(theta) + apply, with the x-hat and
        y all-reduces over `comm`; y (original order) complete on every rank."""
        th = _f64(theta).ravel()
        _check(lib().phm_instantiate_apply_sharded(self._h, comm._h, _dp(th), th.size, x_ptr, y_ptr, m))

    def instantiate_apply_sharded(self, comm: "Comm", theta, x) -> np.ndarray:
        """Host-buffer form of instantiate_apply_sharded_device (synchronous)."""
        th = _f64(theta).ravel()
        xa = _f64(x)
        one = xa.ndim == 1
        xf = np.asfortranarray(xa.reshape(xa.shape[0], -1))
        y = np.empty_like(xf)
        _check(lib().phm_instantiate_apply_sharded_host(self._h, comm._h, _dp(th), th.size, _dp(xf), xf.shape[0],
                                                        _dp(y), xf.shape[1]))
        return y[:, 0] if one else y

    def apply_sharded_device(self, comm: "Comm", x_ptr: int, y_ptr: int, m: int = 1) -> None:
        _check(lib().phm_apply_sharded(self._h, comm._h, x_ptr, y_ptr, m))

    def apply_rows_device(self, x_ptr: int, yrows_ptr: int, m: int = 1) -> None:
        _check(lib().phm_apply_rows_device(self._h, _P(x_ptr), _P(yrows_ptr), m))

    def apply_partial_device(self, x_ptr: int, ypart_ptr: int, m: int = 1) -> None:
        """This shard's full-length partial y (tree order, n x m); sum across ranks."""
        _check(lib().phm_apply_partial_device(self._h, _P(x_ptr), _P(ypart_ptr), m))

    def instantiate_apply_partial_device(self, theta, x_ptr: int, ypart_ptr: int, m: int = 1) -> None:
        th = _f64(theta).ravel()
        _check(lib().phm_instantiate_apply_partial_device(self._h, _dp(th), th.size, _P(x_ptr), _P(ypart_ptr), m))
        self.theta = list(th)

    def far_h(self, i: int) -> np.ndarray:
        r, c = C.c_int64(), C.c_int64()
        _check(lib().phm_instance_far_h(self._h, i, None, C.byref(r), C.byref(c)))
        out = np.empty((r.value, c.value), order="F")
        _check(lib().phm_instance_far_h(self._h, i, out.ctypes.data_as(_DP), None, None))
        return out

    def near_d(self, b: int, shape) -> np.ndarray:
        out = np.empty(int(shape[0]) * int(shape[1]), dtype=np.float64)
        _check(lib().phm_instance_near_d(self._h, b, _dp(out)))
        return out.reshape((int(shape[0]), int(shape[1])), order="F")

    def class_c(self, k: int) -> np.ndarray:
        P = self.parent.info()["P"]
        out = np.empty(P * P, dtype=np.float64)
        _check(lib().phm_instance_class_c(self._h, k, _dp(out)))
        return out.reshape((P, P), order="F")

    def estimate_error(self, probe_rows: int = 200, seed: int = 0, details: bool = False):
        """estimate_error of the reference harness (harness.cpp:183-236)."""
        n = self.parent.n()
        m = min(probe_rows, n)
        err = C.c_double()
        rows = np.empty(m, dtype=np.int64)
        ex, ap, x = np.empty(m), np.empty(m), np.empty(n)
        _check(lib().phm_estimate_error(self._h, probe_rows, seed, C.byref(err), rows.ctypes.data_as(_I64P),
                                        _dp(ex), _dp(ap), _dp(x)))
        if details:
            return err.value, {"rows": rows, "exact": ex, "approx": ap, "x": x}
        return err.value

    def to_dense(self, guard: int = 8192) -> np.ndarray:
        n = self.parent.n()
        if n > guard:
            raise PhmatError("to_dense: matrix exceeds the size guard")
        out = np.empty((n, n), order="F")
        _check(lib().phm_to_dense(self._h, out.ctypes.data_as(_DP), guard))
        return out


# ---------------------------------------------------------------- functions
# --------------------------------------------------------------- multi-GPU
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, _P, C.c_int64, _P, _P)


class Comm:
    """Communicator of the row-sharded step (phm_comm): NCCL, or a Python
    callback ``fn(buf_ptr, count, stream_ptr) -> None`` that leaves the device
    buffer summed over the ranks (tests: gloo on the host)."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().phm_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, ctx: "Context", uid: bytes, rank: int, world: int) -> "Comm":
        h = _P()
        _check(lib().phm_comm_create_nccl(ctx._h, uid, rank, world, C.byref(h)))
        return cls(h)

    @classmethod
    def callback(cls, fn, rank: int, world: int) -> "Comm":
        def tramp(buf, count, stream, user):
            try:
                fn(buf, count, stream)
                return 0
            except Exception:  # reported as a failed exchange
                import traceback

                traceback.print_exc()
                return 1

        cfn = ALLREDUCE_FN(tramp)
        h = _P()
        _check(lib().phm_comm_create_callback(C.cast(cfn, _P), None, rank, world, C.byref(h)))
        return cls(h, keep=cfn)

    @classmethod
    def probe(cls, rank: int, world: int) -> "Comm":
        """No-op exchanges: times one rank's sharded step on one GPU."""
        h = _P()
        _check(lib().phm_comm_create_probe(rank, world, C.byref(h)))
        return cls(h)

    def info(self):
        r, w, k = C.c_int(), C.c_int(), C.c_int()
        _check(lib().phm_comm_info(self._h, C.byref(r), C.byref(w), C.byref(k)))
        return {"rank": r.value, "world": w.value, "nccl": bool(k.value)}

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.phm_comm_destroy(self._h)
            self._h = None


def _points(points) -> np.ndarray:
    p = np.ascontiguousarray(points, dtype=np.float64)
    if p.ndim != 2:
        raise InvalidArgument("points must be an n x d array")
    return p


def _build(points, config: PHConfig, fmt: int, ctx: Optional[Context]) -> ParametricMatrix:
    p = _points(points)
    ctx = ctx or Context.default()
    h = _P()
    cfg = config.to_c(fmt)
    _check(lib().phm_matrix_build(ctx._h, _dp(p), p.shape[0], p.shape[1], C.byref(cfg), C.byref(h)))
    return ParametricMatrix(h, ctx, fmt, config, p.shape[0], p.shape[1])


def offline_h(points, config: PHConfig, ctx: Optional[Context] = None) -> ParametricMatrix:
    """offline_h (phmatrix.hpp:82-91): tree over the unit box, blocks, TT data, upload."""
    return _build(points, config, Format.H, ctx)


def offline_h2(points, config: PHConfig, ctx: Optional[Context] = None) -> ParametricMatrix:
    """offline_h2 (phmatrix.hpp:82-91)."""
    return _build(points, config, Format.H2, ctx)


def offline_structure(points, config: PHConfig, fmt: int = Format.H2) -> ParametricMatrix:
    """Host-only build (no GPU needed): structure and offline TT data only."""
    p = _points(points)
    h = _P()
    cfg = config.to_c(fmt)
    _check(lib().phm_matrix_build_host(_dp(p), p.shape[0], p.shape[1], C.byref(cfg), C.byref(h)))
    return ParametricMatrix(h, None, fmt, config, p.shape[0], p.shape[1])


def _config_from_c(c: _Config) -> PHConfig:
    box = [(c.theta_lo[k], c.theta_hi[k]) for k in range(c.d_theta)]
    return PHConfig(spec=KernelSpec(c.family, box, bool(c.amplitude)), l_max=c.l_max, p_s=c.p_s,
                    p_theta=[c.p_theta[k] for k in range(c.d_theta)], eps=c.eps, eta=c.eta, r_max_far=c.r_max_far,
                    r_max_near=c.r_max_near, seed=c.seed, near_mode=c.near_mode,
                    translation_cache=bool(c.translation_cache), threads=c.threads, shard_rank=c.shard_rank,
                    shard_count=c.shard_count, symmetric_near=bool(c.symmetric_near))


def load_parametric(path: str, ctx: Optional[Context] = None, threads: int = 0) -> ParametricMatrix:
    """load_parametric_h / _h2 (phmatrix.hpp:160-164): HMAT v1 artifact
    written by the reference's `phmat build --artifact` (or save_parametric)."""
    ctx = ctx or Context.default()
    h = _P()
    _check(lib().phm_matrix_load(ctx._h, os.fsencode(path), threads, C.byref(h)))
    c = _Config()
    _check(lib().phm_matrix_config(h, C.byref(c)))
    pm = ParametricMatrix(h, ctx, c.format, _config_from_c(c), 0, 0)
    inf = pm.info()
    pm._n, pm._d = inf["n"], inf["d"]
    return pm


def load_parametric_structure(path: str, threads: int = 0) -> ParametricMatrix:
    """Host-only load of an HMAT v1 artifact (no GPU): structure + TT data."""
    h = _P()
    _check(lib().phm_matrix_load_host(os.fsencode(path), threads, C.byref(h)))
    c = _Config()
    _check(lib().phm_matrix_config(h, C.byref(c)))
    pm = ParametricMatrix(h, None, c.format, _config_from_c(c), 0, 0)
    inf = pm.info()
    pm._n, pm._d = inf["n"], inf["d"]
    return pm


def save_parametric(pm: ParametricMatrix, path: str) -> None:
    """save_parametric (phmatrix.hpp:157-158), HMAT v1."""
    _check(lib().phm_matrix_save(pm._h, os.fsencode(path)))


def artifact_is_h2(path: str) -> bool:
    v = C.c_int()
    _check(lib().phm_artifact_is_h2(os.fsencode(path), C.byref(v)))
    return bool(v.value)


def instantiate(pm: ParametricMatrix, theta) -> InstantiatedMatrix:
    """instantiate(pm, theta) (phmatrix.hpp:133-138): zero kernel evaluations
    in TT / snapshot near mode; domain_error outside the theta box."""
    th = _f64(theta).ravel()
    h = _P()
    _check(lib().phm_instantiate(pm._h, _dp(th), th.size, C.byref(h)))
    return InstantiatedMatrix(pm, h, th)


class Baseline:
    H_ACA, H2_HCA = 1, 2


class _BaselineParent:
    """What an instance needs from its parent for a baseline (no parametric data)."""

    def __init__(self, n: int, d: int, p_s: int, ctx):
        self._n, self.ctx = n, ctx
        self._P = p_s ** d

    def n(self) -> int:
        return self._n

    def info(self) -> dict:
        return {"P": self._P, "n": self._n}


class BaselineMatrix(InstantiatedMatrix):
    """HAcaMatrix / H2HcaMatrix (baselines.hpp:27-82) at one fixed theta:
    apply, to_dense, mean_far_rank, coupling_ratio, build times and kernel
    evaluation counts. Built by h_aca / h2_hca."""

    def info(self) -> dict:
        b = _BaselineInfo()
        _check(lib().phm_baseline_info_get(self._h, C.byref(b)))
        return {k: getattr(b, k) for k, _ in _BaselineInfo._fields_}

    def mean_far_rank(self) -> float:
        return self.info()["mean_far_rank"]

    def coupling_ratio(self) -> float:
        return self.info()["coupling_ratio"]

    def reinstantiate(self, theta) -> None:
        raise LogicError("a baseline matrix is built at a fixed theta")


def _baseline(points, config: PHConfig, method: int, theta, eps, r_max, ctx) -> BaselineMatrix:
    p = _points(points)
    ctx = ctx or Context.default()
    th = _f64(theta).ravel()
    cfg = config.to_c(Format.H if method == Baseline.H_ACA else Format.H2)
    h = _P()
    _check(lib().phm_baseline_build(ctx._h, _dp(p), p.shape[0], p.shape[1], C.byref(cfg), method, _dp(th), th.size,
                                    float(config.eps if eps is None else eps),
                                    int(config.r_max_far if r_max is None else r_max), C.byref(h)))
    return BaselineMatrix(_BaselineParent(p.shape[0], p.shape[1], config.p_s, ctx), h, th)


def h_aca(points, config: PHConfig, theta, eps: Optional[float] = None, r_max: Optional[int] = None,
          ctx: Optional[Context] = None) -> BaselineMatrix:
    """HAcaMatrix(tree, blocks, spec, theta, eps, r_max) (baselines.cpp:52-89):
    tree / blocks / kernel from the config; ACA far blocks, dense near blocks."""
    return _baseline(points, config, Baseline.H_ACA, theta, eps, r_max, ctx)


def h2_hca(points, config: PHConfig, theta, eps: Optional[float] = None, r_max: Optional[int] = None,
           ctx: Optional[Context] = None) -> BaselineMatrix:
    """H2HcaMatrix(tree, blocks, spec, theta, p_s, eps, r_max) (baselines.cpp:133-219)."""
    return _baseline(points, config, Baseline.H2_HCA, theta, eps, r_max, ctx)


def aca_partial(a, eps: float, r_max: int, seed: int):
    """aca_partial (baselines.hpp:22-24) on a dense matrix: (V, Y, capped)."""
    A = np.asfortranarray(np.asarray(a, dtype=np.float64))
    m, n = A.shape
    cap = max(1, min(m, n, r_max))
    V = np.zeros((m, cap), order="F")
    Y = np.zeros((n, cap), order="F")
    rank = C.c_int64()
    capped = C.c_int32()
    _check(lib().phm_aca_partial_dense(A.ctypes.data_as(_DP), m, n, eps, r_max, seed, C.byref(rank), C.byref(capped),
                                       V.ctypes.data_as(_DP), Y.ctypes.data_as(_DP)))
    t = rank.value
    return V[:, :t].copy(order="F"), Y[:, :t].copy(order="F"), bool(capped.value)


def instantiate_batch(pm: ParametricMatrix, thetas) -> List[InstantiatedMatrix]:
    """theta-batched instantiate for sweeps: thetas (count, d_theta) -> count
    instances; in snapshot mode the snapshots are read once for the batch.
    Equal, bit for bit, to [instantiate(pm, t) for t in thetas]."""
    th = np.ascontiguousarray(_f64(thetas).reshape(len(thetas), -1))
    count, dt = th.shape
    hs = (_P * count)()
    _check(lib().phm_instantiate_batch(pm._h, _dp(th), dt, count, C.cast(hs, _P)))
    return [InstantiatedMatrix(pm, _P(hs[b]), th[b]) for b in range(count)]


def reinstantiate_batch(insts: Sequence[InstantiatedMatrix], thetas) -> None:
    """In place: insts[b] re-instantiated at thetas[b], one snapshot pass."""
    th = np.ascontiguousarray(_f64(thetas).reshape(len(insts), -1))
    hs = (_P * len(insts))(*[i._h for i in insts])
    _check(lib().phm_reinstantiate_batch(C.cast(hs, _P), len(insts), _dp(th), th.shape[1]))
    for b, i in enumerate(insts):
        i.theta = list(th[b])


def metrics(pm: ParametricMatrix) -> dict:
    """StructureMetrics (phmatrix.hpp:141-153)."""
    inf = pm.info()
    return {k: inf[k] for k in ("n", "storage_entries", "storage_gb", "nf_ratio", "ff_ratio", "coupling_ratio",
                                "rank", "c_sp", "n_classes", "n_far", "n_near")} | {"m_a": inf["n_classes"]}


def generate_points(n: int, d: int, seed: int) -> np.ndarray:
    """generate_points (harness.cpp:174-181): U[0,1)^d, row-major fill."""
    out = np.empty((n, d), dtype=np.float64)
    _check(lib().phm_generate_points(n, d, seed, _dp(out)))
    return out


def generate_mixture_points(n: int, d: int, clusters: int, sigma: float, seed: int) -> np.ndarray:
    out = np.empty((n, d), dtype=np.float64)
    _check(lib().phm_generate_mixture_points(n, d, clusters, sigma, seed, _dp(out)))
    return out


def generate_normal(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(lib().phm_generate_normal(n, seed, _dp(out)))
    return out


def _unpack_cores(nc, dims, data):
    cores, off = [], 0
    for r0, m, r1 in dims[: 3 * nc].reshape(-1, 3):
        sz = int(r0 * m * r1)
        cores.append(data[off: off + sz].reshape((int(r0), int(m), int(r1)), order="F").copy())
        off += sz
    return cores


def tt_cross(tensor, eps=1e-5, r_max=120, seed=0, round_after=True):
    """TT-cross of a dense tensor (first index fastest; pass a Fortran-ordered
    array or any array whose F-order flattening is the tensor). Returns
    (cores, info) with cores shaped (r0, m, r1)."""
    t = np.asfortranarray(tensor, dtype=np.float64)
    flat = np.ascontiguousarray(t.ravel(order="F"))
    dims = np.array(t.shape, dtype=np.int64)
    nc, ln, ev = C.c_int32(), C.c_int64(), C.c_uint64()
    flags = np.zeros(2, dtype=np.int32)
    est = C.c_double()
    cd = np.zeros(3 * len(dims), dtype=np.int64)
    args = (_dp(flat), dims.ctypes.data_as(_I64P), len(dims), eps, r_max, seed, 1 if round_after else 0,
            C.byref(nc), cd.ctypes.data_as(_I64P))
    _check(lib().phm_tt_cross_dense(*args, None, 0, C.byref(ln), C.byref(ev), flags.ctypes.data_as(_I32P),
                                    C.byref(est)))
    data = np.empty(ln.value, dtype=np.float64)
    _check(lib().phm_tt_cross_dense(*args, _dp(data), ln.value, C.byref(ln), C.byref(ev),
                                    flags.ctypes.data_as(_I32P), C.byref(est)))
    return _unpack_cores(nc.value, cd, data), {"evals": ev.value, "rank_capped": bool(flags[0]),
                                               "converged": bool(flags[1]), "est_rel_error": est.value}


def tt_round(cores, eps=0.0, abs_budget=-1.0):
    dims = np.array([c.shape for c in cores], dtype=np.int64).ravel()
    data = np.ascontiguousarray(np.concatenate([np.asarray(c).ravel(order="F") for c in cores]))
    nc, ln = C.c_int32(), C.c_int64()
    od = np.zeros(3 * len(cores), dtype=np.int64)
    _check(lib().phm_tt_round(len(cores), dims.ctypes.data_as(_I64P), _dp(data), eps, abs_budget, C.byref(nc),
                              od.ctypes.data_as(_I64P), None, 0, C.byref(ln)))
    out = np.empty(ln.value, dtype=np.float64)
    _check(lib().phm_tt_round(len(cores), dims.ctypes.data_as(_I64P), _dp(data), eps, abs_budget, C.byref(nc),
                              od.ctypes.data_as(_I64P), _dp(out), ln.value, C.byref(ln)))
    return _unpack_cores(nc.value, od, out)


def tt_full(cores) -> np.ndarray:
    cur = np.asarray(cores[0]).reshape(-1, cores[0].shape[2], order="F")
    dims = [cores[0].shape[1]]
    for c in cores[1:]:
        r0, m, r1 = c.shape
        cur = (cur @ np.asarray(c).reshape(r0, m * r1, order="F")).reshape(-1, r1, order="F")
        dims.append(m)
    return cur.reshape(dims, order="F")


def theta_draws(lo: float, hi: float, count: int, seed: int) -> np.ndarray:
    """run_experiment's theta samples (harness.cpp:254-260)."""
    out = np.empty(count, dtype=np.float64)
    _check(lib().phm_theta_draws(lo, hi, count, seed, _dp(out)))
    return out
