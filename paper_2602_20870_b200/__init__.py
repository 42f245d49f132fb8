"""B200-native FGFRFT hot path -- Python binding of the C ABI (include/fgfrft_b200.h).

The product is ``libfgfrft_b200.so`` (hand-written sm_100a kernels behind an ``extern "C"``
boundary); the C++ drop-in header ``include/fgfrft/transform.hpp`` is the reference-facing
API. This module is a thin ctypes binding with the same names and error behaviour as the
reference (proj/include/fgfrft/transform.hpp:41-148, sinc.hpp:50-63, errors.hpp:36-62) so
tests and bench.py read like the reference's own tests. There is no CPU fallback: if the
shared library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import math
import os
import warnings
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "ParameterError", "ShapeError", "CapacityError", "NumericalError", "DEFAULT_MEMORY_BUDGET",
    "C128", "C64", "lib", "sinc_coeffs", "fnv1a64", "PowerCache", "build_power_cache",
    "FracOperator", "fgfrft_matrix", "fgfrft_grad", "apply_forward", "apply_inverse",
    "apply_series", "dlda", "mse_step", "launch_count",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfgfrft_b200.so")
DEFAULT_MEMORY_BUDGET = 4 << 30  # transform.hpp:17
C128, C64 = 0, 1
Q, DQ = 0, 1


class ParameterError(ValueError):
    """errors.hpp:36 parameter_error."""


class ShapeError(ParameterError):
    """errors.hpp:40 shape_error."""


class CapacityError(ParameterError):
    """errors.hpp:44 capacity_error."""


class NumericalError(ArithmeticError):
    """errors.hpp:48 numerical_error (also CUDA / NCCL failures)."""


class OptimizerError(NumericalError):
    """errors.hpp optimizer_error: non-finite loss or gradient inside a learner."""


class IoError(RuntimeError):
    """errors.hpp io_error: a file cannot be opened or written."""


class ParseError(IoError):
    """errors.hpp parse_error: a malformed or truncated file."""


_STATUS = {1: ParameterError, 2: ShapeError, 3: CapacityError, 4: NumericalError, 5: NumericalError,
           6: NumericalError, 7: OptimizerError, 8: IoError, 9: ParseError}

_LIB = None


def lib() -> ctypes.CDLL:
    """Load libfgfrft_b200.so (raises if it has not been built: no silent fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() or paper_2602_20870_b200/build.sh")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, i64, u64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    pp = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "fgfrft_last_error": (ctypes.c_char_p, []),
        "fgfrft_version": (ctypes.c_char_p, []),
        "fgfrft_launch_count": (u64, []),
        "fgfrft_profile_enable": (i, [i]),
        "fgfrft_profile_read": (i, [vp, vp, i]),
        "fgfrft_profile_trace": (i, [vp, vp, vp, i, vp]),
        "fgfrft_sinc_coeffs": (i, [d, i, vp, vp]),
        "fgfrft_fnv1a64": (u64, [vp, ctypes.c_size_t]),
        "fgfrft_cache_create": (i, [vp, i64, i, u64, i, i, pp]),
        "fgfrft_cache_create_from_powers": (i, [vp, vp, i64, i, u64, i, i, pp]),
        "fgfrft_cache_destroy": (i, [vp]),
        "fgfrft_cache_info": (i, [vp, vp, vp, vp, vp, vp]),
        "fgfrft_cache_power": (i, [vp, i, vp]),
        "fgfrft_cache_is_real": (i, [vp, vp]),
        "fgfrft_cache_route_info": (i, [vp, vp, vp]),
        "fgfrft_cache_verify": (i, [vp, vp]),
        "fgfrft_cache_set_stream": (i, [vp, vp]),
        "fgfrft_cache_device_slab": (i, [vp, i, pp]),
        "fgfrft_cache_device_bytes": (i, [vp, vp]),
        "fgfrft_synthesize": (i, [vp, vp, i, i, i, vp]),
        "fgfrft_synthesize_dev": (i, [vp, vp, i, i, i, vp]),
        "fgfrft_apply": (i, [vp, vp, i, i, i, vp, i64, vp]),
        "fgfrft_apply_dev": (i, [vp, vp, i, i, i, vp, i64, vp]),
        "fgfrft_apply_matrix": (i, [vp, i64, i, vp, i64, vp, i]),
        "fgfrft_dlda": (i, [vp, vp, i, vp, vp, i64, vp, vp]),
        "fgfrft_dlda_dev": (i, [vp, vp, i, vp, vp, i64, vp, vp]),
        "fgfrft_mse_step": (i, [vp, vp, i, vp, vp, i64, vp, vp, vp]),
        "fgfrft_mse_step_dev": (i, [vp, vp, i, vp, vp, i64, vp, vp, vp]),
        "fgfrft_shard_create": (i, [vp, i64, i, i64, i64, u64, i, pp]),
        "fgfrft_shard_destroy": (i, [vp]),
        "fgfrft_shard_info": (i, [vp, vp, vp, vp, vp, vp]),
        "fgfrft_shard_set_stream": (i, [vp, vp]),
        "fgfrft_shard_synthesize_dev": (i, [vp, vp, i, i, vp]),
        "fgfrft_shard_apply_dev": (i, [vp, vp, i, vp, i64, vp]),
        "fgfrft_shard_mse_partial_dev": (i, [vp, vp, i, vp, vp, i64, vp, vp, vp]),
        "fgfrft_batch_create": (i, [vp, i64, i64, i, i, pp]),
        "fgfrft_batch_destroy": (i, [vp]),
        "fgfrft_batch_set_stream": (i, [vp, vp]),
        "fgfrft_batch_forward_dev": (i, [vp, vp, i, vp, i64, vp]),
        "fgfrft_batch_dlda_dev": (i, [vp, vp, i, vp, vp, i64, vp]),
        "fgfrft_cache_set_engine": (i, [vp, i]),
        "fgfrft_int8_digits": (i, []),
        "fgfrft_step_int8_digits": (i, []),
        "fgfrft_denoise_create": (i, [vp, vp, vp, i64, pp]),
        "fgfrft_denoise_destroy": (i, [vp]),
        "fgfrft_denoise_eval": (i, [vp, d, vp, vp, vp, vp]),
        "fgfrft_denoise_fit": (i, [vp, i, d, d, vp, vp, vp, vp, vp, vp, vp]),
        "fgfrft_cache_orthogonality": (i, [vp, vp]),
        "fgfrft_cache_prepare": (i, [vp]),
        "fgfrft_cache_set_order_window": (i, [vp, d, d]),
        "fgfrft_cache_order_window": (i, [vp, vp, vp, vp]),
        "fgfrft_dgemm_int8_dev": (i, [i, i, i64, i64, i64, vp, i64, vp, i64, vp, i64, i, vp]),
        "fgfrft_spectrum_create": (i, [vp, vp, i64, i, pp]),
        "fgfrft_spectrum_decompose": (i, [vp, i64, i, pp]),
        "fgfrft_spectrum_destroy": (i, [vp]),
        "fgfrft_spectrum_info": (i, [vp, vp, vp]),
        "fgfrft_spectrum_vectors": (i, [vp, vp]),
        "fgfrft_spectrum_set_stream": (i, [vp, vp]),
        "fgfrft_exact": (i, [vp, vp, i, i, vp]),
        "fgfrft_exact_dev": (i, [vp, vp, i, i, vp]),
        "fgfrft_cascade_create": (i, [vp, vp, d, i, pp]),
        "fgfrft_cascade_destroy": (i, [vp]),
        "fgfrft_cascade_eval": (i, [vp, vp, vp, vp]),
        "fgfrft_cascade_learn": (i, [vp, d, i, d, vp, vp, vp, vp]),
        "fgfrft_cache_save": (i, [vp, ctypes.c_char_p]),
        "fgfrft_shard_mse_dlda_partial_dev": (i, [vp, vp, i, vp, vp, i64, vp, vp, vp]),
        "fgfrft_shard_apply_gather_dev": (i, [vp, vp, i, vp, i64, vp, vp, i]),
        "fgfrft_denoise_create_exact": (i, [vp, vp, vp, i64, i, pp]),
        "fgfrft_denoise_create_ex": (i, [vp, vp, vp, i64, i, pp]),
        "fgfrft_zgemm_int8_dev": (i, [i, i, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp]),
        "fgfrft_denoise_reconstruct": (i, [vp, d, vp, vp]),
        "fgfrft_ipc_get": (i, [vp, vp, vp]),
        "fgfrft_ipc_open": (i, [vp, i, pp]),
        "fgfrft_ipc_close": (i, [vp]),
        "fgfrft_cache_load": (i, [ctypes.c_char_p, u64, i, pp]),
        "fgfrft_comm_unique_id": (i, [vp]),
        "fgfrft_comm_create": (i, [vp, i, i, i, pp]),
        "fgfrft_comm_create_all": (i, [i, vp, vp]),
        "fgfrft_comm_destroy": (i, [vp]),
        "fgfrft_comm_info": (i, [vp, vp, vp, vp]),
        "fgfrft_pshard_plan": (i, [i64, i, vp]),
        "fgfrft_pshard_create": (i, [vp, i64, i, u64, vp, pp]),
        "fgfrft_pshard_create_local": (i, [vp, i64, i, u64, i, i, i, pp]),
        "fgfrft_pshard_destroy": (i, [vp]),
        "fgfrft_pshard_info": (i, [vp, vp, vp, vp, vp, vp, vp, vp]),
        "fgfrft_pshard_set_stream": (i, [vp, vp]),
        "fgfrft_pshard_partial_dev": (i, [vp, vp, i, i, vp, i64, vp]),
        "fgfrft_pshard_mse_step_dev": (i, [vp, vp, i, vp, vp, i64, vp, vp]),
        "fgfrft_pshard_mse_step": (i, [vp, vp, i, vp, vp, i64, vp, vp]),
        "fgfrft_pshard_apply_dev": (i, [vp, vp, i, i, vp, i64, vp]),
        "fgfrft_pshard_partial_scatter_dev": (i, [vp, vp, i, i, vp, i64, vp, i]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


def exported_symbols():
    return [
        "fgfrft_last_error", "fgfrft_version", "fgfrft_launch_count", "fgfrft_profile_enable",
        "fgfrft_profile_read", "fgfrft_profile_trace", "fgfrft_sinc_coeffs", "fgfrft_fnv1a64",
        "fgfrft_cache_create", "fgfrft_cache_create_from_powers", "fgfrft_cache_destroy", "fgfrft_cache_info",
        "fgfrft_cache_is_real", "fgfrft_cache_route_info",
        "fgfrft_cache_power", "fgfrft_cache_verify", "fgfrft_cache_set_stream", "fgfrft_cache_device_slab",
        "fgfrft_cache_device_bytes", "fgfrft_synthesize", "fgfrft_synthesize_dev", "fgfrft_apply",
        "fgfrft_apply_dev", "fgfrft_apply_matrix", "fgfrft_dlda", "fgfrft_dlda_dev", "fgfrft_mse_step",
        "fgfrft_mse_step_dev", "fgfrft_shard_create", "fgfrft_shard_destroy", "fgfrft_shard_info",
        "fgfrft_shard_set_stream", "fgfrft_shard_synthesize_dev", "fgfrft_shard_apply_dev",
        "fgfrft_shard_mse_partial_dev", "fgfrft_batch_create", "fgfrft_batch_destroy", "fgfrft_batch_set_stream",
        "fgfrft_batch_forward_dev", "fgfrft_batch_dlda_dev", "fgfrft_dgemm_int8_dev", "fgfrft_cache_set_engine",
        "fgfrft_int8_digits", "fgfrft_step_int8_digits", "fgfrft_cache_orthogonality", "fgfrft_denoise_create", "fgfrft_denoise_destroy",
        "fgfrft_denoise_eval", "fgfrft_denoise_fit",
        "fgfrft_cache_prepare", "fgfrft_cache_set_order_window", "fgfrft_cache_order_window", "fgfrft_spectrum_create", "fgfrft_spectrum_decompose", "fgfrft_spectrum_destroy",
        "fgfrft_spectrum_info", "fgfrft_spectrum_vectors", "fgfrft_spectrum_set_stream", "fgfrft_exact",
        "fgfrft_exact_dev", "fgfrft_cascade_create", "fgfrft_cascade_destroy", "fgfrft_cascade_eval",
        "fgfrft_cascade_learn", "fgfrft_cache_save", "fgfrft_cache_load", "fgfrft_shard_mse_dlda_partial_dev",
        "fgfrft_shard_apply_gather_dev", "fgfrft_ipc_get", "fgfrft_ipc_open", "fgfrft_ipc_close",
        "fgfrft_denoise_create_exact", "fgfrft_denoise_reconstruct", "fgfrft_zgemm_int8_dev",
        "fgfrft_denoise_create_ex", "fgfrft_comm_unique_id", "fgfrft_comm_create", "fgfrft_comm_create_all",
        "fgfrft_comm_destroy", "fgfrft_comm_info", "fgfrft_pshard_plan", "fgfrft_pshard_create",
        "fgfrft_pshard_create_local", "fgfrft_pshard_destroy", "fgfrft_pshard_info", "fgfrft_pshard_set_stream",
        "fgfrft_pshard_partial_dev", "fgfrft_pshard_mse_step_dev", "fgfrft_pshard_mse_step",
        "fgfrft_pshard_apply_dev", "fgfrft_pshard_partial_scatter_dev",
    ]


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().fgfrft_last_error().decode(errors="replace")
        raise _STATUS.get(rc, NumericalError)(msg)


def launch_count() -> int:
    return int(lib().fgfrft_launch_count())


ENGINE_AUTO, ENGINE_DMMA, ENGINE_INT8, ENGINE_INT8_COMBINE = 0, 1, 2, 3

KERNEL_CLASSES = ("synthesis", "dmma_zgemm", "power_dots", "elementwise", "int8_gemm", "slicing", "combine",
                  "node_operators")


def profile_enable(on: bool = True) -> None:
    _check(lib().fgfrft_profile_enable(int(on)))


def profile_read(reset: bool = True):
    """{class: (total_ms, launches)} from CUDA events recorded around each launch."""
    ms = np.zeros(8)
    cnt = np.zeros(8, dtype=np.int64)
    _check(lib().fgfrft_profile_read(_ptr(ms), _ptr(cnt), int(reset)))
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}


def profile_trace(cap: int = 4096):
    """[(class, start_ms, end_ms)] of the recorded launches (call before profile_read(reset=True))."""
    cls = np.zeros(cap, dtype=np.int32)
    t0, t1 = np.zeros(cap), np.zeros(cap)
    cnt = ctypes.c_int()
    _check(lib().fgfrft_profile_trace(_ptr(cls), _ptr(t0), _ptr(t1), cap, ctypes.addressof(cnt)))
    m = min(cnt.value, cap)
    return [(KERNEL_CLASSES[cls[i]], float(t0[i]), float(t1[i])) for i in range(m)]


def _cm(a: np.ndarray) -> np.ndarray:
    """Column-major complex128 view/copy (the Eigen::MatrixXcd layout)."""
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a, dtype=np.complex128)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _alphas(alphas) -> np.ndarray:
    return np.ascontiguousarray(np.atleast_1d(np.asarray(alphas, dtype=np.float64)))


# ----------------------------------------------------------------------------- sinc.hpp

def sinc_coeffs(alpha: float, l: int):
    """sinc.hpp:50-63 -> (c, dc) with entry [n + l] = term n."""
    c = np.empty(max(2 * l + 1, 1))
    dc = np.empty(max(2 * l + 1, 1))
    _check(lib().fgfrft_sinc_coeffs(float(alpha), int(l), _ptr(c), _ptr(dc)))
    return c, dc


def fnv1a64(buf: np.ndarray) -> int:
    b = np.ascontiguousarray(buf)
    return int(lib().fgfrft_fnv1a64(_ptr(b), b.nbytes))


def content_fingerprint(f: np.ndarray) -> int:
    """gft.hpp:46-48 over the column-major bytes."""
    fc = _cm(f)
    return fnv1a64(np.ascontiguousarray(fc.T))


# ----------------------------------------------------------------------------- transform.hpp

class PowerCache:
    """transform.hpp:41-80 on the GPU. ``PowerCache(f, l, memory_budget)`` builds P_k = F^k,
    k = 1..l on device (DMMA GEMM chain). Move-only in spirit: the handle owns device memory."""

    def __init__(self, f: np.ndarray, l: int, memory_budget: int = DEFAULT_MEMORY_BUDGET, dtype: int = C128,
                 device: int = 0, powers: Optional[np.ndarray] = None):
        self._h = ctypes.c_void_p()
        fc = _cm(f)
        if fc.shape[0] != fc.shape[1]:
            raise ShapeError("PowerCache: F must be square")
        n = fc.shape[0]
        if powers is None:
            _check(lib().fgfrft_cache_create(_ptr(fc), n, int(l), int(memory_budget), dtype, device,
                                             ctypes.byref(self._h)))
        else:
            p = np.ascontiguousarray(powers, dtype=np.complex128)  # [l, n, n] slabs of P_k^T (col-major P_k)
            _check(lib().fgfrft_cache_create_from_powers(_ptr(p), _ptr(fc), n, int(l), int(memory_budget), dtype,
                                                         device, ctypes.byref(self._h)))
        self._n, self._l, self.dtype, self.device = n, int(l), dtype, device
        fp = ctypes.c_uint64()
        _check(lib().fgfrft_cache_info(self._h, None, None, ctypes.addressof(fp), None, None))
        self._fp = fp.value

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().fgfrft_cache_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def l(self) -> int:
        return self._l

    def n(self) -> int:
        return self._n

    def fingerprint(self) -> int:
        return self._fp

    def route_info(self):
        """(route, nodes) of the last MSE step: 0 synthesis, 1 power products, 2 node interpolation,
        3 packed (Q, dQ/da from the packed slabs + one Ozaki GEMM [Y; dY] = [Q; dQ] X), 4 the same
        step with Q, dQ/da synthesised on the INT8 tensor cores from the digit cache, 5 the same step
        with Q, dQ/da interpolated from the order window's node operators (nodes = their count)."""
        r, k = ctypes.c_int(), ctypes.c_int()
        _check(lib().fgfrft_cache_route_info(self._h, ctypes.addressof(r), ctypes.addressof(k)))
        return r.value, k.value

    def is_real(self) -> bool:
        v = ctypes.c_int()
        _check(lib().fgfrft_cache_is_real(self._h, ctypes.addressof(v)))
        return bool(v.value)

    def power(self, k: int) -> np.ndarray:
        out = np.empty((self._n, self._n), dtype=np.complex128, order="F")
        _check(lib().fgfrft_cache_power(self._h, int(k), _ptr(out)))
        return out

    def verify(self, f: np.ndarray) -> None:
        fc = _cm(f)
        _check(lib().fgfrft_cache_verify(self._h, _ptr(fc)))

    def set_stream(self, stream_handle: int) -> None:
        _check(lib().fgfrft_cache_set_stream(self._h, ctypes.c_void_p(stream_handle)))

    def set_engine(self, engine: int) -> None:
        """ENGINE_AUTO, ENGINE_DMMA (FP64 tensor cores, synthesis + GEMM per order) or ENGINE_INT8
        (real F: INT8 tensor-core power products, see fgfrft_cache_set_engine)."""
        _check(lib().fgfrft_cache_set_engine(self._h, int(engine)))

    def orthogonality(self) -> float:
        """||F^T F - I||_F / sqrt(n) measured at build (real caches; -1 otherwise)."""
        r = ctypes.c_double()
        _check(lib().fgfrft_cache_orthogonality(self._h, ctypes.addressof(r)))
        return r.value

    def prepare(self) -> None:
        """Build lazily-built device structures (INT8 digit slices of the cache) now."""
        _check(lib().fgfrft_cache_prepare(self._h))

    def set_order_window(self, lo: float, hi: float) -> int:
        """Declare the orders the caller will step with (fgfrft_cache_set_order_window): r exact node
        operators at the Chebyshev nodes of [lo, hi]; one / two-order steps and applies with orders
        inside take them instead of the L packed powers. hi <= lo clears. Returns r."""
        _check(lib().fgfrft_cache_set_order_window(self._h, float(lo), float(hi)))
        return self.order_window()[2]

    def order_window(self):
        """(lo, hi, nodes) of the declared order window (nodes 0: none)."""
        lo, hi, r = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        _check(lib().fgfrft_cache_order_window(self._h, ctypes.addressof(lo), ctypes.addressof(hi),
                                               ctypes.addressof(r)))
        return lo.value, hi.value, r.value

    def device_bytes(self) -> int:
        b = ctypes.c_uint64()
        _check(lib().fgfrft_cache_device_bytes(self._h, ctypes.addressof(b)))
        return b.value

    def save(self, path: str) -> None:
        """Write F, the resident slabs and their checksum (fgfrft_cache_save)."""
        _check(lib().fgfrft_cache_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str, memory_budget: int = DEFAULT_MEMORY_BUDGET, device: int = 0) -> "PowerCache":
        """Rebuild a cache from a file written by save() (no power recursion)."""
        self = cls.__new__(cls)
        self._h = ctypes.c_void_p()
        _check(lib().fgfrft_cache_load(os.fsencode(path), int(memory_budget), int(device), ctypes.byref(self._h)))
        n, l, fp, dt = ctypes.c_int64(), ctypes.c_int(), ctypes.c_uint64(), ctypes.c_int()
        _check(lib().fgfrft_cache_info(self._h, ctypes.addressof(n), ctypes.addressof(l), ctypes.addressof(fp),
                                       ctypes.addressof(dt), None))
        self._n, self._l, self._fp, self.dtype, self.device = n.value, l.value, fp.value, dt.value, device
        return self


def build_power_cache(f, l, memory_budget=DEFAULT_MEMORY_BUDGET, **kw) -> PowerCache:
    """transform.hpp:82-85."""
    return PowerCache(f, l, memory_budget, **kw)


class FracOperator:
    """transform.hpp:89-93: {q, alpha, l}; l = 0 marks an exact spectral operator."""

    def __init__(self, q: np.ndarray, alpha: float, l: int):
        self.q, self.alpha, self.l = q, alpha, l


def _warn_window(alpha: float, l: int) -> None:
    if abs(alpha) > l + 1.0:  # transform.hpp:97-104
        warnings.warn(f"order alpha = {alpha:g} lies outside the series window [-{l + 1}, {l + 1}]; "
                      "coefficient mass concentrates in dropped terms")


def synthesize(cache: PowerCache, alphas, truncation: int = 0, which: int = Q) -> np.ndarray:
    """Multi-order synthesis: returns [A, n, n] with out[a] = Q(alpha_a) (column-major views)."""
    al = _alphas(alphas)
    buf = np.empty((len(al), cache.n(), cache.n()), dtype=np.complex128)  # slab a = Q_a^T row-major
    _check(lib().fgfrft_synthesize(cache.handle, _ptr(al), len(al), int(truncation), which, _ptr(buf)))
    return np.transpose(buf, (0, 2, 1))


def fgfrft_matrix(cache: PowerCache, alpha: float, truncation: int = 0) -> FracOperator:
    """transform.hpp:111-123."""
    l = cache.l() if truncation == 0 else truncation
    if l < 1 or l > cache.l():
        raise ParameterError("fgfrft_matrix: truncation exceeds the cached power set")
    _warn_window(alpha, l)
    return FracOperator(synthesize(cache, [alpha], truncation, Q)[0], float(alpha), l)


def fgfrft_grad(cache: PowerCache, alpha: float) -> np.ndarray:
    """transform.hpp:127-136."""
    _warn_window(alpha, cache.l())
    return synthesize(cache, [alpha], 0, DQ)[0]


def apply_forward(op: FracOperator, x: np.ndarray, device: int = 0) -> np.ndarray:
    """transform.hpp:138-141: Q X on the DMMA GEMM."""
    xc = _cm(x)
    q = _cm(op.q)
    if xc.shape[0] != q.shape[1]:
        raise ShapeError("apply_forward: signal length does not match operator")
    y = np.empty_like(xc, order="F")
    _check(lib().fgfrft_apply_matrix(_ptr(q), q.shape[0], 0, _ptr(xc), xc.shape[1], _ptr(y), device))
    return y


def apply_inverse(op: FracOperator, x: np.ndarray, device: int = 0) -> np.ndarray:
    """transform.hpp:145-148: Q^H X."""
    xc = _cm(x)
    q = _cm(op.q)
    if xc.shape[0] != q.shape[0]:
        raise ShapeError("apply_inverse: signal length does not match operator")
    y = np.empty_like(xc, order="F")
    _check(lib().fgfrft_apply_matrix(_ptr(q), q.shape[0], 1, _ptr(xc), xc.shape[1], _ptr(y), device))
    return y


def apply_series(cache: PowerCache, alphas, x: np.ndarray, truncation: int = 0, inverse: bool = False) -> np.ndarray:
    """Extension: Y_a = Q(alpha_a) X (or Q^H X) for many orders without a host round trip of Q.
    Returns [A, n, b] where out[a] is column-major n x b."""
    al = _alphas(alphas)
    xc = _cm(x)
    if xc.shape[0] != cache.n():
        raise ShapeError("apply_forward: signal length does not match operator")
    b = xc.shape[1]
    y = np.empty((len(al), b, cache.n()), dtype=np.complex128)
    _check(lib().fgfrft_apply(cache.handle, _ptr(al), len(al), int(truncation), int(inverse), _ptr(xc), b, _ptr(y)))
    return np.transpose(y, (0, 2, 1))


def dlda(cache: PowerCache, alphas, g: Sequence[np.ndarray], x: np.ndarray):
    """Extension: s[a, k + L] = Re<G_a, F^k X> and dL/dalpha_a = sum_k c'_k s[a, k + L]."""
    al = _alphas(alphas)
    xc = _cm(x)
    b = xc.shape[1]
    gs = np.stack([np.ascontiguousarray(_cm(gi).T) for gi in g]) if len(al) else np.empty(0)
    if gs.shape != (len(al), b, cache.n()) or xc.shape[0] != cache.n():
        raise ShapeError("dlda: cotangent / signal shape mismatch")
    s = np.empty((len(al), 2 * cache.l() + 1))
    out = np.empty(len(al))
    _check(lib().fgfrft_dlda(cache.handle, _ptr(al), len(al), _ptr(gs), _ptr(xc), b, _ptr(s), _ptr(out)))
    return out, s


def mse_step(cache: PowerCache, alphas, x: np.ndarray, x_clean: np.ndarray, want_y: bool = False):
    """Extension: for each order, loss = ||Q X - Xc||^2/(n b) and dloss/dalpha (host buffers)."""
    al = _alphas(alphas)
    xc = _cm(x)
    xcl = _cm(x_clean)
    if xc.shape != xcl.shape or xc.shape[0] != cache.n():
        raise ShapeError("mse_step: signal shape mismatch")
    b = xc.shape[1]
    loss = np.empty(len(al))
    dl = np.empty(len(al))
    y = np.empty((len(al), b, cache.n()), dtype=np.complex128) if want_y else None
    _check(lib().fgfrft_mse_step(cache.handle, _ptr(al), len(al), _ptr(xc), _ptr(xcl), b,
                                 _ptr(y) if want_y else None, _ptr(loss), _ptr(dl)))
    return loss, dl, (np.transpose(y, (0, 2, 1)) if want_y else None)


class GraphBatch:
    """Config-5 shape: many independent small graphs (n <= 64), complex64, H orders per graph.
    Device buffers are torch tensors; forward/dlda are stream-ordered with torch's current stream."""

    def __init__(self, fs: np.ndarray, l: int, device: int = 0):
        import torch
        self.torch = torch
        fs = np.ascontiguousarray(np.asarray(fs, dtype=np.complex128).transpose(0, 2, 1))  # column-major slabs
        self.graphs, self.n = fs.shape[0], fs.shape[1]
        self.l, self.device = int(l), device
        self._h = ctypes.c_void_p()
        _check(lib().fgfrft_batch_create(fs.ctypes.data, self.graphs, self.n, self.l, device, ctypes.byref(self._h)))
        _check(lib().fgfrft_batch_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)))

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().fgfrft_batch_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, alphas, x):
        """alphas: [G, H] float64 tensor (device); x: [G, C, n] complex64 tensor (device).
        Returns y [G, H, C, n] complex64 (y[g, h] is the column-major n x C block)."""
        t = self.torch
        G, H = alphas.shape
        C = x.shape[1]
        y = t.empty((G, H, C, self.n), dtype=t.complex64, device=x.device)
        _check(lib().fgfrft_batch_forward_dev(self._h, alphas.data_ptr(), H, x.data_ptr(), C, y.data_ptr()))
        return y

    def dlda(self, alphas, g, x):
        t = self.torch
        G, H = alphas.shape
        out = t.empty((G, H), dtype=t.float64, device=x.device)
        _check(lib().fgfrft_batch_dlda_dev(self._h, alphas.data_ptr(), H, g.data_ptr(), x.data_ptr(), x.shape[1],
                                           out.data_ptr()))
        return out


def dgemm_int8(a, b, slices: int = 0):
    """C = A B (real float64 torch CUDA tensors) on the INT8 tensor cores (Ozaki scheme), through
    fgfrft_dgemm_int8_dev. Row-major torch operands are passed as transposed column-major ones;
    the result is column-major (m x n) in memory, returned as a strided (m, n) view."""
    import torch
    assert a.dtype == torch.float64 and b.dtype == torch.float64 and a.is_cuda and b.is_cuda
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    a = a.contiguous()
    b = b.contiguous()
    ct = torch.empty((n, m), dtype=torch.float64, device=a.device)
    _check(lib().fgfrft_dgemm_int8_dev(1, 1, m, n, k, a.data_ptr(), k, b.data_ptr(), n, ct.data_ptr(), m, slices,
                                       ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)))
    return ct.t()


def zgemm_int8(a, b, op_a: str = "N", op_b: str = "N"):
    """C = op(A) op(B) for complex128 torch CUDA tensors on the INT8 tensor cores (one real Ozaki
    GEMM with K doubled), through fgfrft_zgemm_int8_dev. op: "N", "T" or "C" (conjugate
    transpose). Operands are passed as column-major (a torch (r, c) row-major tensor is the
    column-major c x r matrix of its transpose)."""
    import torch
    assert a.dtype == torch.complex128 and b.dtype == torch.complex128 and a.is_cuda and b.is_cuda
    code = {"N": 0, "T": 1, "C": 2}
    # column-major views: A_cm = a^T (shape (a.shape[1], a.shape[0])), likewise B
    acm = a.contiguous()
    bcm = b.contiguous()
    ar, ac = acm.shape[1], acm.shape[0]   # column-major rows / cols
    br, bc = bcm.shape[1], bcm.shape[0]
    m, k = (ar, ac) if op_a == "N" else (ac, ar)
    k2, n = (br, bc) if op_b == "N" else (bc, br)
    assert k == k2
    ct = torch.empty((n, m), dtype=torch.complex128, device=a.device)
    _check(lib().fgfrft_zgemm_int8_dev(code[op_a], code[op_b], m, n, k, acm.data_ptr(), ar, bcm.data_ptr(), br,
                                       ct.data_ptr(), m, ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)))
    return ct  # column-major m x n (i.e. ct.T is C)


class DenoiseProblem:
    """GPU-resident denoising learner (learn.hpp:168-516 on the device): y, x_ref are n x C real
    host arrays; eval(alpha, h) -> (loss, grad_alpha, grad_h); fit(...) runs Adam.
    ``DenoiseProblem(cache, y, x, loss_on_real=False)``: fast backend (Q and dQ synthesised from the
    cache, five GEMMs per evaluation; real or complex F);
    ``DenoiseProblem.exact(eig, y, x, loss_on_real)``: exact backend on a device spectrum."""

    def __init__(self, cache: Optional[PowerCache], y: np.ndarray, x_ref: np.ndarray,
                 eig: Optional["UnitaryEigen"] = None, loss_on_real: bool = False):
        y = np.asfortranarray(np.asarray(y, dtype=np.float64))
        x = np.asfortranarray(np.asarray(x_ref, dtype=np.float64))
        n = cache.n() if cache is not None else eig.n()
        if y.shape != x.shape or y.shape[0] != n:
            raise ShapeError("denoise: signal shape mismatch")
        self.n, self.ch = y.shape
        self.cache, self.eig = cache, eig  # keep the handles alive
        self._h = ctypes.c_void_p()
        if cache is not None:
            _check(lib().fgfrft_denoise_create_ex(cache.handle, y.ctypes.data, x.ctypes.data, self.ch,
                                                  int(bool(loss_on_real)), ctypes.byref(self._h)))
        else:
            _check(lib().fgfrft_denoise_create_exact(eig.handle, y.ctypes.data, x.ctypes.data, self.ch,
                                                     int(bool(loss_on_real)), ctypes.byref(self._h)))

    @classmethod
    def exact(cls, eig: "UnitaryEigen", y: np.ndarray, x_ref: np.ndarray, loss_on_real: bool = False):
        return cls(None, y, x_ref, eig=eig, loss_on_real=loss_on_real)

    def reconstruct(self, alpha: float, h: np.ndarray) -> np.ndarray:
        h = np.ascontiguousarray(h, dtype=np.float64)
        out = np.empty((self.n, self.ch), order="F")
        _check(lib().fgfrft_denoise_reconstruct(self._h, float(alpha), h.ctypes.data, out.ctypes.data))
        return out

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().fgfrft_denoise_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def eval(self, alpha: float, h: np.ndarray):
        h = np.ascontiguousarray(h, dtype=np.float64)
        loss, ga = ctypes.c_double(), ctypes.c_double()
        gh = np.empty(self.n)
        _check(lib().fgfrft_denoise_eval(self._h, float(alpha), h.ctypes.data, ctypes.addressof(loss),
                                         ctypes.addressof(ga), gh.ctypes.data))
        return loss.value, ga.value, gh

    def fit(self, epochs: int, lr: float = 0.01, init_alpha: float = 0.5, want_reconstruction: bool = False):
        tl, ta = np.empty(epochs + 1), np.empty(epochs + 1)
        hb = np.empty(self.n)
        ab, lb, be = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        rec = np.empty((self.n, self.ch), order="F") if want_reconstruction else None
        _check(lib().fgfrft_denoise_fit(self._h, int(epochs), float(lr), float(init_alpha), tl.ctypes.data,
                                        ta.ctypes.data, ctypes.addressof(ab), hb.ctypes.data, ctypes.addressof(lb),
                                        ctypes.addressof(be), rec.ctypes.data if rec is not None else None))
        return {"traj_loss": tl, "traj_alpha": ta, "alpha_best": ab.value, "h_best": hb, "loss_best": lb.value,
                "best_epoch": be.value, "reconstruction": rec}


# ----------------------------------------------------------------------------- spectral.hpp / learn.hpp


class UnitaryEigen:
    """spectral.hpp:19-31 on the GPU: F = V diag(e^{j theta}) V^H, V resident in HBM.

    ``UnitaryEigen(v=..., theta=...)`` stores a recorded spectrum (KnownSpectrum);
    ``eigendecompose_unitary(f)`` computes one on the device."""

    def __init__(self, v: Optional[np.ndarray] = None, theta: Optional[np.ndarray] = None, device: int = 0,
                 _handle=None):
        self._h = ctypes.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            vc = _cm(v)
            th = np.ascontiguousarray(theta, dtype=np.float64)
            if vc.shape[0] != vc.shape[1] or th.shape != (vc.shape[0],):
                raise ShapeError("spectrum: V must be n x n and theta of length n")
            _check(lib().fgfrft_spectrum_create(_ptr(vc), _ptr(th), vc.shape[0], device, ctypes.byref(self._h)))
        n = ctypes.c_int64()
        _check(lib().fgfrft_spectrum_info(self._h, ctypes.addressof(n), None))
        self._n = n.value
        self.device = device

    @property
    def handle(self):
        return self._h

    def n(self) -> int:
        return self._n

    @property
    def theta(self) -> np.ndarray:
        th = np.empty(self._n)
        _check(lib().fgfrft_spectrum_info(self._h, None, _ptr(th)))
        return th

    @property
    def v(self) -> np.ndarray:
        buf = np.empty((self._n, self._n), dtype=np.complex128)  # row-major buffer of V^T
        _check(lib().fgfrft_spectrum_vectors(self._h, _ptr(buf)))
        return buf.T

    def eigenvalues(self) -> np.ndarray:
        return np.exp(1j * self.theta)

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().fgfrft_spectrum_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def eigendecompose_unitary(f: np.ndarray, device: int = 0) -> UnitaryEigen:
    """spectral.hpp:121-155 with the large products and the Hermitian eigensolve on the GPU."""
    fc = _cm(f)
    if fc.shape[0] != fc.shape[1]:
        raise ShapeError("eigendecompose_unitary: F must be square")
    h = ctypes.c_void_p()
    _check(lib().fgfrft_spectrum_decompose(_ptr(fc), fc.shape[0], device, ctypes.byref(h)))
    return UnitaryEigen(device=device, _handle=h)


def exact_matrices(eig: UnitaryEigen, alphas, which: int = Q) -> np.ndarray:
    """[A, n, n]: V diag(e^{j a theta}) V^H (which Q) or its a-derivative (DQ) for every order."""
    al = _alphas(alphas)
    buf = np.empty((len(al), eig.n(), eig.n()), dtype=np.complex128)
    _check(lib().fgfrft_exact(eig.handle, _ptr(al), len(al), which, _ptr(buf)))
    return np.transpose(buf, (0, 2, 1))


def exact_gfrft(eig: UnitaryEigen, alpha: float) -> FracOperator:
    """spectral.hpp:158-166."""
    return FracOperator(exact_matrices(eig, [alpha], Q)[0], float(alpha), 0)


def exact_gfrft_grad(eig: UnitaryEigen, alpha: float) -> np.ndarray:
    """spectral.hpp:169-174."""
    return exact_matrices(eig, [alpha], DQ)[0]


def phase_margin(eig: UnitaryEigen) -> float:
    """spectral.hpp:179-195 (min_k pi - |theta_k|, warning below 0.05 pi)."""
    margin = float(np.min(np.pi - np.abs(eig.theta))) if eig.n() else float(np.pi)
    margin = min(margin, float(np.pi))
    if margin < 0.05 * np.pi:
        warnings.warn(f"phase margin {margin} is below 0.05*pi; series approximation accuracy is at risk")
    return margin


FAST, EXACT = "fast", "exact"


class CascadeProblem:
    """learn.hpp:55-116 on the GPU. ``backend`` "fast" synthesises the layer operators from a
    PowerCache of F (built here with ``truncation`` unless ``cache`` is given); "exact" uses the
    spectrum. eval(alphas) -> (loss, grad)."""

    def __init__(self, f: Optional[np.ndarray], depth: int = 1, target_order: float = 1.5, truncation: int = 10,
                 backend: str = FAST, memory_budget: int = DEFAULT_MEMORY_BUDGET, eig: Optional[UnitaryEigen] = None,
                 cache: Optional[PowerCache] = None, device: int = 0):
        if depth < 1:
            raise ParameterError("CascadeConfig: depth must be >= 1")
        if truncation < 1:
            raise ParameterError("CascadeConfig: truncation must be >= 1")
        if backend not in (FAST, EXACT):
            raise ParameterError(f"unknown backend {backend!r}")
        self.eig = eig if eig is not None else eigendecompose_unitary(f, device)
        self.cache = None
        if backend == FAST:
            self.cache = cache if cache is not None else PowerCache(f, truncation, memory_budget, device=device)
        self.depth, self.backend = int(depth), backend
        self._h = ctypes.c_void_p()
        _check(lib().fgfrft_cascade_create(self.cache.handle if self.cache is not None else None, self.eig.handle,
                                           float(target_order), self.depth, ctypes.byref(self._h)))

    def n(self) -> int:
        return self.eig.n()

    def eval(self, alphas):
        al = _alphas(alphas)
        if len(al) != self.depth:
            raise ShapeError("cascade: need one order per layer")
        loss, grad = ctypes.c_double(), np.empty(self.depth)
        _check(lib().fgfrft_cascade_eval(self._h, _ptr(al), ctypes.addressof(loss), _ptr(grad)))
        return loss.value, grad

    def learn(self, init_order: float = 0.1, epochs: int = 200, lr: float = 0.01):
        """learn_orders (learn.hpp:124-166): trajectory of (loss, alphas) for epochs + 1 points."""
        tl = np.empty(epochs + 1) if epochs >= 1 else np.empty(1)
        ta = np.empty((max(epochs, 0) + 1, self.depth))
        fl, fa = ctypes.c_double(), np.empty(self.depth)
        _check(lib().fgfrft_cascade_learn(self._h, float(init_order), int(epochs), float(lr), _ptr(tl), _ptr(ta),
                                          ctypes.addressof(fl), _ptr(fa)))
        return {"traj_loss": tl, "traj_alphas": ta, "final_loss": fl.value, "final_alphas": fa,
                "final_alpha_sum": float(fa.sum())}

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().fgfrft_cascade_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def learn_orders(f: np.ndarray, depth: int = 1, init_order: float = 0.1, target_order: float = 1.5,
                 truncation: int = 10, epochs: int = 200, lr: float = 0.01, backend: str = FAST, device: int = 0):
    """learn.hpp:124-166 (CascadeConfig fields as keyword arguments)."""
    if epochs < 1:
        raise ParameterError("CascadeConfig: epochs must be >= 1")
    if not lr > 0:
        raise ParameterError("CascadeConfig: lr must be positive")
    prob = CascadeProblem(f, depth, target_order, truncation, backend, device=device)
    try:
        return prob.learn(init_order, epochs, lr)
    finally:
        prob.close()
