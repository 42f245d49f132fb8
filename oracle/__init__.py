"""CPU oracle for the FGFRFT hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` leg may import this package; it is the checker, never the product. The product
path (``paper_2602_20870_b200`` -> ``libfgfrft_b200.so``) neither imports nor links it.

Pinning: the reference C++ library cannot be compiled here (Eigen3,
CLI11, Catch2 absent; no network). Its std-only headers ARE compiled where they lie
(oracle/ref_shim.cpp -> oracle/_ref/), which pins ``sinc_coeffs`` and the input RNG bit-exactly;
the matrix parts are pinned by the reference's own known-answer tests
(test_transform.cpp, test_sinc.cpp, acceptance.cpp criteria 1-6) re-run against this
restatement in tests/test_oracle.py, and by committed golden vectors under tests/golden/.

Restated reference functions (file:line under /root/reference/proj/include/fgfrft/):
  sinc, sinc_deriv, sinc_coeffs      sinc.hpp:15-63          (C, fgfrft_oracle.c)
  content_fingerprint / fnv1a64      gft.hpp:46-48, rng.hpp:59-67 (C)
  PowerCache                         transform.hpp:41-80     (numpy GEMM recursion P_k = F P_{k-1})
  fgfrft_matrix / fgfrft_grad        transform.hpp:21-34, 111-136 (C, 96x96 pair blocks)
  apply_forward / apply_inverse      transform.hpp:138-148   (numpy zgemm)
  eigendecompose_unitary             spectral.hpp:55-155     (numpy eigh, cluster refinement)
  exact_gfrft / exact_gfrft_grad     spectral.hpp:158-174
  phase_margin                       spectral.hpp:179-195
  matrix_errors                      metrics.hpp:21-34
  cascade dL/dalpha (K=1)            learn.hpp:88-92
  Cascade / learn_orders             learn.hpp:55-166 (any depth, fast and exact backends)
  FastDenoiseEngine (real F), Adam   learn.hpp:291-413, learn.hpp:471-516, adam.hpp:34-53
  ExactDenoiseEngine                 learn.hpp:205-289
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import warnings

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_MEMORY_BUDGET = 4 << 30  # transform.hpp:17


class ParameterError(ValueError):
    pass


class ShapeError(ParameterError):
    pass


class CapacityError(ParameterError):
    pass


class NumericalError(ArithmeticError):
    pass


def build() -> str:
    out = os.path.join(_HERE, "liboracle_fgfrft.so")
    src = os.path.join(_HERE, "fgfrft_oracle.c")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "all"])
    return out


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        l = ctypes.CDLL(build())
        d, i, i64, vp = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        l.oracle_sinc.restype = d
        l.oracle_sinc.argtypes = [d]
        l.oracle_sinc_deriv.restype = d
        l.oracle_sinc_deriv.argtypes = [d]
        l.oracle_sinc_coeffs.restype = i
        l.oracle_sinc_coeffs.argtypes = [d, i, vp, vp]
        l.oracle_fnv1a64.restype = ctypes.c_uint64
        l.oracle_fnv1a64.argtypes = [vp, ctypes.c_size_t, ctypes.c_uint64]
        l.oracle_synthesize.argtypes = [vp, i64, i, vp, vp, i]
        l.oracle_power_dots.argtypes = [vp, i64, i, vp, vp]
        l.oracle_max_threads.restype = i
        _LIB = l
    return _LIB


# ----------------------------------------------------------------------------- sinc.hpp

def sinc(x: float) -> float:
    return lib().oracle_sinc(float(x))


def sinc_deriv(x: float) -> float:
    return lib().oracle_sinc_deriv(float(x))


def sinc_coeffs(alpha: float, l: int):
    """sinc.hpp:50-63 -> (c, dc), each 2l+1 doubles with entry [n + l] = term n."""
    if l < 1:
        raise ParameterError("sinc_coeffs: truncation order must be >= 1")
    c = np.empty(2 * l + 1)
    dc = np.empty(2 * l + 1)
    lib().oracle_sinc_coeffs(float(alpha), int(l), c.ctypes.data, dc.ctypes.data)
    return c, dc


def content_fingerprint(f: np.ndarray) -> int:
    """gft.hpp:46-48: FNV-1a-64 over the column-major interleaved complex128 bytes."""
    buf = np.ascontiguousarray(np.asfortranarray(f, dtype=np.complex128).T)
    return int(lib().oracle_fnv1a64(buf.ctypes.data, buf.nbytes, 0xCBF29CE484222325))


# ----------------------------------------------------------------------------- transform.hpp

class PowerCache:
    """transform.hpp:41-80. Slabs are stored as a C-contiguous [l, n, n] array whose slab k-1
    is P_k^T in row-major, i.e. P_k in column-major (the Eigen layout)."""

    def __init__(self, f: np.ndarray, l: int, memory_budget: int = DEFAULT_MEMORY_BUDGET,
                 real_recursion: bool = False):
        """real_recursion: when Im F == 0, run the recursion as real dgemm (a quarter of the flops)
        and store the slabs as complex128. Same products up to summation order (~1 ulp); used only
        to build large oracle caches (bench.py's CPU baseline at config 3) outside timed regions."""
        if l < 1:
            raise ParameterError("PowerCache: truncation order must be >= 1")
        f = np.asfortranarray(f, dtype=np.complex128)
        n = f.shape[0]
        nbytes = l * n * n * 16
        if nbytes > memory_budget:
            raise CapacityError(f"PowerCache: {l} powers of a {n}x{n} matrix need {nbytes} bytes, "
                                f"over the {memory_budget}-byte budget")
        self.l = l
        self.n = n
        self.fingerprint = content_fingerprint(f)
        self.slabs = np.empty((l, n, n), dtype=np.complex128)
        self.slabs[0] = f.T
        if real_recursion and not np.any(f.imag):
            ft = np.ascontiguousarray(f.real.T)
            cur = ft.copy()
            for k in range(2, l + 1):
                cur = cur @ ft
                self.slabs[k - 1] = cur
            return
        for k in range(2, l + 1):
            # P_k = F @ P_{k-1} (left multiply, transform.hpp:58); stored transposed:
            # P_k^T = P_{k-1}^T @ F^T
            np.matmul(self.slabs[k - 2], f.T, out=self.slabs[k - 1])

    def power(self, k: int) -> np.ndarray:
        if k < 1 or k > self.l:
            raise ParameterError("PowerCache: power index out of range")
        return self.slabs[k - 1].T

    def verify(self, f: np.ndarray) -> None:
        if content_fingerprint(f) != self.fingerprint:
            raise NumericalError("PowerCache: fingerprint mismatch, cache is stale for this matrix")


def _warn_window(alpha: float, l: int) -> None:
    if abs(alpha) > l + 1.0:  # transform.hpp:97-104
        warnings.warn(f"order alpha = {alpha} lies outside the series window [-{l + 1}, {l + 1}]; "
                      "coefficient mass concentrates in dropped terms")


def _synth(cache: PowerCache, coef: np.ndarray, l: int, nthreads: int = 1) -> np.ndarray:
    q_t = np.empty((cache.n, cache.n), dtype=np.complex128)  # Q^T row-major == Q column-major
    lib().oracle_synthesize(cache.slabs.ctypes.data, cache.n, l, np.ascontiguousarray(coef).ctypes.data,
                            q_t.ctypes.data, nthreads)
    return q_t.T


def fgfrft_matrix(cache: PowerCache, alpha: float, truncation: int = 0, nthreads: int = 1) -> np.ndarray:
    """transform.hpp:111-123 -> Q (n x n, column-major view)."""
    l = cache.l if truncation == 0 else truncation
    if l < 1 or l > cache.l:
        raise ParameterError("fgfrft_matrix: truncation exceeds the cached power set")
    _warn_window(alpha, l)
    c, _ = sinc_coeffs(alpha, l)
    return _synth(cache, c, l, nthreads)


def fgfrft_grad(cache: PowerCache, alpha: float, nthreads: int = 1) -> np.ndarray:
    """transform.hpp:127-136 -> dQ/dalpha."""
    _warn_window(alpha, cache.l)
    _, dc = sinc_coeffs(alpha, cache.l)
    return _synth(cache, dc, cache.l, nthreads)


def apply_forward(q: np.ndarray, x: np.ndarray) -> np.ndarray:
    """transform.hpp:138-141."""
    if x.shape[0] != q.shape[1]:
        raise ShapeError("apply_forward: signal length does not match operator")
    return q @ x


def apply_inverse(q: np.ndarray, x: np.ndarray) -> np.ndarray:
    """transform.hpp:145-148: Q^H x."""
    if x.shape[0] != q.shape[0]:
        raise ShapeError("apply_inverse: signal length does not match operator")
    return q.conj().T @ x


def power_dots(cache: PowerCache, m: np.ndarray) -> np.ndarray:
    """s_k = Re<M, F^k> for k = -L..L ([k + L] layout), so that Re<G, F^k X> = s_k with
    M = G X^H, and dL/dalpha = sum_k c'_k s_k (definition: learn.hpp:88-92)."""
    mt = np.ascontiguousarray(np.asfortranarray(m, dtype=np.complex128).T)
    out = np.empty(2 * cache.l + 1)
    lib().oracle_power_dots(cache.slabs.ctypes.data, cache.n, cache.l, mt.ctypes.data, out.ctypes.data)
    return out


def dlda_mse(cache: PowerCache, alpha: float, x: np.ndarray, x_clean: np.ndarray):
    """MSE denoising loss L = ||Q^a X - Xc||_F^2 / (N B) and dL/dalpha, evaluated the way the
    reference's cascade does (learn.hpp:82-92 with K=1): dL/da = Re sum conj(G) o (dQ X),
    G = 2 (Y - Xc) / (N B). Returns (loss, dlda, Y)."""
    n, b = x.shape
    q = fgfrft_matrix(cache, alpha)
    y = q @ x
    r = y - x_clean
    loss = float(np.vdot(r, r).real) / (n * b)
    g = 2.0 * r / (n * b)
    dq = fgfrft_grad(cache, alpha)
    dlda = float(np.sum(np.conj(g) * (dq @ x)).real)
    return loss, dlda, y


# ----------------------------------------------------------------------------- spectral.hpp

K_CLUSTER_GAP = 1e-5  # spectral.hpp:43


def _wrap_phase(lam: np.ndarray) -> np.ndarray:
    t = np.arctan2(lam.imag, lam.real)  # spectral.hpp:34-38
    t[t <= -math.pi] = math.pi
    return t


def _refine_clusters(cosv, w, fw, skew):
    """spectral.hpp:55-82."""
    n = w.shape[0]
    lam = np.empty(n, dtype=np.complex128)
    lo = 0
    while lo < n:
        hi = lo
        while hi + 1 < n and cosv[hi + 1] - cosv[hi] <= K_CLUSTER_GAP:
            hi += 1
        k = hi - lo + 1
        if k > 1:
            m = skew(w, lo, k)
            _, u = np.linalg.eigh(m)
            w[:, lo:hi + 1] = w[:, lo:hi + 1] @ u
            fw[:, lo:hi + 1] = fw[:, lo:hi + 1] @ u
        for c in range(lo, hi + 1):
            lam[c] = np.vdot(w[:, c], fw[:, c])
        lo = hi + 1
    return w, fw, lam


def is_real(f: np.ndarray, tol: float = 1e-13) -> bool:
    return float(np.abs(f.imag).max()) <= tol  # gft.hpp:34-36


def eigendecompose_unitary(f: np.ndarray, known=None):
    """spectral.hpp:121-155 -> (V, theta ascending). ``known`` = (V, theta) short-circuit."""
    if known is not None:
        return known
    f = np.asarray(f, dtype=np.complex128)
    if is_real(f):  # spectral.hpp:84-98
        fr = f.real
        s = 0.5 * (fr + fr.T)
        cosv, ev = np.linalg.eigh(s)
        b = 0.5 * (fr - fr.T)
        w = ev.astype(np.complex128)
        fw = (fr @ ev).astype(np.complex128)

        def skew(wcur, lo, k):
            wc = wcur[:, lo:lo + k].real
            return (wc.T @ (b @ wc)).astype(np.complex128) * (-1j)
    else:  # spectral.hpp:100-112
        a = 0.5 * (f + f.conj().T)
        cosv, w = np.linalg.eigh(a)
        b = (f - f.conj().T) * (-0.5j)
        fw = f @ w

        def skew(wcur, lo, k):
            wc = wcur[:, lo:lo + k]
            return wc.conj().T @ (b @ wc)
    w, fw, lam = _refine_clusters(cosv, np.array(w, dtype=np.complex128), np.array(fw), skew)
    theta = _wrap_phase(lam)
    order = np.argsort(theta, kind="stable")
    v = w[:, order]
    theta = theta[order]
    resid = fw[:, order] - np.exp(1j * theta)[None, :] * v
    rel = np.linalg.norm(resid) / max(np.linalg.norm(f), 1e-300)
    if rel > 1e-6:
        raise NumericalError(f"eigendecompose_unitary: reconstruction residual {rel} exceeds 1e-6")
    return v, theta


def exact_gfrft(eig, alpha: float) -> np.ndarray:
    """spectral.hpp:158-166: V diag(e^{j alpha theta}) V^H."""
    v, theta = eig
    return (v * np.exp(1j * alpha * theta)[None, :]) @ v.conj().T


def exact_gfrft_grad(eig, alpha: float) -> np.ndarray:
    """spectral.hpp:169-174."""
    v, theta = eig
    return (v * (1j * theta * np.exp(1j * alpha * theta))[None, :]) @ v.conj().T


def phase_margin(theta: np.ndarray) -> float:
    """spectral.hpp:179-195."""
    margin = float(np.min(math.pi - np.abs(theta))) if len(theta) else math.pi
    margin = min(margin, math.pi)
    if margin < 0.05 * math.pi:
        warnings.warn(f"phase margin {margin} is below 0.05*pi; series approximation accuracy is at risk")
    return margin


# ----------------------------------------------------------------------------- metrics.hpp

def matrix_errors(approx: np.ndarray, reference: np.ndarray):
    """metrics.hpp:21-34 -> dict(mse, mae, nmse)."""
    if approx.shape != reference.shape:
        raise ShapeError("matrix_errors: shape mismatch")
    ref_sq = float(np.vdot(reference, reference).real)
    if ref_sq == 0.0:
        raise NumericalError("matrix_errors: NMSE undefined for all-zero reference")
    d = approx - reference
    cnt = float(d.size)
    sq = float(np.vdot(d, d).real)
    return {"mse": sq / cnt, "mae": float(np.abs(d).sum()) / cnt, "nmse": sq / ref_sq}


# ----------------------------------------------------------------------------- tests/oracles.hpp

def scalar_series(theta: float, alpha: float, l: int) -> complex:
    """tests/oracles.hpp:23-30."""
    acc = 0j
    for n in range(-l, l + 1):
        x = alpha - n
        s = (1.0 if x == 0 else 0.0) if x == round(x) else math.sin(math.pi * x) / (math.pi * x)
        acc += s * complex(math.cos(n * theta), math.sin(n * theta))
    return acc


def truncation_bound(thetas, alpha: float, l: int) -> float:
    """tests/oracles.hpp:31-41."""
    return max(abs(complex(math.cos(alpha * t), math.sin(alpha * t)) - scalar_series(t, alpha, l))
               for t in thetas)


def spectral_norm(m: np.ndarray) -> float:
    return float(np.linalg.svd(m, compute_uv=False)[0])


def matrix_power(f: np.ndarray, m: int) -> np.ndarray:
    """tests/oracles.hpp:50-56."""
    acc = np.eye(f.shape[0], dtype=np.complex128)
    base = f if m >= 0 else f.conj().T
    for _ in range(abs(m)):
        acc = base @ acc
    return acc


def rotation2(phi: float) -> np.ndarray:
    """tests/oracles.hpp:43-48."""
    return np.array([[math.cos(phi), -math.sin(phi)], [math.sin(phi), math.cos(phi)]], dtype=np.complex128)


# ----------------------------------------------------------------------------- large-N checker

def series_apply_recursive(f: np.ndarray, alpha: float, l: int, x: np.ndarray, which: str = "c",
                           inverse: bool = False) -> np.ndarray:
    """Q(alpha) X (or Q^H X) for a FEW columns X without forming any power: the powers act by
    repeated multiplication, F^k X = F (F^{k-1} X) and (F^H)^k X (tests/oracles.hpp:50-56's
    matrix_power, applied to X), weighted by the reference coefficients (sinc.hpp:50-63),
    summed in ascending k like transform.hpp:118-121. which = "c" (Q) or "dc" (dQ/dalpha).
    Cost 2L n^2 |X|: an independent checker at sizes where the dense oracle cannot run."""
    c, dc = sinc_coeffs(alpha, l)
    coef = c if which == "c" else dc
    if inverse:  # Q^H = sum conj(c_k) F^{-k}: swap the roles of +k and -k (real coefficients)
        coef = coef[::-1]
    x = np.asarray(x, dtype=np.complex128)
    if not np.any(f.imag):  # real F (graph GFTs): the same products as real GEMMs on (Re, Im)
        fp, fh = np.ascontiguousarray(f.real), np.ascontiguousarray(f.real.T)

        def mul(m, v):
            return m @ v.real + 1j * (m @ v.imag)
    else:
        fp, fh = np.ascontiguousarray(f), np.ascontiguousarray(f.conj().T)

        def mul(m, v):
            return m @ v
    acc = coef[l] * x
    vp, vm = x, x
    for k in range(1, l + 1):
        vp = mul(fp, vp)
        vm = mul(fh, vm)
        acc = acc + (coef[l + k] * vp + coef[l - k] * vm)
    return acc


def power_dots_recursive(f: np.ndarray, l: int, g: np.ndarray, x: np.ndarray) -> np.ndarray:
    """s_k = Re<G, F^k X>, k = -L..L, by the same recursion (definition of learn.hpp:88-92)."""
    out = np.empty(2 * l + 1)
    fh = np.ascontiguousarray(f.conj().T)
    fp = np.ascontiguousarray(f)
    out[l] = float(np.vdot(g, x).real)
    vp, vm = x.astype(np.complex128), x.astype(np.complex128)
    for k in range(1, l + 1):
        vp = fp @ vp
        vm = fh @ vm
        out[l + k] = float(np.vdot(g, vp).real)
        out[l - k] = float(np.vdot(g, vm).real)
    return out


# ------------------------------------------------------------------ denoising learner (real F)

class FastDenoise:
    """learn.hpp:291-413 FastDenoiseEngine<MatrixXd> (real F) / <MatrixXcd> (complex F): matrix-free
    Q^alpha through iterated products with F / F^H; the signal-side powers F^n y are precomputed
    (learn.hpp:300-305). Complex F: loss on the complex residual, or on its real part with
    loss_on_real (learn.hpp:389-403)."""

    def __init__(self, y: np.ndarray, x: np.ndarray, f: np.ndarray, l: int, loss_on_real: bool = False):
        self.cplx = bool(np.iscomplexobj(f) and np.any(np.imag(f) != 0))
        dt = np.complex128 if self.cplx else float
        self.y, self.x = np.asarray(y, float), np.asarray(x, float)
        self.f = np.asarray(f, dt) if self.cplx else np.asarray(np.real(f), float)
        self.l, self.loss_on_real = int(l), bool(loss_on_real)
        self.spow = self._powers(self.y.astype(dt))

    def _powers(self, v: np.ndarray) -> dict:
        p = {0: v}
        fh = self.f.conj().T
        for m in range(1, self.l + 1):  # at(m) = F at(m-1), at(-m) = F^H at(-(m-1))
            p[m] = self.f @ p[m - 1]
            p[-m] = fh @ p[-(m - 1)]
        return p

    def _run(self, c: np.ndarray, h: np.ndarray):
        l = self.l
        u = c[l] * self.spow[0]
        for m in range(1, l + 1):
            u = u + (c[l + m] * self.spow[m] + c[l - m] * self.spow[-m])
        v = h[:, None] * u
        tpow = self._powers(v)
        w = c[l] * tpow[0]
        for m in range(1, l + 1):  # Q^H v = sum_m c_{-m} F^m v
            w = w + (c[l - m] * tpow[m] + c[l + m] * tpow[-m])
        if self.cplx and self.loss_on_real:
            r = w.real - self.x
            return u, tpow, w, r.astype(np.complex128), float(np.sum(r * r))
        cot = w - self.x
        return u, tpow, w, cot, float(np.vdot(cot, cot).real)

    def eval(self, alpha: float, h: np.ndarray):
        """-> (loss, grad_alpha, grad_h), learn.hpp:306-338."""
        l = self.l
        c, dc = sinc_coeffs(alpha, l)
        u, tpow, w, cot, loss = self._run(c, h)
        gpow = self._powers(cot)
        qr = c[l] * gpow[0]
        for m in range(1, l + 1):
            qr = qr + (c[l + m] * gpow[m] + c[l - m] * gpow[-m])
        grad_h = 2.0 * np.sum((np.conj(qr) * u).real, axis=1)
        dqh_v = dc[l] * tpow[0]
        for m in range(1, l + 1):
            dqh_v = dqh_v + (dc[l - m] * tpow[m] + dc[l + m] * tpow[-m])
        du = dc[l] * self.spow[0]
        for m in range(1, l + 1):
            du = du + (dc[l + m] * self.spow[m] + dc[l - m] * self.spow[-m])
        ga = 2.0 * float(np.sum((np.conj(cot) * dqh_v).real)) + 2.0 * float(np.sum((np.conj(qr) * (h[:, None] * du)).real))
        return loss, ga, grad_h

    def reconstruct(self, alpha: float, h: np.ndarray) -> np.ndarray:
        c, _ = sinc_coeffs(alpha, self.l)
        return np.real(self._run(c, h)[2])


class ExactDenoise:
    """learn.hpp:205-289 ExactDenoiseEngine: F^a = V diag(e^{j a theta}) V^H on the spectrum,
    loss on the complex residual (or its real part with loss_on_real)."""

    def __init__(self, y: np.ndarray, x: np.ndarray, eig, loss_on_real: bool = False):
        self.y, self.x = np.asarray(y, float), np.asarray(x, float)
        self.v, self.theta = eig
        self.loss_on_real = bool(loss_on_real)
        self.ytil = self.v.conj().T @ self.y.astype(np.complex128)

    def _run(self, alpha: float, h: np.ndarray):
        phase = np.exp(1j * alpha * self.theta)
        u = self.v @ (phase[:, None] * self.ytil)
        b = self.v.conj().T @ (h[:, None] * u)
        w = self.v @ (phase.conj()[:, None] * b)
        if self.loss_on_real:
            r = w.real - self.x
            return phase, u, b, w, r.astype(np.complex128), float(np.sum(r * r))
        cot = w - self.x
        return phase, u, b, w, cot, float(np.vdot(cot, cot).real)

    def eval(self, alpha: float, h: np.ndarray):
        """-> (loss, grad_alpha, grad_h), learn.hpp:211-229."""
        phase, u, b, w, cot, loss = self._run(alpha, h)
        vh_r = self.v.conj().T @ cot
        far = self.v @ (phase[:, None] * vh_r)
        grad_h = 2.0 * np.sum((far.conj() * u).real, axis=1)
        jt = 1j * self.theta
        t1 = (-jt * phase.conj())[:, None] * b
        ga = 2.0 * float(np.sum((vh_r.conj() * t1).real))
        q = self.v @ ((jt * phase)[:, None] * self.ytil)
        ga += 2.0 * float(np.sum((far.conj() * (h[:, None] * q)).real))
        return loss, ga, grad_h

    def reconstruct(self, alpha: float, h: np.ndarray) -> np.ndarray:
        return self._run(alpha, h)[3].real


def adam_step(params, m, v, grad, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """adam.hpp:34-53 (step = the new step count)."""
    m = beta1 * m + (1.0 - beta1) * grad
    v = beta2 * v + (1.0 - beta2) * grad * grad
    c1 = 1.0 - beta1 ** step
    c2 = 1.0 - beta2 ** step
    return params - lr * (m / c1) / (np.sqrt(v / c2) + eps), m, v


def denoise_fit(problem: FastDenoise, epochs: int, lr: float, init_alpha: float):
    """learn.hpp:471-516: Adam over [alpha, h] from [init_alpha, 1..1]; returns (trajectory
    [(loss, alpha)] of epochs + 1 entries, alpha_best, h_best, loss_best, best_epoch)."""
    n = problem.y.shape[0]
    params = np.ones(n + 1)
    params[0] = init_alpha
    m, v = np.zeros(n + 1), np.zeros(n + 1)
    traj, best = [], (math.inf, None, -1)
    for epoch in range(epochs + 1):
        loss, ga, gh = problem.eval(float(params[0]), params[1:])
        traj.append((loss, float(params[0])))
        if loss < best[0]:
            best = (loss, params.copy(), epoch)
        if epoch < epochs:
            params, m, v = adam_step(params, m, v, np.concatenate([[ga], gh]), epoch + 1, lr)
    return traj, float(best[1][0]), best[1][1:], best[0], best[2]


# ----------------------------------------------------------------------------- learn.hpp cascade

class Cascade:
    """learn.hpp:55-116 (CascadeProblem): Yhat = Q_K ... Q_1 (X = I), target = exact
    F^{target_order}, loss = |Yhat - target|^2 / N^2, reverse-accumulated order gradients.
    backend "fast": Q from fgfrft_matrix / fgfrft_grad of a PowerCache; "exact": exact_gfrft."""

    def __init__(self, f, depth: int, target_order: float, truncation: int, backend: str = "fast", eig=None,
                 cache=None):
        if depth < 1 or truncation < 1:
            raise ParameterError("CascadeConfig: depth and truncation must be >= 1")
        self.n = f.shape[0]
        self.eig = eig if eig is not None else eigendecompose_unitary(f)
        self.target = exact_gfrft(self.eig, target_order)  # learn.hpp:61
        self.backend = backend
        self.cache = None
        if backend == "fast":
            self.cache = cache if cache is not None else PowerCache(np.asarray(f, dtype=np.complex128), truncation)

    def _op(self, a):
        return fgfrft_matrix(self.cache, a) if self.backend == "fast" else exact_gfrft(self.eig, a)

    def _grad_op(self, a):
        return fgfrft_grad(self.cache, a) if self.backend == "fast" else exact_gfrft_grad(self.eig, a)

    def eval(self, alphas):
        """learn.hpp:72-97."""
        k = len(alphas)
        nn = float(self.n) * float(self.n)
        ops = [self._op(float(a)) for a in alphas]
        prefix = []
        for l in range(k):
            prefix.append(ops[0] if l == 0 else ops[l] @ prefix[l - 1])
        resid = prefix[k - 1] - self.target
        loss = float(np.vdot(resid, resid).real) / nn
        grad = np.empty(k)
        b = resid
        for l in range(k - 1, -1, -1):
            dq = self._grad_op(float(alphas[l]))
            dyhat = dq if l == 0 else dq @ prefix[l - 1]
            grad[l] = 2.0 / nn * float(np.sum(b.conj() * dyhat).real)
            if l > 0:
                b = ops[l].conj().T @ b
        return loss, grad


def learn_orders(problem: Cascade, depth: int, init_order: float, epochs: int, lr: float):
    """learn.hpp:124-166: Adam from init_order; returns (traj_loss [epochs+1], traj_alphas
    [epochs+1, depth], final_loss, final_alphas)."""
    params = np.full(depth, float(init_order))
    m, v = np.zeros(depth), np.zeros(depth)
    tl, ta = [], []
    for epoch in range(epochs):
        loss, grad = problem.eval(params)
        if not math.isfinite(loss):
            raise NumericalError(f"learn_orders: non-finite loss at epoch {epoch}")
        tl.append(loss)
        ta.append(params.copy())
        params, m, v = adam_step(params, m, v, grad, epoch + 1, lr)
    loss, _ = problem.eval(params)
    tl.append(loss)
    ta.append(params.copy())
    return np.array(tl), np.array(ta), loss, params
