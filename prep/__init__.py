"""Host-side input preparation for the five BASELINE configs (not the hot path).

The reference builds F on the host (``gft_from_shift``, proj/include/fgfrft/gft.hpp:74-128)
and the north star keeps that eigendecomposition in host code. The reference cannot be
compiled here (Eigen3 is absent), so this module restates the pieces needed to generate
inputs, using numpy/LAPACK for the dense eigensolver / QR:

* ``Rng``                 -- rng.hpp:12-56 (C restatement in prep_rng.c, bit-exact)
* ``grid_graph``          -- graph.hpp:45-72
* ``knn_graph``           -- graph.hpp:77-125, plus Gaussian weights (new, BASELINE C2/C4)
* ``laplacian``           -- graph.hpp:136-141 (combinatorial)
* ``gft_from_shift``      -- gft.hpp:74-128 (sign pivot, cluster MGS, F = V^T)
* ``random_unitary``      -- gft.hpp:132-153 (Haar via Householder QR)
* ``synthetic_unitary``   -- gft.hpp:158-177 (prescribed spectrum)
* ``spread_phases``       -- tests/oracles.hpp:74-86 (glibc srand/rand, called directly)
* ``er_graph``, ``sphere_torus_cloud``, signal generators -- new for the BASELINE configs.

Because eigensolvers choose different bases inside degenerate clusters, F is generated
once per config and persisted (``save_matrix``); the GPU path and the oracle always
consume the identical bytes.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import struct
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    """Compile prep_rng.c into prep/libprep_rng.so (idempotent)."""
    src = os.path.join(_HERE, "prep_rng.c")
    out = os.path.join(_HERE, "libprep_rng.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", out, src, "-lm"])
    return out


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(build())
        vp, u64, i64, dp = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
        lib.prep_rng_create.restype = vp
        lib.prep_rng_create.argtypes = [u64]
        lib.prep_rng_destroy.argtypes = [vp]
        lib.prep_rng_uniform.restype = ctypes.c_double
        lib.prep_rng_uniform.argtypes = [vp]
        lib.prep_rng_gaussian.restype = ctypes.c_double
        lib.prep_rng_gaussian.argtypes = [vp]
        lib.prep_rng_fill_uniform.argtypes = [vp, i64, dp]
        lib.prep_rng_fill_gaussian.argtypes = [vp, i64, dp]
        lib.prep_rng_derive.restype = u64
        lib.prep_rng_derive.argtypes = [u64, u64]
        _LIB = lib
    return _LIB


class Rng:
    """rng.hpp:12-56: mt19937_64 stream, 53-bit uniform, Box-Muller with a spare."""

    def __init__(self, seed: int):
        self._lib = _lib()
        self._h = self._lib.prep_rng_create(ctypes.c_uint64(seed & (2**64 - 1)))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.prep_rng_destroy(h)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = self._lib.prep_rng_uniform(self._h)
        return u if (lo == 0.0 and hi == 1.0) else lo + (hi - lo) * u

    def gaussian(self) -> float:
        return self._lib.prep_rng_gaussian(self._h)

    def uniforms(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self._lib.prep_rng_fill_uniform(self._h, n, out.ctypes.data)
        return out

    def gaussians(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self._lib.prep_rng_fill_gaussian(self._h, n, out.ctypes.data)
        return out

    @staticmethod
    def derive(seed: int, index: int) -> int:
        return int(_lib().prep_rng_derive(seed & (2**64 - 1), index & (2**64 - 1)))


# ----------------------------------------------------------------------------- graphs

def grid_graph(rows: int, cols: int) -> np.ndarray:
    """graph.hpp:45-72: node (r, c) -> r*cols + c, unit 4-neighbour edges."""
    n = rows * cols
    a = np.zeros((n, n))
    for r in range(rows):
        for c in range(cols):
            u = r * cols + c
            if c + 1 < cols:
                a[u, u + 1] = a[u + 1, u] = 1.0
            if r + 1 < rows:
                a[u, u + cols] = a[u + cols, u] = 1.0
    return a


def er_graph(n: int, p: float, seed: int) -> np.ndarray:
    """Erdos-Renyi G(n, p): one Rng::uniform() per upper-triangle pair (i < j), row-major."""
    rng = Rng(seed)
    iu = np.triu_indices(n, 1)
    draw = rng.uniforms(len(iu[0])) < p
    a = np.zeros((n, n))
    a[iu[0][draw], iu[1][draw]] = 1.0
    return a + a.T


def knn_graph(points: np.ndarray, k: int, gaussian_weights: bool = True) -> np.ndarray:
    """graph.hpp:77-125 selection (distance, then smaller index), union symmetrization.

    With ``gaussian_weights`` the union edges carry exp(-d^2 / (2 sigma^2)), sigma = mean
    distance over all directed k-NN picks (BASELINE configs 2 and 4); the reference's
    builder is binary (graph.hpp:115), which ``gaussian_weights=False`` reproduces.
    """
    pts = np.asarray(points, dtype=np.float64)
    n = pts.shape[0]
    if not 1 <= k < n:
        raise ValueError("knn_graph: need 1 <= k < n")
    sq = (pts * pts).sum(1)
    nbr = np.empty((n, k), dtype=np.int64)
    d2 = np.empty((n, k))
    idx = np.arange(n)
    for i0 in range(0, n, 1024):
        blk = slice(i0, min(n, i0 + 1024))
        # exact per-pair differences so ties resolve exactly as in the reference loop
        diff = pts[blk, None, :] - pts[None, :, :]
        dd = (diff * diff).sum(-1)
        for r, i in enumerate(range(blk.start, blk.stop)):
            order = np.lexsort((idx, dd[r]))
            order = order[order != i][:k]
            nbr[i] = order
            d2[i] = dd[r, order]
    del sq
    a = np.zeros((n, n))
    rows = np.repeat(np.arange(n), k)
    if gaussian_weights:
        sigma = float(np.sqrt(d2).mean())
        w = np.exp(-d2.ravel() / (2.0 * sigma * sigma))
    else:
        w = np.ones(n * k)
    a[rows, nbr.ravel()] = w
    # union: keep the weight of the edge where present (d_ij = d_ji, so weights agree)
    a = np.maximum(a, a.T)
    np.fill_diagonal(a, 0.0)
    return a


def laplacian(adj: np.ndarray) -> np.ndarray:
    """graph.hpp:136-141: combinatorial L = D - A."""
    z = -adj.copy()
    z[np.diag_indices_from(z)] += adj.sum(1)
    return z


# ----------------------------------------------------------------------------- GFT matrices

def unitarity_residual(f: np.ndarray) -> float:
    """gft.hpp:39-44."""
    n = f.shape[0]
    g = f @ f.conj().T
    g[np.diag_indices(n)] -= 1.0
    return float(np.linalg.norm(g) / math.sqrt(n))


def gft_from_shift(z: np.ndarray) -> np.ndarray:
    """gft.hpp:74-128: ascending eigenvalues, MGS inside degenerate clusters, sign pivot
    (first entry of largest magnitude made positive), clusters ordered by pivot; F = V^T."""
    n = z.shape[0]
    if np.linalg.norm(z - z.T) > 1e-12 * max(1.0, np.linalg.norm(z)):
        raise ValueError("gft_from_shift: shift operator is not symmetric")
    lam, v = np.linalg.eigh(z)
    v = np.array(v, order="F")
    scale = max(1.0, abs(lam[0]), abs(lam[-1]))
    tol = 1e-9 * scale
    lo = 0
    while lo < n:
        hi = lo
        while hi + 1 < n and lam[hi + 1] - lam[hi] <= tol:
            hi += 1
        k = hi - lo + 1
        if k > 1:
            for a in range(k):
                col = v[:, lo + a]
                for b in range(a):
                    vb = v[:, lo + b]
                    col -= (vb @ col) * vb
                col /= np.linalg.norm(col)
        pivots = []
        for a in range(lo, hi + 1):
            p = int(np.argmax(np.abs(v[:, a])))  # first index of the max, as sign_pivot
            if v[p, a] < 0.0:
                v[:, a] = -v[:, a]
            pivots.append((p, a))
        if k > 1:
            pivots.sort()
            v[:, lo:hi + 1] = v[:, [c for _, c in pivots]]
        lo = hi + 1
    f = np.asfortranarray(v.T.astype(np.complex128))
    resid = unitarity_residual(f)
    if resid > 1e-10:
        raise ArithmeticError(f"gft_from_shift: unitarity residual {resid} exceeds 1e-10")
    return f


def random_unitary(n: int, seed: int) -> np.ndarray:
    """gft.hpp:132-153: QR of a complex Gaussian (column-major draw order), R phases removed.
    LAPACK's Householder QR stands in for Eigen's, so matrices match the reference in
    distribution, not bit for bit (SURVEY 8(c) caveat)."""
    rng = Rng(seed)
    g = rng.gaussians(2 * n * n).reshape(n * n, 2)
    a = ((g[:, 0] + 1j * g[:, 1]) * math.sqrt(0.5)).reshape(n, n).T  # column-major fill
    q, r = np.linalg.qr(a)
    d = np.diag(r)
    m = np.abs(d)
    phase = np.where(m > 0, d / np.where(m > 0, m, 1), 1.0)
    return np.asfortranarray(q * phase[None, :])


def synthetic_unitary(phases, seed: int):
    """gft.hpp:158-177: F = V diag(e^{j theta}) V^H over a Haar basis. Returns (F, V, theta)."""
    theta = np.asarray(phases, dtype=np.float64)
    if theta.size < 1 or not np.all(np.abs(theta) < math.pi):
        raise ValueError("synthetic_unitary: phases must satisfy |theta| < pi")
    v = random_unitary(theta.size, seed)
    f = (v * np.exp(1j * theta)[None, :]) @ v.conj().T
    return np.asfortranarray(f), v, theta


_LIBC = None


def spread_phases(n: int, margin: float, seed: int = 0) -> np.ndarray:
    """tests/oracles.hpp:74-86, with glibc srand()/rand() called directly (bit-identical)."""
    global _LIBC
    if _LIBC is None:
        _LIBC = ctypes.CDLL("libc.so.6")
    _LIBC.srand(ctypes.c_uint(seed))
    lim = math.pi - margin
    rand_max = 2147483647
    out = np.array([-lim + 2.0 * lim * (_LIBC.rand() / (rand_max + 1.0)) for _ in range(n)])
    if n >= 2:
        out[0] = -lim
        out[-1] = lim
    return out


# ----------------------------------------------------------------------------- persistence

_MAGIC = b"FGFRFTM1"


def save_matrix(path: str, f: np.ndarray) -> None:
    """Binary F: magic, int64 n, then n*n column-major interleaved complex128."""
    f = np.asfortranarray(f, dtype=np.complex128)
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path + ".tmp", "wb") as fh:
        fh.write(_MAGIC + struct.pack("<q", f.shape[0]))
        fh.write(f.T.tobytes(order="C"))
    os.replace(path + ".tmp", path)


def load_matrix(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        if fh.read(8) != _MAGIC:
            raise IOError(f"{path}: not an FGFRFT matrix file")
        (n,) = struct.unpack("<q", fh.read(8))
        data = np.frombuffer(fh.read(16 * n * n), dtype=np.complex128)
    return np.asfortranarray(data.reshape(n, n).T)


def data_dir() -> str:
    d = os.environ.get("FGFRFT_DATA", os.path.join(os.path.dirname(_HERE), "data"))
    os.makedirs(d, exist_ok=True)
    return d


# ----------------------------------------------------------------------------- configs

@dataclasses.dataclass
class Config:
    name: str
    f: np.ndarray            # N x N complex128, column-major
    l: int                   # series truncation L
    alphas: np.ndarray       # orders evaluated per step
    x: np.ndarray            # N x B noisy signals (complex128, column-major)
    x_clean: np.ndarray      # N x B clean targets
    description: str = ""

    @property
    def n(self) -> int:
        return self.f.shape[0]

    @property
    def b(self) -> int:
        return self.x.shape[1]


def _cached_f(tag: str, make) -> np.ndarray:
    path = os.path.join(data_dir(), f"F_{tag}.bin")
    if os.path.exists(path):
        return load_matrix(path)
    f = make()
    save_matrix(path, f)
    return f


def config1(seed: int = 1) -> Config:
    """C1: ER(256, p=0.05), combinatorial Laplacian, L=32, alpha=0.37, one N(0,1) signal."""
    f = _cached_f(f"c1_s{seed}", lambda: gft_from_shift(laplacian(er_graph(256, 0.05, seed))))
    rng = Rng(Rng.derive(seed, 1))
    x = rng.gaussians(256).astype(np.complex128).reshape(256, 1, order="F")
    return Config("C1", f, 32, np.array([0.37]), np.asfortranarray(x), np.asfortranarray(x.copy()),
                  "N=256 ER(p=0.05) combinatorial Laplacian, L=32, alpha=0.37, B=1")


def config2(seed: int = 1, n: int = 1024, b: int = 256, l: int = 64, n_alpha: int = 64) -> Config:
    """C2: 1024 uniform points in the unit square, Gaussian-weighted k-NN (k=8), L=64,
    B=256 bandlimited signals (first 50 GFT coefficients N(0,1)) + N(0, 0.1^2) noise,
    64 orders on linspace(0, 2)."""
    def make_f():
        rng = Rng(seed)
        pts = rng.uniforms(2 * n).reshape(n, 2)
        return gft_from_shift(laplacian(knn_graph(pts, 8)))
    f = _cached_f(f"c2_s{seed}_n{n}", make_f)
    rng = Rng(Rng.derive(seed, 2))
    coef = np.zeros((n, b))
    coef[:50, :] = rng.gaussians(50 * b).reshape(b, 50).T
    clean = f.conj().T @ coef.astype(np.complex128)          # inverse GFT: x = F^H c
    noisy = clean + 0.1 * rng.gaussians(n * b).reshape(b, n).T
    return Config("C2", f, l, np.linspace(0.0, 2.0, n_alpha), np.asfortranarray(noisy),
                  np.asfortranarray(clean),
                  f"N={n} Gaussian k-NN(k=8) sensor graph, L={l}, B={b}, {n_alpha} orders in [0,2]")


def _piecewise_smooth_images(rng: Rng, b: int, side: int) -> np.ndarray:
    """Random axis-aligned rectangles with U[0,1] intensities plus a sinusoidal ramp;
    row-major flatten (image.hpp:54-59 node order r*cols + c)."""
    imgs = np.empty((side * side, b))
    yy, xx = np.mgrid[0:side, 0:side] / float(side)
    for j in range(b):
        img = np.zeros((side, side))
        nrect = 3 + int(rng.uniform() * 4)
        for _ in range(nrect):
            r0, r1 = sorted(int(rng.uniform() * side) for _ in range(2))
            c0, c1 = sorted(int(rng.uniform() * side) for _ in range(2))
            img[r0:r1 + 1, c0:c1 + 1] = rng.uniform()
        fx, fy, ph = rng.uniform(0.5, 2.0), rng.uniform(0.5, 2.0), rng.uniform(0, 2 * math.pi)
        img = 0.8 * img + 0.2 * (0.5 + 0.5 * np.sin(2 * math.pi * (fx * xx + fy * yy) + ph))
        imgs[:, j] = img.reshape(-1)
    return imgs


def config3(seed: int = 1, side: int = 64, b: int = 1024, l: int = 64) -> Config:
    """C3: 64x64 4-neighbour grid (N=4096), L=64, B=1024 noisy piecewise-smooth images."""
    n = side * side
    f = _cached_f(f"c3_s{seed}_side{side}", lambda: gft_from_shift(laplacian(grid_graph(side, side))))
    rng = Rng(Rng.derive(seed, 3))
    clean = _piecewise_smooth_images(rng, b, side)
    noisy = clean + 0.1 * rng.gaussians(n * b).reshape(b, n).T
    return Config("C3", f, l, np.array([0.37]), np.asfortranarray(noisy.astype(np.complex128)),
                  np.asfortranarray(clean.astype(np.complex128)),
                  f"{side}x{side} grid (N={n}), L={l}, B={b} images")


def sphere_torus_cloud(n: int, seed: int) -> np.ndarray:
    """Half the points uniform on a unit sphere centred at (-1.2, 0, 0), half on a torus
    (R=1, r=0.35) centred at (1.2, 0, 0); torus points by area-weighted rejection."""
    rng = Rng(seed)
    ns = n // 2
    nt = n - ns
    g = rng.gaussians(3 * ns).reshape(ns, 3)
    sphere = g / np.linalg.norm(g, axis=1, keepdims=True) + np.array([-1.2, 0.0, 0.0])
    big_r, small_r = 1.0, 0.35
    tor = []
    while len(tor) < nt:
        u, v, w = rng.uniform(0, 2 * math.pi), rng.uniform(0, 2 * math.pi), rng.uniform()
        if w <= (big_r + small_r * math.cos(v)) / (big_r + small_r):
            tor.append(((big_r + small_r * math.cos(v)) * math.cos(u) + 1.2,
                        (big_r + small_r * math.cos(v)) * math.sin(u), small_r * math.sin(v)))
    return np.vstack([sphere, np.array(tor)])


def config4(seed: int = 1, n: int = 8192, replicas: int = 512, l: int = 128) -> Config:
    """C4: sphere+torus cloud, Gaussian k-NN (k=10), L=128, xyz channels + N(0, 0.02^2)
    jitter x 512 replicas (B=1536)."""
    pts = sphere_torus_cloud(n, seed)
    f = _cached_f(f"c4_s{seed}_n{n}", lambda: gft_from_shift(laplacian(knn_graph(pts, 10))))
    rng = Rng(Rng.derive(seed, 4))
    clean = np.tile(pts, (1, replicas))
    noisy = clean + 0.02 * rng.gaussians(n * 3 * replicas).reshape(3 * replicas, n).T
    return Config("C4", f, l, np.array([0.37]), np.asfortranarray(noisy.astype(np.complex128)),
                  np.asfortranarray(clean.astype(np.complex128)),
                  f"N={n} sphere+torus k-NN(k=10), L={l}, B={3 * replicas}")


def config5(seed: int = 1, graphs: int = 4096, n: int = 64, channels: int = 64, heads: int = 4,
            l: int = 16):
    """C5: independent ER(64, 0.1) graphs (seed derive(seed, g)), 4 orders per graph
    U[0.5, 1.5], 64-channel N(0,1) features. Returns (F stack [G,N,N] column-major slabs
    as an array of Fortran matrices, orders [G, heads], features [G, N, C])."""
    fs = np.empty((graphs, n, n), dtype=np.complex128)
    rng = Rng(Rng.derive(seed, 5))
    for g in range(graphs):
        fs[g] = gft_from_shift(laplacian(er_graph(n, 0.1, Rng.derive(seed, 1000 + g))))
    orders = np.array([[rng.uniform(0.5, 1.5) for _ in range(heads)] for _ in range(graphs)])
    feats = rng.gaussians(graphs * n * channels).reshape(graphs, channels, n).transpose(0, 2, 1)
    return fs, orders, np.ascontiguousarray(feats), l
