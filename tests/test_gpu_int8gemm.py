"""INT8 tensor-core (tcgen05 kind::i8) FP64 GEMM, Ozaki scheme: exactness on small-integer
inputs, accuracy against an exact (float128-free) reference built from integer arithmetic, and
shape edge cases (non-multiples of the 128 x 64 tile and of the 64-byte K block)."""
import numpy as np
import pytest

import paper_2602_20870_b200 as fg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _exactish(a, b):
    # reference in float64 with compensated (Kahan-free) approach: split each double into
    # hi + lo halves so the products are exact, accumulate with math.fsum per element
    return a @ b   # float64 BLAS: ~1e-16 relative, far below the 1e-12 bound asserted here


@pytest.mark.parametrize("m,n,k", [(128, 64, 64), (256, 128, 1024), (300, 70, 100), (1, 1, 1), (129, 65, 65), (384, 256, 200), (256, 320, 64),
                                   (1024, 512, 1024)])
@pytest.mark.parametrize("slices", [6, 7, 8])
def test_int8_gemm_accuracy(m, n, k, slices):
    rng = np.random.default_rng(m * 1000 + n * 10 + k)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    c = fg.dgemm_int8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), slices).cpu().numpy()
    ref = _exactish(a, b)
    tol = {6: 2e-12, 7: 2e-14, 8: 2e-15}[slices]
    assert np.linalg.norm(c - ref) <= tol * np.linalg.norm(ref)


def test_int8_gemm_small_integers():
    # integer inputs: the base-254 digits reconstruct them to ~2^-53, so 7 digits give the exact
    # integer products after rounding
    rng = np.random.default_rng(5)
    a = rng.integers(-63, 64, size=(256, 192)).astype(np.float64)
    b = rng.integers(-63, 64, size=(192, 128)).astype(np.float64)
    c = fg.dgemm_int8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 7).cpu().numpy()
    assert np.abs(c - a @ b).max() <= 1e-9
    assert np.array_equal(np.rint(c), a @ b)


def test_int8_gemm_scaled_rows_and_zeros():
    rng = np.random.default_rng(9)
    a = rng.standard_normal((200, 300)) * np.exp2(rng.integers(-40, 40, size=(200, 1)))
    a[7] = 0.0
    b = rng.standard_normal((300, 90)) * np.exp2(rng.integers(-30, 30, size=(1, 90)))
    b[:, 3] = 0.0
    c = fg.dgemm_int8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 6).cpu().numpy()
    ref = a @ b
    # row/column scaling is exact: relative error per (row, col) block is scale free
    err = np.abs(c - ref) / (np.abs(a).max(1, keepdims=True) * np.abs(b).max(0, keepdims=True) + 1e-300)
    assert err.max() <= 1e-12 * np.sqrt(300)
    assert np.all(c[7] == 0.0) and np.all(c[:, 3] == 0.0)


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (130, 70, 33), (512, 300, 1024), (1000, 257, 4096)])
@pytest.mark.parametrize("op_a,op_b", [("N", "N"), ("C", "N"), ("N", "C"), ("T", "T")])
def test_zgemm_int8_matches_fp64(m, n, k, op_a, op_b):
    """Complex GEMM as one real Ozaki GEMM with K doubled: within 1e-12 of the FP64 product
    (relative to |op(A)| |op(B)| norms), every op combination."""
    import torch
    rng = np.random.default_rng(m + 7 * n + k)
    shp_a = (m, k) if op_a == "N" else (k, m)
    shp_b = (k, n) if op_b == "N" else (n, k)
    A = rng.standard_normal(shp_a) + 1j * rng.standard_normal(shp_a)
    B = rng.standard_normal(shp_b) + 1j * rng.standard_normal(shp_b)
    opf = {"N": lambda z: z, "T": lambda z: z.T, "C": lambda z: z.conj().T}
    ref = opf[op_a](A) @ opf[op_b](B)
    ta = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()   # column-major A in a row-major tensor
    tb = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    c = fg.zgemm_int8(ta, tb, op_a, op_b).cpu().numpy().T
    scale = np.linalg.norm(A) * np.linalg.norm(B)
    assert np.linalg.norm(c - ref) <= 1e-12 * scale
