"""GPU parity: every hot-path entry point of libfgfrft_b200.so against the CPU oracle on the
same inputs, plus the reference's known-answer tests re-run through the C ABI.

Tolerances (BASELINE north star): complex128 within 1e-10 relative Frobenius; the series
synthesis is evaluated in the reference's operation order without FMA contraction, so it is
asserted BIT-EXACT against the oracle. dL/dalpha: |g - g_ref| <= 1e-10 * sum_k |c'_k s_k|.
"""
import ctypes
import math

import os

import numpy as np
import pytest

import oracle as O
import paper_2602_20870_b200 as fg
import prep

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _cache_pair(f, l, **kw):
    return fg.PowerCache(f, l, **kw), O.PowerCache(f, l, kw.get("memory_budget", O.DEFAULT_MEMORY_BUDGET))


# --------------------------------------------------------------------------- power cache (K1)

@pytest.mark.parametrize("n,l", [(1, 3), (2, 4), (24, 10), (48, 10), (100, 7), (256, 8)])
def test_cache_build_matches_oracle(n, l):
    f = prep.random_unitary(n, 77 + n)
    g, o = _cache_pair(f, l)
    assert g.fingerprint() == o.fingerprint == fg.content_fingerprint(f)
    assert np.array_equal(g.power(1), f)                   # P_1 = F copied bit-exactly
    for k in range(2, l + 1):
        assert rel(g.power(k), o.power(k)) <= 1e-12
        step = f @ g.power(k - 1)
        assert np.linalg.norm(g.power(k) - step) <= 1e-9 * np.linalg.norm(step)   # test_transform.cpp:33-42
    assert prep.unitarity_residual(g.power(l)) <= 1e-8


def test_cache_identity_and_rotation():  # test_transform.cpp:20-31
    c = fg.PowerCache(np.eye(8, dtype=complex), 3)
    for k in (1, 2, 3):
        assert np.abs(c.power(k) - np.eye(8)).max() == 0.0
    r = fg.PowerCache(O.rotation2(math.pi / 4), 4)
    assert np.abs(r.power(4) + np.eye(2)).max() < 1e-14


def test_cache_fingerprint_and_errors():  # test_transform.cpp:44-58
    f, other = prep.random_unitary(16, 5), prep.random_unitary(16, 6)
    c = fg.PowerCache(f, 4)
    c.verify(f)
    with pytest.raises(fg.NumericalError):
        c.verify(other)
    for k in (0, 5):
        with pytest.raises(fg.ParameterError):
            c.power(k)
    with pytest.raises(fg.CapacityError):
        fg.PowerCache(prep.random_unitary(64, 1), 10, 1024)
    fg.PowerCache(prep.random_unitary(64, 1), 2, 8 << 20)


# --------------------------------------------------------------------------- synthesis (K2)

@pytest.mark.parametrize("n,l", [(1, 2), (2, 10), (24, 10), (40, 10), (33, 5), (64, 24), (97, 12), (256, 32)])
def test_synthesis_bit_exact(n, l):
    f = prep.random_unitary(n, 1000 + n)
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l, powers=o.slabs)  # identical cache bytes -> bit-exact comparison
    alphas = [0.37, -0.7, 1.5, 0.0, 2.0, 3.3, 1.0000004]
    qs = fg.synthesize(g, alphas)
    for a, q in zip(alphas, qs):
        assert np.array_equal(q, O.fgfrft_matrix(o, a)), a
    dqs = fg.synthesize(g, alphas, which=fg.DQ)
    for a, dq in zip(alphas, dqs):
        assert np.array_equal(dq, O.fgfrft_grad(o, a)), a


def test_synthesis_truncation_and_sweep_chunks():
    """>= 8 orders take the DMMA sweep kernel: ~1e-16 relative (DMMA accumulation order), and
    integer orders stay exact (0 * p = 0, 1 * p = p)."""
    f = prep.random_unitary(70, 3)
    o = O.PowerCache(f, 16)
    g = fg.PowerCache(f, 16, powers=o.slabs)
    alphas = list(np.linspace(0, 2, 11))
    for t in (1, 5, 16):
        qs = fg.synthesize(g, alphas, truncation=t)
        for a, q in zip(alphas, qs):
            assert rel(q, O.fgfrft_matrix(o, a, t)) <= 1e-14
        assert np.array_equal(qs[0], np.eye(70)) and np.array_equal(qs[5], O.fgfrft_matrix(o, 1.0, t))
    for t in (1, 16):
        for a, q in zip(alphas[:3], fg.synthesize(g, alphas[:3], truncation=t)):  # scalar path: bit-exact
            assert np.array_equal(q, O.fgfrft_matrix(o, a, t))
    with pytest.raises(fg.ParameterError):
        fg.synthesize(g, [0.5], truncation=17)


def test_kats_through_the_c_abi():
    # order 0 -> identity exactly (test_transform.cpp:60-65)
    c = fg.PowerCache(prep.random_unitary(32, 9), 6)
    assert np.linalg.norm(fg.fgfrft_matrix(c, 0.0).q - np.eye(32)) == 0.0
    # integer orders (test_transform.cpp:67-75)
    f = prep.random_unitary(24, 31)
    c = fg.PowerCache(f, 10)
    for m in range(-3, 4):
        e = O.matrix_power(f, m)
        assert np.linalg.norm(fg.fgfrft_matrix(c, float(m)).q - e) <= 1e-10 * np.linalg.norm(e)
    # conjugate symmetry, bit-exact here (test_transform.cpp:77-85 bounds it by 1e-14)
    c = fg.PowerCache(prep.random_unitary(40, 13), 10)
    for a in (0.3, 0.7, 1.5, 2.2):
        assert np.array_equal(fg.fgfrft_matrix(c, -a).q, fg.fgfrft_matrix(c, a).q.conj().T)
    # spectral-error identity (test_transform.cpp:98-112)
    f, v, th = prep.synthetic_unitary(prep.spread_phases(64, 0.05 * math.pi, 23), 40)
    eig = O.eigendecompose_unitary(f)
    c = fg.PowerCache(f, 24)
    for a, l in ((0.5, 10), (0.3, 16), (0.85, 12), (1.4, 20), (0.15, 24)):
        lhs = O.spectral_norm(fg.fgfrft_matrix(c, a, l).q - O.exact_gfrft(eig, a))
        assert lhs == pytest.approx(O.truncation_bound(th, a, l), abs=1e-8)
    # gradient vs finite differences (test_transform.cpp:151-160)
    f, _, _ = prep.synthetic_unitary(prep.spread_phases(32, 0.1 * math.pi, 3), 15)
    c = fg.PowerCache(f, 10)
    for a in (0.15, 0.55, 1.0, 1.5):
        fd = (fg.fgfrft_matrix(c, a + 1e-4).q - fg.fgfrft_matrix(c, a - 1e-4).q) / 2e-4
        assert rel(fg.fgfrft_grad(c, a), fd) <= 1e-6
    # identity spectrum gradient (test_transform.cpp:162-174)
    c = fg.PowerCache(np.eye(6, dtype=complex), 8)
    assert np.abs(fg.fgfrft_grad(c, 0.0)).max() == 0.0


def test_window_warning():
    c = fg.PowerCache(prep.random_unitary(8, 3), 4)
    with pytest.warns(UserWarning, match="window"):
        fg.fgfrft_matrix(c, 9.0)
    assert fg.fgfrft_matrix(c, 0.5, 2).l == 2


# --------------------------------------------------------------------------- apply (K3)

@pytest.mark.parametrize("n,b", [(1, 1), (8, 3), (40, 1), (130, 70), (256, 1), (300, 257)])
def test_apply_matrix_matches_oracle(n, b):
    rng = np.random.default_rng(n)
    q = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    op = fg.FracOperator(np.asfortranarray(q), 0.3, 4)
    assert rel(fg.apply_forward(op, x), O.apply_forward(q, x)) <= 1e-13
    assert rel(fg.apply_inverse(op, x), O.apply_inverse(q, x)) <= 1e-13
    with pytest.raises(fg.ShapeError):
        fg.apply_forward(op, np.zeros((n + 1, 1)))


def test_apply_series_matches_oracle():
    f = prep.random_unitary(150, 8)
    o = O.PowerCache(f, 12)
    g = fg.PowerCache(f, 12)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((150, 33)) + 1j * rng.standard_normal((150, 33))
    alphas = [0.0, 0.37, 1.0, 1.9]
    ys = fg.apply_series(g, alphas, x)
    yi = fg.apply_series(g, alphas, x, inverse=True)
    for a, y, z in zip(alphas, ys, yi):
        q = O.fgfrft_matrix(o, a)
        assert rel(y, q @ x) <= 1e-12
        assert rel(z, q.conj().T @ x) <= 1e-12
    assert np.array_equal(ys[0], x.astype(complex)) or rel(ys[0], x) <= 1e-15   # order 0 is the identity


def test_forward_inverse_roundtrip():  # test_transform.cpp:176-203
    f, v, th = prep.synthetic_unitary(prep.spread_phases(64, 0.05 * math.pi, 23), 40)
    c = fg.PowerCache(f, 12)
    rng = prep.Rng(55)
    x = np.array([complex(rng.gaussian(), rng.gaussian()) for _ in range(64)]).reshape(64, 1)
    q0 = fg.fgfrft_matrix(c, 0.0)
    assert np.linalg.norm(fg.apply_forward(q0, x) - x) == 0.0
    q1 = fg.fgfrft_matrix(c, 1.0)
    assert np.linalg.norm(fg.apply_inverse(q1, fg.apply_forward(q1, x)) - x) <= 1e-10 * np.linalg.norm(x)


# --------------------------------------------------------------------------- dL/dalpha (K4)

def test_dlda_matches_oracle():
    f = prep.random_unitary(90, 21)
    o = O.PowerCache(f, 9)
    g = fg.PowerCache(f, 9)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((90, 17)) + 1j * rng.standard_normal((90, 17))
    alphas = [0.37, 1.2, -0.4, 0.0, 2.0]
    gs = [rng.standard_normal((90, 17)) + 1j * rng.standard_normal((90, 17)) for _ in alphas]
    dl, s = fg.dlda(g, alphas, gs, x)
    for i, a in enumerate(alphas):
        s_ref = O.power_dots(o, gs[i] @ x.conj().T)
        assert np.abs(s[i] - s_ref).max() <= 1e-10 * np.abs(s_ref).sum()
        _, dc = O.sinc_coeffs(a, 9)
        ref = float(np.sum(np.conj(gs[i]) * (O.fgfrft_grad(o, a) @ x)).real)
        assert abs(dl[i] - ref) <= 1e-10 * np.sum(np.abs(dc * s_ref))


def test_mse_step_config1():
    cfg = prep.config1()
    o = O.PowerCache(cfg.f, cfg.l)
    g = fg.PowerCache(cfg.f, cfg.l)
    rng = np.random.default_rng(5)
    clean = cfg.x + 0.1 * rng.standard_normal(cfg.x.shape)
    loss, dl, y = fg.mse_step(g, cfg.alphas, cfg.x, clean, want_y=True)
    lr, dr, yr = O.dlda_mse(o, cfg.alphas[0], cfg.x, clean)
    assert rel(y[0], yr) <= 1e-10
    assert loss[0] == pytest.approx(lr, rel=1e-10)
    _, dc = O.sinc_coeffs(cfg.alphas[0], cfg.l)
    s_ref = O.power_dots(o, (2 * (yr - clean) / yr.size) @ cfg.x.conj().T)
    assert abs(dl[0] - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))


def test_cpp_dropin_header_suite():
    """The reference's transform/sinc test cases compiled against include/fgfrft/*.hpp."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_dropin")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.parametrize("n,l,n_alpha", [(40, 5, 8), (97, 70, 67), (256, 64, 64), (33, 130, 9)])
def test_synthesis_sweep_dmma_path(n, l, n_alpha):
    """DMMA sweep synthesis (several power chunks, > 64 orders, ragged n) vs the oracle; DQ too."""
    f = prep.random_unitary(n, 900 + n)
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l, powers=o.slabs)
    alphas = list(np.linspace(-2.2, 2.3, n_alpha))
    qs = fg.synthesize(g, alphas)
    dqs = fg.synthesize(g, alphas, which=fg.DQ)
    for i in range(0, n_alpha, max(1, n_alpha // 9)):
        assert rel(qs[i], O.fgfrft_matrix(o, alphas[i])) <= 1e-14
        assert rel(dqs[i], O.fgfrft_grad(o, alphas[i])) <= 1e-13
    # conjugate symmetry across the sweep: Q(-a) = Q(a)^H to 1e-14 elementwise
    sym = fg.synthesize(g, [-a for a in alphas[:8]])
    for i in range(8):
        assert np.abs(sym[i] - qs[i].conj().T).max() <= 1e-14


@pytest.mark.parametrize("n,l,n_alpha,b", [(90, 9, 8, 17), (150, 70, 67, 5), (33, 3, 64, 40)])
def test_dlda_sweep_dmma_path(n, l, n_alpha, b):
    """>= 8 orders route to the DMMA split-K contraction (several power / order chunks)."""
    f = prep.random_unitary(n, 500 + n)
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    alphas = list(np.linspace(-1.3, 2.1, n_alpha))
    gs = [rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b)) for _ in alphas]
    dl, s = fg.dlda(g, alphas, gs, x)
    for i in range(0, n_alpha, max(1, n_alpha // 7)):
        s_ref = O.power_dots(o, gs[i] @ x.conj().T)
        assert np.abs(s[i] - s_ref).max() <= 1e-10 * np.abs(s_ref).sum()
        _, dc = O.sinc_coeffs(alphas[i], l)
        assert abs(dl[i] - float(np.dot(dc, s_ref))) <= 1e-10 * np.sum(np.abs(dc * s_ref))


# --------------------------------------------------------------------------- complex64 path

@pytest.mark.parametrize("n,l,b", [(64, 8, 5), (150, 16, 33), (256, 32, 64)])
def test_complex64_path_within_1e4_of_fp64_oracle(n, l, b):
    """North star: the optional complex64 path within 1e-4 of the fp64 oracle. The c64 cache is
    built in complex128 (DMMA) and demoted per power; synthesis, FP32 GEMM and the gradient
    contraction run on complex64 data."""
    f = prep.random_unitary(n, 70 + n)
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l, dtype=fg.C64)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    alphas = [0.37, -0.8, 1.0, 0.0]
    for a, q in zip(alphas, fg.synthesize(g, alphas)):
        assert rel(q, O.fgfrft_matrix(o, a)) <= 1e-4
    ys = fg.apply_series(g, alphas, x)
    yi = fg.apply_series(g, alphas, x, inverse=True)
    loss, dl, _ = fg.mse_step(g, alphas, x, xc)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        assert rel(ys[i], q @ x) <= 1e-4
        assert rel(yi[i], q.conj().T @ x) <= 1e-4
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(loss[i] - lr) <= 1e-4 * lr
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (q @ x - xc) / (n * b)) @ x.conj().T)
        assert abs(dl[i] - dr) <= 1e-4 * np.sum(np.abs(dc * s_ref))
    assert np.array_equal(fg.synthesize(g, [0.0])[0], np.eye(n))  # order 0 still exact
    with pytest.raises(fg.ParameterError):
        fg.PowerCache(prep.random_unitary(7, 1), 2, dtype=fg.C64)  # odd n: TMA alignment


# --------------------------------------------------------------------------- real-F path

@pytest.mark.parametrize("n,l,b", [(64, 8, 5), (100, 12, 33), (256, 32, 17)])
def test_real_f_path_matches_complex_path_and_oracle(n, l, b, monkeypatch):
    """Graph-derived F is real: the cache is stored real and the real kernels run. They must agree
    with the oracle (bit-exact single-order synthesis) and with the forced complex path."""
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 7 + n)))
    assert np.all(f.imag == 0)
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    assert g.is_real()
    monkeypatch.setenv("FGFRFT_NO_REAL", "1")
    gc = fg.PowerCache(f, l)
    monkeypatch.delenv("FGFRFT_NO_REAL")
    assert not gc.is_real()
    ge = fg.PowerCache(f, l, powers=o.slabs)
    assert ge.is_real()
    g.set_engine(fg.ENGINE_DMMA)  # this test pins the synthesis + DMMA GEMM route
    gc.set_engine(fg.ENGINE_DMMA)
    for k in (1, 2, l):
        assert rel(g.power(k), o.power(k)) <= 1e-13
        assert np.all(g.power(k).imag == 0)
    for a in (0.37, -1.1, 0.0, 2.0):  # scalar exact path on identical cache bytes
        q = fg.synthesize(ge, [a])[0]
        assert np.array_equal(q, O.fgfrft_matrix(o, a))
        assert np.array_equal(fg.synthesize(ge, [a], which=fg.DQ)[0], O.fgfrft_grad(o, a))
    alphas = list(np.linspace(-0.5, 1.9, 12))  # sweep: DMMA kernels
    qs, qc = fg.synthesize(g, alphas), fg.synthesize(gc, alphas)
    for i, a in enumerate(alphas):
        assert rel(qs[i], O.fgfrft_matrix(o, a)) <= 1e-13
        assert rel(qs[i], qc[i]) <= 1e-13
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    for al in ([0.37], alphas):
        y, yc = fg.apply_series(g, al, x), fg.apply_series(gc, al, x)
        yi = fg.apply_series(g, al, x, inverse=True)
        loss, dl, _ = fg.mse_step(g, al, x, xc)
        lc, dlc, _ = fg.mse_step(gc, al, x, xc)
        for i, a in enumerate(al):
            q = O.fgfrft_matrix(o, a)
            assert rel(y[i], q @ x) <= 1e-13 and rel(y[i], yc[i]) <= 1e-13
            assert rel(yi[i], q.T @ x) <= 1e-13
            lr, dr, _ = O.dlda_mse(o, a, x, xc)
            assert abs(loss[i] - lr) <= 1e-12 * lr and abs(loss[i] - lc[i]) <= 1e-12 * lr
            _, dc = O.sinc_coeffs(a, l)
            s_ref = O.power_dots(o, (2.0 * (q @ x - xc) / (n * b)) @ x.conj().T)
            tol = 1e-10 * np.sum(np.abs(dc * s_ref))
            assert abs(dl[i] - dr) <= tol and abs(dl[i] - dlc[i]) <= tol


# --------------------------------------------------------------------------- power-product route (INT8)

@pytest.mark.parametrize("n,l,b,n_alpha", [(64, 8, 5, 9), (100, 12, 33, 12), (256, 32, 17, 40), (200, 64, 3, 70)])
def test_power_route_matches_oracle(n, l, b, n_alpha):
    """Real F, order sweep through Z_k = F^k X on the INT8 tensor cores (Ozaki, 7 digits) and the
    DMMA combination: F^a X, the MSE loss and dL/dalpha within the north-star bar (1e-10) of the
    oracle's series; typically ~1e-13."""
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 11 + n)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    assert g.is_real()
    assert 0 <= g.orthogonality() <= 1e-12  # graph GFT: the Gram form of the step is used
    g.set_engine(fg.ENGINE_INT8)
    rng = np.random.default_rng(n + b)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    alphas = list(np.linspace(-0.9, 2.0, n_alpha))
    loss, dl, y = fg.mse_step(g, alphas, x, xc, want_y=True)
    worst = 0.0
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        yr = q @ x
        e = rel(y[i], yr)
        worst = max(worst, e)
        assert e <= 1e-10
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(loss[i] - lr) <= 1e-10 * lr
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (yr - xc) / (n * b)) @ x.conj().T)
        assert abs(dl[i] - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))
    assert worst <= 5e-12  # the INT8 products are far inside the bar
    # the DMMA engine on the same handle agrees
    g.set_engine(fg.ENGINE_DMMA)
    loss2, dl2, y2 = fg.mse_step(g, alphas, x, xc, want_y=True)
    assert np.max(np.abs(loss2 - loss) / loss) <= 1e-10
    assert all(rel(y2[i], y[i]) <= 1e-10 for i in range(len(alphas)))


@pytest.mark.parametrize("n,l,b", [(96, 8, 7), (300, 16, 40), (512, 24, 129)])
def test_int8_synthesis_route_matches_oracle(n, l, b):
    """Real F, few orders (synthesis route) with the INT8 engine: op(Q) X and Re(G X^H) are Ozaki
    GEMMs on the INT8 tensor cores; forward, inverse, loss and dL/dalpha within 1e-10 of the
    oracle, and within 1e-10 of the DMMA engine."""
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.08, 3 + n)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    g.set_engine(fg.ENGINE_INT8)
    rng = np.random.default_rng(b)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    alphas = [0.37, -1.3]  # 2 orders < L / 2: synthesis route
    y = fg.apply_series(g, alphas, x)
    yi = fg.apply_series(g, alphas, x, inverse=True)
    loss, dl, _ = fg.mse_step(g, alphas, x, xc)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        assert rel(y[i], q @ x) <= 2e-12
        assert rel(yi[i], q.T @ x) <= 2e-12
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(loss[i] - lr) <= 1e-10 * lr
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (q @ x - xc) / (n * b)) @ x.conj().T)
        assert abs(dl[i] - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))
    g.set_engine(fg.ENGINE_DMMA)
    y2 = fg.apply_series(g, alphas, x)
    loss2, dl2, _ = fg.mse_step(g, alphas, x, xc)
    assert all(rel(y2[i], y[i]) <= 2e-12 for i in range(2))
    assert np.max(np.abs(loss2 - loss) / loss) <= 1e-10


@pytest.mark.parametrize("n,l,b,n_alpha", [(64, 8, 5, 9), (256, 32, 17, 40)])
def test_power_route_apply_and_dlda(n, l, b, n_alpha):
    """Order sweeps of apply_forward / apply_inverse and of the dL/dalpha contraction through the
    power products (INT8 engine): within 1e-10 of the oracle; Q(a)^T X is Q(-a) X."""
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 21 + n)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    g.set_engine(fg.ENGINE_INT8)
    rng = np.random.default_rng(7 * n + b)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    gr = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    alphas = list(np.linspace(-1.7, 2.3, n_alpha))
    y = fg.apply_series(g, alphas, x)
    yi = fg.apply_series(g, alphas, x, inverse=True)
    dl, s = fg.dlda(g, alphas, np.broadcast_to(gr, (n_alpha, n, b)), x)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        assert rel(y[i], q @ x) <= 1e-11
        assert rel(yi[i], q.T @ x) <= 1e-11
        s_ref = O.power_dots(o, gr @ x.conj().T)
        _, dc = O.sinc_coeffs(a, l)
        assert np.max(np.abs(s[i] - s_ref)) <= 1e-10 * np.max(np.abs(s_ref))
        assert abs(dl[i] - float(np.dot(dc, s_ref))) <= 1e-10 * np.sum(np.abs(dc * s_ref))


def test_power_route_non_orthogonal_real_f():
    """A real but non-orthogonal F (0.97 x a graph GFT): the power-product MSE step must not use the
    Gram identity; s_k = Re<G, F^k X> is contracted directly and matches the oracle."""
    n, l, b = 128, 16, 9
    f = 0.97 * prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 5)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    assert g.orthogonality() > 1e-3
    g.set_engine(fg.ENGINE_INT8)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = 0.9 * x
    alphas = list(np.linspace(0.1, 1.9, 20))
    loss, dl, _ = fg.mse_step(g, alphas, x, xc)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(loss[i] - lr) <= 1e-10 * lr
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (q @ x - xc) / (n * b)) @ x.conj().T)
        assert abs(dl[i] - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))


@pytest.mark.parametrize("n,l,b,n_alpha", [(256, 32, 17, 40), (128, 64, 6, 64)])
def test_int8_combine_engine(n, l, b, n_alpha):
    """Experimental engine: the per-order combination Y = C Z also on the INT8 tensor cores (Z as
    base-254 digits bounded by the column norms of X), Gram form of s_k. Within 1e-10 of the
    oracle and of the DMMA engine."""
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 31 + n)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    g.set_engine(fg.ENGINE_INT8_COMBINE)
    rng = np.random.default_rng(n * b)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    alphas = list(np.linspace(-0.4, 1.8, n_alpha))
    loss, dl, y = fg.mse_step(g, alphas, x, xc, want_y=True)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        yr = q @ x
        assert rel(y[i], yr) <= 1e-11
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(loss[i] - lr) <= 1e-10 * lr
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (yr - xc) / (n * b)) @ x.conj().T)
        assert abs(dl[i] - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))


@pytest.mark.parametrize("n,l,b", [(256, 32, 1), (100, 12, 7), (64, 8, 32), (1024, 16, 3)])
def test_fused_small_batch_apply(n, l, b):
    """Small signal batches (2B <= 64): fused synthesis + product, Q(alpha) never leaves the SM.
    Forward and inverse against the oracle (1e-12) and against the synthesis + DMMA GEMM route."""
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 41 + n)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l)
    rng = np.random.default_rng(n + 3 * b)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    alphas = [0.37, 1.0, -0.81]
    launches = fg.launch_count()
    y = fg.apply_series(g, alphas, x)
    yi = fg.apply_series(g, alphas, x, inverse=True)
    assert fg.launch_count() - launches <= 2 * 4   # fused + reduce per call (+ coefficient upload)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        assert rel(y[i], q @ x) <= 1e-12
        assert rel(yi[i], q.T @ x) <= 1e-12
    g.set_engine(fg.ENGINE_DMMA)
    y2 = fg.apply_series(g, alphas, x)
    assert all(rel(y2[i], y[i]) <= 1e-13 for i in range(len(alphas)))


# --------------------------------------------------------------------------- on-disk cache (8(f) rank 4)

@pytest.mark.parametrize("kind,dtype", [("real", fg.C128), ("complex", fg.C128), ("complex", fg.C64)])
def test_cache_save_load_round_trip(tmp_path, kind, dtype):
    n, l = (300, 12) if kind == "real" else (130, 9)
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.05, 4))) if kind == "real" else prep.random_unitary(n, 8)
    g = fg.PowerCache(f, l, dtype=dtype)
    path = str(tmp_path / "cache.fgc")
    g.save(path)
    h = fg.PowerCache.load(path)
    assert (h.n(), h.l(), h.fingerprint(), h.dtype) == (n, l, g.fingerprint(), dtype)
    assert h.is_real() == g.is_real()
    if kind == "real":
        assert h.orthogonality() == pytest.approx(g.orthogonality(), rel=1e-9)
    for k in (1, l // 2, l):
        assert np.array_equal(h.power(k), g.power(k))
    alphas = [0.31, 1.2]
    assert np.array_equal(fg.synthesize(h, alphas), fg.synthesize(g, alphas))
    h.verify(f) if dtype == fg.C128 else None
    # budget check as in the constructor; corruption and truncation are detected
    with pytest.raises(fg.CapacityError):
        fg.PowerCache.load(path, memory_budget=1024)
    raw = bytearray(open(path, "rb").read())
    bad = str(tmp_path / "bad.fgc")
    raw2 = bytearray(raw)
    raw2[-100] ^= 0x40  # a slab byte
    open(bad, "wb").write(raw2)
    with pytest.raises(fg.NumericalError):
        fg.PowerCache.load(bad)
    open(bad, "wb").write(raw[: len(raw) // 2])
    with pytest.raises(fg.ParseError):
        fg.PowerCache.load(bad)
    raw3 = bytearray(raw)
    raw3[0] = ord("X")
    open(bad, "wb").write(raw3)
    with pytest.raises(fg.ParseError):
        fg.PowerCache.load(bad)
    with pytest.raises(fg.IoError):
        fg.PowerCache.load(str(tmp_path / "missing.fgc"))


def test_complex64_api_over_real_f_runs_the_real_fp64_path():
    """A real F under dtype C64: powers stored as real doubles (same 8 bytes per element), the real
    FP64 kernels run, and the *_dev entry points take / return complex64 device buffers."""
    import torch
    n, l, b = 512, 16, 48
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.03, 5)))
    g64 = fg.PowerCache(f, l, dtype=fg.C64)
    g128 = fg.PowerCache(f, l)
    dt = ctypes.c_int()
    fg._check(fg.lib().fgfrft_cache_info(g64.handle, None, None, None, ctypes.addressof(dt), None))
    assert dt.value == fg.C64 and g64.is_real() and g64.device_bytes() == g128.device_bytes()
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))).astype(np.complex64)
    xc = (x + 0.1 * rng.standard_normal((n, b))).astype(np.complex64)
    alphas = np.array([0.37, 1.21])
    lib = fg.lib()
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    xcd = torch.from_numpy(np.ascontiguousarray(xc.T)).cuda()
    y = torch.empty((2, b, n), dtype=torch.complex64, device="cuda")
    fg._check(lib.fgfrft_apply_dev(g64.handle, alphas.ctypes.data, 2, 0, 0, xd.data_ptr(), b, y.data_ptr()))
    q = torch.empty((2, n, n), dtype=torch.complex64, device="cuda")
    fg._check(lib.fgfrft_synthesize_dev(g64.handle, alphas.ctypes.data, 2, 0, 0, q.data_ptr()))
    loss = torch.empty(2, dtype=torch.float64, device="cuda")
    dl = torch.empty(2, dtype=torch.float64, device="cuda")
    fg._check(lib.fgfrft_mse_step_dev(g64.handle, alphas.ctypes.data, 2, xd.data_ptr(), xcd.data_ptr(), b, None,
                                      loss.data_ptr(), dl.data_ptr()))
    torch.cuda.synchronize()
    x128, xc128 = x.astype(np.complex128), xc.astype(np.complex128)
    y_ref = fg.apply_series(g128, alphas, x128)
    q_ref = fg.synthesize(g128, alphas)
    l_ref, d_ref, _ = fg.mse_step(g128, alphas, x128, xc128)
    ys = y.cpu().numpy().transpose(0, 2, 1)
    for i in range(2):
        assert rel(ys[i], y_ref[i]) <= 1e-6                       # complex64 rounding of the output only
        assert rel(q.cpu().numpy()[i].T, q_ref[i]) <= 1e-6
    assert np.allclose(loss.cpu().numpy(), l_ref, rtol=1e-12)   # FP64 arithmetic on the same inputs
    assert np.allclose(dl.cpu().numpy(), d_ref, rtol=1e-9, atol=1e-14)
    # host-buffer entry points return complex128 as before
    assert rel(fg.apply_series(g64, alphas, x128)[0], y_ref[0]) <= 1e-14


def test_concurrent_handles_from_threads():
    """Distinct handles used from concurrent host threads (ctypes releases the GIL): results equal
    the sequential ones; one handle shared by two threads is serialised by the handle."""
    import threading
    fa = prep.gft_from_shift(prep.laplacian(prep.er_graph(600, 0.02, 1)))
    fb = prep.random_unitary(300, 2)
    rng = np.random.default_rng(3)
    xa = rng.standard_normal((600, 40)) + 1j * rng.standard_normal((600, 40))
    xb = rng.standard_normal((300, 20)) + 1j * rng.standard_normal((300, 20))
    ga, gb = fg.PowerCache(fa, 16), fg.PowerCache(fb, 12)
    alphas = list(np.linspace(0.1, 1.9, 12))
    ref_a = fg.mse_step(ga, alphas, xa, xa + 0.1)
    ref_b = fg.apply_series(gb, alphas[:3], xb)
    out, errs = {}, []

    def work(key, fn):
        try:
            for _ in range(5):
                out[key] = fn()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=("a", lambda: fg.mse_step(ga, alphas, xa, xa + 0.1))),
          threading.Thread(target=work, args=("b", lambda: fg.apply_series(gb, alphas[:3], xb))),
          threading.Thread(target=work, args=("a2", lambda: fg.mse_step(ga, alphas, xa, xa + 0.1)))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for key in ("a", "a2"):
        assert np.array_equal(out[key][0], ref_a[0]) and np.array_equal(out[key][1], ref_a[1])
    assert np.array_equal(out["b"], ref_b)


@pytest.mark.parametrize("n,l,b,lo,hi,na", [(512, 16, 40, 0.0, 2.0, 64), (600, 24, 33, -0.7, 0.4, 16),
                                             (520, 12, 64, 1.0, 4.5, 20), (1024, 64, 48, 0.2, 0.3, 32),
                                             (512, 10, 40, -3.0, 3.0, 40)])
def test_node_route_sweeps_match_oracle(n, l, b, lo, hi, na):
    """Order sweeps on a real F through the node route (Chebyshev interpolation of Q(a) over the
    sweep's interval, INT8 node operators; wide intervals fall back to the power route) against
    the oracle: F^a X, Q(a)^H X, loss and dL/da within 1e-10."""
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 6.0 / n, n + l)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l, powers=o.slabs)
    rng = np.random.default_rng(n + na)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    alphas = list(np.linspace(lo, hi, na))
    loss, dl, ym = fg.mse_step(g, alphas, x, xc, want_y=True)
    route, nodes = g.route_info()
    assert route in (1, 2)
    ys = fg.apply_series(g, alphas, x)
    yi = fg.apply_series(g, alphas, x, inverse=True)
    for i in range(0, na, max(1, na // 8)):
        a = alphas[i]
        q = O.fgfrft_matrix(o, a)
        assert rel(ys[i], q @ x) <= 1e-10
        assert rel(yi[i], q.T @ x) <= 1e-10
        assert rel(ym[i], q @ x) <= 1e-10
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(loss[i] - lr) <= 1e-10 * lr
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (q @ x - xc) / (n * b)) @ x.conj().T)
        assert abs(dl[i] - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))
    # (the element-pair node operators, FGFRFT_NODE_PAIRS=1, hold 32 nodes: wider sweeps fall back)
    if hi - lo <= (4.0 if os.environ.get("FGFRFT_NODE_PAIRS") == "1" else 6.0):
        assert route == 2 and nodes <= 11 + 5 * (hi - lo), nodes
