"""Seeded random shapes through every route of the C ABI (synthesis / fused small-batch apply /
INT8 and DMMA GEMMs / power products / one-pass Q + dQ step / complex64 bridge) against the
oracle: ragged n (not multiples of the 32-tile or the 128-row INT8 tile), tiny and odd sizes,
1..12 orders, real and complex F."""
import numpy as np
import pytest

import oracle as O
import paper_2602_20870_b200 as fg
import prep

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 2, 3, 17, 33, 64, 95, 130, 257, 513, 600]))
    l = int(rng.integers(1, 20))
    b = int(rng.choice([1, 2, 7, 32, 33, 70]))
    na = int(rng.integers(1, 13))
    real = bool(rng.integers(0, 2)) and n >= 3
    engine = int(rng.choice([fg.ENGINE_AUTO, fg.ENGINE_DMMA, fg.ENGINE_INT8]))
    if real:
        f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, min(1.0, 4.0 / n), seed)))
    else:
        f = prep.random_unitary(n, seed)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    alphas = list(rng.uniform(-1.5, 2.5, na))
    return n, l, b, f, x, xc, alphas, engine


@pytest.mark.parametrize("seed", range(24))
def test_random_shapes_all_routes(seed):
    n, l, b, f, x, xc, alphas, engine = _case(seed)
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l, powers=o.slabs)
    if g.is_real():
        g.set_engine(engine)
    ys = fg.apply_series(g, alphas, x)
    yi = fg.apply_series(g, alphas, x, inverse=True)
    loss, dl, ym = fg.mse_step(g, alphas, x, xc, want_y=True)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        tol = 1e-10
        assert rel(ys[i], q @ x) <= tol, (i, a)
        assert rel(yi[i], q.conj().T @ x) <= tol, (i, a)
        assert rel(ym[i], q @ x) <= tol
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(loss[i] - lr) <= 1e-10 * lr
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (q @ x - xc) / (n * b)) @ x.conj().T)
        assert abs(dl[i] - dr) <= 1e-10 * max(np.sum(np.abs(dc * s_ref)), 1e-300)
    d2, s = fg.dlda(g, alphas, [2.0 * (O.fgfrft_matrix(o, a) @ x - xc) / (n * b) for a in alphas], x)
    for i, a in enumerate(alphas):
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (O.fgfrft_matrix(o, a) @ x - xc) / (n * b)) @ x.conj().T)
        assert np.abs(s[i] - s_ref).max() <= 1e-10 * max(np.abs(s_ref).sum(), 1e-300)


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_complex64_real_f(seed):
    """complex64 API over a real F (real-double storage): within 1e-10 of the oracle through the
    host entry points (complex128 host buffers, FP64 arithmetic)."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.choice([34, 96, 258, 520]))
    l, b = int(rng.integers(2, 16)), int(rng.choice([1, 9, 40]))
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 4.0 / n, seed)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l, dtype=fg.C64)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    alphas = list(rng.uniform(-1.0, 2.0, int(rng.integers(1, 5))))
    ys = fg.apply_series(g, alphas, x)
    for i, a in enumerate(alphas):
        assert rel(ys[i], O.fgfrft_matrix(o, a) @ x) <= 1e-10
