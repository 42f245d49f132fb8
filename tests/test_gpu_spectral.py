"""Exact GFRFT and eigendecomposition on the GPU and the cascaded order
learner (rank 2), against the oracle restatements of spectral.hpp:121-174 and learn.hpp:55-166,
plus the reference's own known-answer tests (test_spectral.cpp, test_learn.cpp)."""
import math

import numpy as np
import pytest

import oracle as O
import paper_2602_20870_b200 as fg
import prep

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _grid_gft(side):
    return prep.gft_from_shift(prep.laplacian(prep.grid_graph(side, side)))


# --------------------------------------------------------------------------- spectrum / exact

@pytest.mark.parametrize("kind,n", [("haar", 24), ("haar", 200), ("grid", 8), ("er", 300), ("synthetic", 96)])
def test_decomposition_matches_oracle(kind, n):
    if kind == "haar":
        f = prep.random_unitary(n, 5)
    elif kind == "grid":
        f = _grid_gft(n)
    elif kind == "er":
        f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.05, 9)))
    else:
        f, _, _ = prep.synthetic_unitary(prep.spread_phases(n, 0.2, 4), 21)
    ve, te = O.eigendecompose_unitary(f)
    eig = fg.eigendecompose_unitary(f)
    assert np.max(np.abs(eig.theta - te)) <= 1e-10
    assert np.all(np.diff(eig.theta) >= 0)
    v = eig.v
    # V unitary, F V = V diag(e^{j theta}), the operators agree with the oracle's
    assert rel(v.conj().T @ v, np.eye(f.shape[0])) <= 1e-12
    assert rel(f @ v, v * np.exp(1j * eig.theta)[None, :]) <= 1e-9
    for a in (0.3, 1.0, -0.7):
        assert rel(fg.exact_gfrft(eig, a).q, O.exact_gfrft((ve, te), a)) <= 1e-10
        assert rel(fg.exact_gfrft_grad(eig, a), O.exact_gfrft_grad((ve, te), a)) <= 1e-10


def test_identity_and_rotation_spectra():  # test_spectral.cpp:34-40, 64-71
    eig = fg.eigendecompose_unitary(np.eye(16))
    assert np.all(eig.theta == 0.0)
    c, s = math.cos(math.pi / 4), math.sin(math.pi / 4)
    eig = fg.eigendecompose_unitary(np.array([[c, -s], [s, c]]))
    assert np.max(np.abs(eig.theta - np.array([-math.pi / 4, math.pi / 4]))) <= 1e-14
    # alpha = 0.5 of a pi/4 rotation is a pi/8 rotation (test_spectral.cpp:114-119)
    q = fg.exact_gfrft(eig, 0.5).q
    c8, s8 = math.cos(math.pi / 8), math.sin(math.pi / 8)
    assert np.max(np.abs(q - np.array([[c8, -s8], [s8, c8]]))) <= 1e-14


def test_known_spectrum_and_exact_orders():  # test_spectral.cpp:42-47, 96-127
    f, v, theta = prep.synthetic_unitary(prep.spread_phases(40, 0.2, 4), 21)
    eig = fg.UnitaryEigen(v=v, theta=theta)
    assert np.array_equal(eig.theta, theta)
    assert rel(fg.exact_gfrft(eig, 1.0).q, f) <= 1e-12
    assert rel(fg.exact_gfrft(eig, 0.0).q, np.eye(40)) <= 1e-13
    assert rel(fg.exact_gfrft(eig, 2.0).q, f @ f) <= 1e-12
    q = fg.exact_matrices(eig, [0.3, 0.4, 0.7])
    assert rel(q[0] @ q[1], q[2]) <= 1e-12
    # finite differences of the exact operator (test_spectral.cpp:129-150)
    h = 1e-4
    fd = (fg.exact_gfrft(eig, 0.6 + h).q - fg.exact_gfrft(eig, 0.6 - h).q) / (2 * h)
    assert rel(fg.exact_gfrft_grad(eig, 0.6), fd) <= 1e-6


def test_non_unitary_input_fails():  # test_spectral.cpp:174-180
    a = np.eye(8)
    a[0, 1] = 0.5
    with pytest.raises(fg.NumericalError):
        fg.eigendecompose_unitary(a)


def test_phase_margin_warns():  # test_spectral.cpp:152-172
    f, v, theta = prep.synthetic_unitary(prep.spread_phases(16, 0.01, 2), 3)
    with pytest.warns(UserWarning):
        m = fg.phase_margin(fg.UnitaryEigen(v=v, theta=theta))
    assert abs(m - 0.01) <= 1e-12


# --------------------------------------------------------------------------- cascade

@pytest.mark.parametrize("backend", [fg.FAST, fg.EXACT])
@pytest.mark.parametrize("kind,n,k,l", [("haar", 24, 1, 8), ("haar", 24, 3, 8), ("haar", 64, 2, 10),
                                        ("grid", 12, 3, 16), ("haar", 256, 2, 20)])
def test_cascade_eval_matches_oracle(backend, kind, n, k, l):
    f = prep.random_unitary(n, 3) if kind == "haar" else _grid_gft(n)
    eig = O.eigendecompose_unitary(f)
    ref = O.Cascade(f, k, 1.5, l, backend, eig=eig)
    prob = fg.CascadeProblem(f, k, 1.5, l, backend, eig=fg.UnitaryEigen(v=eig[0], theta=eig[1]))
    rng = prep.Rng(71 + k)
    for _ in range(4):
        al = np.array([rng.uniform(-0.5, 1.8) for _ in range(k)])
        loss, grad = prob.eval(al)
        lr, gr = ref.eval(al)
        assert abs(loss - lr) <= 1e-10 * max(lr, 1e-300) + 1e-14
        assert np.max(np.abs(grad - gr)) <= 1e-9 * max(np.max(np.abs(gr)), 1e-3)


@pytest.mark.parametrize("backend", [fg.FAST, fg.EXACT])
def test_cascade_gradients_finite_differences(backend):  # acceptance.cpp:154-180
    f = prep.random_unitary(64, 5)
    prob = fg.CascadeProblem(f, 2, 1.5, 10, backend)
    rng = prep.Rng(500)
    for _ in range(5):
        al = np.array([rng.uniform(-0.5, 2.0), rng.uniform(-0.5, 2.0)])
        _, grad = prob.eval(al)
        for l in range(2):
            def loss_at(a, l=l):
                aa = al.copy()
                aa[l] = a
                return prob.eval(aa)[0]
            fd = (loss_at(al[l] + 1e-4) - loss_at(al[l] - 1e-4)) / 2e-4
            assert abs(grad[l] - fd) / max(abs(fd), 1e-12) <= 1e-5


def test_learn_orders_matches_oracle_loop():
    f = prep.random_unitary(48, 21)
    eig = O.eigendecompose_unitary(f)
    ref = O.Cascade(f, 2, 1.5, 30, "fast", eig=eig)
    tl, ta, fl, fa = O.learn_orders(ref, 2, 0.1, 40, 0.01)
    prob = fg.CascadeProblem(f, 2, 1.5, 30, fg.FAST, eig=fg.UnitaryEigen(v=eig[0], theta=eig[1]))
    out = prob.learn(0.1, 40, 0.01)
    assert np.max(np.abs(out["traj_loss"] - tl) / tl) <= 1e-8
    assert np.max(np.abs(out["traj_alphas"] - ta)) <= 1e-9
    assert abs(out["final_loss"] - fl) <= 1e-8 * fl


@pytest.mark.parametrize("k", [1, 2])
def test_learned_orders_additivity(k):  # test_learn.cpp:104-120
    # seed 5: see test_oracle.py::test_cascade_learned_orders_additivity for the choice
    out = fg.learn_orders(prep.random_unitary(48, 5), depth=k, init_order=0.1, target_order=1.5, truncation=30,
                          epochs=200, lr=0.01, backend=fg.FAST)
    assert out["final_loss"] <= 1e-4
    assert abs(out["final_alpha_sum"] - 1.5) <= 0.01


def test_exact_backend_stationary_at_target():  # test_learn.cpp:90-102
    out = fg.learn_orders(prep.random_unitary(20, 8), depth=1, init_order=0.7, target_order=0.7, epochs=10,
                          backend=fg.EXACT)
    assert out["final_loss"] == 0.0  # Q and the target are the same device computation
    assert np.all(out["traj_loss"] == 0.0)
    assert np.all(out["traj_alphas"][:, 0] == 0.7)


def test_cascade_errors():
    f = prep.random_unitary(16, 2)
    with pytest.raises(fg.ParameterError):
        fg.CascadeProblem(f, 0, 1.5, 8)
    prob = fg.CascadeProblem(f, 2, 1.5, 8)
    with pytest.raises(fg.ShapeError):
        prob.eval([0.1])
    with pytest.raises(fg.ParameterError):
        prob.learn(0.1, 0, 0.01)


# --------------------------------------------------------------------------- acceptance 3-4 fully on the GPU

def test_series_vs_exact_errors_on_gpu_three_digits():  # acceptance.cpp:81-101 + north star "3 digits"
    f = prep.random_unitary(1000, 42)
    alphas = [0.15, 0.35, 0.55, 0.75, 0.95]
    eig = fg.eigendecompose_unitary(f)
    cache = fg.PowerCache(f, 10)
    qs = fg.synthesize(cache, alphas)
    ex = fg.exact_matrices(eig, alphas)
    ve, te = O.eigendecompose_unitary(f)
    oc = O.PowerCache(f, 10)
    gpu = [O.matrix_errors(qs[i], ex[i]) for i in range(len(alphas))]
    ref = [O.matrix_errors(O.fgfrft_matrix(oc, a, nthreads=8), O.exact_gfrft((ve, te), a)) for a in alphas]
    for g, r in zip(gpu, ref):
        for key in ("mse", "nmse", "mae"):
            assert float(f"{g[key]:.3e}") == float(f"{r[key]:.3e}")
    nmse = sum(e["nmse"] for e in gpu) / len(gpu)
    mae = sum(e["mae"] for e in gpu) / len(gpu)
    assert 2.05e-2 / 3 <= nmse <= 2.05e-2 * 3
    assert 4.00e-3 / 3 <= mae <= 4.00e-3 * 3


def test_monotone_convergence_on_gpu():  # acceptance.cpp:103-117
    f, v, th = prep.synthetic_unitary(prep.spread_phases(512, 0.1 * math.pi, 23), 63)
    eig = fg.UnitaryEigen(v=v, theta=th)
    exact = fg.exact_gfrft(eig, 0.5).q
    cache = fg.PowerCache(f, 30)
    prev = None
    for l in (10, 20, 30):
        q = fg.fgfrft_matrix(cache, 0.5, l).q
        nmse = np.linalg.norm(q - exact) ** 2 / np.linalg.norm(exact) ** 2
        if prev is not None:
            assert nmse <= 0.9 * prev
        prev = nmse
