"""GPU-resident denoising learner: evaluations and short Adam fits against
the oracle restatement of the reference's fast engine (learn.hpp:291-516, adam.hpp:34-53)."""
import numpy as np
import pytest

import oracle as O
import paper_2602_20870_b200 as fg
import prep

pytestmark = pytest.mark.gpu


def _problem(n, l, ch, seed):
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.08, seed)))
    rng = np.random.default_rng(seed)
    coef = np.zeros((n, ch))
    coef[: n // 8] = rng.standard_normal((n // 8, ch))
    x = f.real.T @ coef                       # smooth (band-limited) clean signals
    y = x + 0.1 * rng.standard_normal((n, ch))
    return f, x, y


@pytest.mark.parametrize("n,l,ch", [(128, 8, 3), (256, 32, 16), (512, 64, 64)])
def test_denoise_eval_matches_reference_engine(n, l, ch):
    f, x, y = _problem(n, l, ch, 5 + n)
    ref = O.FastDenoise(y, x, f.real, l)
    g = fg.PowerCache(f, l)
    dp = fg.DenoiseProblem(g, y, x)
    rng = np.random.default_rng(n)
    for alpha in (0.5, 0.83, -0.4):
        h = 1.0 + 0.1 * rng.standard_normal(n)
        loss, ga, gh = dp.eval(alpha, h)
        lr, gar, ghr = ref.eval(alpha, h)
        assert abs(loss - lr) <= 1e-10 * lr
        assert abs(ga - gar) <= 1e-9 * max(1.0, abs(gar))
        assert np.linalg.norm(gh - ghr) <= 1e-9 * np.linalg.norm(ghr)


def test_denoise_fit_matches_reference_loop():
    n, l, ch, epochs = 128, 16, 4, 12
    f, x, y = _problem(n, l, ch, 77)
    ref = O.FastDenoise(y, x, f.real, l)
    traj, ab, hb, lb, be = O.denoise_fit(ref, epochs, 0.01, 0.5)
    g = fg.PowerCache(f, l)
    dp = fg.DenoiseProblem(g, y, x)
    out = dp.fit(epochs, lr=0.01, init_alpha=0.5, want_reconstruction=True)
    tl = np.array([t[0] for t in traj])
    ta = np.array([t[1] for t in traj])
    assert np.max(np.abs(out["traj_loss"] - tl) / tl) <= 1e-8
    assert np.max(np.abs(out["traj_alpha"] - ta)) <= 1e-9
    assert out["best_epoch"] == be
    assert abs(out["alpha_best"] - ab) <= 1e-9 and abs(out["loss_best"] - lb) <= 1e-8 * lb
    assert np.max(np.abs(out["h_best"] - hb)) <= 1e-8
    rec = ref.reconstruct(ab, hb)
    assert np.linalg.norm(out["reconstruction"] - rec) <= 1e-8 * np.linalg.norm(rec)
    assert out["traj_loss"][-1] < out["traj_loss"][0]  # it learns


def test_denoise_rejects_complex64_cache():
    f = prep.random_unitary(64, 3)
    g = fg.PowerCache(f, 4, dtype=fg.C64)
    with pytest.raises(fg.ParameterError):
        fg.DenoiseProblem(g, np.zeros((64, 2)), np.zeros((64, 2)))
    with pytest.raises(fg.ShapeError):
        fg.DenoiseProblem(fg.PowerCache(f, 4), np.zeros((63, 2)), np.zeros((63, 2)))


def test_denoise_fit_non_finite_loss_reports_epoch():  # learn.hpp:499-505 (optimizer_error)
    n, l, ch = 64, 6, 2
    f, x, y = _problem(n, l, ch, 11)
    y = y.copy()
    y[3, 1] = np.nan
    dp = fg.DenoiseProblem(fg.PowerCache(f, l), y, x)
    loss, ga, gh = dp.eval(0.5, np.ones(n))
    assert not np.isfinite(loss)                 # a single evaluation just reports it
    with pytest.raises(fg.OptimizerError, match="non-finite loss at epoch 0"):
        dp.fit(5, lr=0.01, init_alpha=0.5)


@pytest.mark.parametrize("kind,loss_on_real", [("grid", False), ("synthetic", False), ("synthetic", True)])
def test_exact_denoise_backend_matches_oracle(kind, loss_on_real):  # learn.hpp:205-289, acceptance.cpp:183-226
    if kind == "grid":
        f = prep.gft_from_shift(prep.laplacian(prep.grid_graph(8, 8)))
        ve, te = O.eigendecompose_unitary(f)
    else:
        f, ve, te = prep.synthetic_unitary(prep.spread_phases(48, 0.2, 4), 21)
    n = f.shape[0]
    rng = np.random.default_rng(600)
    x = rng.standard_normal((n, 3))
    y = x + 0.5 * rng.standard_normal((n, 3))
    ref = O.ExactDenoise(y, x, (ve, te), loss_on_real)
    dp = fg.DenoiseProblem.exact(fg.UnitaryEigen(v=ve, theta=te), y, x, loss_on_real)
    for alpha in (-1.0, 0.37, 1.6):
        h = 1.0 + 0.3 * rng.standard_normal(n)
        loss, ga, gh = dp.eval(alpha, h)
        lr, gar, ghr = ref.eval(alpha, h)
        assert abs(loss - lr) <= 1e-10 * lr
        assert abs(ga - gar) <= 1e-9 * max(1.0, abs(gar))
        assert np.linalg.norm(gh - ghr) <= 1e-9 * np.linalg.norm(ghr)
        assert np.linalg.norm(dp.reconstruct(alpha, h) - ref.reconstruct(alpha, h)) <= 1e-10 * np.linalg.norm(y)
        # finite differences of the device loss (acceptance.cpp:201-220)
        fd = (dp.eval(alpha + 1e-4, h)[0] - dp.eval(alpha - 1e-4, h)[0]) / 2e-4
        assert abs(ga - fd) / max(abs(fd), 1e-12) <= 1e-5


def test_exact_denoise_fit_matches_reference_loop():
    f, ve, te = prep.synthetic_unitary(prep.spread_phases(40, 0.2, 4), 21)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((40, 2))
    y = x + 0.3 * rng.standard_normal((40, 2))
    ref = O.ExactDenoise(y, x, (ve, te))
    traj, ab, hb, lb, be = O.denoise_fit(ref, 15, 0.01, 0.5)
    dp = fg.DenoiseProblem.exact(fg.UnitaryEigen(v=ve, theta=te), y, x)
    out = dp.fit(15, lr=0.01, init_alpha=0.5, want_reconstruction=True)
    tl = np.array([t[0] for t in traj])
    assert np.max(np.abs(out["traj_loss"] - tl) / tl) <= 1e-8
    assert out["best_epoch"] == be
    assert np.linalg.norm(out["reconstruction"] - ref.reconstruct(ab, hb)) <= 1e-8 * np.linalg.norm(y)


@pytest.mark.parametrize("loss_on_real", [False, True])
@pytest.mark.parametrize("n", [48, 520])
def test_fast_denoise_complex_f_matches_oracle(n, loss_on_real):  # FastDenoiseEngine<MatrixXcd>
    f = prep.random_unitary(n, 13)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 3))
    y = x + 0.4 * rng.standard_normal((n, 3))
    l = 10
    ref = O.FastDenoise(y, x, f, l, loss_on_real)
    dp = fg.DenoiseProblem(fg.PowerCache(f, l), y, x, loss_on_real=loss_on_real)
    for alpha in (0.3, 1.1):
        h = 1.0 + 0.2 * rng.standard_normal(n)
        loss, ga, gh = dp.eval(alpha, h)
        lr, gar, ghr = ref.eval(alpha, h)
        assert abs(loss - lr) <= 1e-10 * lr
        assert abs(ga - gar) <= 1e-9 * max(1.0, abs(gar))
        assert np.linalg.norm(gh - ghr) <= 1e-9 * np.linalg.norm(ghr)
        assert np.linalg.norm(dp.reconstruct(alpha, h) - ref.reconstruct(alpha, h)) <= 1e-10 * np.linalg.norm(y)
