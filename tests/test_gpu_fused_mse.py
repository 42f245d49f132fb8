"""GPU parity of the fused MSE step (ozgemm CM 1 with OzOut::lpart, packed.cu
fused_mse_finish_kernel): on the device-resident step the product GEMM takes each M tile of Q rows
and then the matching dQ tile, stores Y, never stores dY, and accumulates |Y - Xc|^2 and
Re conj(Y - Xc) dY in its epilogue. Checked against the oracle (transform.hpp:111-148, the
learn.hpp:88-92 loss / gradient form) at the north star's 1e-10 bar, against the separate
elementwise pass (FGFRFT_FUSED_MSE=0) on identical products, with padded rows (n % 128 != 0) and
padded signal columns (2b % 64 != 0), one and two orders (integer and negative ones too), with and without the Y output, on the
packed and the order-window routes, and run to run bit for bit.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2602_20870_b200 as fg
import prep

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def problem():
    n, l, b = 1000, 16, 37
    rng0 = prep.Rng(21)
    pts = rng0.uniforms(2 * n).reshape(n, 2)
    f = prep.gft_from_shift(prep.laplacian(prep.knn_graph(pts, 8)))
    rng = np.random.default_rng(9)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * (rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b)))
    old = os.environ.pop("FGFRFT_DSYNTH", None)
    g = fg.PowerCache(f, l, memory_budget=4 << 30)
    yield f, l, x, xc, g, O.PowerCache(f, l)
    g.close()
    if old is not None:
        os.environ["FGFRFT_DSYNTH"] = old


def dev_step(g, alphas, x, xc, want_y, fused=True):
    import torch
    al = np.ascontiguousarray(alphas, dtype=np.float64)
    a, (n, b) = len(al), x.shape
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    xcd = torch.from_numpy(np.ascontiguousarray(xc.T)).cuda()
    lo = torch.empty(a, dtype=torch.float64, device="cuda")
    dl = torch.empty(a, dtype=torch.float64, device="cuda")
    yd = torch.full((a, b, n), float("nan"), dtype=torch.complex128, device="cuda") if want_y else None
    g.set_stream(torch.cuda.current_stream().cuda_stream)
    old = os.environ.get("FGFRFT_FUSED_MSE")
    os.environ["FGFRFT_FUSED_MSE"] = "1" if fused else "0"
    try:
        fg._check(fg.lib().fgfrft_mse_step_dev(g.handle, al.ctypes.data, a, xd.data_ptr(), xcd.data_ptr(), b,
                                               yd.data_ptr() if want_y else None, lo.data_ptr(), dl.data_ptr()))
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("FGFRFT_FUSED_MSE", None)
        else:
            os.environ["FGFRFT_FUSED_MSE"] = old
    y = yd.cpu().numpy().transpose(0, 2, 1) if want_y else None
    return lo.cpu().numpy(), dl.cpu().numpy(), y


@pytest.mark.parametrize("alphas", [[0.37], [0.25, 1.75], [2.0], [-1.3, 0.04]])
@pytest.mark.parametrize("want_y", [True, False])
def test_fused_step_matches_oracle(problem, alphas, want_y):
    f, l, x, xc, g, o = problem
    loss, dl, y = dev_step(g, alphas, x, xc, want_y)
    assert g.route_info()[0] == 3
    for i, a in enumerate(alphas):
        lr, dr, yr = O.dlda_mse(o, a, x, xc)
        if want_y:
            assert rel(y[i], yr) <= 1e-10
        assert abs(loss[i] - lr) <= 1e-10 * lr
        s = O.power_dots(o, 2.0 * (yr - xc) @ x.conj().T / x.size)
        _, dc = O.sinc_coeffs(a, l)
        assert abs(dl[i] - dr) <= 1e-10 * max(np.sum(np.abs(dc * s)), 1e-300)


def test_fused_matches_separate_pass_and_is_deterministic(problem):
    f, l, x, xc, g, o = problem
    al = [0.81, -0.4]
    l1, d1, y1 = dev_step(g, al, x, xc, True)
    l2, d2, y2 = dev_step(g, al, x, xc, True)
    l0, d0, y0 = dev_step(g, al, x, xc, True, fused=False)
    assert np.array_equal(l1, l2) and np.array_equal(d1, d2) and np.array_equal(y1, y2)
    assert np.array_equal(y1, y0)  # the same products; only the loss sums are grouped differently
    assert np.allclose(l1, l0, rtol=1e-13, atol=0)
    assert np.allclose(d1, d0, rtol=1e-11, atol=1e-300)
    # the host-buffer step (separate pass, X in column chunks) agrees too
    lh, dh, _ = fg.mse_step(g, al, x, xc)
    assert np.allclose(l1, lh, rtol=1e-13, atol=0)
    assert np.allclose(d1, dh, rtol=1e-11, atol=1e-300)


def test_fused_step_on_the_order_window(problem):
    f, l, x, xc, g, o = problem
    g.set_order_window(0.0, 2.0)
    try:
        for a in (0.37, 1.9):
            loss, dl, y = dev_step(g, [a], x, xc, True)
            assert g.route_info()[0] == 5
            lr, dr, yr = O.dlda_mse(o, a, x, xc)
            assert rel(y[0], yr) <= 1e-10
            assert abs(loss[0] - lr) <= 1e-10 * lr
            s = O.power_dots(o, 2.0 * (yr - xc) @ x.conj().T / x.size)
            _, dc = O.sinc_coeffs(a, l)
            assert abs(dl[0] - dr) <= 1e-10 * max(np.sum(np.abs(dc * s)), 1e-300)
    finally:
        g.set_order_window(0.0, 0.0)
