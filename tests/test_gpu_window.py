"""GPU parity of the order-window route (fgfrft_cache_set_order_window): Q(a), dQ/da of orders
inside a declared window interpolated from exact FP64 node operators at its Chebyshev nodes (the
node-route criterion: coefficients to 4e-15 of the largest), then the packed step's Ozaki GEMM and
loss pass -- against the oracle (transform.hpp:111-148, learn.hpp:88-92 form) at the 1e-10 bar.
Orders outside the window, a cleared window and the memory budget keep the packed route."""
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
    n, l, b = 1024, 24, 80
    rng = prep.Rng(11)
    pts = rng.uniforms(2 * n).reshape(n, 2)
    f = prep.gft_from_shift(prep.laplacian(prep.knn_graph(pts, 8)))
    r = np.random.default_rng(5)
    x = r.standard_normal((n, b)) + 1j * r.standard_normal((n, b))
    xc = x + 0.1 * r.standard_normal((n, b))
    g = fg.PowerCache(f, l, memory_budget=8 << 30)
    nodes = g.set_order_window(0.0, 2.0)
    return f, l, x, xc, g, O.PowerCache(f, l), nodes


def test_window_nodes(problem):
    f, l, x, xc, g, o, nodes = problem
    lo, hi, r = g.order_window()
    assert (lo, hi) == (0.0, 2.0) and r == nodes and 10 <= r <= 24


@pytest.mark.parametrize("alphas", [[0.37], [0.0], [2.0], [1.3], [0.25, 1.75], [0.04]])
def test_window_mse_step_matches_oracle(problem, alphas):
    f, l, x, xc, g, o, nodes = problem
    loss, dl, y = fg.mse_step(g, alphas, x, xc, want_y=True)
    assert g.route_info() == (5, nodes)
    for i, a in enumerate(alphas):
        lr, dr, yr = O.dlda_mse(o, a, x, xc)
        assert rel(y[i], yr) <= 1e-10
        assert abs(loss[i] - lr) <= 1e-10 * lr
        s = O.power_dots(o, 2.0 * (yr - xc) @ x.conj().T / x.size)
        _, dc = O.sinc_coeffs(a, l)
        assert abs(dl[i] - dr) <= 1e-10 * max(np.sum(np.abs(dc * s)), 1e-300)


def test_window_apply_and_inverse(problem):
    f, l, x, xc, g, o, nodes = problem
    for alphas, inverse in (([0.1, 0.9], False), ([0.3, 1.1, 1.6, 1.9], False), ([0.6], True)):
        y = fg.apply_series(g, alphas, x, inverse=inverse)  # inverse: Q(-a) lies outside: packed route
        for i, a in enumerate(alphas):
            q = O.fgfrft_matrix(o, a)
            assert rel(y[i], (q.conj().T if inverse else q) @ x) <= 1e-10


def test_window_outside_and_cleared_take_the_packed_route(problem):
    f, l, x, xc, g, o, nodes = problem
    lr, dr, yr = O.dlda_mse(o, 2.5, x, xc)
    loss, dl, y = fg.mse_step(g, [2.5], x, xc, want_y=True)
    assert g.route_info()[0] == 3
    assert rel(y[0], yr) <= 1e-10 and abs(loss[0] - lr) <= 1e-10 * lr
    g.set_order_window(0.0, 0.0)
    assert g.order_window()[2] == 0
    fg.mse_step(g, [0.37], x, xc)
    assert g.route_info()[0] == 3
    assert g.set_order_window(0.0, 2.0) == nodes  # rebuilt: the same nodes


def test_window_host_and_device_steps_agree(problem):
    import torch
    f, l, x, xc, g, o, nodes = problem
    loss_h, dl_h, _ = fg.mse_step(g, [0.81], x, xc)  # host buffers (chunked H2D)
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    xcd = torch.from_numpy(np.ascontiguousarray(xc.T)).cuda()
    lo = torch.empty(1, dtype=torch.float64, device="cuda")
    dl = torch.empty(1, dtype=torch.float64, device="cuda")
    al = np.array([0.81])
    fg._check(fg.lib().fgfrft_mse_step_dev(g.handle, al.ctypes.data, 1, xd.data_ptr(), xcd.data_ptr(), x.shape[1],
                                           None, lo.data_ptr(), dl.data_ptr()))
    torch.cuda.synchronize()
    assert g.route_info()[0] == 5
    # same products; the host form's separate loss pass and the fused epilogue sum in different
    # (each deterministic) orders
    assert abs(float(lo[0]) - loss_h[0]) <= 1e-14 * abs(loss_h[0])
    assert abs(float(dl[0]) - dl_h[0]) <= 1e-12 * abs(dl_h[0])


def test_window_budget_and_validation():
    n, l = 512, 8
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.02, 4)))
    g = fg.PowerCache(f, l, memory_budget=l * n * n * 16 + (1 << 20))  # no room for the node operators
    with pytest.raises(fg.CapacityError):
        g.set_order_window(0.0, 2.0)
    assert g.order_window()[2] == 0
    with pytest.raises(fg.ParameterError):
        fg.PowerCache(f, l).set_order_window(-40.0, 40.0)  # more than 48 nodes
    h = fg.PowerCache(prep.random_unitary(n, 3), l)  # complex F: no packed route
    with pytest.raises(fg.ParameterError):
        h.set_order_window(0.0, 1.0)


def test_window_inverse_inside_and_truncation_fallback():
    """A window around zero serves the inverse apply (Q(a)^H = Q(-a), -a inside the window); a
    truncated apply cannot use the full-L node operators and falls back to the packed route."""
    n, l, b = 512, 16, 70
    f = prep.gft_from_shift(prep.laplacian(prep.grid_graph(16, 32)))
    o = O.PowerCache(f, l)
    g = fg.PowerCache(f, l, memory_budget=4 << 30)
    assert g.set_order_window(-1.0, 1.0) > 0
    r = np.random.default_rng(9)
    x = r.standard_normal((n, b)) + 1j * r.standard_normal((n, b))
    for alphas in ([0.3], [0.7, -0.45]):
        y = fg.apply_series(g, alphas, x, inverse=True)
        for i, a in enumerate(alphas):
            q = O.fgfrft_matrix(o, a)
            assert rel(y[i], q.conj().T @ x) <= 1e-10
    yt = fg.apply_series(g, [0.3], x, truncation=9)
    assert rel(yt[0], O.fgfrft_matrix(o, 0.3, truncation=9) @ x) <= 1e-10
    xc = x + 0.05 * r.standard_normal((n, b))
    loss, dl, _ = fg.mse_step(g, [-0.8], x, xc)
    assert g.route_info()[0] == 5
    lr, dr, _ = O.dlda_mse(o, -0.8, x, xc)
    assert abs(loss[0] - lr) <= 1e-10 * lr
