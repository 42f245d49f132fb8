"""GPU parity of the packed step route (csrc/packed.cu, csrc/ozgemm.cu dsynth_kernel): one, two
or four orders over a real cache with a large signal batch -- Q(a), dQ/da synthesised either from
the packed 40-bit fixed-point slabs (FP64 decode, route 3) or on the INT8 tensor cores from the
element-row digit cache (route 4), one Ozaki GEMM [Y; dY] = [Q; dQ] X, loss and dL/da from one
elementwise pass -- against the oracle (transform.hpp:111-148, learn.hpp:88-92 form) at the 1e-10
relative bar of the north star. Every test runs under both synthesis engines (FGFRFT_DSYNTH).
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2602_20870_b200 as fg
import prep

pytestmark = pytest.mark.gpu

ROUTES = {"packed": 3, "dsynth": 4}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _graph_f(n, seed):
    rng = prep.Rng(seed)
    pts = rng.uniforms(2 * n).reshape(n, 2)
    return prep.gft_from_shift(prep.laplacian(prep.knn_graph(pts, 8)))


@pytest.fixture(scope="module", params=["packed", "dsynth"])
def engine(request):
    old = os.environ.get("FGFRFT_DSYNTH")
    os.environ["FGFRFT_DSYNTH"] = "1" if request.param == "dsynth" else "0"
    yield ROUTES[request.param]
    if old is None:
        os.environ.pop("FGFRFT_DSYNTH", None)
    else:
        os.environ["FGFRFT_DSYNTH"] = old


@pytest.fixture(scope="module")
def problem(engine):
    n, l, b = 1024, 24, 80
    f = _graph_f(n, 11)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    return f, l, x, xc, fg.PowerCache(f, l, memory_budget=8 << 30), O.PowerCache(f, l), engine


@pytest.mark.parametrize("alphas", [[0.37], [0.04], [-1.3], [0.25, 1.75], [2.0]])
def test_packed_mse_step_matches_oracle(problem, alphas):
    f, l, x, xc, g, o, route = problem
    loss, dl, y = fg.mse_step(g, alphas, x, xc, want_y=True)
    assert g.route_info()[0] == route
    for i, a in enumerate(alphas):
        lr, dr, yr = O.dlda_mse(o, a, x, xc)
        assert rel(y[i], yr) <= 1e-10
        assert abs(loss[i] - lr) <= 1e-10 * lr
        s = O.power_dots(o, 2.0 * (yr - xc) @ x.conj().T / x.size)
        _, dc = O.sinc_coeffs(a, l)
        assert abs(dl[i] - dr) <= 1e-10 * max(np.sum(np.abs(dc * s)), 1e-300)


@pytest.mark.parametrize("alphas,inverse", [([0.37], False), ([0.37], True), ([0.1, 0.9], False),
                                            ([0.1, 0.5, 1.2, -0.7], True)])
def test_packed_apply_matches_oracle(problem, alphas, inverse):
    f, l, x, xc, g, o, route = problem
    y = fg.apply_series(g, alphas, x, inverse=inverse)
    for i, a in enumerate(alphas):
        q = O.fgfrft_matrix(o, a)
        yr = (q.conj().T if inverse else q) @ x
        assert rel(y[i], yr) <= 1e-10


def test_packed_apply_truncation(problem):
    f, l, x, xc, g, o, route = problem
    y = fg.apply_series(g, [0.6], x, truncation=9)
    assert rel(y[0], O.fgfrft_matrix(o, 0.6, truncation=9) @ x) <= 1e-10


def test_packed_integer_order_is_the_power(problem):
    f, l, x, xc, g, o, route = problem
    y = fg.apply_series(g, [3.0, 0.0], x)
    # c_k(3) is an exact Kronecker row (sinc.hpp:16): Y = P_3 X up to the 40-bit quantisation of P_3
    # in the cache (<= 2^-39 of each tile's / element row's largest entry) and the 5-digit (39.9-bit)
    # Ozaki product -- two ~2^-40 roundings, ~2e-11 relative; the series bar is 1e-10
    assert rel(y[0], o.power(3) @ x) <= 5e-11
    assert rel(y[1], x) <= 1e-13


def test_packed_route_respects_memory_budget(engine):
    """The packed slabs are auxiliary: with a budget that only covers the reference count
    L n^2 16 bytes (transform.hpp:46-53) they are not built and the exact route runs."""
    n, l, b = 512, 8, 40
    f = _graph_f(n, 3)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((n, b)) + 0j
    xc = x.copy()
    tight = fg.PowerCache(f, l, memory_budget=l * n * n * 16)
    roomy = fg.PowerCache(f, l, memory_budget=1 << 30)
    lt, dt_, _ = fg.mse_step(tight, [0.4], x, xc)
    assert tight.route_info()[0] not in (3, 4)
    lr, dr, _ = fg.mse_step(roomy, [0.4], x, xc)
    assert roomy.route_info()[0] == engine
    assert abs(lt[0] - lr[0]) <= 1e-10 * lr[0]
    assert abs(dt_[0] - dr[0]) <= 1e-9 * max(1.0, abs(dr[0]))


def test_packed_host_and_device_steps_agree(problem):
    """fgfrft_mse_step (host buffers: X copied in column chunks overlapping the synthesis) and
    fgfrft_mse_step_dev (device-resident X) run the same products: identical results."""
    import torch
    f, l, x, xc, g, o, route = problem
    n, b = x.shape
    al = np.array([0.81, -0.4])
    loss_h, dl_h, _ = fg.mse_step(g, al, x, xc)
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    xcd = torch.from_numpy(np.ascontiguousarray(xc.T)).cuda()
    lo = torch.empty(2, dtype=torch.float64, device="cuda")
    dl = torch.empty(2, dtype=torch.float64, device="cuda")
    g.set_stream(torch.cuda.current_stream().cuda_stream)
    fg._check(fg.lib().fgfrft_mse_step_dev(g.handle, al.ctypes.data, 2, xd.data_ptr(), xcd.data_ptr(), b, None,
                                           lo.data_ptr(), dl.data_ptr()))
    torch.cuda.synchronize()
    assert np.allclose(lo.cpu().numpy(), loss_h, rtol=1e-14, atol=0)
    assert np.allclose(dl.cpu().numpy(), dl_h, rtol=1e-12, atol=1e-300)


def test_node_sweep_snaps_order_zero_and_narrow_sweeps_fall_back():
    """Node-interpolated sweeps (real F, 16-64 orders): alpha = 0 returns X bit for bit (Q(0) = I,
    test_transform.cpp:60-65); a narrow sweep (width 0.01) whose derivative weights
    would amplify the node operators' INT8 error takes the power route and stays at 1e-10."""
    n, l, b = 512, 10, 40
    f = _graph_f(n, 23)
    g = fg.PowerCache(f, l, memory_budget=4 << 30)
    o = O.PowerCache(f, l)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    wide = np.linspace(0.0, 2.0, 24)
    loss, dl, y = fg.mse_step(g, wide, x, xc, want_y=True)
    assert g.route_info()[0] == 2
    assert np.array_equal(y[0], x)
    assert loss[0] == np.vdot(x - xc, x - xc).real / (n * b) or abs(loss[0] - np.vdot(x - xc, x - xc).real / (n * b)) \
        <= 1e-15 * loss[0]
    narrow = np.linspace(0.7, 0.71, 32)
    loss, dl, _ = fg.mse_step(g, narrow, x, xc)
    assert g.route_info()[0] == 1  # power products: no derivative-weight amplification
    for i in (0, 13, 31):
        a = float(narrow[i])
        lr, dr, yr = O.dlda_mse(o, a, x, xc)
        s = O.power_dots(o, 2.0 * (yr - xc) @ x.conj().T / x.size)
        _, dc = O.sinc_coeffs(a, l)
        assert abs(loss[i] - lr) <= 1e-10 * lr
        assert abs(dl[i] - dr) <= 1e-10 * np.sum(np.abs(dc * s))


def test_tensor_core_synthesis_matches_packed_synthesis():
    """The two synthesis engines on one cache: Y = Q(a) X from the digit cache (5 digits per element
    row over the powers) and from the packed 40-bit tiles agree to their common quantisation
    (~2^-40 of the entries), odd n (ragged edge tiles) and a truncated series included."""
    n, l, b = 1000, 20, 80
    f = _graph_f(n, 31)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    o = O.PowerCache(f, l)
    old = os.environ.get("FGFRFT_DSYNTH")
    try:
        out = {}
        for eng in ("0", "1"):
            os.environ["FGFRFT_DSYNTH"] = eng
            g = fg.PowerCache(f, l, memory_budget=8 << 30)
            out[eng] = (fg.apply_series(g, [0.43, -1.2], x), fg.apply_series(g, [0.8], x, truncation=7))
        for a, ya, yb in zip([0.43, -1.2], out["0"][0], out["1"][0]):
            yr = O.fgfrft_matrix(o, a) @ x
            assert rel(yb, yr) <= 1e-10 and rel(ya, yr) <= 1e-10
            assert rel(ya, yb) <= 1e-10
        yr = O.fgfrft_matrix(o, 0.8, truncation=7) @ x
        assert rel(out["1"][1][0], yr) <= 1e-10 and rel(out["0"][1][0], yr) <= 1e-10
    finally:
        if old is None:
            os.environ.pop("FGFRFT_DSYNTH", None)
        else:
            os.environ["FGFRFT_DSYNTH"] = old


@pytest.mark.parametrize("alpha", [0.37, -1.3, 1.0])
def test_digit_emission_matches_the_slicing_pass(problem, alpha):
    """One order on whole 128-row tiles: psynth writes [Q; dQ]'s Ozaki digits itself, scaled per row
    by the exponents prow_bound_kernel derives from the powers' row / column maxima (packed.cu), in
    place of FP64 Q + row maxima + the slicing pass (FGFRFT_PSYNTH_DIGITS=0). The bound is looser
    than the exact row maximum by a few bits, so the two differ in the last digits only; both hold
    the oracle's 1e-10 bar."""
    f, l, x, xc, g, o, route = problem
    if route != 3:
        pytest.skip("digit emission is the packed FP64-decode synthesis' (route 3)")
    old = os.environ.get("FGFRFT_PSYNTH_DIGITS")
    try:
        os.environ["FGFRFT_PSYNTH_DIGITS"] = "0"
        l0, d0, y0 = fg.mse_step(g, [alpha], x, xc, want_y=True)
        os.environ["FGFRFT_PSYNTH_DIGITS"] = "1"
        l1, d1, y1 = fg.mse_step(g, [alpha], x, xc, want_y=True)
    finally:
        if old is None:
            os.environ.pop("FGFRFT_PSYNTH_DIGITS", None)
        else:
            os.environ["FGFRFT_PSYNTH_DIGITS"] = old
    assert g.route_info()[0] == 3
    assert rel(y1[0], y0[0]) <= 1e-11
    lr, dr, yr = O.dlda_mse(o, alpha, x, xc)
    assert rel(y1[0], yr) <= 1e-10
    assert abs(l1[0] - lr) <= 1e-10 * lr
    s = O.power_dots(o, 2.0 * (yr - xc) @ x.conj().T / x.size)
    _, dc = O.sinc_coeffs(alpha, l)
    assert abs(d1[0] - dr) <= 1e-10 * max(np.sum(np.abs(dc * s)), 1e-300)
