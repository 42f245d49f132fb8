"""The drop-in headers are ADDITIVE: a reference caller compiles unchanged.

* `demos/fractional_power.cpp` of the reference (graph builder + gft_from_shift + spectral +
  PowerCache + fgfrft_matrix + matrix_errors) compiles, byte for byte from /root/reference,
  against include/ (here: no Eigen, so the standalone restatements of graph/gft/rng/metrics are
  used; with Eigen the headers forward to the reference's own via #include_next).
* tests/cpp/bench_pattern.cpp (the bench.hpp:150-180 call pattern) compiles.
* The no-Eigen gft_from_shift / random_unitary agree with prep/ (numpy restatement).
The compiled binaries themselves run on the GPU in test_gpu_dropin_demo.py.
"""
import os
import subprocess

import numpy as np
import pytest

import prep

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DEMO = "/root/reference/proj/demos/fractional_power.cpp"
LIBDIR = os.path.join(ROOT, "paper_2602_20870_b200")


def _compile(src, out, extra=()):
    cmd = ["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), "-o", out, src, *extra]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.skipif(not os.path.exists(REF_DEMO), reason="reference checkout absent")
def test_reference_demo_compiles_unchanged(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libfgfrft_b200.so")):
        pytest.skip("library not built")
    _compile(REF_DEMO, str(tmp_path / "demo"), ["-L" + LIBDIR, "-lfgfrft_b200"])


def test_bench_call_pattern_compiles(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libfgfrft_b200.so")):
        pytest.skip("library not built")
    _compile(os.path.join(ROOT, "tests", "cpp", "bench_pattern.cpp"), str(tmp_path / "bp"),
             ["-L" + LIBDIR, "-lfgfrft_b200"])


def test_no_eigen_gft_matches_prep(tmp_path):
    exe = str(tmp_path / "gft")
    _compile(os.path.join(ROOT, "tests", "cpp", "gft_fallback.cpp"), exe)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    n = int(out[0])
    f = np.array([float(v) for v in out[1:1 + n * n]]).reshape(n, n)
    lap = prep.laplacian(prep.grid_graph(5, 6))
    assert np.abs(f @ f.T - np.eye(n)).max() < 1e-12
    lam = np.sort(np.linalg.eigvalsh(lap))
    assert np.abs(f.T @ np.diag(lam) @ f - lap).max() < 1e-11         # F = V^T, ascending lambda
    fr = prep.gft_from_shift(lap).real
    gaps = np.diff(lam)
    simple = [k for k in range(n) if (k == 0 or gaps[k - 1] > 1e-6) and (k == n - 1 or gaps[k] > 1e-6)]
    assert len(simple) > n // 3
    for k in simple:  # same eigenvector; the same sign unless the sign pivot (first largest |v_i|)
        # is an exact tie of symmetric entries, where rounding picks the pivot (also in the reference)
        d = min(np.abs(f[k] - fr[k]).max(), np.abs(f[k] + fr[k]).max())
        assert d < 1e-10
        a = np.abs(fr[k])
        if np.sum(a >= a.max() * (1 - 1e-12)) == 1:
            assert np.abs(f[k] - fr[k]).max() < 1e-10
    h = np.array([complex(*map(float, line.split())) for line in out[1 + n * n:1 + n * n + 49]]).reshape(7, 7)
    hr = prep.random_unitary(7, 11)
    assert np.abs(h - hr).max() < 1e-12                                  # the unique Q with R_kk > 0
