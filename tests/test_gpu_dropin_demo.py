"""The C++ reference callers built against the drop-in headers by __graft_entry__.build() run on
the GPU: the reference's own demos/fractional_power.cpp (compiled byte for byte from the reference
checkout) and tests/cpp/bench_pattern.cpp (bench.hpp:150-180's call pattern)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
CPP = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")


def test_reference_demo_runs():
    exe = os.path.join(CPP, "ref_demo_fractional_power")
    if not os.path.exists(exe):
        pytest.skip("reference demo not built (no reference checkout at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    rows = [ln.split() for ln in out.stdout.splitlines()[2:] if ln.strip()]
    assert len(rows) == 5
    for alpha, e10, e20 in rows:
        e10, e20 = float(e10), float(e20)
        assert 0.0 <= e20 <= e10 < 1.0  # more terms, smaller truncation error (test_transform.cpp:114-127)


def test_bench_pattern_runs():
    exe = os.path.join(CPP, "bench_pattern")
    if not os.path.exists(exe):
        pytest.skip("bench_pattern not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
