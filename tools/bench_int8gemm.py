"""Times the INT8 tensor-core FP64 GEMM (fgfrft_dgemm_int8_dev, slicing included) against the
DMMA real GEMM path and torch (cuBLAS DGEMM) on Z-route shapes: C (m x n) = A (m x k) B (k x n)."""
import json
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_20870_b200 as fg  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


shapes = [(16384, 512, 1024), (131072, 512, 1024), (4096, 2048, 4096)]
for m, n, k in shapes:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    ref = a @ b
    res = {"m": m, "n": n, "k": k}
    for s in (7, 8):
        c = fg.dgemm_int8(a, b, s)
        res[f"relerr_s{s}"] = float((c - ref).norm() / ref.norm())
        t = timed(lambda: fg.dgemm_int8(a, b, s))
        res[f"ms_s{s}"] = t
        fg.profile_enable(True)
        fg.profile_read(reset=True)
        fg.dgemm_int8(a, b, s)
        prof = fg.profile_read(reset=True)
        fg.profile_enable(False)
        res[f"gemm_ms_s{s}"] = prof["int8_gemm"][0]
        res[f"slice_ms_s{s}"] = prof["slicing"][0]
        res[f"kernel_int8_tops_s{s}"] = 2.0 * m * n * k * (s * (s + 1) // 2) / prof["int8_gemm"][0] / 1e9
        res[f"fp64eq_tflops_s{s}"] = 2.0 * m * n * k / t / 1e9
        res[f"int8_tops_s{s}"] = 2.0 * m * n * k * (s * (s + 1) // 2) / t / 1e9
    t = timed(lambda: a @ b)
    res["cublas_dgemm_ms"] = t
    res["cublas_dgemm_tflops"] = 2.0 * m * n * k / t / 1e9
    print(json.dumps(res), flush=True)
