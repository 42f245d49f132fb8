"""The paper's Table II on one B200 (the only published timings of this path):
online construction of F^alpha from the cached powers (L = 10) against the exact
eigendecomposition-based operator, N = 1000 .. 8000, Haar-random complex unitary F.

  python tools/bench_table2.py [--ns 1000,2000,...,8000] [--out profiles/r01_table2.jsonl]

Per N: fgfrft_matrix (one order, device output; HBM-bound: L slabs read + 1 written) and
exact_gfrft (V diag(e^{j a theta}) V^H: one DMMA ZGEMM, 8 N^3 flops) given the spectrum, both
timed with CUDA events (median of 5 groups of 5 after 3 warm-ups); the GPU eigendecomposition
(once per F) and the DMMA cache build are reported beside them. Paper numbers: i5-12600KF,
PyTorch 2.6.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402

PAPER = {1000: (0.0068, 0.0130), 2000: (0.0366, 0.0866), 3000: (0.0845, 0.3245), 4000: (0.1586, 0.7227),
         5000: (0.2484, 1.3942), 6000: (0.3582, 2.3962), 7000: (0.4952, 3.7579), 8000: (0.8120, 5.5446)}


def timed(stream, fn, reps=5, warm=3, groups=5):
    with torch.cuda.stream(stream):
        for _ in range(warm):
            fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(groups):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        out.append(e0.elapsed_time(e1) / reps)
    return float(np.median(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="1000,2000,3000,4000,5000,6000,7000,8000")
    ap.add_argument("--l", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--record", default=None, help="also write the reference CLI's bench.csv + bench.manifest "
                    "(commands.hpp:140-165 format) under this prefix")
    args = ap.parse_args()
    records = []
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        hbm = 6650.0
    lib = fg.lib()
    fh = open(args.out, "a") if args.out else None
    for n in (int(v) for v in args.ns.split(",")):
        t0 = time.perf_counter()
        f = prep.random_unitary(n, 1)
        prep_s = time.perf_counter() - t0
        stream = torch.cuda.Stream()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cache = fg.PowerCache(f, args.l, memory_budget=64 << 30)
        torch.cuda.synchronize()
        build_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        eig = fg.eigendecompose_unitary(f)
        eig_s = time.perf_counter() - t0
        cache.set_stream(stream.cuda_stream)
        fg._check(lib.fgfrft_spectrum_set_stream(eig.handle, ctypes_stream(stream)))
        q = torch.empty((n, n), dtype=torch.complex128, device="cuda")
        al = np.array([0.37])
        t_series = timed(stream, lambda: fg._check(lib.fgfrft_synthesize_dev(cache.handle, al.ctypes.data, 1, 0, 0,
                                                                            q.data_ptr())))
        t_exact = timed(stream, lambda: fg._check(lib.fgfrft_exact_dev(eig.handle, al.ctypes.data, 1, 0,
                                                                      q.data_ptr())), reps=2, groups=3)
        byts = (args.l + 1) * n * n * 16.0
        ps, pe = PAPER.get(n, (None, None))
        rec = {"n": n, "l": args.l, "series_ms": t_series, "series_gbs": byts / (t_series * 1e-3) / 1e9,
               "series_frac_hbm": byts / (t_series * 1e-3) / 1e9 / hbm, "exact_ms": t_exact,
               "exact_tflops": 8.0 * n ** 3 / (t_exact * 1e-3) / 1e12, "speedup_series_vs_exact": t_exact / t_series,
               "gpu_eig_s": eig_s, "cache_build_s": build_s, "prep_s": prep_s,
               "paper_series_s": ps, "paper_exact_s": pe,
               "speedup_vs_paper_series": (ps / (t_series * 1e-3)) if ps else None}
        records.append({"n": n, "l": args.l, "fast_s": t_series * 1e-3, "exact_s": t_exact * 1e-3,
                        "speedup": t_exact / t_series, "repeats": 25})
        line = json.dumps(rec)
        print(line, flush=True)
        if fh:
            fh.write(line + "\n")
            fh.flush()
        del q, cache, eig
        torch.cuda.empty_cache()
    if args.record:
        from paper_2602_20870_b200 import formats
        formats.write_bench(args.record, records,
                            [("n-list", args.ns), ("l", str(args.l)), ("repeats", "25"), ("warmups", "3"),
                             ("alpha", "0.37"), ("seed", "1"), ("haar", "1"), ("out", args.record),
                             ("device", "B200")], 1)


def ctypes_stream(stream):
    import ctypes
    return ctypes.c_void_p(stream.cuda_stream)


if __name__ == "__main__":
    main()
