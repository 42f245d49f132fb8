"""Per-config measurements on one B200 (BASELINE configs C1-C4; C5 in its own kernel).

For each config: device cache build (K1, FP64 TFLOP/s), single-order synthesis GB/s vs HBM
peak (K2), series apply F^a X (K2 + DMMA GEMM, signal-nodes/s and GEMM TFLOP/s), and the full
forward + MSE + dL/da step. CUDA events on the library stream, >= 3 warm-ups, inputs larger
than L2 (every cache here is >= 34 MB; C2-C4 >> 126 MB L2). Writes one JSON line per config.

  python tools/bench_configs.py [--configs 1,2,3,4] [--out profiles/r01_configs.jsonl]
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


def timed(stream, fn, reps=5, warm=3):
    with torch.cuda.stream(stream):
        for _ in range(warm):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def run(name, cfg, peaks, budget):
    n, b, L = cfg.n, cfg.b, cfg.l
    A = len(cfg.alphas)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cache = fg.PowerCache(cfg.f, L, memory_budget=budget)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    cache.set_stream(stream.cuda_stream)
    lib = fg.lib()
    al = np.ascontiguousarray(cfg.alphas, dtype=np.float64)
    one = al[:1].copy()
    q = torch.empty((1, n, n), dtype=torch.complex128, device="cuda")
    t_syn = timed(stream, lambda: fg._check(lib.fgfrft_synthesize_dev(cache.handle, one.ctypes.data, 1, 0, 0,
                                                                       q.data_ptr())))
    syn_bytes = (L + 1) * n * n * 16.0
    del q
    x = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda()
    xc = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda()
    y = torch.empty((A, b, n), dtype=torch.complex128, device="cuda")
    t_app = timed(stream, lambda: fg._check(lib.fgfrft_apply_dev(cache.handle, al.ctypes.data, A, 0, 0, x.data_ptr(),
                                                                  b, y.data_ptr())))
    loss = torch.empty(A, dtype=torch.float64, device="cuda")
    dl = torch.empty(A, dtype=torch.float64, device="cuda")
    t_step = timed(stream, lambda: fg._check(lib.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, A, x.data_ptr(),
                                                                      xc.data_ptr(), b, None, loss.data_ptr(),
                                                                      dl.data_ptr())))
    out = {
        "config": name, "n": n, "l": L, "b": b, "orders": A, "cache_gb": L * n * n * 16 / 1e9,
        "cache_build": {"s": build_s, "tflops": (L - 1) * 8.0 * n ** 3 / build_s / 1e12},
        "synthesis_one_order": {"ms": t_syn, "gbs": syn_bytes / (t_syn * 1e-3) / 1e9,
                                "frac_hbm": syn_bytes / (t_syn * 1e-3) / 1e9 / peaks["hbm"]},
        "apply": {"ms": t_app, "signal_nodes_per_s": n * b * A / (t_app * 1e-3),
                  "gemm_tflops_equiv": 8.0 * n * n * b * A / (t_app * 1e-3) / 1e12},
        "mse_step": {"ms": t_step, "signal_nodes_per_s": n * b * A / (t_step * 1e-3)},
    }
    cache.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        hbm = 6650.0
    peaks = {"hbm": hbm}
    gens = {"1": (prep.config1, 1 << 30), "2": (prep.config2, 8 << 30), "3": (prep.config3, 32 << 30),
            "4": (prep.config4, 140 << 30)}
    fh = open(args.out, "a") if args.out else None
    for c in args.configs.split(","):
        gen, budget = gens[c]
        t0 = time.perf_counter()
        cfg = gen()
        prep_s = time.perf_counter() - t0
        res = run("C" + c, cfg, peaks, budget)
        res["prep_s"] = prep_s
        line = json.dumps(res)
        print(line, flush=True)
        if fh:
            fh.write(line + "\n")
            fh.flush()


if __name__ == "__main__":
    main()
