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


def timed(stream, fn, reps=5, warm=3, groups=5):
    """Median over `groups` CUDA-event-timed groups of `reps` calls (ms per call)."""
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


def run(name, cfg, peaks, budget, dtype=0):
    n, b, L = cfg.n, cfg.b, cfg.l
    es = 16 if dtype == 0 else 8
    ct = torch.complex128 if dtype == 0 else torch.complex64
    A = len(cfg.alphas)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cache = fg.PowerCache(cfg.f, L, memory_budget=budget, dtype=dtype)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    cache.set_stream(stream.cuda_stream)
    lib = fg.lib()
    al = np.ascontiguousarray(cfg.alphas, dtype=np.float64)
    one = al[:1].copy()
    q = torch.empty((1, n, n), dtype=ct, device="cuda")
    t_syn = timed(stream, lambda: fg._check(lib.fgfrft_synthesize_dev(cache.handle, one.ctypes.data, 1, 0, 0,
                                                                       q.data_ptr())))
    real = cache.is_real()
    syn_bytes = (L * (8.0 if real else float(es)) + float(es)) * n * n
    del q
    x = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda().to(ct)
    xc = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda().to(ct)
    y = torch.empty((A, b, n), dtype=ct, device="cuda")
    t_app = timed(stream, lambda: fg._check(lib.fgfrft_apply_dev(cache.handle, al.ctypes.data, A, 0, 0, x.data_ptr(),
                                                                  b, y.data_ptr())))
    loss = torch.empty(A, dtype=torch.float64, device="cuda")
    dl = torch.empty(A, dtype=torch.float64, device="cuda")
    t_step = timed(stream, lambda: fg._check(lib.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, A, x.data_ptr(),
                                                                      xc.data_ptr(), b, None, loss.data_ptr(),
                                                                      dl.data_ptr())))
    out = {
        "config": name, "dtype": "c128" if dtype == 0 else "c64", "real_f": real, "n": n, "l": L, "b": b,
        "orders": A, "cache_gb": L * n * n * (8 if real else es) / 1e9,
        "cache_build": {"s": build_s, "tflops": (L - 1) * (2.0 if real else 8.0) * n ** 3 / build_s / 1e12},
        "synthesis_one_order": {"ms": t_syn, "gbs": syn_bytes / (t_syn * 1e-3) / 1e9,
                                "frac_hbm": syn_bytes / (t_syn * 1e-3) / 1e9 / peaks["hbm"]},
        "apply": {"ms": t_app, "signal_nodes_per_s": n * b * A / (t_app * 1e-3),
                  "gemm_tflops_equiv": (4.0 if real else 8.0) * n * n * b * A / (t_app * 1e-3) / 1e12},
        "mse_step": {"ms": t_step, "signal_nodes_per_s": n * b * A / (t_step * 1e-3)},
    }
    cache.close()
    return out


def run_c5(peaks):
    """C5: 4096 ER(64, 0.1) graphs, L=16, 4 orders per graph, 64 channels, complex64.
    Step = forward Y_gh = F_g^{a_gh} X_g for all graphs/heads + dL/da_gh for a cotangent G."""
    t0 = time.perf_counter()
    fs, orders, feats, l = prep.config5()
    prep_s = time.perf_counter() - t0
    G, n, C = feats.shape
    H = orders.shape[1]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch = fg.GraphBatch(fs, l)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    a_d = torch.from_numpy(orders).cuda()
    x_d = torch.from_numpy(np.ascontiguousarray(feats.transpose(0, 2, 1)).astype(np.complex64)).cuda()
    g_d = torch.randn((G, H, C, n), dtype=torch.complex64, device="cuda")
    t_fwd = timed(stream, lambda: batch.forward(a_d, x_d))
    t_bwd = timed(stream, lambda: batch.dlda(a_d, g_d, x_d))
    nodes = G * H * n * C
    real = bool(np.all(np.imag(fs) == 0))
    e = 4 if real else 8  # real F: float slabs, real Q; complex F: complex64 slabs
    # FP32 flops per graph. Real F: synthesis 2 FMAs (P, P^T) per element, power and head = 4 L n^2 H;
    # Y = Q X real x complex = 4 n^2 C H; Re M = Gr Xr^T + Gi Xi^T = 4 n^2 C H; dots 4 L n^2 H.
    # Complex F: every product complex (4 real FMAs): twice each.
    per = 4 * l * n * n * H + 4 * n * n * C * H
    flops_fwd = G * per * (1 if real else 2)
    flops_bwd = G * per * (1 if real else 2)
    cache_bytes = G * l * 64 * 64 * e
    sig = G * C * n * 8  # one complex64 n x C block per graph
    fwd_bytes = cache_bytes + sig + H * sig  # powers + X read, Y_h written
    bwd_bytes = cache_bytes + sig + H * sig  # powers + X + G_h read
    peak = _hbm_peak()
    return {"config": "C5", "graphs": G, "n": n, "l": l, "heads": H, "channels": C, "dtype": "c64",
            "real_f": real, "cache_gb": cache_bytes / 1e9, "prep_s": prep_s, "cache_build_s": build_s,
            "forward": {"ms": t_fwd, "signal_nodes_per_s": nodes / (t_fwd * 1e-3), "hbm_gb": fwd_bytes / 1e9,
                        "hbm_gbs": fwd_bytes / (t_fwd * 1e-3) / 1e9,
                        "frac_hbm": fwd_bytes / (t_fwd * 1e-3) / 1e9 / peak,
                        "fp32_tflops": flops_fwd / (t_fwd * 1e-3) / 1e12},
            "dlda": {"ms": t_bwd, "hbm_gb": bwd_bytes / 1e9, "hbm_gbs": bwd_bytes / (t_bwd * 1e-3) / 1e9,
                     "frac_hbm": bwd_bytes / (t_bwd * 1e-3) / 1e9 / peak,
                     "fp32_tflops": flops_bwd / (t_bwd * 1e-3) / 1e12},
            "step": {"ms": t_fwd + t_bwd, "signal_nodes_per_s": nodes / ((t_fwd + t_bwd) * 1e-3)},
            "peak_hbm_gbs": peak}


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        for k in ("hbm_gbs", "hbm_copy_gbs", "copy_gbs"):
            if k in d:
                return float(d[k])
    except Exception:
        pass
    return 6549.1


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
        if c == "5":
            line = json.dumps(run_c5(peaks))
            print(line, flush=True)
            if fh:
                fh.write(line + "\n")
            continue
        dtype = 1 if c.endswith("c64") else 0
        gen, budget = gens[c.replace("c64", "")]
        t0 = time.perf_counter()
        cfg = gen()
        prep_s = time.perf_counter() - t0
        res = run("C" + c, cfg, peaks, budget, dtype)
        res["prep_s"] = prep_s
        line = json.dumps(res)
        print(line, flush=True)
        if fh:
            fh.write(line + "\n")
            fh.flush()


if __name__ == "__main__":
    main()
