"""Exact GFRFT / eigendecomposition on the GPU and the cascaded order learner (SURVEY 8(f) ranks
2-3) on BASELINE-shaped graphs, with the reference algorithm (oracle restatement, numpy/OpenBLAS
on all host cores) timed beside them.

  python tools/bench_spectral.py [--shapes c2,c3] [--epochs 20] [--cpu-eig]

Per shape (c2: the N=1024 sensor graph, c3: the 64x64 grid, N=4096):
  * eig: fgfrft_spectrum_decompose (cuSOLVER Hermitian stage + cluster refinement + products);
  * exact: one order of V diag(e^{j a theta}) V^H (scaling + one DMMA ZGEMM, 8 N^3 flops) against
    the series synthesis fgfrft_matrix (L = 64, HBM-bound) -- the paper's Table II comparison;
  * cascade: one evaluation (loss + K gradients) per backend and depth, and learn_orders epochs.
Host wall clock around synchronous library calls (each call ends with a device sync).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402


def timed(fn, reps=5, warm=1):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def run(tag, f, l, epochs, cpu_eig):
    import oracle as O
    n = f.shape[0]
    out = {"shape": tag, "n": n, "l": l, "cpu_cores": os.cpu_count()}
    t0 = time.perf_counter()
    eig = fg.eigendecompose_unitary(f)
    out["gpu_eig_s_first"] = time.perf_counter() - t0
    out["gpu_eig_s"] = timed(lambda: fg.eigendecompose_unitary(f).close(), reps=3)
    if cpu_eig:
        t0 = time.perf_counter()
        ve, te = O.eigendecompose_unitary(f)
        out["cpu_eig_s"] = time.perf_counter() - t0
        out["eig_theta_maxdiff"] = float(np.max(np.abs(eig.theta - te)))
    ve, te = eig.v, eig.theta
    # exact operator vs series synthesis, one order
    t_ex = timed(lambda: fg.exact_matrices(eig, [0.37]))
    cache = fg.PowerCache(f, l, memory_budget=64 << 30)
    t_se = timed(lambda: fg.synthesize(cache, [0.37]))
    t_cpu_ex = timed(lambda: O.exact_gfrft((ve, te), 0.37), reps=3)
    out.update({"gpu_exact_ms": t_ex * 1e3, "gpu_exact_tflops": 8.0 * n ** 3 / t_ex / 1e12,
                "gpu_series_ms": t_se * 1e3, "cpu_exact_ms": t_cpu_ex * 1e3,
                "note": "host wall clock incl. the n x n complex128 download per call"})
    # device-only timing of the exact operator (no download)
    import torch
    buf = torch.empty((8, n, n), dtype=torch.complex128, device="cuda")
    al = np.linspace(0.1, 1.9, 8)

    def ex_dev():
        fg._check(fg.lib().fgfrft_exact_dev(eig.handle, al.ctypes.data, 8, fg.Q, buf.data_ptr()))
        torch.cuda.synchronize()
    out["gpu_exact_dev_ms_per_order"] = timed(ex_dev) * 1e3 / 8
    out["gpu_exact_dev_tflops"] = 8.0 * n ** 3 / (out["gpu_exact_dev_ms_per_order"] * 1e-3) / 1e12
    del buf
    # cascade
    casc = []
    for backend in (fg.FAST, fg.EXACT):
        for k in (1, 2, 3):
            prob = fg.CascadeProblem(f, k, 1.5, l, backend, eig=eig, cache=cache if backend == fg.FAST else None)
            al = np.full(k, 1.5 / k) + 0.05
            t_eval = timed(lambda: prob.eval(al))
            rec = {"backend": backend, "depth": k, "gpu_eval_ms": t_eval * 1e3,
                   "gemms_per_eval": 3 * (k - 1) + (2 * k if backend == fg.EXACT else 0)}
            if epochs > 0:
                t0 = time.perf_counter()
                res = prob.learn(0.1, epochs, 0.01)
                rec["gpu_ms_per_epoch"] = (time.perf_counter() - t0) / (epochs + 1) * 1e3
                rec["loss_first"], rec["loss_last"] = float(res["traj_loss"][0]), float(res["traj_loss"][-1])
            if k <= 2 and n <= 1024:
                ref = O.Cascade(f, k, 1.5, l, backend, eig=(ve, te),
                                cache=None if backend == fg.EXACT else O.PowerCache(f, l, 64 << 30))
                t_ref = timed(lambda: ref.eval(al), reps=1, warm=0)
                lr_, gr = ref.eval(al)
                lg, gg = prob.eval(al)
                rec.update({"cpu_reference_eval_ms": t_ref * 1e3, "speedup_vs_cpu_eval": t_ref / t_eval,
                            "parity_loss_rel": abs(lg - lr_) / max(lr_, 1e-300),
                            "parity_grad_abs": float(np.max(np.abs(gg - gr)))})
            prob.close()
            casc.append(rec)
    out["cascade"] = casc
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="c2,c3")
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--cpu-eig", action="store_true")
    args = ap.parse_args()
    for s in args.shapes.split(","):
        if s == "c2":
            print(json.dumps(run("c2", prep.config2().f, 64, args.epochs, args.cpu_eig)), flush=True)
        elif s == "c3":
            print(json.dumps(run("c3", prep.config3().f, 64, args.epochs, args.cpu_eig)), flush=True)


if __name__ == "__main__":
    main()
