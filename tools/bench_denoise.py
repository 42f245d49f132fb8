"""GPU-resident denoising learner (learn.hpp:291-516 on the device) on BASELINE-shaped graphs.

  python tools/bench_denoise.py [--epochs 20] [--shapes c2,c3]

c2: the config-2 sensor graph (N=1024), L=64, C=256 channels; c3: the 64x64 grid (N=4096), L=64,
C=1024 channels (the image-denoising shape). One epoch = one evaluation (loss, d/dalpha, d/dh:
Q and dQ/dalpha synthesised from the cache in one pass, five n x n x C GEMMs on the INT8 engine)
+ the Adam step, all on the device. Wall clock around the synchronous `fit`; the reference
algorithm (oracle restatement, numpy/OpenBLAS on all host cores) is timed for one evaluation
beside it.
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


def run(tag, f, l, ch, epochs):
    n = f.shape[0]
    rng = np.random.default_rng(1)
    coef = np.zeros((n, ch))
    coef[: n // 16] = rng.standard_normal((n // 16, ch))
    x = f.real.T @ coef
    y = x + 0.1 * rng.standard_normal((n, ch))
    cache = fg.PowerCache(f, l, memory_budget=64 << 30)
    dp = fg.DenoiseProblem(cache, y, x)
    dp.fit(2, lr=0.01)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = dp.fit(epochs, lr=0.01, init_alpha=0.5)
    dt = time.perf_counter() - t0
    per_epoch = dt / (epochs + 1)
    # reference algorithm, one evaluation
    import oracle as O
    t0 = time.perf_counter()
    ref = O.FastDenoise(y, x, f.real, l)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    lr_, ga, _ = ref.eval(0.5, np.ones(n))
    t_ref = time.perf_counter() - t0
    lg, gg, _ = dp.eval(0.5, np.ones(n))
    flops_epoch = 5 * 2.0 * n * n * ch  # u, du, w, dQ^T v, Q r (FP64-equivalent)
    synth_bytes = (l + 2) * n * n * 8.0  # L real slabs read, Q and dQ written
    return {"shape": tag, "n": n, "l": l, "channels": ch, "epochs": epochs,
            "gpu_ms_per_epoch": per_epoch * 1e3, "gpu_gemm_tflops_equiv_if_gemm_only": flops_epoch / per_epoch / 1e12,
            "synthesis_bytes_per_epoch": synth_bytes,
            "cpu_reference_ms_per_eval": t_ref * 1e3, "cpu_setup_s": t_setup, "cpu_cores": os.cpu_count(),
            "speedup_vs_cpu_eval": t_ref / per_epoch, "loss_first": float(out["traj_loss"][0]),
            "loss_last": float(out["traj_loss"][-1]), "alpha_best": out["alpha_best"],
            "parity_eval_rel": abs(lg - lr_) / lr_, "parity_grad_alpha_abs": abs(gg - ga)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--shapes", default="c2,c3")
    args = ap.parse_args()
    for s in args.shapes.split(","):
        if s == "c2":
            cfg = prep.config2()
            print(json.dumps(run("c2", cfg.f, 64, 256, args.epochs)), flush=True)
        elif s == "c3":
            cfg = prep.config3()
            print(json.dumps(run("c3", cfg.f, 64, 1024, args.epochs)), flush=True)


if __name__ == "__main__":
    main()
