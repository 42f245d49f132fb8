"""The reference CLI's accuracy sweep (commands.hpp:98-122, bench.hpp accuracy_sweep) on one B200:
for every (n, l, alpha, seed), the series operator F^alpha from the cached powers (fgfrft_matrix,
the bit-exact synthesis kernels) against the exact one V diag(e^{j alpha theta}) V^H from the GPU
eigendecomposition, their matrix_errors (metrics.hpp:21-34), written as the reference's sweep.csv
+ sweep.manifest (paper_2602_20870_b200.formats).

  python tools/sweep.py [--ns 256,1024] [--alphas 0.15,0.35,0.55,0.75,0.95] [--ls 10,20,30] \\
                        [--seeds 1] [--out sweep]

F per (n, seed): the reference's synthetic unitary for sweeps (prep.random_unitary, Haar).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402
from paper_2602_20870_b200 import formats  # noqa: E402


def matrix_errors(approx, reference):
    """metrics.hpp:21-34: MSE = ||D||^2 / N^2, MAE = sum |D| / N^2, NMSE = ||D||^2 / ||ref||^2."""
    d = approx - reference
    sq = float(np.vdot(d, d).real)
    return {"mse": sq / d.size, "mae": float(np.abs(d).sum()) / d.size,
            "nmse": sq / float(np.vdot(reference, reference).real)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="256,1024")
    ap.add_argument("--alphas", default="0.15,0.35,0.55,0.75,0.95")
    ap.add_argument("--ls", default="10,20,30")
    ap.add_argument("--seeds", default="1")
    ap.add_argument("--out", default="sweep")
    args = ap.parse_args()
    ns = [int(v) for v in args.ns.split(",")]
    alphas = [float(v) for v in args.alphas.split(",")]
    ls = [int(v) for v in args.ls.split(",")]
    seeds = [int(v) for v in args.seeds.split(",")]
    records = []
    for n in ns:
        for seed in seeds:
            f = prep.random_unitary(n, seed)
            eig = fg.eigendecompose_unitary(f)
            for l in ls:
                cache = fg.PowerCache(f, l, memory_budget=64 << 30)
                for a in alphas:
                    e = matrix_errors(fg.fgfrft_matrix(cache, a).q, fg.exact_gfrft(eig, a).q)
                    records.append({"n": n, "l": l, "alpha": a, "seed": seed, **e})
                    print(f"sweep n={n} l={l} alpha={a} seed={seed} nmse={e['nmse']:.4g}", flush=True)
                cache.close()
            eig.close()
    csv_path, man = formats.write_sweep(args.out, records,
                                        [("n-list", args.ns), ("alpha-list", args.alphas), ("l-list", args.ls),
                                         ("seeds", args.seeds), ("out", args.out), ("device", "B200")], seeds[0])
    print(f"sweep: {len(records)} rows -> {csv_path}, {man}")


if __name__ == "__main__":
    main()
