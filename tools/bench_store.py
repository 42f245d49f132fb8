"""On-disk power cache (fgfrft_cache_save / _load): throughput against a fresh
build of the same cache.

  python tools/bench_store.py [--shape c3] [--dir /tmp]

c2: N=1024 sensor graph, L=64 (0.54 GB real cache); c3: 64x64 grid, L=64 (8.6 GB).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="c2,c3")
    ap.add_argument("--dir", default="/tmp")
    args = ap.parse_args()
    for shape in args.shape.split(","):
        f = (prep.config2() if shape == "c2" else prep.config3()).f
        t0 = time.perf_counter()
        g = fg.PowerCache(f, 64, memory_budget=64 << 30)
        t_build = time.perf_counter() - t0
        path = os.path.join(args.dir, f"fgfrft_{shape}.fgc")
        t0 = time.perf_counter()
        g.save(path)
        t_save = time.perf_counter() - t0
        size = os.path.getsize(path)
        t0 = time.perf_counter()
        h = fg.PowerCache.load(path, memory_budget=64 << 30)
        t_load = time.perf_counter() - t0
        same = bool((h.power(64) == g.power(64)).all())
        os.remove(path)
        print(json.dumps({"shape": shape, "n": g.n(), "l": 64, "file_gb": size / 1e9, "build_s": t_build,
                          "save_s": t_save, "save_gbs": size / t_save / 1e9, "load_s": t_load,
                          "load_gbs": size / t_load / 1e9, "powers_identical": same}), flush=True)
        del g, h


if __name__ == "__main__":
    main()
