import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2602_20870_b200 as fg, prep, oracle as O
n, l, b = int(sys.argv[1]), int(sys.argv[2]), 80
rng = prep.Rng(3); pts = rng.uniforms(2 * n).reshape(n, 2)
f = prep.gft_from_shift(prep.laplacian(prep.knn_graph(pts, 8)))
g = fg.PowerCache(f, l, memory_budget=4 << 30)
x = np.random.default_rng(1).standard_normal((n, b)) + 0j
y = fg.apply_series(g, [0.3], x)
o = O.PowerCache(f, l)
yr = O.fgfrft_matrix(o, 0.3) @ x
print("dbg", os.environ.get("FGFRFT_DS_DEBUG"), "rel", np.linalg.norm(y[0] - yr) / np.linalg.norm(yr), flush=True)
