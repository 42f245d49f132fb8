"""Input preparation: the restated reference Rng is bit-exact (golden streams from the
reference's rng.hpp via oracle/_ref), and the graph / GFT builders keep the reference's
invariants (gft.hpp:74-128, graph.hpp:45-125)."""
import json
import math
import os

import numpy as np

import prep

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_rng_streams_match_reference():
    data = json.load(open(os.path.join(GOLDEN, "rng_stream.json")))
    for st in data["streams"]:
        r = prep.Rng(int(st["seed"]))
        got = [r.uniform() if k == 0 else r.gaussian() for k in st["kinds"]]
        assert [float(v).hex() for v in got] == st["values"]
    for d in data["derive"]:
        assert prep.Rng.derive(int(d["seed"]), int(d["index"])) == int(d["value"])


def test_grid_graph_structure():
    a = prep.grid_graph(3, 4)
    assert a.shape == (12, 12) and np.array_equal(a, a.T)
    assert a[0, 1] == 1 and a[0, 4] == 1 and a[3, 4] == 0  # no wraparound (graph.hpp:45-72)
    assert a.sum() == 2 * (3 * 3 + 2 * 4)


def test_gft_from_shift_is_orthogonal_and_sign_fixed():
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(64, 0.1, 3)))
    assert prep.unitarity_residual(f) < 1e-12
    v = f.T.real
    for j in range(v.shape[1]):
        p = int(np.argmax(np.abs(v[:, j])))
        assert v[p, j] > 0


def test_knn_union_and_weights():
    rng = prep.Rng(1)
    pts = rng.uniforms(2 * 50).reshape(50, 2)
    a = prep.knn_graph(pts, 4)
    assert np.array_equal(a, a.T) and np.all(np.diag(a) == 0)
    assert np.all((a > 0).sum(1) >= 4) and np.all(a <= 1.0)
    b = prep.knn_graph(pts, 4, gaussian_weights=False)
    assert np.array_equal(b > 0, a > 0) and set(np.unique(b)) <= {0.0, 1.0}


def test_spread_phases_extremes():
    ph = prep.spread_phases(64, 0.05 * math.pi, 23)
    lim = math.pi - 0.05 * math.pi
    assert ph[0] == -lim and ph[-1] == lim and np.all(np.abs(ph) <= lim)


def test_config1_shapes(tmp_path, monkeypatch):
    monkeypatch.setenv("FGFRFT_DATA", str(tmp_path))
    c = prep.config1()
    assert c.f.shape == (256, 256) and c.x.shape == (256, 1) and c.l == 32
    assert prep.unitarity_residual(c.f) < 1e-10
    assert os.path.exists(os.path.join(str(tmp_path), "F_c1_s1.bin"))
    assert np.array_equal(prep.load_matrix(os.path.join(str(tmp_path), "F_c1_s1.bin")), c.f)
