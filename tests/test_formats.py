"""The reference's run-record formats restated in paper_2602_20870_b200/formats.py (io.hpp:172-300,
commands.hpp:98-165): shortest round-trip doubles, CRLF CSV with fixed headers, key=value manifests
and their parse errors. CPU only."""
import math

import pytest

from paper_2602_20870_b200 import formats as F


@pytest.mark.parametrize("v,s", [(0.5, "0.5"), (0.1, "0.1"), (1.0, "1"), (1e-300, "1e-300"), (123456.0, "123456"),
                                 (1.0 / 3.0, "0.3333333333333333"), (2.0 / 3.0, "0.6666666666666666"),
                                 (0.55, "0.55"), (-2.5e-7, "-2.5e-07"), (0.0, "0")])
def test_format_double_shortest_round_trip(v, s):
    assert F.format_double(v) == s
    assert float(F.format_double(v)) == v


def test_format_double_round_trips_every_double_sampled():
    import random
    rng = random.Random(7)
    for _ in range(2000):
        v = rng.uniform(-1, 1) * 10.0 ** rng.randint(-300, 300)
        assert float(F.format_double(v)) == v
    assert F.format_double(math.pi) == "3.141592653589793"


def test_sweep_and_bench_files(tmp_path):
    recs = [{"n": 256, "l": 32, "alpha": 0.37, "seed": 1, "mse": 1.25e-5, "mae": 2.5e-3, "nmse": 3.1e-3},
            {"n": 1024, "l": 64, "alpha": 1.5, "seed": 1, "mse": 4e-6, "mae": 1e-3, "nmse": 2e-3}]
    csv_path, man = F.write_sweep(str(tmp_path / "sweep"), recs, [("n-list", "256,1024"), ("out", "sweep")], 1)
    raw = open(csv_path, "rb").read()
    assert raw.startswith(b"n,l,alpha,seed,mse,mae,nmse\r\n256,32,0.37,1,1.25e-05,0.0025,0.0031\r\n")
    rows = F.read_csv(csv_path)
    assert rows[0] == F.SWEEP_HEADER and len(rows) == 3 and rows[2][2] == "1.5"
    m = F.read_manifest(man)
    assert m.command == "sweep" and m.seed == 1 and m.outputs == [csv_path]
    assert m.flags == [("n-list", "256,1024"), ("out", "sweep")]
    b_csv, b_man = F.write_bench(str(tmp_path / "bench"),
                                 [{"n": 1000, "l": 10, "fast_s": 3.9e-5, "exact_s": 2e-4, "speedup": 5.1, "repeats": 25}],
                                 [("l", "10")], 1)
    assert F.read_csv(b_csv) == [F.BENCH_HEADER, ["1000", "10", "3.9e-05", "0.0002", "5.1", "25"]]
    assert F.read_manifest(b_man).command == "bench"


def test_manifest_parse_error_names_the_line(tmp_path):
    p = tmp_path / "bad.manifest"
    p.write_text("command=sweep\nversion=1\nno-equals-here\n")
    with pytest.raises(F.FormatError, match="line 3"):
        F.read_manifest(str(p))
    with pytest.raises(F.FormatError):
        F.read_manifest(str(tmp_path / "missing.manifest"))
