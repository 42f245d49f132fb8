"""The reference's run-record formats (second half): the sweep / bench CSV
files and the run manifest the reference CLI writes next to them, so a sweep or bench run on the
B200 leaves the same files a reference run does (and the reference's own readers accept them).

Restated from `io.hpp:172-186` (format_double: the shortest %g that round-trips, else %.17g),
`io.hpp:203-250` (CsvWriter: RFC 4180 numeric payloads, fixed header, CRLF rows; read_csv drops a
trailing CR and blank lines), `io.hpp:252-300` (RunManifest: flat key=value, `flag.<k>`,
`output.<i>`; a line without '=' is a parse_error naming the line) and the column sets of
`commands.hpp:98-122` (sweep: n, l, alpha, seed, mse, mae, nmse) and `commands.hpp:140-165`
(bench: n, l, fast_s, exact_s, speedup, repeats). Host code only; no GPU involved.
"""
from __future__ import annotations

import datetime
from dataclasses import dataclass, field
from typing import Iterable, List, Sequence, Tuple

SWEEP_HEADER = ["n", "l", "alpha", "seed", "mse", "mae", "nmse"]
BENCH_HEADER = ["n", "l", "fast_s", "exact_s", "speedup", "repeats"]
VERSION = "0.1.0-b200"


class FormatError(ValueError):
    """Raised where the reference raises io_error / parse_error."""


def format_double(v: float) -> str:
    """Shortest %.{p}g (p = 1..16) that reads back to v, else %.17g (io.hpp:175-186)."""
    v = float(v)
    for prec in range(1, 17):
        s = "%.*g" % (prec, v)
        if float(s) == v:
            return s
    return "%.17g" % v


class CsvWriter:
    """io.hpp:203-223: header first, cells joined by ',', rows ended by CRLF."""

    def __init__(self, path: str, header: Sequence[str]):
        self.path = path
        try:
            self._fh = open(path, "w", newline="")
        except OSError as ex:
            raise FormatError(f"cannot open {path} for writing") from ex
        self.write_row(header)

    def write_row(self, cells: Sequence[str]) -> None:
        self._fh.write(",".join(cells) + "\r\n")

    def close(self) -> None:
        self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def read_csv(path: str) -> List[List[str]]:
    """io.hpp:225-246."""
    try:
        with open(path, "rb") as fh:
            data = fh.read().decode()
    except OSError as ex:
        raise FormatError(f"cannot open {path}") from ex
    rows = []
    for line in data.split("\n"):
        if line.endswith("\r"):
            line = line[:-1]
        if line:
            rows.append(line.split(","))
    return rows


@dataclass
class RunManifest:
    """io.hpp:253-260."""
    command: str = ""
    version: str = ""
    seed: int = 0
    timestamp: str = ""
    flags: List[Tuple[str, str]] = field(default_factory=list)
    outputs: List[str] = field(default_factory=list)


def write_manifest(path: str, m: RunManifest) -> None:
    """io.hpp:262-272."""
    lines = [f"command={m.command}", f"version={m.version}", f"seed={m.seed}", f"timestamp={m.timestamp}"]
    lines += [f"flag.{k}={v}" for k, v in m.flags]
    lines += [f"output.{i}={o}" for i, o in enumerate(m.outputs)]
    try:
        with open(path, "w", newline="") as fh:
            fh.write("\n".join(lines) + "\n")
    except OSError as ex:
        raise FormatError(f"cannot open {path} for writing") from ex


def read_manifest(path: str) -> RunManifest:
    """io.hpp:274-300 (unknown keys are ignored, as there)."""
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError as ex:
        raise FormatError(f"cannot open {path}") from ex
    m = RunManifest()
    for lineno, line in enumerate(text.split("\n"), 1):
        if not line:
            continue
        if "=" not in line:
            raise FormatError(f"manifest parse error at line {lineno}: missing '='")
        key, value = line.split("=", 1)
        if key == "command":
            m.command = value
        elif key == "version":
            m.version = value
        elif key == "seed":
            m.seed = int(value) if value.isdigit() else 0
        elif key == "timestamp":
            m.timestamp = value
        elif key.startswith("flag."):
            m.flags.append((key[5:], value))
        elif key.startswith("output."):
            m.outputs.append(value)
    return m


def timestamp_utc() -> str:
    """ISO-8601 UTC second resolution (the reference's detail::timestamp_utc)."""
    return datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")


def _join(values: Iterable) -> str:
    return ",".join(format_double(v) if isinstance(v, float) else str(v) for v in values)


def write_sweep(out: str, records: Sequence[dict], flags: Sequence[Tuple[str, str]], seed: int) -> Tuple[str, str]:
    """`out`.csv (SWEEP_HEADER rows: dicts with n, l, alpha, seed, mse, mae, nmse) + `out`.manifest."""
    csv_path = out + ".csv"
    with CsvWriter(csv_path, SWEEP_HEADER) as w:
        for r in records:
            w.write_row([str(int(r["n"])), str(int(r["l"])), format_double(r["alpha"]), str(int(r["seed"])),
                         format_double(r["mse"]), format_double(r["mae"]), format_double(r["nmse"])])
    man = out + ".manifest"
    write_manifest(man, RunManifest("sweep", VERSION, int(seed), timestamp_utc(), list(flags), [csv_path]))
    return csv_path, man


def write_bench(out: str, records: Sequence[dict], flags: Sequence[Tuple[str, str]], seed: int) -> Tuple[str, str]:
    """`out`.csv (BENCH_HEADER rows: dicts with n, l, fast_s, exact_s, speedup, repeats) + `out`.manifest."""
    csv_path = out + ".csv"
    with CsvWriter(csv_path, BENCH_HEADER) as w:
        for r in records:
            w.write_row([str(int(r["n"])), str(int(r["l"])), format_double(r["fast_s"]), format_double(r["exact_s"]),
                         format_double(r["speedup"]), str(int(r["repeats"]))])
    man = out + ".manifest"
    write_manifest(man, RunManifest("bench", VERSION, int(seed), timestamp_utc(), list(flags), [csv_path]))
    return csv_path, man


join = _join
