"""Benchmark run records, their CSV form and the matrix text files of the reference CLI.

Mirrors include/rsylv/run_record.hpp + src/run_record.cpp:35-86 (RunRecord, csv_header,
to_csv_row, parse_csv_row, write_csv, read_csv) and src/matrix_io.cpp:10-67 (format_double,
parse_double, write_matrix / read_matrix and the *_file variants). Numbers are written as the
SHORTEST round-trip decimal exactly like std::to_chars (fixed or scientific, whichever is
shorter, fixed on a tie), so a CSV written here is byte-identical to the reference's for equal
values and a reparse reproduces every value bitwise (tests/test_cli_host.py pins the format
against the reference's own format_double).
"""
from __future__ import annotations

import dataclasses
import math
from typing import IO, Iterable

import numpy as np


def _shortest_digits(v: float) -> tuple[str, int]:
    """Shortest round-trip significant digits of |v| > 0 and the decimal exponent E such that
    |v| = 0.d1d2...dk * 10^E (Python's repr is the shortest round-trip form)."""
    r = repr(abs(v))
    mant, _, exp = r.partition("e")
    e10 = int(exp) if exp else 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    # position of the decimal point relative to the first significant digit
    lead = len(ip.lstrip("0")) if ip.strip("0") else -(len(fp) - len(fp.lstrip("0")))
    digits = digits.rstrip("0") or "0"
    return digits, lead + e10


def format_double(v: float) -> str:
    """std::to_chars(double) shortest form (matrix_io.cpp:10-14)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    d, e = _shortest_digits(v)  # |v| = 0.d * 10^e
    k = len(d)
    # fixed notation
    if e >= k:  # an integer: to_chars prints its exact decimal value in fixed form
        fixed = str(int(abs(v)))
    elif e > 0:
        fixed = d[:e] + "." + d[e:]
    else:
        fixed = "0." + "0" * (-e) + d
    # scientific notation, printf %e style exponent (sign, at least two digits)
    x = e - 1
    sci = d[0] + ("." + d[1:] if k > 1 else "") + "e" + ("-" if x < 0 else "+") + f"{abs(x):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def parse_double(s: str) -> float:
    """std::from_chars(double) on the whole token (matrix_io.cpp:16-24): malformed -> ValueError."""
    t = s.strip()
    if t != s or not t or t[0] == "+" or t.lower() in ("infinity", "-infinity"):
        raise ValueError(f"parse_double: malformed value '{s}'")
    try:
        return float(t)
    except ValueError:
        raise ValueError(f"parse_double: malformed value '{s}'") from None


@dataclasses.dataclass
class RunRecord:
    """include/rsylv/run_record.hpp:15-31, plus the number of GPUs (the CSV keeps the reference's
    14 columns unless written with gpus=True)."""
    solver: str = ""
    m: int = 0
    n: int = 0
    tile_size: int = 0
    workers: int = 0
    mu: float = 0.0
    nu: float = 0.0
    omega: float = 0.0
    alpha: float = 1.0
    wall_time_seconds: float = 0.0
    residual: float = 0.0
    min_local_alpha: float = 1.0
    scaling_events: int = 0
    median: bool = False
    gpus: int = 1


_HEADER = ("solver,m,n,tile_size,workers,mu,nu,omega,alpha,"
           "wall_time_seconds,residual,min_local_alpha,scaling_events,median")


def csv_header(gpus: bool = False) -> str:
    """run_record.cpp:35-38 (+ ",gpus" when requested)."""
    return _HEADER + (",gpus" if gpus else "")


def to_csv_row(r: RunRecord, gpus: bool = False) -> str:
    """run_record.cpp:40-48."""
    f = [r.solver, str(int(r.m)), str(int(r.n)), str(int(r.tile_size)), str(int(r.workers)),
         format_double(r.mu), format_double(r.nu), format_double(r.omega),
         format_double(r.alpha), format_double(r.wall_time_seconds), format_double(r.residual),
         format_double(r.min_local_alpha), str(int(r.scaling_events)), "1" if r.median else "0"]
    if gpus:
        f.append(str(int(r.gpus)))
    return ",".join(f)


def parse_csv_row(line: str) -> RunRecord:
    """run_record.cpp:50-69 (14 fields; 15 with the gpus column)."""
    f = line.split(",")
    if len(f) not in (14, 15):
        raise ValueError("parse_csv_row: expected 14 fields")

    def count(s: str) -> int:
        if not s.isdigit():
            raise ValueError(f"parse_csv_row: bad count '{s}'")
        return int(s)

    return RunRecord(solver=f[0], m=count(f[1]), n=count(f[2]), tile_size=count(f[3]),
                     workers=count(f[4]), mu=parse_double(f[5]), nu=parse_double(f[6]),
                     omega=parse_double(f[7]), alpha=parse_double(f[8]),
                     wall_time_seconds=parse_double(f[9]), residual=parse_double(f[10]),
                     min_local_alpha=parse_double(f[11]), scaling_events=count(f[12]),
                     median=f[13] == "1", gpus=count(f[14]) if len(f) == 15 else 1)


def write_csv(fh: IO[str], rows: Iterable[RunRecord], gpus: bool = False) -> None:
    """run_record.cpp:71-74."""
    fh.write(csv_header(gpus) + "\n")
    for r in rows:
        fh.write(to_csv_row(r, gpus) + "\n")


def read_csv(fh: IO[str]) -> list[RunRecord]:
    """run_record.cpp:76-86: header must match exactly (either form); blank lines skipped."""
    lines = fh.read().split("\n")
    if not lines or lines == [""]:
        return []
    if lines[0] not in (csv_header(False), csv_header(True)):
        raise ValueError("read_csv: unexpected header")
    return [parse_csv_row(ln) for ln in lines[1:] if ln]


def write_matrix(fh: IO[str], a) -> None:
    """matrix_io.cpp:26-36: 'rows cols' then one row per line, space separated."""
    a = np.asarray(a, dtype=np.float64)
    fh.write(f"{a.shape[0]} {a.shape[1]}\n")
    for i in range(a.shape[0]):
        fh.write(" ".join(format_double(x) for x in a[i]) + "\n")


def read_matrix(fh: IO[str]) -> np.ndarray:
    """matrix_io.cpp:38-51."""
    toks = fh.read().split()
    if len(toks) < 2:
        raise ValueError("read_matrix: missing 'rows cols' header")
    rows, cols = int(toks[0]), int(toks[1])
    if len(toks) < 2 + rows * cols:
        raise ValueError("read_matrix: truncated matrix body")
    vals = [parse_double(t) for t in toks[2:2 + rows * cols]]
    return np.asfortranarray(np.array(vals, dtype=np.float64).reshape(rows, cols))


def write_matrix_file(path: str, a) -> None:
    with open(path, "w") as fh:
        write_matrix(fh, a)


def read_matrix_file(path: str) -> np.ndarray:
    with open(path) as fh:
        return read_matrix(fh)
