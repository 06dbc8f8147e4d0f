"""On-disk formats either side of the LTS path (io-formats).

SFG  text:   line 1 ``SFG <d> <nx> <ny> [<nz>]``, then whitespace-separated
             finite decimal values, x-fastest order (reference
             triangulation.py:8 vertex ids).
SFGB binary: the same header line (magic ``SFGB``) terminated by ``\\n``, then
             the values as raw little-endian float64 (SPEC's "raw
             little-endian float64 variant" for the 10^8-vertex benchmarks).
Preserve list: one vertex id per line (``read_preserve_list``).

The hot path computes in float32 (BASELINE north_star); ``read_field``
returns the values as float32 for it.  Written float32 values carry 9
significant digits, so ``read_sfg(write_sfg(g))`` cast to float32 is the
identity on float32 fields.  Errors follow the reference's ValueError
classes: ``FieldError`` for count mismatches / non-finite values (with the
line number), ``MeshError`` for a malformed header.
"""
from __future__ import annotations

import numpy as np

from .errors import FieldError, MeshError

_MAGIC_TEXT = "SFG"
_MAGIC_BIN = "SFGB"


def _parse_header(line: str, magic: str):
    parts = line.split()
    if not parts or parts[0] != magic:
        raise MeshError(f"line 1: expected '{magic} <d> <nx> <ny> [<nz>]', got {line[:60]!r}")
    try:
        d = int(parts[1])
        dims = tuple(int(x) for x in parts[2:])
    except (IndexError, ValueError):
        raise MeshError(f"line 1: malformed header {line[:60]!r}") from None
    if d not in (2, 3) or len(dims) != d or any(x < 1 for x in dims):
        raise MeshError(f"line 1: dimension {d} with sizes {dims} is not a 2D/3D grid")
    return dims


def _header(magic: str, dims) -> str:
    return f"{magic} {len(dims)} " + " ".join(str(int(x)) for x in dims)


def _check_finite(values: np.ndarray, where: str):
    bad = ~np.isfinite(values)
    if bad.any():
        raise FieldError(f"{where}: value {int(np.argmax(bad))} is not finite")


def read_sfg(text: str):
    """SFG text -> (dims (nx, ny[, nz]), float64 values, x-fastest)."""
    lines = text.splitlines()
    if not lines:
        raise MeshError("line 1: empty input")
    dims = _parse_header(lines[0], _MAGIC_TEXT)
    n = int(np.prod(dims))
    vals = []
    for ln, line in enumerate(lines[1:], start=2):
        for tok in line.split():
            try:
                vals.append(float(tok))
            except ValueError:
                raise FieldError(f"line {ln}: {tok[:30]!r} is not a decimal value") from None
            if len(vals) > n:
                raise FieldError(f"line {ln}: more than {n} values for grid {dims}")
    if len(vals) != n:
        raise FieldError(f"line {len(lines)}: {len(vals)} values for grid {dims} (expected {n})")
    v = np.asarray(vals, dtype=np.float64)
    _check_finite(v, "values")
    return dims, v


def write_sfg(dims, values) -> str:
    """(dims, values) -> SFG text; float32 values with 9 significant digits,
    float64 values in shortest round-trip form."""
    v = np.asarray(values).ravel()
    if v.size != int(np.prod(dims)):
        raise FieldError(f"{v.size} values for grid {tuple(dims)}")
    if v.dtype == np.float32:
        # 9 significant digits: the decimal lies well inside the float32's
        # rounding interval, so parsing it as float64 and casting back is exact
        body = ["%.9g" % x for x in v.astype(np.float64)]
    else:
        body = [repr(float(x)) for x in v.astype(np.float64)]
    rows = [" ".join(body[i:i + 16]) for i in range(0, len(body), 16)]
    return _header(_MAGIC_TEXT, dims) + "\n" + "\n".join(rows) + "\n"


def read_sfgb(data: bytes):
    """SFGB bytes -> (dims, float64 values)."""
    nl = data.find(b"\n")
    if nl < 0:
        raise MeshError("line 1: missing SFGB header")
    dims = _parse_header(data[:nl].decode("ascii", "replace"), _MAGIC_BIN)
    n = int(np.prod(dims))
    body = data[nl + 1:]
    if len(body) != 8 * n:
        raise FieldError(f"SFGB body holds {len(body)} bytes for grid {dims} (expected {8 * n})")
    v = np.frombuffer(body, dtype="<f8").astype(np.float64)
    _check_finite(v, "values")
    return dims, v


def write_sfgb(dims, values) -> bytes:
    v = np.ascontiguousarray(np.asarray(values, dtype="<f8").ravel())
    if v.size != int(np.prod(dims)):
        raise FieldError(f"{v.size} values for grid {tuple(dims)}")
    return (_header(_MAGIC_BIN, dims) + "\n").encode("ascii") + v.tobytes()


def read_field(path: str):
    """SFG or SFGB file -> (dims, float32 values) for the hot path."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data.startswith(_MAGIC_BIN.encode()):
        dims, v = read_sfgb(data)
    else:
        dims, v = read_sfg(data.decode("utf-8"))
    return dims, v.astype(np.float32)


def write_field(path: str, dims, values):
    """Write SFGB when the path ends in .sfgb, SFG text otherwise."""
    if path.endswith(".sfgb"):
        with open(path, "wb") as fh:
            fh.write(write_sfgb(dims, values))
    else:
        with open(path, "w") as fh:
            fh.write(write_sfg(dims, values))


def read_preserve_list(text: str, n: int) -> np.ndarray:
    """One vertex id per line (blank lines and '#' comments ignored)."""
    ids = []
    for ln, line in enumerate(text.splitlines(), start=1):
        s = line.split("#", 1)[0].strip()
        if not s:
            continue
        try:
            v = int(s)
        except ValueError:
            raise FieldError(f"line {ln}: {s[:30]!r} is not a vertex id") from None
        if v < 0 or v >= n:
            raise FieldError(f"line {ln}: vertex id {v} is outside [0, {n})")
        ids.append(v)
    return np.unique(np.asarray(ids, dtype=np.int64))


def write_preserve_list(ids) -> str:
    return "".join(f"{int(v)}\n" for v in np.asarray(ids).ravel())
