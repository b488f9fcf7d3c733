"""Instance and solution files (the formats of hm/io.py:1-20), read strictly.

Instance files are whitespace-separated UTF-8 text; ``#`` comment lines and
blank lines are skipped:

* canonical (``.usaphmp``): ``n p``, ``chi alpha delta``, n distance rows,
  n flow rows;
* coordinate (``.coords``): ``n p``, ``chi alpha delta``, n ``x y`` rows
  (Euclidean distances, computed as in generate_urand), n flow rows.

Solution files: ``n p``, the p hub indices, the n allocation entries, all
1-based.  Every malformed input raises ``ParseError`` (a ValueError) whose
message starts with the offending line number, so a caller can point at it.
Distance and flow values must be finite and non-negative; the distance
diagonal must be zero; factors must be positive; nothing may follow the last
expected row.
"""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

from .io import euclidean_distances
from .model import Instance, Solution

CANONICAL = "canonical"
COORDINATE = "coordinate"
FORMAT_BY_SUFFIX = {".usaphmp": CANONICAL, ".coords": COORDINATE}


class ParseError(ValueError):
    """hm/io.py:43-46: a malformed file; ``line`` is the 1-based line number
    (None when the problem is not tied to one line)."""

    def __init__(self, msg: str, line: int | None = None):
        self.line = line
        super().__init__(msg if line is None else f"line {line}: {msg}")


def _text(source) -> str:
    if isinstance(source, Path):
        raise TypeError("pass file contents or a stream; load_instance takes paths")
    if isinstance(source, (bytes, bytearray)):
        return bytes(source).decode("utf-8")
    if isinstance(source, str):
        return source
    data = source.read()
    return data.decode("utf-8") if isinstance(data, bytes) else data


class _Rows:
    """The logical (non-blank, non-comment) lines of a file, with numbers."""

    def __init__(self, text: str):
        self._rows = [(no, ln.strip()) for no, ln in enumerate(text.splitlines(), start=1)
                      if ln.strip() and not ln.strip().startswith("#")]
        self._at = 0
        self.line = 0

    def take(self, what: str) -> list[str]:
        if self._at >= len(self._rows):
            raise ParseError(f"unexpected end of file, expected {what}")
        self.line, text = self._rows[self._at]
        self._at += 1
        return text.split()

    def finish(self) -> None:
        if self._at < len(self._rows):
            no, text = self._rows[self._at]
            raise ParseError(f"unexpected trailing content: {text[:40]!r}", no)

    def numbers(self, count: int, what: str, nonnegative: bool = True) -> np.ndarray:
        tokens = self.take(what)
        if len(tokens) != count:
            raise ParseError(f"expected {count} values for {what}, got {len(tokens)}", self.line)
        try:
            vals = np.array([float(t) for t in tokens], dtype=np.float64)
        except ValueError:
            raise ParseError(f"non-numeric token in {what}", self.line) from None
        if not np.all(np.isfinite(vals)):
            raise ParseError(f"non-finite value in {what}", self.line)
        if nonnegative and np.any(vals < 0):
            raise ParseError(f"negative value in {what}", self.line)
        return vals

    def sizes(self) -> tuple[int, int]:
        tokens = self.take("header 'n p'")
        if len(tokens) != 2:
            raise ParseError(f"expected 'n p', got {len(tokens)} tokens", self.line)
        try:
            n, p = int(tokens[0]), int(tokens[1])
        except ValueError:
            raise ParseError("n and p must be integers", self.line) from None
        return n, p


def format_for_path(path) -> str:
    suffix = Path(path).suffix.lower()
    if suffix not in FORMAT_BY_SUFFIX:
        raise ValueError(f"cannot infer format from suffix {suffix!r}; "
                         f"expected .usaphmp or .coords")
    return FORMAT_BY_SUFFIX[suffix]


def parse_instance(source, format: str = CANONICAL, name: str = "") -> Instance:
    if format not in (CANONICAL, COORDINATE):
        raise ValueError(f"unknown format {format!r}")
    rows = _Rows(_text(source))
    n, p = rows.sizes()
    if n < 1:
        raise ParseError(f"node count must be positive, got {n}", rows.line)
    if not 1 <= p <= n:
        raise ParseError(f"hub count p={p} outside [1, {n}]", rows.line)
    factors = rows.numbers(3, "cost factors 'chi alpha delta'")
    if np.any(factors <= 0):
        raise ParseError("cost factors must be positive", rows.line)
    if format == CANONICAL:
        dist = np.empty((n, n), dtype=np.float64)
        for i in range(n):
            dist[i] = rows.numbers(n, f"distance row {i + 1}")
            if dist[i, i] != 0.0:
                raise ParseError(f"distance diagonal entry {i + 1} must be zero", rows.line)
    else:
        xy = np.empty((n, 2), dtype=np.float64)
        for i in range(n):
            xy[i] = rows.numbers(2, f"coordinate pair {i + 1}", nonnegative=False)
        dist = euclidean_distances(xy)
    flow = np.empty((n, n), dtype=np.float64)
    for i in range(n):
        flow[i] = rows.numbers(n, f"flow row {i + 1}")
    rows.finish()
    chi, alpha, delta = (float(v) for v in factors)
    return Instance(n=n, p=p, dist=dist, flow=flow, chi=chi, alpha=alpha, delta=delta, name=name)


def load_instance(path, format: str | None = None) -> Instance:
    path = Path(path)
    return parse_instance(path.read_bytes(), format=format or format_for_path(path),
                          name=path.stem)


def serialize_instance(inst: Instance) -> bytes:
    """Canonical bytes; every float printed with repr (round-trips exactly)."""
    lines = [f"{inst.n} {inst.p}", f"{inst.chi!r} {inst.alpha!r} {inst.delta!r}"]
    lines += [" ".join(repr(v) for v in row) for row in inst.dist.tolist()]
    lines += [" ".join(repr(v) for v in row) for row in inst.flow.tolist()]
    return ("\n".join(lines) + "\n").encode("utf-8")


def save_instance(path, inst: Instance) -> None:
    Path(path).write_bytes(serialize_instance(inst))


def read_solution(source) -> tuple[int, int, Solution]:
    """(n, p, Solution) with 0-based arrays."""
    rows = _Rows(_text(source))
    n, p = rows.sizes()
    if n < 1 or not 1 <= p <= n:
        raise ParseError(f"bad sizes n={n}, p={p}", rows.line)
    parsed = []
    for count, what in ((p, "hub indices"), (n, "allocation entries")):
        vals = rows.numbers(count, what)
        if np.any(vals != np.floor(vals)):
            raise ParseError(f"non-integer token in {what}", rows.line)
        parsed.append(vals.astype(np.int64))
    rows.finish()
    hub_idx, alloc = parsed
    for label, vals in (("hub index", hub_idx), ("allocation entry", alloc)):
        if np.any(vals < 1) or np.any(vals > n):
            raise ParseError(f"{label} outside [1, {n}]")
    hub = np.zeros(n, dtype=bool)
    hub[hub_idx - 1] = True
    return n, p, Solution(hub=hub, alloc=alloc - 1)


def write_solution(sol: Solution, p: int | None = None) -> bytes:
    hubs = sol.hubs
    lines = [f"{sol.hub.shape[0]} {hubs.size if p is None else p}",
             " ".join(str(int(h) + 1) for h in hubs),
             " ".join(str(int(a) + 1) for a in sol.alloc)]
    return ("\n".join(lines) + "\n").encode("utf-8")


def sha256_hex(data: bytes) -> str:
    return hashlib.sha256(data).hexdigest()
