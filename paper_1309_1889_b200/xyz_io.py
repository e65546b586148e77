"""Extended-XYZ particle files and CSV output: the data formats on
either side of the path, as the reference writes and reads them.

  paramd::load_system / save_system / TrajectoryWriter / format_real
                                   include/paramd/xyz_io.hpp:17-30, src/xyz_io.cpp:1-120
  paramd::validate_system          src/system.cpp:10-33
  paramd::csv_num / CsvWriter      include/paramd/csv.hpp:11-34

Format: line 1 N; line 2 "box <bx> <by> <bz>" then free tokens; then N lines
"element x y z q vx vy vz mass".  Reals are written with %.17g, so files round-trip
bitwise, and byte-identical to the reference's for the same system.  Parse errors
carry the reference's messages and line numbers.  Host-side code: no GPU involved.
"""
from __future__ import annotations

import math

import numpy as np

from . import ConfigError, Error, ParticleSystem


class ParseError(Error):  # errors.hpp:22-24
    pass


def format_real(v: float) -> str:
    """%.17g (src/xyz_io.cpp:13-17)."""
    return "%.17g" % float(v)


csv_num = format_real  # csv.hpp:11-15


def validate_system(s: ParticleSystem, require_in_box: bool) -> None:
    """src/system.cpp:10-33, same checks and messages, in the same order."""
    n = len(s.positions)
    if n == 0:
        raise ConfigError("system must contain at least one particle")
    if len(s.velocities) != n or len(s.charges) != n or len(s.masses) != n:
        raise ConfigError(f"system field lengths differ: positions={n} velocities={len(s.velocities)} "
                          f"charges={len(s.charges)} masses={len(s.masses)}")
    b = s.box
    if not (b[0] > 0.0 and b[1] > 0.0 and b[2] > 0.0):
        raise ConfigError("box extents must be positive")
    finite = (np.isfinite(s.positions).all(axis=1) & np.isfinite(s.velocities).all(axis=1)
              & np.isfinite(s.charges) & np.isfinite(s.masses))
    nonpos = ~(s.masses > 0.0)
    outside = np.zeros(n, dtype=bool)
    if require_in_box:
        p = s.positions
        outside = (p[:, 0] < 0.0) | (p[:, 0] > b[0]) | (p[:, 1] < 0.0) | (p[:, 1] > b[1]) | \
                  (p[:, 2] < 0.0) | (p[:, 2] > b[2])
    bad = ~finite | nonpos | outside
    if bad.any():  # the first failing particle, with the first failing check
        i = int(np.argmax(bad))
        if not finite[i]:
            raise ConfigError(f"non-finite value at particle {i}")
        if nonpos[i]:
            raise ConfigError(f"non-positive mass at particle {i}")
        raise ConfigError(f"particle {i} outside the box")


def _strtod_full(tok: str):
    """std::strtod consuming the whole token, else None."""
    t = tok.strip()
    if t != tok or not t or "_" in t:  # Python float() accepts digit separators, strtod does not
        return None
    try:
        return float(t)
    except ValueError:
        low = t.lower()
        if low.startswith("0x") or low.startswith("-0x") or low.startswith("+0x"):
            try:
                return float.fromhex(t)
            except ValueError:
                return None
        return None


def _parse_real(tok: str, lineno: int) -> float:  # src/xyz_io.cpp:30-39
    v = _strtod_full(tok)
    if v is None:
        raise ParseError(f"line {lineno}: expected a number, got '{tok}'")
    if not math.isfinite(v):
        raise ParseError(f"line {lineno}: non-finite value '{tok}'")
    return v


def load_system(path: str) -> ParticleSystem:
    """paramd::load_system (src/xyz_io.cpp:43-86)."""
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise Error(f"cannot open {path} for reading")
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # getline: a trailing newline does not start another line
    if not lines:
        raise ParseError("line 1: empty file")
    first = lines[0]
    head = first.rstrip(" \t\r")
    try:
        j = 0
        while j < len(head) and head[j] in " \t\n\v\f\r":
            j += 1
        body = head[j:]
        if body.startswith(("+", "-")):
            digits = body[1:]
        else:
            digits = body
        if not digits or not digits.isdigit():
            raise ValueError
        n = int(body)
    except ValueError:
        n = 0
        raise ParseError(f"line 1: expected a positive particle count, got '{first}'") from None
    if n < 1:
        raise ParseError(f"line 1: expected a positive particle count, got '{first}'")
    if len(lines) < 2:
        raise ParseError("line 2: missing comment line")
    comment = lines[1].split()
    if len(comment) < 4 or comment[0] != "box":
        raise ParseError("line 2: expected 'box <x> <y> <z>' at the start of the comment")
    box = np.array([_parse_real(comment[k], 2) for k in (1, 2, 3)])
    pos = np.zeros((n, 3))
    vel = np.zeros((n, 3))
    q = np.zeros(n)
    m = np.zeros(n)
    for i in range(n):
        lineno = 3 + i
        if lineno - 1 >= len(lines):
            raise ParseError(f"line {lineno}: unexpected end of file ({i} of {n} rows read)")
        tok = lines[lineno - 1].split()
        if len(tok) != 9:
            raise ParseError(f"line {lineno}: expected 9 fields, got {len(tok)}")
        vals = [_parse_real(t, lineno) for t in tok[1:]]
        pos[i] = vals[0:3]
        q[i] = vals[3]
        vel[i] = vals[4:7]
        m[i] = vals[7]
    s = ParticleSystem(pos, vel, q, m, box)
    validate_system(s, True)
    return s


def _frame_text(s: ParticleSystem, extra: str) -> str:  # src/xyz_io.cpp:90-103
    out = [f"{s.size()}\n", "box " + " ".join(format_real(v) for v in s.box) + extra + "\n"]
    for i in range(s.size()):
        p, v = s.positions[i], s.velocities[i]
        out.append("X " + " ".join(format_real(x) for x in (p[0], p[1], p[2], s.charges[i], v[0], v[1], v[2],
                                                              s.masses[i])) + "\n")
    return "".join(out)


def save_system(s: ParticleSystem, path: str) -> None:
    """paramd::save_system (src/xyz_io.cpp:107-111)."""
    try:
        f = open(path, "w", newline="")
    except OSError:
        raise Error(f"cannot open {path} for writing")
    with f:
        f.write(_frame_text(s, ""))


class TrajectoryWriter:
    """paramd::TrajectoryWriter (src/xyz_io.cpp:113-120): appends frames whose comment
    carries the box, step and time."""

    def __init__(self, path: str):
        try:
            self._f = open(path, "w", newline="")
        except OSError:
            raise Error(f"cannot open {path} for writing")

    def write_frame(self, s: ParticleSystem, step: int, time_fs: float) -> None:
        self._f.write(_frame_text(s, f" step={int(step)} time={format_real(time_fs)}"))
        self._f.flush()

    def close(self):
        self._f.close()


class CsvWriter:
    """paramd::CsvWriter (csv.hpp:17-34)."""

    def __init__(self, path: str):
        try:
            self._f = open(path, "w", newline="")
        except OSError:
            raise Error(f"cannot open {path} for writing")

    def row(self, cells) -> None:
        self._f.write(",".join(cells) + "\n")
        self._f.flush()

    def close(self):
        self._f.close()
