"""Run configuration files of the cavity harness: ``sforge::cli::run_config``,
``parse_run_config`` and ``load_run_config`` (inc/config.hpp:28-260).

A flat ``key = value`` document; ``#`` starts a comment anywhere; every key has
a default; unknown, repeated or malformed keys are errors naming the line,
with the reference's texts. Numbers follow ``std::stod`` / ``std::stol``
(longest valid prefix, then "trailing characters" if anything is left).
"""
from __future__ import annotations

import re
from dataclasses import dataclass

from ._lib import ConfigError, SfError
from .sim import FluidParams, SolverConfig


class ConfigFileError(SfError):
    """cli::config_error (config.hpp:23-26)."""

    def __init__(self, msg: str):
        super().__init__(1, msg)


_WS = " \t\n\v\f\r"


@dataclass
class RunConfig:
    nx: int = 33
    ny: int = 33
    nz: int = 3
    re: float = 100.0
    sigma: float = 0.5
    omega: float = 1.7
    tolerance: float = 1e-6
    max_sweeps: int = 500
    alpha: float = 0.0
    density: float = 1.0
    lid_speed: float = 1.0
    symmetry_z: bool = True
    steady_tol: float = 1e-6
    max_steps: int = 200000
    output_cadence: int = 0
    workers: int = 1
    mode: str = "plain"
    tile: tuple = (0, 0, 0)
    ghost: int = 1
    profiles_out: str = "profiles.csv"
    residuals_out: str = "residuals.csv"
    fields_out: str = ""

    def solver(self) -> SolverConfig:
        """run_config::solver (config.hpp:72-84): the unit cavity box."""
        return SolverConfig(extents=(self.nx, self.ny, self.nz), reynolds=self.re, sigma=self.sigma,
                            omega=self.omega, tolerance=self.tolerance, max_sweeps=_i32(self.max_sweeps),
                            symmetry_z=self.symmetry_z)

    def fluid(self) -> FluidParams:
        """run_config::fluid (config.hpp:86-93)."""
        return FluidParams(viscosity=self.lid_speed * 1.0 / self.re, density=self.density,
                           lid_speed=self.lid_speed, blend=self.alpha)


def _i32(v: int) -> int:  # static_cast<int> of a long
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v >= 1 << 31 else v


# strtod's subject sequence (decimal, hexadecimal, inf/infinity, nan[(...)])
_DEC = r"[+-]?(?:\d+\.?\d*(?:[eE][+-]?\d+)?|\.\d+(?:[eE][+-]?\d+)?)"
_HEX = r"[+-]?0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?"
_SPECIAL = r"[+-]?(?:[iI][nN][fF](?:[iI][nN][iI][tT][yY])?|[nN][aA][nN](?:\([0-9A-Za-z_]*\))?)"
_FLOAT = re.compile("(?:%s|%s|%s)" % (_HEX, _SPECIAL, _DEC))
_INT = re.compile(r"[+-]?\d+")
_LONG_MAX = 2 ** 63 - 1


def _bad(line: int, key: str, why: str):
    raise ConfigFileError("line %d: bad value for '%s': %s" % (line, key, why))


def _strtod_prefix(s: str):
    t = s.lstrip(_WS)
    m = _FLOAT.match(t)
    if not m:
        return None, 0
    tok = m.group(0)
    # a hex prefix without digits ("0x") is the decimal 0 followed by 'x'
    if re.fullmatch(r"[+-]?0[xX]\.?", tok):
        tok = tok[: tok.index("0") + 1]
    lo = tok.lower().lstrip("+-")
    if lo.startswith("0x"):
        t2 = tok if "p" in lo else tok + "p0"
        val = float.fromhex(t2)
    elif lo.startswith("inf") or lo.startswith("nan"):
        val = float(tok.split("(")[0].lower().replace("infinity", "inf"))
    else:
        val = float(tok)
        if val in (float("inf"), float("-inf")):
            return "range", 0  # std::stod throws out_of_range on overflow
    return val, len(s) - len(t) + len(tok)


def _to_double(line: int, key: str, v: str) -> float:
    val, used = _strtod_prefix(v)
    if val is None or val == "range":
        _bad(line, key, "expected a number, got '%s'" % v)
    if used != len(v):
        _bad(line, key, "trailing characters in '%s'" % v)
    return val


def _to_long(line: int, key: str, v: str) -> int:
    t = v.lstrip(_WS)
    m = _INT.match(t)
    if not m or not -_LONG_MAX - 1 <= int(m.group(0)) <= _LONG_MAX:
        _bad(line, key, "expected an integer, got '%s'" % v)
    if len(v) - len(t) + len(m.group(0)) != len(v):
        _bad(line, key, "trailing characters in '%s'" % v)
    return int(m.group(0))


def _to_bool(line: int, key: str, v: str) -> bool:
    if v in ("true", "yes", "on", "1"):
        return True
    if v in ("false", "no", "off", "0"):
        return False
    _bad(line, key, "expected true/false, got '%s'" % v)


def _to_tile(line: int, key: str, v: str):
    parts = v.split(",")
    if parts and parts[-1] == "":  # std::getline yields no empty last field
        parts = parts[:-1]
    out = []
    for p in parts:
        if len(out) == 3:
            _bad(line, key, "expected three comma-separated integers")
        out.append(_i32(_to_long(line, key, p.strip(_WS))))
    if len(out) != 3:
        _bad(line, key, "expected three comma-separated integers")
    return tuple(out)


def parse_run_config(text: str) -> RunConfig:
    """cli::parse_run_config (config.hpp:166-249)."""
    rc = RunConfig()
    seen = set()
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines = lines[:-1]
    for n, raw in enumerate(lines, start=1):
        h = raw.find("#")
        if h >= 0:
            raw = raw[:h]
        t = raw.strip(_WS)
        if not t:
            continue
        eq = t.find("=")
        if eq < 0:
            raise ConfigFileError("line %d: expected 'key = value', got '%s'" % (n, t))
        key, value = t[:eq].strip(_WS), t[eq + 1:].strip(_WS)
        if not key:
            raise ConfigFileError("line %d: missing key before '='" % n)
        if key in seen:
            raise ConfigFileError("line %d: duplicate key '%s'" % (n, key))
        seen.add(key)
        if key in ("nx", "ny", "nz"):
            v = _to_long(n, key, value)
            if v < 1:
                _bad(n, key, "grid extent must be at least 1")
            setattr(rc, key, v)
        elif key == "re":
            rc.re = _to_double(n, key, value)
            if not rc.re > 0.0:
                _bad(n, key, "Reynolds number must be positive")
        elif key == "sigma":
            rc.sigma = _to_double(n, key, value)
            if not (0.0 < rc.sigma < 1.0):
                _bad(n, key, "must lie in (0,1)")
        elif key == "omega":
            rc.omega = _to_double(n, key, value)
            if not (1.0 <= rc.omega < 2.0):
                _bad(n, key, "must lie in [1,2)")
        elif key == "tolerance":
            rc.tolerance = _to_double(n, key, value)
            if not rc.tolerance > 0.0:
                _bad(n, key, "must be positive")
        elif key == "max_sweeps":
            rc.max_sweeps = _to_long(n, key, value)
            if rc.max_sweeps < 1:
                _bad(n, key, "must be at least 1")
        elif key == "alpha":
            rc.alpha = _to_double(n, key, value)
            if not (0.0 <= rc.alpha <= 1.0):
                _bad(n, key, "must lie in [0,1]")
        elif key in ("density", "lid_speed", "steady_tol"):
            setattr(rc, key, _to_double(n, key, value))
            if not getattr(rc, key) > 0.0:
                _bad(n, key, "must be positive")
        elif key == "symmetry_z":
            rc.symmetry_z = _to_bool(n, key, value)
        elif key == "max_steps":
            rc.max_steps = _to_long(n, key, value)
            if rc.max_steps < 1:
                _bad(n, key, "must be at least 1")
        elif key == "output_cadence":
            rc.output_cadence = _to_long(n, key, value)
            if rc.output_cadence < 0:
                _bad(n, key, "must be non-negative")
        elif key in ("workers", "ghost"):
            setattr(rc, key, _i32(_to_long(n, key, value)))
            if getattr(rc, key) < 1:
                _bad(n, key, "must be at least 1")
        elif key == "mode":
            if value not in ("plain", "overlap"):
                _bad(n, key, "expected plain or overlap, got '%s'" % value)
            rc.mode = value
        elif key == "tile":
            rc.tile = _to_tile(n, key, value)
            if any(x < 0 for x in rc.tile):
                _bad(n, key, "tile extents must be non-negative")
        elif key in ("profiles_out", "residuals_out", "fields_out"):
            setattr(rc, key, value)
        else:
            raise ConfigFileError("line %d: unknown key '%s'" % (n, key))
    if _i32(rc.max_sweeps) < 1:  # solver_config::validate (cfd.hpp:55-65) after the int narrowing
        raise ConfigError(1, "max_sweeps must be at least 1")  # a cfd_error: not prefixed with the path
    return rc


def load_run_config(path: str) -> RunConfig:
    """cli::load_run_config (config.hpp:251-260)."""
    try:
        with open(path, newline="") as f:
            text = f.read()
    except OSError:
        raise ConfigFileError("cannot open config file '%s'" % path) from None
    try:
        return parse_run_config(text)
    except ConfigFileError as e:
        raise ConfigFileError("%s: %s" % (path, e)) from None
