"""load_config: flat `key = value` text with [sections]
("flat key=value text with sections, documented schema"),
every unknown key an error, parse errors with line / column, semantic errors
with the key path; `--set section.key=value` overrides.

Schema (section.key: type, default):

    [case]     name: circular | pseudo2d | humps | hump_dambreak | monai | river | dem   (required)
               dem_path: str (name = dem; Esri ASCII, top row first)
               eta0: float 0.0 (name = dem: initial free surface; h = max(0, eta0 - z))
               seed: int (monai / river generators)
    [grid]     L: int (required, 1..13)   epsilon: float (required, >= 0)
               band: neighbours | parents | none   (D3)
    [physics]  cfl 0.5, g 9.80665, manning (case default), h_dry 1e-6
    [time]     t_end: float (case default)   dt_fallback: float 1e-3
               output_times: comma list of floats (ascending)
    [boundary] west / east / north / south: reflective | transmissive | inflow (case default)
    [output]   dir: str "out"   snapshots: bool true   step_report: bool true
               gauges: "name x y; name x y; ..."   gauge_every: int 1 (steps)
    [solver]   kind: adaptive | uniform   device: int 0

Host plumbing only (no GPU work): the engine is built by `build_state`.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import cases
from .abi import (BAND_NEIGHBOURS, BAND_NONE, BAND_PARENTS, BC_INFLOW, BC_REFLECTIVE, BC_TRANSMISSIVE, SimConfig)


class ConfigError(ValueError):
    """A located config error: `where` is 'path:line:col' or a key path."""

    def __init__(self, where: str, msg: str):
        super().__init__(f"{where}: {msg}")
        self.where = where


CASES = {
    "circular": cases.circular_dambreak,
    "pseudo2d": cases.pseudo2d_dambreak,
    "humps": cases.quiescent_humps,
    "hump_dambreak": cases.hump_dambreak,
    "monai": cases.monai_runup,
    "river": cases.river_flood,
    "dem": None,
}
_BANDS = {"neighbours": BAND_NEIGHBOURS, "parents": BAND_PARENTS, "none": BAND_NONE}
_BCS = {"reflective": BC_REFLECTIVE, "transmissive": BC_TRANSMISSIVE, "inflow": BC_INFLOW}
_BOOL = {"true": True, "yes": True, "1": True, "false": False, "no": False, "0": False}

# section -> key -> (parser, default); default None = optional / case default
_SCHEMA = {
    "case": {"name": ("case", None), "dem_path": ("str", None), "eta0": ("float", 0.0), "seed": ("int", None)},
    "grid": {"L": ("int", None), "epsilon": ("float", None), "band": ("band", BAND_NEIGHBOURS)},
    "physics": {"cfl": ("float", 0.5), "g": ("float", 9.80665), "manning": ("float", None), "h_dry": ("float", 1e-6)},
    "time": {"t_end": ("float", None), "dt_fallback": ("float", 1e-3), "output_times": ("floats", ())},
    "boundary": {k: ("bc", None) for k in ("west", "east", "north", "south")},
    "output": {"dir": ("str", "out"), "snapshots": ("bool", True), "step_report": ("bool", True),
               "gauges": ("gauges", ()), "gauge_every": ("int", 1)},
    "solver": {"kind": ("solver", "adaptive"), "device": ("int", 0)},
}
REQUIRED = ("case.name", "grid.L", "grid.epsilon")


def _parse_value(kind: str, raw: str, where: str):
    s = raw.strip()
    try:
        if kind == "int":
            return int(s)
        if kind == "float":
            v = float(s)
            if not np.isfinite(v):
                raise ValueError
            return v
        if kind == "str":
            if not s:
                raise ValueError
            return s
        if kind == "bool":
            return _BOOL[s.lower()]
        if kind == "floats":
            return tuple(float(x) for x in s.split(",") if x.strip())
        if kind == "case":
            if s not in CASES:
                raise ConfigError(where, f"unknown case {s!r} (one of {', '.join(CASES)})")
            return s
        if kind == "band":
            return _BANDS[s.lower()]
        if kind == "bc":
            return _BCS[s.lower()]
        if kind == "solver":
            if s not in ("adaptive", "uniform"):
                raise ValueError
            return s
        if kind == "gauges":
            out = []
            for part in s.split(";"):
                f = part.split()
                if not f:
                    continue
                if len(f) != 3:
                    raise ValueError
                out.append((f[0], float(f[1]), float(f[2])))
            return tuple(out)
    except ConfigError:
        raise
    except (ValueError, KeyError):
        pass
    raise ConfigError(where, f"invalid {kind} value {raw.strip()!r}")


@dataclass
class RunConfig:
    """SimConfig external form plus the output plan."""

    values: dict = field(default_factory=dict)  # "section.key" -> parsed value

    def get(self, key: str):
        if key in self.values:
            return self.values[key]
        sec, k = key.split(".", 1)
        return _SCHEMA[sec][k][1]


def _set(values: dict, key: str, raw: str, where: str) -> None:
    if "." not in key:
        raise ConfigError(where, f"key {key!r} outside a section")
    sec, k = key.split(".", 1)
    if sec not in _SCHEMA:
        raise ConfigError(where, f"unknown section [{sec}]")
    if k not in _SCHEMA[sec]:
        raise ConfigError(where, f"unknown key {sec}.{k}")
    values[f"{sec}.{k}"] = _parse_value(_SCHEMA[sec][k][0], raw, f"{where} ({sec}.{k})")


def parse_config(text: str, source: str = "<config>", overrides=()) -> RunConfig:
    """Parse + validate (total: every input gives a RunConfig or a ConfigError)."""
    values: dict = {}
    sec = None
    for ln, line in enumerate(text.splitlines(), 1):
        body = line.split("#", 1)[0]
        s = body.strip()
        if not s:
            continue
        col = len(body) - len(body.lstrip()) + 1
        where = f"{source}:{ln}:{col}"
        if s.startswith("["):
            if not s.endswith("]") or len(s) < 3:
                raise ConfigError(where, f"malformed section header {s!r}")
            sec = s[1:-1].strip()
            if sec not in _SCHEMA:
                raise ConfigError(where, f"unknown section [{sec}]")
            continue
        if "=" not in s:
            raise ConfigError(where, f"expected key = value, got {s!r}")
        k, v = s.split("=", 1)
        k = k.strip()
        if not k:
            raise ConfigError(where, "empty key")
        if sec is None:
            raise ConfigError(where, f"key {k!r} before any [section]")
        _set(values, f"{sec}.{k}", v, where)
    for o in overrides:
        if "=" not in o:
            raise ConfigError(f"--set {o}", "expected section.key=value")
        k, v = o.split("=", 1)
        _set(values, k.strip(), v, f"--set {o}")
    rc = RunConfig(values)
    validate(rc)
    return rc


def load_config(path: str, overrides=()) -> RunConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise ConfigError(str(path), f"cannot read: {e.strerror}") from None
    return parse_config(text, str(path), overrides)


def validate(rc: RunConfig) -> None:
    for k in REQUIRED:
        if rc.get(k) is None:
            raise ConfigError(k, "required key missing")
    L = rc.get("grid.L")
    if not 1 <= L <= 13:
        raise ConfigError("grid.L", f"L = {L} outside [1, 13] (z-index must stay below 2^28, zorder.hpp:21)")
    if not rc.get("grid.epsilon") >= 0.0:
        raise ConfigError("grid.epsilon", f"epsilon = {rc.get('grid.epsilon')} must be >= 0")
    if not 0.0 < rc.get("physics.cfl") <= 1.0:
        raise ConfigError("physics.cfl", "CFL number must be in (0, 1]")
    for k in ("physics.g", "physics.h_dry", "time.dt_fallback"):
        if not rc.get(k) > 0.0:
            raise ConfigError(k, "must be > 0")
    if rc.get("physics.manning") is not None and rc.get("physics.manning") < 0.0:
        raise ConfigError("physics.manning", "must be >= 0")
    te = rc.get("time.t_end")
    if te is not None and te < 0.0:
        raise ConfigError("time.t_end", "must be >= 0")
    ot = rc.get("time.output_times")
    if any(b <= a for a, b in zip(ot, ot[1:])) or any(t < 0 for t in ot):
        raise ConfigError("time.output_times", "must be non-negative and ascending")
    if rc.get("output.gauge_every") < 1:
        raise ConfigError("output.gauge_every", "must be >= 1")
    if rc.get("case.name") == "dem" and rc.get("case.dem_path") is None:
        raise ConfigError("case.dem_path", "required for case dem")


def build_state(rc: RunConfig):
    """(SimConfig, h, qx, qy, z) of the configured case with every override applied."""
    name = rc.get("case.name")
    L, eps, band = rc.get("grid.L"), rc.get("grid.epsilon"), rc.get("grid.band")
    if name == "dem":
        from . import io

        r = io.read_esri(rc.get("case.dem_path"))
        W = max(r.ncols, r.nrows) * r.cellsize
        z, ina = io.load_dem(r, L, r.xllcorner, r.yllcorner, W)
        h = np.where(ina, 0.0, np.maximum(0.0, rc.get("case.eta0") - z))
        cfg = SimConfig(L=L, epsilon=eps, width=W, x0=r.xllcorner, y0=r.yllcorner, band_mode=band,
                        bc=(BC_TRANSMISSIVE,) * 4, inactive=ina if ina.any() else None, name="dem")
        qx = np.zeros_like(h)
        qy = np.zeros_like(h)
    else:
        kw = dict(L=L, epsilon=eps, band_mode=band)
        if rc.get("case.seed") is not None:
            if name not in ("monai", "river"):
                raise ConfigError("case.seed", f"case {name} takes no seed")
            kw["seed"] = rc.get("case.seed")
        cfg, h, qx, qy, z = CASES[name](**kw)
    cfg.cfl = rc.get("physics.cfl")
    cfg.g = rc.get("physics.g")
    cfg.h_dry = rc.get("physics.h_dry")
    cfg.dt_fallback = rc.get("time.dt_fallback")
    if rc.get("physics.manning") is not None:
        cfg.manning = rc.get("physics.manning")
    if rc.get("time.t_end") is not None:
        cfg.t_end = rc.get("time.t_end")
    ot = tuple(t for t in rc.get("time.output_times") if t <= cfg.t_end)
    cfg.output_times = ot
    bc = list(cfg.bc)
    for k, key in enumerate(("west", "east", "north", "south")):
        if rc.get(f"boundary.{key}") is not None:
            bc[k] = rc.get(f"boundary.{key}")
    cfg.bc = tuple(bc)
    if BC_INFLOW in bc and len(cfg.inflow_t) == 0:
        raise ConfigError("boundary", "an inflow edge needs a case with an inflow series (monai, river)")
    try:
        cfg.validate()
    except ValueError as e:
        raise ConfigError("config", str(e)) from None
    return cfg, h, qx, qy, z


def out_dir(rc: RunConfig) -> str:
    return os.path.abspath(rc.get("output.dir"))
