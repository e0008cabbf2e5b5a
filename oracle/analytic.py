"""Independent physics oracles of the cases module.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): the checkers behind
acceptance criteria A5 (Stoker exact solution, §3.2 / Fig. 13) and
the circular dam-break benchmark profile ("FV1 numerical
solution to 1D radial form of the 2D shallow water equations"). They share
no code with the engine or with oracle/hwfv1_oracle.cpp: the engine and the
CPU restatement agree bit for bit, so these are the checks that the pinned
scheme itself solves the right equations.
"""
from __future__ import annotations

import math

import numpy as np

G = 9.80665


# ---------------------------------------------------------------- Stoker
def stoker_middle(hL: float, hR: float, g: float = G, tol: float = 1e-12):
    """Intermediate state (h_m, u_m, shock speed s) of the wet-bed dam break
    (SPEC.md:504-512): the left rarefaction gives u_m = 2 (sqrt(g hL) -
    sqrt(g h_m)); the right-moving shock into still water gives
    u_m = (h_m - hR) sqrt(g (h_m + hR) / (2 h_m hR)). h_m in (hR, hL) is the
    root of their difference, found by bisection to `tol` (abs. in h)."""
    if not hL > hR >= 0.0:
        raise ValueError("Stoker oracle needs hL > hR >= 0")
    if hR == 0.0:  # dry bed: Ritter, no middle state
        return 0.0, 2.0 * math.sqrt(g * hL), 2.0 * math.sqrt(g * hL)
    cL = math.sqrt(g * hL)

    def f(hm):
        return 2.0 * (cL - math.sqrt(g * hm)) - (hm - hR) * math.sqrt(g * (hm + hR) / (2.0 * hm * hR))

    a, b = hR, hL
    fa = f(a)
    it = 0
    while b - a > tol:
        m = 0.5 * (a + b)
        fm = f(m)
        if (fm > 0.0) == (fa > 0.0):
            a, fa = m, fm
        else:
            b = m
        it += 1
        if it > 200:
            raise RuntimeError("Stoker bisection did not converge")
    hm = 0.5 * (a + b)
    um = 2.0 * (cL - math.sqrt(g * hm))
    s = hm * um / (hm - hR)
    return hm, um, s


def rankine_hugoniot_residual(hL: float, hR: float, g: float = G) -> float:
    """Momentum jump residual across the Stoker shock (SPEC.md:518 self-check):
    s [hu] - [h u^2 + g h^2 / 2], relative to the momentum flux scale."""
    hm, um, s = stoker_middle(hL, hR, g)
    res = s * (hm * um) - (hm * um * um + 0.5 * g * (hm * hm - hR * hR))
    return abs(res) / (0.5 * g * hL * hL)


def stoker(hL: float, hR: float, x0: float, t: float, x, g: float = G):
    """Exact depth and velocity of the dam break at time t, positions x."""
    x = np.asarray(x, dtype=np.float64)
    if t <= 0.0:
        return np.where(x < x0, hL, hR), np.zeros_like(x)
    if hL == hR:
        return np.full_like(x, hL), np.zeros_like(x)
    hm, um, s = stoker_middle(hL, hR, g)
    cL, cm = math.sqrt(g * hL), math.sqrt(g * hm)
    xi = (x - x0) / t
    h = np.empty_like(x)
    u = np.empty_like(x)
    left = xi < -cL
    fan = (xi >= -cL) & (xi < um - cm)
    mid = (xi >= um - cm) & (xi < s)
    right = xi >= s
    h[left], u[left] = hL, 0.0
    c = (2.0 * cL - xi[fan]) / 3.0
    h[fan], u[fan] = c * c / g, 2.0 * (xi[fan] + cL) / 3.0
    h[mid], u[mid] = hm, um
    h[right], u[right] = hR, 0.0
    return h, u


# ---------------------------------------------------------------- radial
def _hll_1d(hL, uL, hR, uR, g):
    """HLL flux (h, hu) of the 1D SWE with the same wave speeds as the engine
    (two-rarefaction estimates), vectorised; dry sides handled."""
    cL, cR = np.sqrt(g * hL), np.sqrt(g * hR)
    us = 0.5 * (uL + uR) + (cL - cR)
    cs = np.maximum(0.5 * (cL + cR) + 0.25 * (uL - uR), 0.0)
    SL = np.minimum(uL - cL, us - cs)
    SR = np.maximum(uR + cR, us + cs)
    dryL, dryR = hL <= 0.0, hR <= 0.0
    SL = np.where(dryL, uR - 2.0 * cR, SL)
    SR = np.where(dryL, uR + cR, SR)
    SL = np.where(dryR & ~dryL, uL - cL, SL)
    SR = np.where(dryR & ~dryL, uL + 2.0 * cL, SR)
    FL = np.stack([hL * uL, hL * uL * uL + 0.5 * g * hL * hL])
    FR = np.stack([hR * uR, hR * uR * uR + 0.5 * g * hR * hR])
    UL, UR = np.stack([hL, hL * uL]), np.stack([hR, hR * uR])
    den = np.where(SR - SL == 0.0, 1.0, SR - SL)
    Fs = (SR * FL - SL * FR + SL * SR * (UR - UL)) / den
    F = np.where(SL >= 0.0, FL, np.where(SR <= 0.0, FR, Fs))
    return np.where((dryL & dryR)[None, :], 0.0, F)


class Radial:
    """1D FV1 solver of the radially symmetric shallow water equations
    (SPEC.md:513-521): cells [r_{i-1/2}, r_{i+1/2}] of equal width on
    [0, R_max], conservative r-weighted form
        d/dt (V_i U_i) = -(r_{i+1/2} F_{i+1/2} - r_{i-1/2} F_{i-1/2}) + (0, g h_i^2 / 2 dr),
    V_i = (r_{i+1/2}^2 - r_{i-1/2}^2) / 2, HLL fluxes, forward Euler, CFL 0.5.
    No flux through r = 0; the outer edge is a wall (closed) or transmissive.
    Flat frictionless bed."""

    def __init__(self, h0, r_max: float, n: int, g: float = G, outer: str = "transmissive"):
        self.g, self.n, self.outer = g, n, outer
        self.dr = r_max / n
        self.re = np.arange(n + 1) * self.dr  # faces
        self.rc = 0.5 * (self.re[:-1] + self.re[1:])
        self.V = 0.5 * (self.re[1:] ** 2 - self.re[:-1] ** 2)
        self.h = np.asarray(h0(self.rc), dtype=np.float64).copy()
        self.q = np.zeros(n)
        self.t = 0.0

    def mass(self) -> float:
        return float(np.sum(self.V * self.h))

    def step(self, t_stop: float, cfl: float = 0.5) -> None:
        g = self.g
        u = np.where(self.h > 1e-12, self.q / np.maximum(self.h, 1e-300), 0.0)
        smax = float(np.max(np.abs(u) + np.sqrt(g * self.h)))
        dt = min(cfl * self.dr / smax, t_stop - self.t)
        # ghost states: reflective at r = 0 (flux weight r = 0 anyway) and at a
        # closed outer wall, copy when transmissive
        hl = np.concatenate(([self.h[0]], self.h))
        ul = np.concatenate(([-u[0]], u))
        hr = np.concatenate((self.h, [self.h[-1]]))
        ur = np.concatenate((u, [-u[-1] if self.outer == "wall" else u[-1]]))
        F = _hll_1d(hl, ul, hr, ur, g)  # at faces 0..n
        rF = F * self.re[None, :]
        src = 0.5 * g * self.h * self.h * self.dr
        self.h = self.h - dt * (rF[0, 1:] - rF[0, :-1]) / self.V
        self.q = self.q + dt * (-(rF[1, 1:] - rF[1, :-1]) + src) / self.V
        self.h = np.maximum(self.h, 0.0)
        self.t += dt

    def run(self, t_end: float) -> None:
        while self.t < t_end:
            self.step(t_end)

    def profile(self, r):
        """Depth at radii r (linear interpolation between cell centres)."""
        return np.interp(np.asarray(r, dtype=np.float64), self.rc, self.h)


def circular_reference(t_end: float = 3.5, radius: float = 2.5, h_in: float = 2.5, h_out: float = 0.5,
                       r_max: float = 40.0, n: int = 8192, g: float = G) -> Radial:
    """The circular dam-break benchmark centreline: the radial
    solver on [0, 40] m at 8192 cells (4096 over the [0, 20] m half-width the
    2D box spans; >= 4096 as SPEC.md:514 asks), transmissive far edge, run to
    t_end."""
    s = Radial(lambda r: np.where(r < radius, h_in, h_out), r_max, n, g)
    s.run(t_end)
    return s
