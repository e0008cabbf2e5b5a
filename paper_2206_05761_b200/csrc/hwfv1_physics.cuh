// hwfv1_physics.cuh — per-cell / per-face arithmetic of the HWFV1 step on
// sm_100a: Haar encode (Eqs. 3a-d),
// significance, hydrostatic reconstruction,
// HLL, the spatial operator + forward Euler (SPEC.md:313-321,
// Eq. 2), Manning friction, CFL and the
// boundary ghost states.
//
// Numerics contract (D1, D2, D7, D11, D12): every expression is
// written in the association order pinned in DESIGN.md, the translation unit
// is compiled with --fmad=false, and only IEEE-correctly-rounded operations
// (+ - * / sqrt) are used, so results are bit-identical to the CPU oracle.
// The hierarchy is stored in PHYSICAL units (cell averages) instead of the
// spec's scale coefficients s = p * 2^(L-n); the two differ by exact powers of
// two, so every comparison and every stored bit maps one-to-one.
#pragma once
#include <cstdint>

namespace hwfv1 {

struct PhysParams {
    double g, half_g, hdry, nM, g_nM2;
};

__device__ __forceinline__ double absd(double x) { return x < 0.0 ? -x : x; }
__device__ __forceinline__ double max2(double a, double b) { return a > b ? a : b; }

// de-singularised velocity, pinned as q * (1/h) (D2)
__device__ __forceinline__ double vel(double h, double q, double hdry) { return (h >= hdry) ? q * (1.0 / h) : 0.0; }

// hydrostatic reconstruction of one side: max(0, (h+z)-zf), below h_dry -> 0
__device__ __forceinline__ double recon(double h, double z, double zf, double hdry) {
    const double t = (h + z) - zf;
    double hs = (t > 0.0) ? t : 0.0;
    if (hs < hdry) hs = 0.0;
    return hs;
}

// A cell as seen by a face: depth, bed, and its velocities / celerity formed
// once per cell (the per-face recomputation in the oracle gives the same bits:
// vel() and sqrt() of identical inputs).
struct CellV {
    double h, qx, qy, z;  // physical state
    double ux, uy;        // vel(h, qx), vel(h, qy)
    double c;             // sqrt(g h)
};
__device__ __forceinline__ CellV make_cell(double4 s, const PhysParams& p) {
    CellV c;
    c.h = s.x; c.qx = s.y; c.qy = s.z; c.z = s.w;
    c.ux = 0.0;
    c.uy = 0.0;
    c.c = 0.0;  // only read when the reconstructed depth equals a wet h (face())
    if (s.x >= p.hdry) {  // dry cells need no reciprocal / square root
        const double rh = 1.0 / s.x;  // one reciprocal serves both components
        c.ux = s.y * rh;
        c.uy = s.z * rh;
        c.c = sqrt(p.g * s.x);
    }
    return c;
}

// HLL flux in the face-normal frame (h, q_n, q_t); identical expression
// order to oracle/hwfv1_oracle.cpp hll(). cLc / cRc are sqrt(g h) of the
// cells, reused when the reconstructed depth equals the cell depth.
__device__ __forceinline__ void hll(double hL, double uL, double vL, double hR, double uR, double vR, double cL,
                                    double cR, const PhysParams& p, double F[3]) {
    if (hL == 0.0 && hR == 0.0) {
        F[0] = 0.0; F[1] = 0.0; F[2] = 0.0;
        return;
    }
    const double qL = hL * uL, qR = hR * uR;
    const double tL = hL * vL, tR = hR * vR;
    double SL, SR;
    if (hL == 0.0) {
        SL = uR - 2.0 * cR;
        SR = uR + cR;
    } else if (hR == 0.0) {
        SL = uL - cL;
        SR = uL + 2.0 * cL;
    } else {
        const double us = (0.5 * (uL + uR)) + (cL - cR);
        double cs = (0.5 * (cL + cR)) + (0.25 * (uL - uR));
        if (cs < 0.0) cs = 0.0;
        const double a = uL - cL, b = us - cs;
        SL = (a < b) ? a : b;
        const double c = uR + cR, d = us + cs;
        SR = (c > d) ? c : d;
    }
    const double FL0 = qL, FL1 = (qL * uL) + (p.half_g * (hL * hL)), FL2 = qL * vL;
    const double FR0 = qR, FR1 = (qR * uR) + (p.half_g * (hR * hR)), FR2 = qR * vR;
    if (SL >= 0.0) {
        F[0] = FL0; F[1] = FL1; F[2] = FL2;
    } else if (SR <= 0.0) {
        F[0] = FR0; F[1] = FR1; F[2] = FR2;
    } else {
        const double inv = 1.0 / (SR - SL);
        const double sls = SL * SR;
        F[0] = (((SR * FL0) - (SL * FR0)) + (sls * (hR - hL))) * inv;
        F[1] = (((SR * FL1) - (SL * FR1)) + (sls * (qR - qL))) * inv;
        F[2] = (((SR * FL2) - (SL * FR2)) + (sls * (tR - tL))) * inv;
    }
}

// One face between left cell L and right cell R; xface selects the normal
// (x: normal qx / tangential qy; y: normal qy / tangential qx). Returns the
// flux and the reconstructed depths.
__device__ __forceinline__ void face(const CellV& L, const CellV& R, bool xface, const PhysParams& p, double F[3],
                                     double& hLs, double& hRs) {
    const double zf = (L.z > R.z) ? L.z : R.z;
    hLs = recon(L.h, L.z, zf, p.hdry);
    hRs = recon(R.h, R.z, zf, p.hdry);
    if (hLs == 0.0 && hRs == 0.0) {
        F[0] = 0.0; F[1] = 0.0; F[2] = 0.0;
        return;
    }
    // sqrt(g h*) (= the cell's c when the reconstruction kept its depth; a
    // reconstructed depth is 0 or >= h_dry, so a dry cell's c is never read)
    const double cL = (hLs == 0.0) ? 0.0 : ((hLs == L.h) ? L.c : sqrt(p.g * hLs));
    const double cR = (hRs == 0.0) ? 0.0 : ((hRs == R.h) ? R.c : sqrt(p.g * hRs));
    if (xface) hll(hLs, L.ux, L.uy, hRs, R.ux, R.uy, cL, cR, p, F);
    else hll(hLs, L.uy, L.ux, hRs, R.uy, R.ux, cL, cR, p, F);
}

// Deterministic inverse cube root (D2): same bit-level seed and
// division-free Newton steps as the oracle, IEEE ops only.
__device__ __forceinline__ double rcbrt_det(double x) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    b = 0x553EF0FF289DD796ull - b / 3ull;
    double y = __longlong_as_double(static_cast<long long>(b));
    const double third = 1.0 / 3.0;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        const double t = (x * y) * (y * y);
        y = y + ((y * (1.0 - t)) * third);
    }
    return y;
}

// CFL rate of one cell, (max(|u|,|v|) + sqrt(gh)) / dx, 0 when dry; the
// step's dt is C / (max rate) (D13).
__device__ __forceinline__ double cfl_rate(double h, double qx, double qy, double inv_dx, const PhysParams& p) {
    if (!(h >= p.hdry)) return 0.0;
    const double rh = 1.0 / h;
    const double aq = max2(absd(qx), absd(qy));
    const double s = (aq * rh) + sqrt(p.g * h);
    return s * inv_dx;
}

// Boundary ghost state (D10); dir W=0,E=1,N=2,S=3. The
// ghost's velocities follow exactly from the interior's (negation and copy
// are exact); an inflow ghost gets fresh ones.
__device__ __forceinline__ CellV boundary_cell(const CellV& own, int kind, int dir, double inflow_value, int mode,
                                               const PhysParams& p) {
    CellV o = own;
    const bool xface = (dir == 0 || dir == 1);
    if (kind == 0) {  // reflective: negate the normal discharge
        // vel(h, -q): -(q/h) when wet (exact), +0 when dry (as the oracle)
        if (xface) { o.qx = -own.qx; o.ux = (own.h >= p.hdry) ? -own.ux : 0.0; }
        else { o.qy = -own.qy; o.uy = (own.h >= p.hdry) ? -own.uy : 0.0; }
    } else if (kind == 2) {  // inflow
        double hg;
        if (mode == 1) {
            const double d = inflow_value - own.z;
            hg = (d > 0.0) ? d : 0.0;
        } else {
            hg = inflow_value;
        }
        const double un = xface ? own.ux : own.uy;
        double4 g4;
        g4.x = hg;
        g4.w = own.z;
        if (xface) { g4.y = hg * un; g4.z = 0.0; }
        else { g4.y = 0.0; g4.z = hg * un; }
        o = make_cell(g4, p);
    }
    return o;
}

// FV1 leaf update (spatial operator + Euler + clamp + friction); nb = W, E,
// N, S neighbour cells. Returns (h, qx, qy). Same pinned expressions as
// oracle fv1_cell().
__device__ __forceinline__ void fv1_cell(const CellV& own, const CellV nb[4], double idx, double dt,
                                         const PhysParams& p, double& hn, double& qxn, double& qyn) {
    const double h = own.h;
    const double hh = h * h;
    double FE[3], FW[3], GN[3], GS[3], hLs, hRs;
    face(own, nb[1], true, p, FE, hLs, hRs);
    FE[1] = FE[1] + (p.half_g * (hh - (hLs * hLs)));
    face(nb[0], own, true, p, FW, hLs, hRs);
    FW[1] = FW[1] + (p.half_g * (hh - (hRs * hRs)));
    face(own, nb[2], false, p, GN, hLs, hRs);
    GN[1] = GN[1] + (p.half_g * (hh - (hLs * hLs)));
    face(nb[3], own, false, p, GS, hLs, hRs);
    GS[1] = GS[1] + (p.half_g * (hh - (hRs * hRs)));

    const double Lh = (-((FE[0] - FW[0]) * idx)) - ((GN[0] - GS[0]) * idx);
    const double Lqx = (-((FE[1] - FW[1]) * idx)) - ((GN[2] - GS[2]) * idx);
    const double Lqy = (-((FE[2] - FW[2]) * idx)) - ((GN[1] - GS[1]) * idx);

    hn = h + (dt * Lh);
    qxn = own.qx + (dt * Lqx);
    qyn = own.qy + (dt * Lqy);
    if (hn < 0.0) hn = 0.0;
    if (hn < p.hdry) {
        qxn = 0.0;
        qyn = 0.0;
    } else if (p.nM > 0.0) {
        const double qm = sqrt((qxn * qxn) + (qyn * qyn));
        if (qm > 0.0) {
            const double Cf = p.g_nM2 * rcbrt_det(hn);
            const double rh = 1.0 / hn;
            const double den = 1.0 + (((dt * Cf) * qm) * (rh * rh));
            const double r = 1.0 / den;
            qxn = qxn * r;
            qyn = qyn * r;
        }
    }
}

// L_c from the face-flux differences, forward Euler, clamp, friction (the
// tail of fv1_cell; shared by the per-leaf and the strip path of k_fv1)
// rh_out: 1 / hn when hn >= h_dry (friction's reciprocal, reused by the CFL
// rate of the same state: cfl_rate_rh), else 0
__device__ __forceinline__ void fv1_finish(const CellV& own, double dFx0, double dFx1, double dFx2, double dGy0,
                                           double dGy1, double dGy2, double idx, double dt, const PhysParams& p,
                                           double& hn, double& qxn, double& qyn, double& rh_out) {
    const double Lh = (-(dFx0 * idx)) - (dGy0 * idx);
    const double Lqx = (-(dFx1 * idx)) - (dGy2 * idx);
    const double Lqy = (-(dFx2 * idx)) - (dGy1 * idx);
    hn = own.h + (dt * Lh);
    qxn = own.qx + (dt * Lqx);
    qyn = own.qy + (dt * Lqy);
    if (hn < 0.0) hn = 0.0;
    rh_out = 0.0;
    if (hn < p.hdry) {
        qxn = 0.0;
        qyn = 0.0;
    } else {
        const double rh = 1.0 / hn;
        rh_out = rh;
        if (p.nM > 0.0) {
            const double qm = sqrt((qxn * qxn) + (qyn * qyn));
            if (qm > 0.0) {
                const double Cf = p.g_nM2 * rcbrt_det(hn);
                const double den = 1.0 + (((dt * Cf) * qm) * (rh * rh));
                const double r = 1.0 / den;
                qxn = qxn * r;
                qyn = qyn * r;
            }
        }
    }
}
__device__ __forceinline__ void fv1_finish(const CellV& own, double dFx0, double dFx1, double dFx2, double dGy0,
                                           double dGy1, double dGy2, double idx, double dt, const PhysParams& p,
                                           double& hn, double& qxn, double& qyn) {
    double rh;
    fv1_finish(own, dFx0, dFx1, dFx2, dGy0, dGy1, dGy2, idx, dt, p, hn, qxn, qyn, rh);
}
// cfl_rate with the state's reciprocal depth already formed (rh = 1 / h when
// h >= h_dry): the same bits as cfl_rate
__device__ __forceinline__ double cfl_rate_rh(double h, double qx, double qy, double rh, double inv_dx,
                                              const PhysParams& p) {
    if (!(h >= p.hdry)) return 0.0;
    const double aq = max2(absd(qx), absd(qy));
    const double s = (aq * rh) + sqrt(p.g * h);
    return s * inv_dx;
}

// Same update as fv1_cell, with the neighbours produced one face at a time
// by `get(d)` so only one neighbour is live (register pressure / occupancy).
template <class GetNb>
__device__ __forceinline__ void fv1_cell_seq(const CellV& own, GetNb&& get, double idx, double dt,
                                             const PhysParams& p, double& hn, double& qxn, double& qyn, double& rh) {
    const double h = own.h;
    const double hh = h * h;
    double hLs, hRs, F[3];
    double dFx0, dFx1, dFx2, dGy0, dGy1, dGy2;
    {
        const CellV e = get(1);
        face(own, e, true, p, F, hLs, hRs);
        const double FE0 = F[0], FE1 = F[1] + (p.half_g * (hh - (hLs * hLs))), FE2 = F[2];
        const CellV w = get(0);
        face(w, own, true, p, F, hLs, hRs);
        const double FW1 = F[1] + (p.half_g * (hh - (hRs * hRs)));
        dFx0 = FE0 - F[0];
        dFx1 = FE1 - FW1;
        dFx2 = FE2 - F[2];
    }
    {
        const CellV nn = get(2);
        face(own, nn, false, p, F, hLs, hRs);
        const double GN0 = F[0], GN1 = F[1] + (p.half_g * (hh - (hLs * hLs))), GN2 = F[2];
        const CellV ss = get(3);
        face(ss, own, false, p, F, hLs, hRs);
        const double GS1 = F[1] + (p.half_g * (hh - (hRs * hRs)));
        dGy0 = GN0 - F[0];
        dGy1 = GN1 - GS1;
        dGy2 = GN2 - F[2];
    }
    fv1_finish(own, dFx0, dFx1, dFx2, dGy0, dGy1, dGy2, idx, dt, p, hn, qxn, qyn, rh);
}

}  // namespace hwfv1
