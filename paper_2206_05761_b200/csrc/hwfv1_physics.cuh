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

// de-singularised velocity
__device__ __forceinline__ double vel(double h, double q, double hdry) { return (h >= hdry) ? q / h : 0.0; }

// hydrostatic reconstruction of one side: max(0, (h+z)-zf), below h_dry -> 0
__device__ __forceinline__ double recon(double h, double z, double zf, double hdry) {
    const double t = (h + z) - zf;
    double hs = (t > 0.0) ? t : 0.0;
    if (hs < hdry) hs = 0.0;
    return hs;
}

// HLL flux in the face-normal frame (h, q_n, q_t); identical expression
// order to oracle/hwfv1_oracle.cpp hll().
__device__ __forceinline__ void hll(double hL, double uL, double vL, double hR, double uR, double vR,
                                    const PhysParams& p, double F[3]) {
    if (hL == 0.0 && hR == 0.0) {
        F[0] = 0.0; F[1] = 0.0; F[2] = 0.0;
        return;
    }
    const double qL = hL * uL, qR = hR * uR;
    const double tL = hL * vL, tR = hR * vR;
    const double cL = sqrt(p.g * hL), cR = sqrt(p.g * hR);
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

// One face, cells given in the normal frame as (h, q_n, q_t, z).
__device__ __forceinline__ void face(double Lh, double Ln, double Lt, double Lz, double Rh, double Rn, double Rt,
                                     double Rz, const PhysParams& p, double F[3], double& hLs, double& hRs) {
    const double zf = (Lz > Rz) ? Lz : Rz;
    hLs = recon(Lh, Lz, zf, p.hdry);
    hRs = recon(Rh, Rz, zf, p.hdry);
    const double uL = vel(Lh, Ln, p.hdry), vL = vel(Lh, Lt, p.hdry);
    const double uR = vel(Rh, Rn, p.hdry), vR = vel(Rh, Rt, p.hdry);
    hll(hLs, uL, vL, hRs, uR, vR, p, F);
}

// Deterministic cube root (D2): same bit-level seed and Newton
// iterations as the oracle, IEEE ops only.
__device__ __forceinline__ double cbrt_det(double x) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    b = b / 3ull + 0x2A9F7893782DA1CEull;
    double y = __longlong_as_double(static_cast<long long>(b));
#pragma unroll
    for (int it = 0; it < 5; ++it) y = ((2.0 * y) + (x / (y * y))) / 3.0;
    return y;
}

// CFL bound of one cell; +inf when dry.
__device__ __forceinline__ double cfl_cell(double h, double qx, double qy, double dx, const PhysParams& p) {
    if (!(h >= p.hdry)) return __longlong_as_double(0x7FF0000000000000ll);
    const double au = absd(qx / h), av = absd(qy / h);
    const double s = ((au > av) ? au : av) + sqrt(p.g * h);
    return dx / s;
}

// Boundary ghost state; own = physical (h, qx, qy, z); dir W=0,E=1,N=2,S=3.
__device__ __forceinline__ double4 boundary_state(double4 own, int kind, int dir, double inflow_value, int mode,
                                                  double hdry) {
    double4 o = own;
    const bool xface = (dir == 0 || dir == 1);
    if (kind == 0) {  // reflective
        if (xface) o.y = -own.y; else o.z = -own.z;
    } else if (kind == 2) {  // inflow
        double hg;
        if (mode == 1) {
            const double d = inflow_value - own.w;
            hg = (d > 0.0) ? d : 0.0;
        } else {
            hg = inflow_value;
        }
        const double un = xface ? vel(own.x, own.y, hdry) : vel(own.x, own.z, hdry);
        o.x = hg;
        if (xface) { o.y = hg * un; o.z = 0.0; }
        else { o.y = 0.0; o.z = hg * un; }
    }
    return o;
}

// FV1 leaf update (spatial operator + Euler + clamp + friction). nb[d] are
// the W, E, N, S neighbour states (physical). Returns (h, qx, qy).
__device__ __forceinline__ void fv1_cell(const double4 own, const double4 nb[4], double dx, double dt,
                                         const PhysParams& p, double& hn, double& qxn, double& qyn) {
    const double h = own.x, qx = own.y, qy = own.z;
    double FE[3], FW[3], GN[3], GS[3], hLs, hRs;
    // east face: own is left, x-frame (h, qx, qy, z)
    face(own.x, own.y, own.z, own.w, nb[1].x, nb[1].y, nb[1].z, nb[1].w, p, FE, hLs, hRs);
    FE[1] = FE[1] + (p.half_g * ((h * h) - (hLs * hLs)));
    // west face: own is right
    face(nb[0].x, nb[0].y, nb[0].z, nb[0].w, own.x, own.y, own.z, own.w, p, FW, hLs, hRs);
    FW[1] = FW[1] + (p.half_g * ((h * h) - (hRs * hRs)));
    // north face: own is left (south cell), y-frame (h, qy, qx, z)
    face(own.x, own.z, own.y, own.w, nb[2].x, nb[2].z, nb[2].y, nb[2].w, p, GN, hLs, hRs);
    GN[1] = GN[1] + (p.half_g * ((h * h) - (hLs * hLs)));
    // south face: own is right
    face(nb[3].x, nb[3].z, nb[3].y, nb[3].w, own.x, own.z, own.y, own.w, p, GS, hLs, hRs);
    GS[1] = GS[1] + (p.half_g * ((h * h) - (hRs * hRs)));

    const double Lh = (-((FE[0] - FW[0]) / dx)) - ((GN[0] - GS[0]) / dx);
    const double Lqx = (-((FE[1] - FW[1]) / dx)) - ((GN[2] - GS[2]) / dx);
    const double Lqy = (-((FE[2] - FW[2]) / dx)) - ((GN[1] - GS[1]) / dx);

    hn = h + (dt * Lh);
    qxn = qx + (dt * Lqx);
    qyn = qy + (dt * Lqy);
    if (hn < 0.0) hn = 0.0;
    if (hn < p.hdry) {
        qxn = 0.0;
        qyn = 0.0;
    } else if (p.nM > 0.0) {
        const double u = qxn / hn, v = qyn / hn;
        const double sp = sqrt((u * u) + (v * v));
        if (sp > 0.0) {
            const double Cf = p.g_nM2 / cbrt_det(hn);
            const double den = 1.0 + (((dt * Cf) * sp) / hn);
            qxn = qxn / den;
            qyn = qyn / den;
        }
    }
}

}  // namespace hwfv1
