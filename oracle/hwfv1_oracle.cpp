// oracle/hwfv1_oracle.cpp — CPU-HWFV1 oracle. TEST INFRASTRUCTURE ONLY.
//
// A literal, readable restatement of /root/reference/SPEC.md (modules zorder,
// mra, traversal, swe, engine) and PAPER.md Algs. 1-5, Eqs. 2-4, plus the
// gap decisions D1-D16 of DESIGN.md. It is the parity checker for the sm_100a
// kernels and the timed CPU-HWFV1 baseline. Nothing in the product links it.
//
// Style: storage follows the spec literally — one flat HierarchyField per
// quantity in z-index order holding SCALE COEFFICIENTS s (physical value
// s * 2^(n-L)), a RecordedGrid of 4^L entries, a
// compacted LeafAssembly with materialised neighbour descriptors
// (SPEC.md:219-224). Parallelism is restricted to SPEC's execution contract
// (SPEC.md:444): writer-exclusive maps, exact min reductions, and a scan-based
// compaction, so results are bitwise independent of the worker count
// (A8).
//
// Floating point: compiled with -ffp-contract=off (no FMA, D2);
// every expression below is written in the exact association order pinned in
// DESIGN.md so the GPU kernels (compiled --fmad=false) can be compared bit for
// bit.
#include "oracle.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

namespace {

// ============================================================== zorder
// Restated with plain bit loops (independent of the product's dilated
// arithmetic). Reference: zorder.hpp:24-66, 69-131.
uint32_t o_interleave(uint32_t i, uint32_t j) {
    uint32_t m = 0;
    for (int b = 0; b < 14 && ((i | j) >> b) != 0u; ++b) {
        m |= ((i >> b) & 1u) << (2 * b);
        m |= ((j >> b) & 1u) << (2 * b + 1);
    }
    return m;
}
void o_deinterleave(uint32_t m, uint32_t* i, uint32_t* j) {
    uint32_t a = 0, c = 0;
    for (int b = 0; b < 14 && (m >> (2 * b)) != 0u; ++b) {
        a |= ((m >> (2 * b)) & 1u) << b;
        c |= ((m >> (2 * b + 1)) & 1u) << b;
    }
    *i = a;
    *j = c;
}
// level_offset as the running sum 1 + 4 + ... + 4^(n-1),
// tabulated once for n = 0..14 (the oracle calls it per cell and per leaf)
struct OffsetTable {
    uint32_t v[15];
    OffsetTable() {
        uint32_t s = 0, p = 1;
        for (int n = 0; n < 15; ++n) {
            v[n] = s;
            s += p;
            p *= 4u;
        }
    }
};
const OffsetTable kOffsets;
inline uint32_t o_offset(int n) { return kOffsets.v[n]; }
// level_of (zorder.hpp:83-87): the level whose z-range holds z
inline int o_level_of(uint32_t z) {
    int n = 0;
    while (n < 13 && kOffsets.v[n + 1] <= z) ++n;
    return n;
}
// same_level_neighbour: decode, shift, re-encode; false off-grid.
bool o_neighbour(int n, uint32_t m, int dir, uint32_t* out) {
    uint32_t i, j;
    o_deinterleave(m, &i, &j);
    const uint32_t side = 1u << n;
    switch (dir) {
        case 0: if (i == 0) return false; --i; break;          // West
        case 1: if (i + 1 >= side) return false; ++i; break;   // East
        case 2: if (j + 1 >= side) return false; ++j; break;   // North
        case 3: if (j == 0) return false; --j; break;          // South
        default: return false;
    }
    *out = o_interleave(i, j);
    return true;
}

// ============================================================== mra arithmetic
// D1: the Haar filters H0=H1=G0=1/sqrt2, G1=-1/sqrt2 applied
// twice (2-D) factor to 1/2; the factored form is used so constants are
// preserved exactly. Child order k = (j_bit<<1)|i_bit.
inline void encode4(double s0, double s1, double s2, double s3, double* s, double* da, double* db, double* dg) {
    *s = 0.5 * ((s0 + s1) + (s2 + s3));
    *da = 0.5 * ((s0 + s1) - (s2 + s3));
    *db = 0.5 * ((s0 + s2) - (s1 + s3));
    *dg = 0.5 * ((s0 + s3) - (s1 + s2));
}
inline void decode4(double s, double da, double db, double dg, double c[4]) {
    c[0] = 0.5 * ((s + da) + (db + dg));
    c[1] = 0.5 * ((s + da) - (db + dg));
    c[2] = 0.5 * ((s - da) + (db - dg));
    c[3] = 0.5 * ((s - da) - (db - dg));
}
inline double absd(double x) { return x < 0.0 ? -x : x; }
inline double max2(double a, double b) { return a > b ? a : b; }
// significance, D6/D7, literally: the normalised
// detail of one quantity is d_norm = max(|dα|,|dβ|,|dγ|) / s_max (a quantity
// with s_max < 1e-12 contributes d_norm = 0), a cell's d_norm is the max over
// h, qx, qy, and the cell is significant when d_norm >= 2^(n-L) eps.
// D8: the cell is near-threshold when |d_norm - thr| <= 1e-12 thr.
inline double dnorm(double da, double db, double dg, double smax) {
    if (smax < 1e-12) return 0.0;
    return max2(max2(absd(da), absd(db)), absd(dg)) / smax;
}
inline double sig_threshold(int n, int L, double eps) { return std::ldexp(eps, n - L); }
inline bool near_threshold(double dn, double thr) { return absd(dn - thr) <= 1e-12 * thr; }
inline bool significant(double da, double db, double dg, double smax, int n, int L, double eps) {
    return dnorm(da, db, dg, smax) >= sig_threshold(n, L, eps);
}

// ============================================================== swe physics
struct Phys {
    double g, hdry, nM;
};
// de-singularised velocity, pinned as q * (1/h): one reciprocal
// per cell serves both components (D2)
inline double vel(double h, double q, double hdry) { return (h >= hdry) ? q * (1.0 / h) : 0.0; }
// hydrostatic reconstruction of one side (D11): max(0, eta - zf),
// depths below h_dry are treated as exactly dry.
inline double recon(double h, double z, double zf, double hdry) {
    const double t = (h + z) - zf;
    double hs = (t > 0.0) ? t : 0.0;
    if (hs < hdry) hs = 0.0;
    return hs;
}
// HLL flux (D12) in the face-normal frame: (h, q_n, q_t).
void hll(double hL, double uL, double vL, double hR, double uR, double vR, double g, double F[3]) {
    if (hL == 0.0 && hR == 0.0) {
        F[0] = F[1] = F[2] = 0.0;
        return;
    }
    const double qL = hL * uL, qR = hR * uR;
    const double tL = hL * vL, tR = hR * vR;
    const double cL = std::sqrt(g * hL), cR = std::sqrt(g * hR);
    double SL, SR;
    if (hL == 0.0) {  // dry left
        SL = uR - 2.0 * cR;
        SR = uR + cR;
    } else if (hR == 0.0) {  // dry right
        SL = uL - cL;
        SR = uL + 2.0 * cL;
    } else {  // two-rarefaction estimates
        const double us = (0.5 * (uL + uR)) + (cL - cR);
        double cs = (0.5 * (cL + cR)) + (0.25 * (uL - uR));
        if (cs < 0.0) cs = 0.0;
        const double a = uL - cL, b = us - cs;
        SL = (a < b) ? a : b;
        const double c = uR + cR, d = us + cs;
        SR = (c > d) ? c : d;
    }
    const double hg = 0.5 * g;
    const double FL0 = qL, FL1 = (qL * uL) + (hg * (hL * hL)), FL2 = qL * vL;
    const double FR0 = qR, FR1 = (qR * uR) + (hg * (hR * hR)), FR2 = qR * vR;
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
// One face: left / right cells as (h, q_n, q_t, z) in the normal frame.
// Returns the HLL flux of the reconstructed pair and the reconstructed depths.
void face(const double Lc[4], const double Rc[4], const Phys& p, double F[3], double* hLs, double* hRs) {
    const double zf = (Lc[3] > Rc[3]) ? Lc[3] : Rc[3];
    *hLs = recon(Lc[0], Lc[3], zf, p.hdry);
    *hRs = recon(Rc[0], Rc[3], zf, p.hdry);
    const double uL = vel(Lc[0], Lc[1], p.hdry), vL = vel(Lc[0], Lc[2], p.hdry);
    const double uR = vel(Rc[0], Rc[1], p.hdry), vR = vel(Rc[0], Rc[2], p.hdry);
    hll(*hLs, uL, vL, *hRs, uR, vR, p.g, F);
}
// Deterministic inverse cube root (D2): bit-level seed + 4 division-free
// Newton steps y <- y + y(1 - h y^3)/3, IEEE ops only, so CPU and GPU agree
// bit for bit (libm cbrt and libdevice cbrt do not).
double rcbrt_det(double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    b = 0x553EF0FF289DD796ull - b / 3u;
    double y;
    std::memcpy(&y, &b, 8);
    const double third = 1.0 / 3.0;
    for (int it = 0; it < 4; ++it) {
        const double t = (x * y) * (y * y);
        y = y + ((y * (1.0 - t)) * third);
    }
    return y;
}
double cbrt_det(double x) { return 1.0 / rcbrt_det(x); }
// semi-implicit Manning friction on a wet post-Euler state:
// q /= 1 + dt * C_f * |q| / h^2 with C_f = g n^2 h^(-1/3) (|u| = |q|/h).
void friction(double h, double* qx, double* qy, double dt, const Phys& p) {
    const double qm = std::sqrt((*qx * *qx) + (*qy * *qy));
    if (qm > 0.0) {
        const double Cf = (p.g * (p.nM * p.nM)) * rcbrt_det(h);
        const double rh = 1.0 / h;
        const double den = 1.0 + (((dt * Cf) * qm) * (rh * rh));
        const double r = 1.0 / den;
        *qx = *qx * r;
        *qy = *qy * r;
    }
}
// CFL rate of one cell: (max(|u|,|v|) + sqrt(gh)) / dx,
// 0 when dry; dt = C / max rate (D13 pin: one reciprocal per cell, none per
// reduction element).
double cfl_cell(double h, double qx, double qy, double dx, double g, double hdry) {
    if (!(h >= hdry)) return 0.0;
    const double rh = 1.0 / h;
    const double aq = max2(absd(qx), absd(qy));
    const double s = (aq * rh) + std::sqrt(g * h);
    return s * (1.0 / dx);
}
// linear interpolation of the inflow series, last value held
double series_value(double t, const double* ts, const double* vs, int n) {
    if (n <= 0) return 0.0;
    if (t <= ts[0]) return vs[0];
    if (t >= ts[n - 1]) return vs[n - 1];
    int k = 0;
    while (k + 1 < n && ts[k + 1] <= t) ++k;
    return vs[k] + ((vs[k + 1] - vs[k]) * ((t - ts[k]) / (ts[k + 1] - ts[k])));
}
// boundary ghost state (D10). own = physical (h, qx, qy, z).
void boundary_state(const double own[4], int kind, int dir, double t, const double* ts, const double* vs, int n,
                    int mode, double hdry, double out[4]) {
    out[0] = own[0]; out[1] = own[1]; out[2] = own[2]; out[3] = own[3];
    const bool xface = (dir == 0 || dir == 1);
    if (kind == SWAMP_BC_REFLECTIVE) {
        if (xface) out[1] = -own[1]; else out[2] = -own[2];
    } else if (kind == SWAMP_BC_INFLOW) {
        const double v = series_value(t, ts, vs, n);
        double hg;
        if (mode == SWAMP_INFLOW_ETA) {
            const double d = v - own[3];
            hg = (d > 0.0) ? d : 0.0;
        } else {
            hg = v;
        }
        const double un = xface ? vel(own[0], own[1], hdry) : vel(own[0], own[2], hdry);
        out[0] = hg;
        if (xface) { out[1] = hg * un; out[2] = 0.0; }
        else { out[1] = 0.0; out[2] = hg * un; }
    }
}
// The FV1 leaf update (SPEC.md:313-321 + Eq. 2 + 322-330 + D11): own and the
// four W,E,N,S neighbour states are physical (h, qx, qy, z). Writes new
// (h, qx, qy). Returns false on a non-finite result.
bool fv1_cell(const double own[4], const double nb[4][4], double dx, double dt, const Phys& p, double out[3]) {
    const double idx = 1.0 / dx;
    const double h = own[0], qx = own[1], qy = own[2];
    const double hg = 0.5 * p.g;
    double FE[3], FW[3], GN[3], GS[3], hLs, hRs;
    {  // east face: own is the left cell, x-frame (h, qx, qy, z)
        const double Lc[4] = {own[0], own[1], own[2], own[3]};
        const double Rc[4] = {nb[1][0], nb[1][1], nb[1][2], nb[1][3]};
        face(Lc, Rc, p, FE, &hLs, &hRs);
        FE[1] = FE[1] + (hg * ((h * h) - (hLs * hLs)));
    }
    {  // west face: own is the right cell
        const double Lc[4] = {nb[0][0], nb[0][1], nb[0][2], nb[0][3]};
        const double Rc[4] = {own[0], own[1], own[2], own[3]};
        face(Lc, Rc, p, FW, &hLs, &hRs);
        FW[1] = FW[1] + (hg * ((h * h) - (hRs * hRs)));
    }
    {  // north face: own is the left (south) cell, y-frame (h, qy, qx, z)
        const double Lc[4] = {own[0], own[2], own[1], own[3]};
        const double Rc[4] = {nb[2][0], nb[2][2], nb[2][1], nb[2][3]};
        face(Lc, Rc, p, GN, &hLs, &hRs);
        GN[1] = GN[1] + (hg * ((h * h) - (hLs * hLs)));
    }
    {  // south face: own is the right (north) cell
        const double Lc[4] = {nb[3][0], nb[3][2], nb[3][1], nb[3][3]};
        const double Rc[4] = {own[0], own[2], own[1], own[3]};
        face(Lc, Rc, p, GS, &hLs, &hRs);
        GS[1] = GS[1] + (hg * ((h * h) - (hRs * hRs)));
    }
    // spatial operator L_c: -(F_e - F_w)/dx - (G_n - G_s)/dx,
    // with 1/dx formed once (D2 pin)
    const double Lh = (-((FE[0] - FW[0]) * idx)) - ((GN[0] - GS[0]) * idx);
    const double Lqx = (-((FE[1] - FW[1]) * idx)) - ((GN[2] - GS[2]) * idx);
    const double Lqy = (-((FE[2] - FW[2]) * idx)) - ((GN[1] - GS[1]) * idx);
    // forward Euler (Eq. 2)
    double hn = h + (dt * Lh);
    double qxn = qx + (dt * Lqx);
    double qyn = qy + (dt * Lqy);
    if (hn < 0.0) hn = 0.0;  // D11 positivity clamp
    if (hn < p.hdry) {       // dry: q = 0
        qxn = 0.0;
        qyn = 0.0;
    } else if (p.nM > 0.0) {
        friction(hn, &qxn, &qyn, dt, p);
    }
    out[0] = hn;
    out[1] = qxn;
    out[2] = qyn;
    return std::isfinite(hn) && std::isfinite(qxn) && std::isfinite(qyn);
}

constexpr uint32_t kBoundaryBase = SWAMP_BOUNDARY_BASE;

}  // namespace

// ====================================================================== engine state
struct oracle_state {
    swamp_config cfg;
    std::vector<double> inflow_t, inflow_v, out_times;
    int L = 0;
    bool uniform = false;
    std::vector<double> s[4];                  // HierarchyField per quantity (h, qx, qy, z), s-units
    std::vector<uint8_t> sig, sig_prev, dem;   // over detail cells (levels 0..L-1)
    std::vector<uint8_t> ina;                  // over all cells: every finest descendant inactive (D16)
    bool has_ina = false;
    std::vector<double> det[3][3];             // DetailField (dα,dβ,dγ) of h, qx, qy
    double smax[4] = {0, 0, 0, 0};
    std::vector<uint32_t> recorded;            // RecordedGrid
    std::vector<uint32_t> leaves, nbr[4];      // LeafAssembly
    double t = 0.0, dt = 0.0, t_next = 0.0;
    int64_t step = 0;
    int64_t cnt_tree = 0, cnt_new = 0;
    // near-threshold cells (D8): of the last step's re-encode (cells on the
    // previous tree), summed over steps, initialise's flow / DEM evaluations
    int64_t near_last = 0, cnt_near = 0, near_init = 0, near_dem = 0;
    std::string err;
};

namespace {

inline uint32_t Z(int n, uint32_t m) { return o_offset(n) + m; }
// phys = s 2^(n-L), exact; the powers of two are tabulated
// (2^-13 .. 2^13) and multiplied, which equals ldexp bit for bit (no
// overflow / subnormals here)
struct Pow2Table {
    double v[27];
    Pow2Table() {
        for (int k = -13; k <= 13; ++k) v[k + 13] = std::ldexp(1.0, k);
    }
};
const Pow2Table kPow2;
inline double to_phys(double s, int n, int L) { return s * kPow2.v[n - L + 13]; }
inline double from_phys(double p, int n, int L) { return p * kPow2.v[L - n + 13]; }

// significance pipeline after (re)encoding: flow | DEM -> band -> closure
// (D3, D5). `evaluated` marks the cells whose
// details were (re)computed (the previous tree; null = every cell): the
// near-threshold count (D8) is over those; the others have zero details.
int64_t flag_tree(oracle_state& S, const uint8_t* evaluated) {
    const int L = S.L;
    const double eps = S.cfg.epsilon;
    const size_t nd = o_offset(L);
    std::vector<uint8_t> pre(nd, 0);
    int64_t nnear = 0;
#pragma omp parallel for schedule(static) reduction(+ : nnear)
    for (int64_t zi = 0; zi < (int64_t)nd; ++zi) {
        const int n = o_level_of((uint32_t)zi);
        double dq[3];
        for (int q = 0; q < 3; ++q) dq[q] = dnorm(S.det[q][0][zi], S.det[q][1][zi], S.det[q][2][zi], S.smax[q]);
        const double dn = max2(max2(dq[0], dq[1]), dq[2]);
        const double thr = sig_threshold(n, L, eps);
        if ((!evaluated || evaluated[zi]) && near_threshold(dn, thr)) ++nnear;
        pre[zi] = (dn >= thr || S.dem[zi]) ? 1 : 0;
    }
    std::vector<uint8_t> band(pre);
    const int mode = S.cfg.band_mode;
    if (mode == SWAMP_BAND_NEIGHBOURS || mode == SWAMP_BAND_PARENTS) {
        // scatter form of SPEC.md:195, evaluated as a gather so each output
        // cell has one writer
        for (int n = 0; n < L; ++n) {
            const uint32_t cnt = 1u << (2 * n);
            if (mode == SWAMP_BAND_NEIGHBOURS) {
#pragma omp parallel for schedule(static)
                for (int64_t m = 0; m < (int64_t)cnt; ++m) {
                    uint8_t b = pre[Z(n, (uint32_t)m)];
                    for (int d = 0; d < 4; ++d) {
                        uint32_t nb;
                        if (o_neighbour(n, (uint32_t)m, d, &nb)) b |= pre[Z(n, nb)];
                    }
                    band[Z(n, (uint32_t)m)] = b;
                }
            } else if (n + 1 < L) {
                // cell (n, p) is marked when a level-(n+1) significant cell has
                // a same-level neighbour among p's children
#pragma omp parallel for schedule(static)
                for (int64_t p = 0; p < (int64_t)cnt; ++p) {
                    uint8_t b = pre[Z(n, (uint32_t)p)];
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t c = 4u * (uint32_t)p + (uint32_t)k;
                        for (int d = 0; d < 4; ++d) {
                            uint32_t nb;
                            if (o_neighbour(n + 1, c, d, &nb)) b |= pre[Z(n + 1, nb)];
                        }
                    }
                    band[Z(n, (uint32_t)p)] = b;
                }
            }
        }
    }
    // ancestor closure, levels L-1 -> 0
    S.sig = band;
    for (int n = L - 2; n >= 0; --n) {
        const uint32_t cnt = 1u << (2 * n);
#pragma omp parallel for schedule(static)
        for (int64_t m = 0; m < (int64_t)cnt; ++m) {
            uint8_t v = S.sig[Z(n, (uint32_t)m)];
            for (int k = 0; k < 4; ++k) v |= S.sig[Z(n + 1, 4u * (uint32_t)m + (uint32_t)k)];
            S.sig[Z(n, (uint32_t)m)] = v ? 1 : 0;
        }
    }
    return nnear;
}

// zero_details_and_reencode: for levels L-1 -> 0, cells on
// the previous tree recompute s and details from their 4 children; details
// elsewhere are zero. `all` = full bottom-up encode (initialise, Alg. 1).
void reencode(oracle_state& S, bool all, bool with_z) {
    const int L = S.L;
    const int nq = with_z ? 4 : 3;
    int64_t tree = 0;
    for (int n = L - 1; n >= 0; --n) {
        const uint32_t cnt = 1u << (2 * n);
#pragma omp parallel for schedule(static) reduction(+ : tree)
        for (int64_t m = 0; m < (int64_t)cnt; ++m) {
            const uint32_t zi = Z(n, (uint32_t)m);
            const bool on = all || S.sig_prev[zi];
            const uint32_t c0 = Z(n + 1, 4u * (uint32_t)m);
            for (int q = 0; q < nq; ++q) {
                double s = 0, da = 0, db = 0, dg = 0;
                if (on) {
                    const std::vector<double>& v = S.s[q];
                    encode4(v[c0], v[c0 + 1], v[c0 + 2], v[c0 + 3], &s, &da, &db, &dg);
                    S.s[q][zi] = s;
                }
                if (q < 3) {
                    S.det[q][0][zi] = da;
                    S.det[q][1][zi] = db;
                    S.det[q][2][zi] = dg;
                }
            }
            if (on) ++tree;
        }
    }
    S.cnt_tree = tree;
}

// decode_tree under D4: levels 0 -> L-1; a significant cell
// that was not on the previous tree writes its 4 children with Eqs. 4a-d and
// zero details (its details are zero after the restricted re-encode).
void decode_new(oracle_state& S) {
    const int L = S.L;
    int64_t nnew = 0;
    for (int n = 0; n < L; ++n) {
        const uint32_t cnt = 1u << (2 * n);
#pragma omp parallel for schedule(static) reduction(+ : nnew)
        for (int64_t m = 0; m < (int64_t)cnt; ++m) {
            const uint32_t zi = Z(n, (uint32_t)m);
            if (!(S.sig[zi] && !S.sig_prev[zi])) continue;
            ++nnew;
            const uint32_t c0 = Z(n + 1, 4u * (uint32_t)m);
            for (int q = 0; q < 3; ++q) {
                double c[4];
                decode4(S.s[q][zi], 0.0, 0.0, 0.0, c);
                for (int k = 0; k < 4; ++k) S.s[q][c0 + k] = c[k];
            }
        }
    }
    S.cnt_new = nnew;
}

// parallel_tree_traversal (Alg. 5)
void ptt(int L, const uint8_t* sig, uint32_t* recorded) {
    const int64_t N = int64_t(1) << (2 * L);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < N; ++m) {
        int n = 0;
        uint32_t c = 0;
        while (n < L && sig[Z(n, c)]) {
            c = 4u * c + (((uint32_t)m >> (2 * (L - n - 1))) & 3u);
            ++n;
        }
        recorded[m] = Z(n, c);
    }
}

// compact_leaves: keep run-first entries; scan-based.
int64_t compact(const uint32_t* rec, int64_t N, uint32_t* out) {
    const int nt = omp_get_max_threads();
    std::vector<int64_t> cnt(nt + 1, 0);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const int T = omp_get_num_threads();
        const int64_t a = N * t / T, b = N * (t + 1) / T;
        int64_t c = 0;
        for (int64_t m = a; m < b; ++m) c += (m == 0 || rec[m] != rec[m - 1]);
        cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
        for (int k = 1; k <= T; ++k) cnt[k] += cnt[k - 1];
        if (out) {
            int64_t o = cnt[t];
            for (int64_t m = a; m < b; ++m)
                if (m == 0 || rec[m] != rec[m - 1]) out[o++] = rec[m];
        }
    }
    return cnt[nt];
}

// find_neighbours
bool neighbours(int L, const uint32_t* rec, const uint32_t* leaves, int64_t N, const int32_t bc[4],
                uint32_t* nbr4 /* [4][N] */) {
    bool ok = true;
#pragma omp parallel for schedule(static) reduction(&& : ok)
    for (int64_t i = 0; i < N; ++i) {
        const uint32_t zl = leaves[i];
        const int n = o_level_of(zl);
        const uint32_t m = zl - o_offset(n);
        for (int d = 0; d < 4; ++d) {
            uint32_t nb;
            uint32_t desc;
            if (!o_neighbour(n, m, d, &nb)) {
                desc = kBoundaryBase + (uint32_t)bc[d];
            } else {
                const uint32_t r = rec[(uint64_t)nb << (2 * (L - n))];
                const int lr = o_level_of(r);
                // the recorded entry must be a leaf covering that finest cell
                const uint32_t mr = r - o_offset(lr);
                if (lr > L || (mr >> 0) >= (1u << (2 * lr))) ok = false;
                desc = (lr >= n) ? Z(n, nb) : r;
            }
            nbr4[(int64_t)d * N + i] = desc;
        }
    }
    return ok;
}

void rebuild_grid(oracle_state& S) {
    const int L = S.L;
    const int64_t NF = int64_t(1) << (2 * L);
    S.recorded.assign(NF, 0);
    ptt(L, S.sig.data(), S.recorded.data());
    const int64_t N = compact(S.recorded.data(), NF, nullptr);
    S.leaves.assign(N, 0);
    compact(S.recorded.data(), NF, S.leaves.data());
    for (int d = 0; d < 4; ++d) S.nbr[d].assign(N, 0);
    std::vector<uint32_t> tmp(4 * N);
    if (!neighbours(L, S.recorded.data(), S.leaves.data(), N, S.cfg.bc, tmp.data()))
        S.err = "find_neighbours: malformed recorded grid";
    for (int d = 0; d < 4; ++d) std::memcpy(S.nbr[d].data(), tmp.data() + d * N, N * sizeof(uint32_t));
}

// physical state (h, qx, qy, z) of hierarchy cell z-index zi
inline void cell_phys(const oracle_state& S, uint32_t zi, double out[4]) {
    const int n = o_level_of(zi);
    for (int q = 0; q < 4; ++q) out[q] = to_phys(S.s[q][zi], n, S.L);
}

// first output time strictly after t, or t_end (D13)
double next_stop(const oracle_state& S, double t) {
    double ts = S.cfg.t_end;
    for (double o : S.out_times)
        if (o > t && o < ts) ts = o;
    return ts;
}

// cfl_timestep: C * min over wet leaves, fallback when all
// dry, clipped to the next output time / t_end. Sets dt and t_next.
bool set_dt(oracle_state& S, double maxrate) {
    double dtc = (maxrate == 0.0) ? S.cfg.dt_fallback : S.cfg.cfl / maxrate;
    const double stop = next_stop(S, S.t);
    if (S.t + dtc >= stop) {
        S.dt = stop - S.t;
        S.t_next = stop;
    } else {
        S.dt = dtc;
        S.t_next = S.t + dtc;
    }
    if (S.t < S.cfg.t_end && !(S.dt > 0.0 && std::isfinite(S.dt))) {
        S.err = "cfl_timestep: dt <= 0 or non-finite";
        return false;
    }
    return true;
}

double leaves_max_rate(const oracle_state& S) {
    const int64_t N = (int64_t)S.leaves.size();
    double mn = 0.0;
#pragma omp parallel for schedule(static) reduction(max : mn)
    for (int64_t i = 0; i < N; ++i) {
        if (S.has_ina && S.ina[S.leaves[i]]) continue;  // D16
        double u[4];
        cell_phys(S, S.leaves[i], u);
        const int n = o_level_of(S.leaves[i]);
        const double v = cfl_cell(u[0], u[1], u[2], std::ldexp(S.cfg.width, -n), S.cfg.g, S.cfg.h_dry);
        mn = v > mn ? v : mn;
    }
    return mn;
}

// FV1 over the leaf assembly, writer-exclusive into U_new, then the write-back
// (from_physical into each leaf's own slot; D15 semantics: all
// updates read the pre-update state).
bool fv1_all(oracle_state& S, double* maxrate) {
    const int64_t N = (int64_t)S.leaves.size();
    const int L = S.L;
    const Phys p{S.cfg.g, S.cfg.h_dry, S.cfg.manning};
    std::vector<double> U(3 * N);
    double mn = 0.0;
    bool ok = true;
    const double dt = S.dt, t = S.t;
#pragma omp parallel for schedule(static) reduction(max : mn) reduction(&& : ok)
    for (int64_t i = 0; i < N; ++i) {
        const uint32_t zl = S.leaves[i];
        const int n = o_level_of(zl);
        double own[4], nb[4][4];
        cell_phys(S, zl, own);
        const double dx = std::ldexp(S.cfg.width, -n);
        double out[3];
        if (S.has_ina && S.ina[zl]) {  // D16: an inactive leaf keeps its state, no CFL
            U[3 * i + 0] = own[0];
            U[3 * i + 1] = own[1];
            U[3 * i + 2] = own[2];
            continue;
        }
        for (int d = 0; d < 4; ++d) {
            const uint32_t desc = S.nbr[d][i];
            if (desc >= kBoundaryBase)
                boundary_state(own, (int)(desc - kBoundaryBase), d, t, S.inflow_t.data(), S.inflow_v.data(),
                               (int)S.inflow_t.size(), S.cfg.inflow_mode, p.hdry, nb[d]);
            else if (S.has_ina && S.ina[desc])  // D16: an inactive neighbour is a reflective wall
                boundary_state(own, SWAMP_BC_REFLECTIVE, d, t, nullptr, nullptr, 0, S.cfg.inflow_mode, p.hdry, nb[d]);
            else
                cell_phys(S, desc, nb[d]);
        }
        if (!fv1_cell(own, nb, dx, dt, p, out)) ok = false;
        U[3 * i + 0] = out[0];
        U[3 * i + 1] = out[1];
        U[3 * i + 2] = out[2];
        const double c = cfl_cell(out[0], out[1], out[2], dx, p.g, p.hdry);
        mn = c > mn ? c : mn;
    }
    if (!ok) {
        S.err = "spatial_operator: non-finite state";
        return false;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        const uint32_t zl = S.leaves[i];
        const int n = o_level_of(zl);
        for (int q = 0; q < 3; ++q) S.s[q][zl] = from_phys(U[3 * i + q], n, L);
    }
    *maxrate = mn;
    return true;
}

}  // namespace

// =========================================================================== C ABI
extern "C" {

int oracle_set_threads(int n) {
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
}

static int create_impl(const swamp_config* cfg, const double* h, const double* qx, const double* qy, const double* z,
                       bool uniform, oracle_state** out) {
    if (!cfg || !out || cfg->L < 1 || cfg->L > 13 || !(cfg->epsilon >= 0.0) || !(cfg->width > 0.0)) return SWAMP_E_ARG;
    auto* S = new oracle_state();
    S->cfg = *cfg;
    S->uniform = uniform;
    if (cfg->inflow_n > 0) {
        S->inflow_t.assign(cfg->inflow_t, cfg->inflow_t + cfg->inflow_n);
        S->inflow_v.assign(cfg->inflow_v, cfg->inflow_v + cfg->inflow_n);
    }
    if (cfg->n_outputs > 0) S->out_times.assign(cfg->output_times, cfg->output_times + cfg->n_outputs);
    S->cfg.inflow_t = S->cfg.inflow_v = S->cfg.output_times = nullptr;
    const int L = cfg->L;
    S->L = L;
    const size_t NH = o_offset(L + 1), ND = o_offset(L);
    const uint32_t side = 1u << L;
    for (int q = 0; q < 4; ++q) S->s[q].assign(NH, 0.0);
    for (int q = 0; q < 3; ++q)
        for (int k = 0; k < 3; ++k) S->det[q][k].assign(ND, 0.0);
    S->sig.assign(ND, 0);
    S->sig_prev.assign(ND, 1);
    S->dem.assign(ND, 0);
    // initial discretisation at level L (from_physical at L = identity)
    const double* src[4] = {h, qx, qy, z};
    for (uint32_t j = 0; j < side; ++j)
        for (uint32_t i = 0; i < side; ++i) {
            const uint32_t zi = Z(L, o_interleave(i, j));
            for (int q = 0; q < 4; ++q) S->s[q][zi] = src[q][(size_t)j * side + i];
        }
    // D16: inactive finest cells; a cell is inactive when every finest
    // descendant is, "mixed" when some but not all are
    std::vector<uint8_t> any;
    if (cfg->inactive) {
        S->has_ina = true;
        S->ina.assign(NH, 0);
        any.assign(NH, 0);
        for (uint32_t j = 0; j < side; ++j)
            for (uint32_t i = 0; i < side; ++i) {
                const uint32_t zi = Z(L, o_interleave(i, j));
                S->ina[zi] = any[zi] = cfg->inactive[(size_t)j * side + i] ? 1 : 0;
            }
        for (int n = L - 1; n >= 0; --n)
            for (uint32_t m = 0; m < (1u << (2 * n)); ++m) {
                const uint32_t zi = Z(n, m), c0 = Z(n + 1, 4u * m);
                S->ina[zi] = S->ina[c0] & S->ina[c0 + 1] & S->ina[c0 + 2] & S->ina[c0 + 3];
                any[zi] = any[c0] | any[c0 + 1] | any[c0 + 2] | any[c0 + 3];
            }
    }
    // s_max per quantity from |s^(L)| over the active cells
    for (int q = 0; q < 4; ++q) {
        double mx = 0.0;
        for (uint32_t m = 0; m < side * side; ++m)
            if (!S->has_ina || !S->ina[Z(L, m)]) mx = max2(mx, absd(S->s[q][Z(L, m)]));
        S->smax[q] = mx;
    }
    for (int q = 0; q < 4; ++q)
        for (uint32_t m = 0; m < side * side; ++m)
            if (!std::isfinite(S->s[q][Z(L, m)])) {
                delete S;
                return SWAMP_E_NONFINITE;
            }
    S->t = 0.0;
    S->step = 0;
    if (uniform) {
        // uniform 2^L x 2^L FV1: the full tree, no MRA
        std::fill(S->sig.begin(), S->sig.end(), 1);
        rebuild_grid(*S);
    } else {
        // full bottom-up encode of every level (Alg. 1), z included once
        reencode(*S, /*all=*/true, /*with_z=*/true);
        // preprocess_dem: static mask from z's MRA
        {
            std::vector<double> dz[3];
            for (int k = 0; k < 3; ++k) dz[k].assign(ND, 0.0);
            for (int n = L - 1; n >= 0; --n)
                for (uint32_t m = 0; m < (1u << (2 * n)); ++m) {
                    const uint32_t zi = Z(n, m), c0 = Z(n + 1, 4u * m);
                    double s, a, b, g;
                    encode4(S->s[3][c0], S->s[3][c0 + 1], S->s[3][c0 + 2], S->s[3][c0 + 3], &s, &a, &b, &g);
                    const double dn = dnorm(a, b, g, S->smax[3]), thr = sig_threshold(n, L, cfg->epsilon);
                    S->dem[zi] = dn >= thr ? 1 : 0;
                    if (near_threshold(dn, thr)) ++S->near_dem;
                    // D16: mixed active / inactive cells are always refined, so
                    // every leaf is wholly active or wholly inactive
                    if (S->has_ina && any[zi] && !S->ina[zi]) S->dem[zi] = 1;
                }
        }
        S->near_init = flag_tree(*S, nullptr);
        // nothing is newly significant at t=0 (sig_prev = all): no decode
        rebuild_grid(*S);
    }
    if (!S->err.empty()) {
        delete S;
        return SWAMP_E_STATE;
    }
    if (!set_dt(*S, leaves_max_rate(*S))) {
        delete S;
        return SWAMP_E_DT;
    }
    *out = S;
    return SWAMP_OK;
}

int oracle_create(const swamp_config* cfg, const double* h, const double* qx, const double* qy, const double* z,
                  oracle_state** out) {
    return create_impl(cfg, h, qx, qy, z, false, out);
}

// uniform-solver handle: same create, full tree, no MRA
int oracle_create_uniform(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                          const double* z, oracle_state** out) {
    return create_impl(cfg, h, qx, qy, z, true, out);
}

int oracle_destroy(oracle_state* s) {
    delete s;
    return SWAMP_OK;
}

// step_adaptive
int oracle_step(oracle_state* S) {
    if (!S) return SWAMP_E_ARG;
    if (S->uniform) return oracle_step_uniform(S);
    if (!(S->t < S->cfg.t_end)) return SWAMP_OK;
    S->sig_prev = S->sig;
    reencode(*S, false, false);   // zero_details_and_reencode
    S->near_last = flag_tree(*S, S->sig_prev.data());  // significance | DEM | band, closure
    S->cnt_near += S->near_last;
    decode_new(*S);               // decode_tree (D4)
    rebuild_grid(*S);             // PTT, compaction, neighbours
    if (!S->err.empty()) return SWAMP_E_STATE;
    double mn;
    if (!fv1_all(*S, &mn)) return SWAMP_E_NONFINITE;  // FV1 + friction + write-back
    S->t = S->t_next;             // t += dt (exactly the clipped stop time when clipped)
    S->step += 1;
    if (!set_dt(*S, mn)) return SWAMP_E_DT;
    return SWAMP_OK;
}

// step_uniform: same flux/source path on every finest cell.
int oracle_step_uniform(oracle_state* S) {
    if (!S) return SWAMP_E_ARG;
    if (!(S->t < S->cfg.t_end)) return SWAMP_OK;
    double mn;
    if (!fv1_all(*S, &mn)) return SWAMP_E_NONFINITE;
    S->t = S->t_next;
    S->step += 1;
    if (!set_dt(*S, mn)) return SWAMP_E_DT;
    return SWAMP_OK;
}

int oracle_info(const oracle_state* S, double* t, double* dt, int64_t* step, int64_t* n_leaves) {
    if (!S) return SWAMP_E_ARG;
    if (t) *t = S->t;
    if (dt) *dt = S->dt;
    if (step) *step = S->step;
    if (n_leaves) *n_leaves = (int64_t)S->leaves.size();
    return SWAMP_OK;
}

int oracle_copy_leaves(const oracle_state* S, uint32_t* leaves, uint32_t* w, uint32_t* e, uint32_t* n, uint32_t* so,
                       int64_t cap, int64_t* count) {
    if (!S) return SWAMP_E_ARG;
    const int64_t N = (int64_t)S->leaves.size();
    if (count) *count = N;
    if (cap < N) return (leaves || w || e || n || so) ? SWAMP_E_ARG : SWAMP_OK;
    if (leaves) std::memcpy(leaves, S->leaves.data(), N * 4);
    uint32_t* outs[4] = {w, e, n, so};
    for (int d = 0; d < 4; ++d)
        if (outs[d]) std::memcpy(outs[d], S->nbr[d].data(), N * 4);
    return SWAMP_OK;
}

int oracle_export_tree(const oracle_state* S, double* h, double* qx, double* qy, double* z, uint8_t* sig) {
    if (!S) return SWAMP_E_ARG;
    double* outs[4] = {h, qx, qy, z};
    for (int q = 0; q < 4; ++q)
        if (outs[q]) std::memcpy(outs[q], S->s[q].data(), S->s[q].size() * 8);
    if (sig) std::memcpy(sig, S->sig.data(), S->sig.size());
    return SWAMP_OK;
}

// zero-detail expansion to the finest grid
int oracle_export_finest(const oracle_state* S, double* h, double* qx, double* qy) {
    if (!S) return SWAMP_E_ARG;
    const int L = S->L;
    const uint32_t side = 1u << L;
    double* outs[3] = {h, qx, qy};
    for (uint32_t j = 0; j < side; ++j)
        for (uint32_t i = 0; i < side; ++i) {
            const uint32_t r = S->recorded[o_interleave(i, j)];
            const int n = o_level_of(r);
            for (int q = 0; q < 3; ++q)
                if (outs[q]) outs[q][(size_t)j * side + i] = to_phys(S->s[q][r], n, L);
        }
    return SWAMP_OK;
}

int oracle_counters(const oracle_state* S, int64_t* out4) {
    if (!S || !out4) return SWAMP_E_ARG;
    out4[0] = (int64_t)S->leaves.size();
    out4[1] = S->cnt_tree;
    out4[2] = S->cnt_new;
    out4[3] = int64_t(1) << (2 * S->L);
    return SWAMP_OK;
}

int oracle_near_threshold(const oracle_state* S, int64_t* out4) {
    if (!S || !out4) return SWAMP_E_ARG;
    out4[0] = S->near_last;
    out4[1] = S->cnt_near;
    out4[2] = S->near_init;
    out4[3] = S->near_dem;
    return SWAMP_OK;
}

const char* oracle_last_error(const oracle_state* S) { return S ? S->err.c_str() : "null state"; }

int oracle_import_tree(oracle_state* S, const double* h, const double* qx, const double* qy, const uint8_t* sig,
                       double t, double dt, double t_next, int64_t step) {
    if (!S) return SWAMP_E_ARG;
    const double* src[3] = {h, qx, qy};
    for (int q = 0; q < 3; ++q) std::memcpy(S->s[q].data(), src[q], S->s[q].size() * 8);
    std::memcpy(S->sig.data(), sig, S->sig.size());
    S->t = t;
    S->dt = dt;
    S->t_next = t_next;
    S->step = step;
    rebuild_grid(*S);
    return S->err.empty() ? SWAMP_OK : SWAMP_E_STATE;
}

// ------------------------------------------------------------- per-op KATs
uint32_t oracle_morton_encode(uint32_t i, uint32_t j) { return o_interleave(i, j); }
void oracle_morton_decode(uint32_t m, uint32_t* i, uint32_t* j) { o_deinterleave(m, i, j); }
int64_t oracle_neighbour(int n, uint32_t m, int dir) {
    uint32_t nb;
    return o_neighbour(n, m, dir, &nb) ? (int64_t)nb : -1;
}
void oracle_encode4(const double c[4], double out[4]) { encode4(c[0], c[1], c[2], c[3], &out[0], &out[1], &out[2], &out[3]); }
void oracle_decode4(const double in[4], double c[4]) { decode4(in[0], in[1], in[2], in[3], c); }
int oracle_significance(const double d[3], double smax, int n, int L, double eps) {
    return significant(d[0], d[1], d[2], smax, n, L, eps) ? 1 : 0;
}
void oracle_hll(double hL, double uL, double vL, double hR, double uR, double vR, double g, double F[3]) {
    hll(hL, uL, vL, hR, uR, vR, g, F);
}
void oracle_face(const double Lc[4], const double Rc[4], double g, double hdry, double F[3], double hs[2]) {
    const Phys p{g, hdry, 0.0};
    face(Lc, Rc, p, F, &hs[0], &hs[1]);
}
void oracle_fv1_cell(const double own[4], const double nb[16], double dx, double dt, double g, double hdry, double nM,
                     double out[3]) {
    const Phys p{g, hdry, nM};
    double n4[4][4];
    for (int d = 0; d < 4; ++d)
        for (int q = 0; q < 4; ++q) n4[d][q] = nb[4 * d + q];
    fv1_cell(own, n4, dx, dt, p, out);
}
void oracle_friction(double h, double qx, double qy, double dt, double g, double nM, double hdry, double out[2]) {
    const Phys p{g, hdry, nM};
    if (h >= hdry && nM > 0.0) friction(h, &qx, &qy, dt, p);
    out[0] = qx;
    out[1] = qy;
}
double oracle_cfl_cell(double h, double qx, double qy, double dx, double g, double hdry) {
    return cfl_cell(h, qx, qy, dx, g, hdry);
}
double oracle_cbrt(double x) { return cbrt_det(x); }
void oracle_boundary(const double own[4], int kind, int dir, double t, const double* ts, const double* vs, int n,
                     int mode, double hdry, double out[4]) {
    boundary_state(own, kind, dir, t, ts, vs, n, mode, hdry, out);
}
void oracle_ptt(int L, const uint8_t* sig, uint32_t* recorded) { ptt(L, sig, recorded); }
int64_t oracle_compact(const uint32_t* recorded, int64_t n, uint32_t* leaves) { return compact(recorded, n, leaves); }
int oracle_neighbours(int L, const uint32_t* recorded, const uint32_t* leaves, int64_t N, const int32_t bc[4],
                      uint32_t* nbr4) {
    return neighbours(L, recorded, leaves, N, bc, nbr4) ? SWAMP_OK : SWAMP_E_STATE;
}
// recursive depth-first traversal (Alg. 2's identification rule)
static void dft(int L, const uint8_t* sig, int n, uint32_t m, std::vector<uint32_t>& out) {
    if (n < L && sig[Z(n, m)]) {
        for (uint32_t k = 0; k < 4; ++k) dft(L, sig, n + 1, 4u * m + k, out);
    } else {
        out.push_back(Z(n, m));
    }
}
int64_t oracle_dft_leaves(int L, const uint8_t* sig, uint32_t* leaves) {
    std::vector<uint32_t> out;
    dft(L, sig, 0, 0, out);
    if (leaves) std::memcpy(leaves, out.data(), out.size() * 4);
    return (int64_t)out.size();
}

}  // extern "C"
