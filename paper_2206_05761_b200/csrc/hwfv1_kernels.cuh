// hwfv1_kernels.cuh — the sm_100a kernels of one adaptive HWFV1 time step
// (Alg. 3):
//
//   K1 k_encode    zero_details_and_reencode + significance (+ DEM mask at t=0)
//                  level-fused over a level-R subtree per CTA, 4 lanes per
//                  parent at the finest level (warp shuffles), shared memory
//                  above; the last CTA finishes levels < R.
//   K2 k_band      safety band + ancestor closure per subtree, leaf count per
//                  subtree; the last CTA closes levels < R and scans the
//                  per-subtree leaf counts into output offsets.
//   K3 k_traverse  decode (projection of newly significant cells, D4) +
//                  parallel tree traversal (Alg. 5) + stream compaction.
//   K5 k_fv1       neighbour finding by Morton arithmetic + flag walk, FV1
//                  (HLL, hydrostatic reconstruction, friction), write-back,
//                  CFL min; the last CTA advances t and computes the next dt.
//
// Storage: the hierarchy is an array of double4 cells
// {h, qx, qy, z} in PHYSICAL units, one Morton-ordered slice per level with
// every level base 256-B aligned; two copies ping-pong (D15). Significance is
// one byte per detail cell and per level, two copies ping-pong (previous /
// current tree). All control state (t, dt, parity, leaf count, error word)
// lives on the device so a step is a fixed kernel sequence (CUDA-graph
// capturable); every kernel is a no-op once t >= t_end.
#pragma once
#include <cstddef>
#include <cstdint>

#include "hwfv1_physics.cuh"
#include "swamp/zorder.hpp"

namespace hwfv1 {

namespace zo = swamp::zorder;

constexpr int kThreads = 256;
constexpr int kMaxL = 13;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kNoSrc = 0xFFFFFFFFu;
constexpr int kMaxParts = 8;

enum Stage : int { kStageImport = 0, kStageEncode = 1, kStageBand = 2, kStageTraverse = 3, kStageFV1 = 5, kStageDt = 6 };
enum ErrCode : int { kErrNone = 0, kErrNonFinite = -3, kErrDt = -4, kErrBarrier = -7 };
enum : int { kStageBarrier = 7 };

struct Ctl {
    // ---- line 0: read once per CTA (cta_head) by every kernel of a step
    double t;        // current simulation time
    double dt;       // dt of the next step
    double t_next;   // time after the next step (exact stop time when clipped)
    double dt_used;  // dt of the last step taken
    long long step;
    int parity;                     // current cell buffer / previous-tree flags
    uint32_t n_leaves;              // leaves of the grid built by the last K2/K3
    uint32_t n_leaves_A;            // of which level-L leaves (listed first, in sibling quadruples)
    uint32_t a_lo, a_hi, b_lo, b_hi; // this partition's slices of the A (level-L) and B lists
    uint32_t n_leaves_used;         // leaves the last FV1 updated
    // quiet lists (Params::qsplit): the leaves of subtrees whose neighbourhood
    // is dry, after the active ones of each list: level-L quads at
    // [qa_lo, qa_lo + qa_n), coarser leaves at [qb_lo, qb_lo + qb_n)
    uint32_t qa_lo, qa_n, qb_lo, qb_n;
    // ---- atomically updated fields, each on its own 128-B line so that the
    //      per-CTA atomics do not queue in front of the line-0 reads
    alignas(128) unsigned long long rate_bits[2];  // CFL max-rate accumulators (bits of a non-negative double), by step parity
    unsigned int done_k1, done_k5;
    alignas(128) unsigned long long cnt_tree;    // cells re-encoded by K1 and the top-level encodes (cumulative)
    unsigned long long cnt_fused;                // level-(L-1) cells re-encoded by FV1 (cumulative)
    unsigned long long cnt_quiet;                // leaves FV1 updated by the dry-subtree shortcut (cumulative)
    unsigned long long cnt_tiled;                // leaves FV1 updated on its tile path (cumulative)
    unsigned long long cnt_skip;                 // leaves of stable quiet subtrees FV1 skipped (cumulative, in cnt_quiet)
    unsigned long long cnt_k1skip;               // re-encoded cells K1 skipped in stable quiet subtrees (cumulative, in cnt_tree)
    alignas(128) unsigned long long cnt_new;     // newly significant cells decoded by the last K3
    unsigned long long cnt_updates;              // leaf updates of all steps so far (sum of N)
    alignas(128) unsigned long long k3_ready;    // K3's top CTA published its results (epoch)
    alignas(128) unsigned int k2_done;           // fused K2+K3: subtree CTAs whose band / closure / counts are out
    alignas(128) unsigned int fv1_tail;          // FV1 (STAGE 5): dynamic tail chunks taken this step
    unsigned int fv1_tjob;                       // FV1 tile path: strip jobs taken this step
    uint32_t n_stile;                            // subtrees on FV1's tile path this step (K3's top)
    alignas(128) unsigned long long smax_bits[4];
    int err_code;
    uint32_t err_z;
    int err_q;
    int err_stage;
    // near-threshold cells (D8; copied into the host mirror with
    // this line): of the last completed step, and summed over all steps
    unsigned long long near_last;
    unsigned long long cnt_near;
    // per-step accumulators by step parity (K1, K2's top CTA, the previous
    // FV1's fused level-(L-1) re-encode), initialise's flow / z counts
    alignas(128) unsigned long long near_step[2];
    unsigned long long near_init, near_dem;
    alignas(128) unsigned long long bar_seq;     // cross-partition barriers passed (k_part_barrier; peers read it)
    alignas(128) unsigned long long dbg[64];     // per-phase globaltimer stamps of probe CTAs (diagnostics)
    // stage timeline (globaltimer ns), double-buffered by step parity, one
    // line per kernel k (K1, K2, K3, K5): [0] = ~(first CTA start), [2] = last
    // CTA done (atomicMax); K5 zeroes the next buffer
    alignas(128) unsigned long long tl[2][4][16];
    // last member: the step whose state the host mirror holds (written into
    // the mapped host mirror only, after the rest of the struct)
    alignas(128) unsigned long long rep_seq;
};

// Programmatic dependent launch: every kernel of the step is launched with
// programmatic stream serialisation; it lets its successor be scheduled as
// soon as all of its CTAs are running (pdl_trigger) and waits for its
// predecessor's completion + memory flush before touching any state
// (pdl_wait). Hides the launch gap behind the last-CTA tails.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// diagnostics: phase stamps of the first and last CTA of a kernel into
// dbg[base + 8 * (last) + k] (k = 7: entry)
struct Probe {
    Ctl* c;
    int slot;
    __device__ __forceinline__ Probe(Ctl* ctl, int base) : c(ctl), slot(-1) {
        if (blockIdx.x == 0) slot = base;
        else if (blockIdx.x == gridDim.x - 1) slot = base + 8;
    }
    __device__ __forceinline__ void operator()(int k, unsigned long long t = 0) const {
        if (slot >= 0 && threadIdx.x == 0) c->dbg[slot + k] = t ? t : gtimer();
    }
};

__device__ __forceinline__ void tl_start(Ctl* c, int buf, int k) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicMax(&c->tl[buf][k][0], ~gtimer());
}
__device__ __forceinline__ void tl_end(Ctl* c, int buf, int k) {
    if (threadIdx.x == 0) atomicMax(&c->tl[buf][k][2], gtimer());
}

struct Params {
    int L, R, K, n_tiles;
    int band_mode;
    int bc[4];
    int inflow_mode, inflow_n, n_out;
    double W, cfl, t_end, dt_fallback;
    double tau[kMaxL + 1];    // e_n = eps 2^(2n-2L+2); 0 >= tau[n]: significance of a zero-detail cell (eps == 0)
    double lvl[kMaxL + 1][4]; // significance table per level {lo, hi, tol, e_n} (sig_class; D7, D8)
    double dx[kMaxL + 1];     // W * 2^-n
    double inv_dx[kMaxL + 1]; // 1.0 / dx[n] (IEEE division, as the oracle)
    // device table: s_max per quantity [0..3], 1 / s_max [4..7] (0 when s_max <
    // 1e-12; screening only), filled on the device after the import
    // (k_smax_table), so the step graphs can be built before it completes
    const double* __restrict__ smx;
    PhysParams phys;
    const double* inflow_t;
    const double* inflow_v;
    const double* out_times;
    unsigned long long base[kMaxL + 2];   // double4 offset of level n
    unsigned long long fbase[kMaxL + 1];  // flag byte offset of level n
    double4* cells[2];
    uint8_t* sig[2];
    uint8_t* pre;
    uint8_t* dem;
    uint32_t* leaves;     // hot-path leaf list: level-L leaves, then the coarser ones
    uint32_t* leaves_x;   // Morton-ordered leaf list for exports
    uint32_t* tile_cnt;
    uint32_t* tile_off;
    uint32_t* tile_lvl;   // traversal depth of each subtree (R = reached) | kEmit
    uint32_t* tile_src;   // decode source of a reached subtree root, or kNoSrc
    // hot-path K3: the top's results for subtree t as four self-tagged words
    // (epoch << 32 | A offset, B offset, depth, decode source), 32 B per
    // subtree: each subtree CTA polls only its own record (4 per line)
    unsigned long long* k3_rec;
    // FV1 dry shortcut (one partition): wet[b][t] = some leaf of subtree t
    // ended the step with h >= h_dry (b = step parity); tact[t] bit 0 =
    // subtree t or a face-adjacent one is wet, or t touches an inflow edge
    uint8_t* wet[2];
    uint8_t* tact;
    // quadrant wet marks (qact = 1: one partition, split K3): qwet[b][4 t + q]
    // = a leaf of quadrant q (the level-(R+1) cell, Morton child q) of subtree
    // t ended the step wet. The dry-shortcut activity of a subtree with a
    // refined root then asks only whether the two quadrants of each neighbour
    // that face it hold wet cells (a leaf's flux neighbour across the edge
    // lies in one of them, or is a leaf covering it); a subtree whose root is
    // not refined asks whether its neighbours hold any
    uint8_t* qwet[2];
    int qact;
    // quiet split (one partition, split K3, no inactive cells): K3's top
    // places the leaves of reached subtrees whose neighbourhood is dry after
    // the active ones in lists A and B (Ctl::qa_*, qb_*); FV1 updates them
    // in a lean pass (a quad per thread, no gathers, no shuffles)
    int qsplit;
    // stable-quiet skip (qskip = 1, with qsplit): per subtree, K2 flags a tree
    // change (tchg: its final flags differ from the previous tree's), K3's top
    // keeps qstate = consecutive steps quiet, reached and unchanged (<= 3).
    // With qstate >= 2 the subtree's leaves, level-(L-1) parents and pre
    // flags in the buffer FV1 writes already hold what FV1 would write (they
    // are FV1's output of two steps ago, and the quiet update is idempotent
    // on dry leaves): FV1 skips the subtree and the next K1 skips its
    // re-encode (its values in that buffer are K1's of two steps ago, from
    // the same children). The counts they would add (near-threshold cells,
    // re-encodes) are cached per subtree: qnk1 = K1's {near, tree}, qnfv =
    // the quiet pass's near count. DESIGN.md §8.
    int qskip;
    uint8_t* tchg;
    uint8_t* qstate;
    uint32_t* qnk1;
    uint32_t* qnfv;
    // inactive cells (D16), levels 0..L at slo(n): bit 0 = every finest
    // descendant inactive, bit 1 = some are; static, every partition holds
    // the whole array
    uint8_t* ina;
    int has_ina;
    // FV1 tile path (one partition, K = 6, no inactive cells): active fully
    // refined subtrees, listed by K3's top in stile[0 .. ctl->n_stile)
    int tiles;
    uint32_t* stile;
    Ctl* ctl_mirror;      // one partition: the host's pinned Ctl mirror (UVA), written at the step's end
    Ctl* rep_ring;        // one partition, advance_reports' graphs: pinned ring of step reports (slot = step & mask)
    uint32_t rep_ring_mask;
    uint32_t fv1_tail16;  // FV1 STAGE 5: sixteenths of the grid-stride windows taken dynamically at the end
    // FV1 STAGE 3, short leaf lists: 4 (or 2) lanes per leaf, one face (pair)
    // each, when 4 (2) lanes per leaf fit fv1_fp_cap16 / 16 of the grid's
    // threads (0: off)
    uint32_t fv1_fp_cap16;
    // Morton-subtree partitions: this partition owns level-R
    // subtrees [tile_lo, tile_hi); cells on levels >= R belong to their
    // subtree's partition, cells above R are replicated except that a leaf's
    // value is current only in the partition of its first subtree. pcells /
    // psig / ppre / ptile_cnt / pctl are every partition's arrays (peer
    // pointers across GPUs; index 0 = self when G = 1).
    int G, part;
    int top_mode;         // levels < R after t = 0: 0 none (R = 0), 1 extra CTA of K2, 2 k_encode_top
    int top_band;         // top_mode 1, one partition: K2's extra CTA also bands the top cells (K3 skips it)
    uint32_t tile_lo, tile_hi, tiles_per_part;  // this partition's subtrees [tile_lo, tile_hi), their count
    uint32_t pbound[kMaxParts + 1];             // partition g owns [pbound[g], pbound[g + 1]) (rebalanced)
    uint32_t pb_align;                          // largest of 16 / 4 / 1 dividing every boundary
    double4* pcells[kMaxParts][2];
    uint8_t* psig[kMaxParts][2];
    uint8_t* ppre[kMaxParts];
    uint8_t* pdem[kMaxParts];   // (repartitioning only)
    uint8_t* pwet[kMaxParts][2];
    uint32_t* ptile_cnt[kMaxParts];
    Ctl* pctl[kMaxParts];
};

// offset of level k in a padded flag layout (every level 16-B aligned): the
// global flag arrays (== Params::fbase, host-checked) and the per-tile
// shared-memory slices (k = n - R) use the same one,
// every level 16-B aligned: 0, 16, 32, 48, 112, 368, 1392, ... ; slo(K) = size
__host__ __device__ __forceinline__ uint32_t slo(int k) {
    return k < 3 ? 16u * static_cast<uint32_t>(k) : 27u + (0x55555555u >> (32 - 2 * k));  // 48 + (4^k - 64) / 3
}

// double4 offset of level n in a cell buffer: every level slice rounded up
// to 8 cells (256 B): 0, 8, 16, 32, 96, 352, ... (host-checked == Params::base)
__host__ __device__ __forceinline__ unsigned long long cbase(int n) {
    return n < 2 ? 8ull * static_cast<unsigned>(n) : 11ull + (0x55555555u >> (32 - 2 * n));  // 16 + (4^n - 16) / 3
}
// 1 / dx_n = 2^n / W exactly: the exponent of 1/W plus n (host-checked == Params::inv_dx)
__device__ __forceinline__ double inv_dx_of(const Params& P, int n) {
    return __longlong_as_double(__double_as_longlong(P.inv_dx[0]) + (static_cast<long long>(n) << 52));
}

// ------------------------------------------------------------------ memory ops
__device__ __forceinline__ double4 ld4(const double4* p) {
    double4 v;
    asm("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ double4 ld4_nc(const double4* p) {
    double4 v;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ double4 ld4_cg(const double4* p) {
    double4 v;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st4(double4* p, double4 v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}
__device__ __forceinline__ uint8_t ldcg_u8(const uint8_t* p) {
    unsigned short v;
    asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return static_cast<uint8_t>(v);
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ldcg_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t lo(int n, int R) { return ((1u << (2 * (n - R))) - 1u) / 3u; }

// partition owning cell (n, m): the one holding its (first) level-R subtree
// partition owning cell (n, m): the owner of its (first) level-R subtree,
// from the subtree boundaries (host twin: swamp_partition_owner)
__host__ __device__ __forceinline__ int owner_in(const uint32_t* pbound, int G, int R, int n, uint32_t m) {
    if (G == 1) return 0;
    const uint32_t t = (n >= R) ? (m >> (2 * (n - R))) : (m << (2 * (R - n)));
    int g = 0;
    while (g + 1 < G && t >= pbound[g + 1]) ++g;
    return g;
}
__device__ __forceinline__ int owner_of(const Params& P, int n, uint32_t m) { return owner_in(P.pbound, P.G, P.R, n, m); }
__device__ __forceinline__ double4* cell_ptr(const Params& P, int buf, int n, uint32_t m) {
    return P.pcells[owner_of(P, n, m)][buf] + cbase(n) + m;
}
// significance byte of (n, m) in copy `which`; levels above R are replicated
__device__ __forceinline__ uint8_t sig_at(const Params& P, int which, int n, uint32_t m) {
    const int g = (n < P.R) ? P.part : owner_of(P, n, m);
    return P.psig[g][which][slo(n) + m];
}

__device__ __forceinline__ void report_error(Ctl* c, int code, uint32_t z, int q, int stage) {
    if (atomicCAS(&c->err_code, 0, code) == 0) {
        c->err_z = z;
        c->err_q = q;
        c->err_stage = stage;
    }
}

// ------------------------------------------------------ encode helpers (Eqs. 3)
struct Red {
    double par, dmax;
};
// parent = 0.25*((c0+c1)+(c2+c3)) and max |detail| of 4 children, physical units
__device__ __forceinline__ Red red4(double c0, double c1, double c2, double c3) {
    const double a = c0 + c1, b = c2 + c3;
    const double par = 0.25 * (a + b);
    const double da = a - b;
    const double db = (c0 + c2) - (c1 + c3);
    const double dg = (c0 + c3) - (c1 + c2);
    return {par, max2(max2(absd(da), absd(db)), absd(dg))};
}
// Significance (D6, D7), SPEC's division
// form: d_norm = max over h, qx, qy of max|d_q| / s_max_q (a quantity with
// s_max < 1e-12 contributes 0) is compared with eps 2^(n-L) (>=). In
// physical units (D = 2^(n+2-L) d on the same 4 children, exact powers of
// two) that is fl(max|D_q| / s_max_q) >= e_n = eps 2^(2n-2L+2), the same
// rounding. A cell is near-threshold (north star: counted and reported)
// when |d_norm - e_n| <= 1e-12 e_n. The per-level table T = {lo, hi, tol,
// e_n}: an approximate d_norm (one multiply by 1 / s_max per quantity,
// within a few ulps) below lo = e_n (1 - 1e-11) is certainly neither
// significant nor near, above hi = e_n (1 + 1e-11) certainly significant
// and not near; only inside that window are the IEEE divisions formed, so
// the flags and counts equal the literal division form bit for bit.
// Returns bit 0 = significant, bit 1 = near-threshold.
__device__ __forceinline__ unsigned sig_exact(double dh, double dqx, double dqy, double e, double tol, double s0,
                                           double s1, double s2) {
    const double nh = (s0 < 1e-12) ? 0.0 : dh / s0;
    const double nx = (s1 < 1e-12) ? 0.0 : dqx / s1;
    const double ny = (s2 < 1e-12) ? 0.0 : dqy / s2;
    const double dn = max2(max2(nh, nx), ny);
    return (dn >= e ? 1u : 0u) | (absd(dn - e) <= tol ? 2u : 0u);
}
__device__ __forceinline__ unsigned sig_class(double dh, double dqx, double dqy, const double* T, const Params& P) {
    const double* S = P.smx;
    const double a = max2(max2(dh * __ldg(S + 4), dqx * __ldg(S + 5)), dqy * __ldg(S + 6));
    if (a < T[0]) return 0u;
    if (a > T[1]) return 1u;
    return sig_exact(dh, dqx, dqy, T[3], T[2], __ldg(S + 0), __ldg(S + 1), __ldg(S + 2));
}
// the static DEM mask's significance of z (initialise only; exact)
__device__ __forceinline__ unsigned sig_class_z(double dz, const double* T, const Params& P) {
    const double s3 = __ldg(P.smx + 3);
    const double dn = (s3 < 1e-12) ? 0.0 : dz / s3;
    return (dn >= T[3] ? 1u : 0u) | (absd(dn - T[3]) <= T[2] ? 2u : 0u);
}

struct Enc {
    double4 par;
    bool flow, zflag;
    bool near, znear;  // near-threshold d_norm of the flow quantities / of z
};
// WITH_Z: also threshold z's details (the static DEM mask, t = 0 only)
template <bool WITH_Z = true>
__device__ __forceinline__ Enc encode_children(const double4 c[4], const Params& P, int n) {
    const Red h = red4(c[0].x, c[1].x, c[2].x, c[3].x);
    const Red qx = red4(c[0].y, c[1].y, c[2].y, c[3].y);
    const Red qy = red4(c[0].z, c[1].z, c[2].z, c[3].z);
    Enc e;
    const unsigned s = sig_class(h.dmax, qx.dmax, qy.dmax, P.lvl[n], P);
    e.flow = s & 1u;
    e.near = s & 2u;
    if (WITH_Z) {
        const Red z = red4(c[0].w, c[1].w, c[2].w, c[3].w);
        e.par = make_double4(h.par, qx.par, qy.par, z.par);
        const unsigned sz = sig_class_z(z.dmax, P.lvl[n], P);
        e.zflag = sz & 1u;
        e.znear = sz & 2u;
    } else {
        const double a = c[0].w + c[1].w, b = c[2].w + c[3].w;
        e.par = make_double4(h.par, qx.par, qy.par, 0.25 * (a + b));
        e.zflag = e.znear = false;
    }
    return e;
}

// encode + flow significance with the level's table staged in shared memory
// (thr4 = Params::lvl[n]; same arithmetic as encode_children<false>)
__device__ __forceinline__ Enc encode_children_t(const double4 c[4], const double* thr4, const Params& P) {
    const Red h = red4(c[0].x, c[1].x, c[2].x, c[3].x);
    const Red qx = red4(c[0].y, c[1].y, c[2].y, c[3].y);
    const Red qy = red4(c[0].z, c[1].z, c[2].z, c[3].z);
    const double a = c[0].w + c[1].w, b = c[2].w + c[3].w;
    Enc e;
    const unsigned sg = sig_class(h.dmax, qx.dmax, qy.dmax, thr4, P);
    e.flow = sg & 1u;
    e.near = sg & 2u;
    e.par = make_double4(h.par, qx.par, qy.par, 0.25 * (a + b));
    e.zflag = e.znear = false;
    return e;
}
// per-level thresholds staged in shared memory (indexed constant-bank loads
// with a runtime level miss the constant cache on the critical path)
__device__ __forceinline__ void stage_thresholds(const Params& P, double (*s_thr)[4]) {
    const int t = static_cast<int>(threadIdx.x);
    if (t < 4 * P.L) {
        const int n = t >> 2, q = t & 3;
        s_thr[n][q] = P.lvl[n][q];
    }
}

__device__ __forceinline__ bool active(const Ctl* c, const Params& P) {
    return *((volatile const double*)&c->t) < P.t_end;
}

// Per-CTA view of the control block: thread 0 reads t / parity / step once
// and broadcasts them through shared memory, so a grid of 1000+ CTAs makes
// one request per CTA to the control line instead of one per warp.
struct Head {
    int active, parity, buf;  // buf = timeline buffer (step parity)
    long long step;
};
// (one 16-B aligned block: the vectorised shared loads cover only it)
struct __align__(16) HeadSlot {
    int h[4];  // active, parity, buf, (pad)
    long long step;
};
__device__ __forceinline__ Head cta_head(const Ctl* c, const Params& P, bool force) {
    __shared__ HeadSlot s;
    if (threadIdx.x == 0) {
        const double t = *((volatile const double*)&c->t);
        s.h[0] = (force || t < P.t_end) ? 1 : 0;
        s.h[1] = *((volatile const int*)&c->parity);
        s.step = *((volatile const long long*)&c->step);
        s.h[2] = static_cast<int>(s.step & 1);
        s.h[3] = 0;
    }
    __syncthreads();
    return {s.h[0], s.h[1], s.h[2], s.step};
}

// one warp: a step's report into host pinned memory — line 0 (t, dt, step,
// leaf counts), the error line and the step's stage stamps (timeline buffer
// `slot`), then rep_seq = step behind a system-scope fence
__device__ __forceinline__ void report_to(const Ctl* ctl, Ctl* dstc, int slot) {
    __syncwarp();
    const unsigned l = threadIdx.x & 31;
    const volatile unsigned long long* src = reinterpret_cast<const volatile unsigned long long*>(ctl);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(dstc);
    const unsigned w = (l < 16) ? l : static_cast<unsigned>(offsetof(Ctl, smax_bits) / 8) + (l - 16);
    dst[w] = src[w];
    if (l < 8) {
        const unsigned t = static_cast<unsigned>(offsetof(Ctl, tl) / 8) + 64u * static_cast<unsigned>(slot) +
                           16u * (l >> 1) + 2u * (l & 1u);
        dst[t] = src[t];
    }
    __syncwarp();
    if (l == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile unsigned long long*>(&dstc->rep_seq) =
            static_cast<unsigned long long>(*reinterpret_cast<const volatile long long*>(&ctl->step));
    }
}

// Block-wide sum of unsigned values (256 threads).
template <int NT = kThreads>
__device__ __forceinline__ unsigned block_sum(unsigned v, unsigned* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    unsigned s = 0;
    if (threadIdx.x < 32) {
        s = (l < NT / 32) ? scratch[l] : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        if (l == 0) scratch[0] = s;
    }
    __syncthreads();
    s = scratch[0];
    __syncthreads();
    return s;
}
// Block-wide exclusive scan (256 threads); returns prefix, *total = sum.
template <int NT = kThreads>
__device__ __forceinline__ unsigned block_exscan(unsigned v, unsigned* scratch, unsigned* total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(kFull, x, o);
        if (l >= o) x += y;
    }
    __syncthreads();
    if (l == 31) scratch[w] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned s = (l < NT / 32) ? scratch[l] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFull, s, o);
            if (l >= o) s += y;
        }
        if (l < NT / 32) scratch[l] = s;  // inclusive warp totals
    }
    __syncthreads();
    const unsigned warp_prefix = (w == 0) ? 0u : scratch[w - 1];
    *total = scratch[NT / 32 - 1];
    __syncthreads();
    return warp_prefix + x - v;
}

// Block-wide exclusive scan of 64-bit values (two 32-bit counts packed as
// hi:lo, neither total reaching 2^32); returns the prefix, *total = sum.
template <int NT = kThreads>
__device__ __forceinline__ unsigned long long block_exscan64(unsigned long long v, unsigned long long* scratch,
                                                             unsigned long long* total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, x, o);
        if (l >= o) x += y;
    }
    __syncthreads();
    if (l == 31) scratch[w] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long s = (l < NT / 32) ? scratch[l] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFull, s, o);
            if (l >= o) s += y;
        }
        if (l < NT / 32) scratch[l] = s;
    }
    __syncthreads();
    const unsigned long long warp_prefix = (w == 0) ? 0ull : scratch[w - 1];
    *total = scratch[NT / 32 - 1];
    __syncthreads();
    return warp_prefix + x - v;
}
// three independent 64-bit exclusive scans sharing one set of barriers
// (scratch: 3 * NT / 32 words); *total[k] = sums
template <int NT = kThreads>
__device__ __forceinline__ void block_exscan64x3(const unsigned long long v[3], unsigned long long* scratch,
                                                 unsigned long long out[3], unsigned long long total[3]) {
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    unsigned long long x[3] = {v[0], v[1], v[2]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const unsigned long long y = __shfl_up_sync(kFull, x[k], o);
            if (l >= o) x[k] += y;
        }
    __syncthreads();
    if (l == 31)
#pragma unroll
        for (int k = 0; k < 3; ++k) scratch[k * NW + w] = x[k];
    __syncthreads();
    if (threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            unsigned long long s = (l < NW) ? scratch[k * NW + l] : 0ull;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(kFull, s, o);
                if (l >= o) s += y;
            }
            if (l < NW) scratch[k * NW + l] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        out[k] = ((w == 0) ? 0ull : scratch[k * NW + w - 1]) + x[k] - v[k];
        total[k] = scratch[k * NW + NW - 1];
    }
    __syncthreads();
}

// last-CTA election: every CTA fences its global writes, then bumps a counter
__device__ __forceinline__ bool last_block(unsigned int* counter, int* s_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        *s_flag = (prev == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    const bool last = *s_flag != 0;
    if (last) __threadfence();
    return last;
}


// near-threshold counts of one CTA (block_sum of flow | z << 16): initialise
// -> near_init / near_dem; a step -> the slot of the step they belong to
// (by step parity; FV1's finalizing CTA folds it into cnt_near / near_last)
__device__ __forceinline__ void add_near(Ctl* ctl, bool init, int slot, unsigned packed) {
    if (threadIdx.x != 0 || packed == 0u) return;
    const unsigned long long f = packed & 0xFFFFu, z = packed >> 16;
    if (init) {
        if (f) atomicAdd(&ctl->near_init, f);
        if (z) atomicAdd(&ctl->near_dem, z);
    } else if (f) {
        atomicAdd(&ctl->near_step[slot], f);
    }
}

// ------------------------------------------------------- TMA bulk copies (1D)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* mbar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mbar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy through the TMA unit (cp.async.bulk, SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(mbar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------ cp.async staging (LDGSTS)
// Every MRA kernel stages what it reads into shared memory with asynchronous
// copies issued up front, so a CTA pays ONE global round trip instead of one
// per level loop iteration (the loads of a runtime-bounded level loop are
// otherwise serialised behind the stores that consume them). cp.async takes
// any global address, including NVLink peer pointers of other partitions.
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }



// stage `bytes` (a multiple of 16, both ends 16-B aligned) into shared memory
template <int NT = kThreads>
__device__ __forceinline__ void stage16(void* s, const void* g, uint32_t bytes) {
    for (uint32_t q = 16u * threadIdx.x; q < bytes; q += 16u * NT)
        cp_async16(static_cast<uint8_t*>(s) + q, static_cast<const uint8_t*>(g) + q);
}

// stage the flag bytes of tile j, levels R..L-1, into the slo layout. Level R
// (one byte) cannot be copied asynchronously: it is returned (thread 0 only)
// and must be stored by the caller after cp_async_wait_all.
// (KT = K known at compile time: the level loop unrolled, offsets constant
// or one table load — the runtime loop's index arithmetic was ~12 % of K2)
template <int KT = 0>
__device__ __forceinline__ uint8_t stage_tile_flags(uint8_t* s, const uint8_t* base, const Params& P, uint32_t j) {
    const int K = KT ? KT : P.K, R = P.R;
    uint8_t v0 = 0;
    if (threadIdx.x == 0) v0 = base[P.fbase[R] + j];
    if (K > 1 && threadIdx.x == 32) cp_async4(s + slo(1), base + P.fbase[R + 1] + 4ull * j);
    if constexpr (KT > 0) {
#pragma unroll
        for (int k = 2; k < KT; ++k) {
            constexpr uint32_t one = 1u;
            const uint32_t cnt = one << (2 * k);
            stage16(s + slo(k), base + P.fbase[R + k] + static_cast<unsigned long long>(j) * cnt, cnt);
        }
    } else {
        for (int k = 2; k < K; ++k) {
            const uint32_t cnt = 1u << (2 * k);
            stage16(s + slo(k), base + slo(R + k) + static_cast<unsigned long long>(j) * cnt, cnt);
        }
    }
    return v0;
}

// ---------------------------------------------------------------- K1 warp part
__device__ __forceinline__ double4 shfl4(double4 v, int src) {
    return make_double4(__shfl_sync(kFull, v.x, src), __shfl_sync(kFull, v.y, src), __shfl_sync(kFull, v.z, src),
                        __shfl_sync(kFull, v.w, src));
}
__device__ __forceinline__ bool byte_of(uint32_t w, int k) { return ((w >> (8 * k)) & 0xFFu) != 0u; }

// Encode of 4 children held by lanes lane, lane+s, lane+2s, lane+3s (result
// meaningful at the gathering lane); one component at a time to keep few
// values live. Same arithmetic as encode_children.
// ZPAR = false: the parent's z is not formed (z is static: both cell buffers
// hold the full hierarchy's z from initialise and every re-encode of it
// gives the same bits, so a caller that stores only h, qx, qy — store_hqq —
// leaves the right z in place; Enc::par.w is then 0)
template <bool INIT, bool ZPAR = true>
__device__ __forceinline__ Enc encode_lanes(double4 v, int s, const Params& P, int n) {
    const int lane = threadIdx.x & 31;
    auto red = [&](double x) {
        const double x1 = __shfl_sync(kFull, x, (lane + s) & 31);
        const double x2 = __shfl_sync(kFull, x, (lane + 2 * s) & 31);
        const double x3 = __shfl_sync(kFull, x, (lane + 3 * s) & 31);
        return red4(x, x1, x2, x3);
    };
    const Red h = red(v.x);
    const Red qx = red(v.y);
    const Red qy = red(v.z);
    const Red z = (INIT || ZPAR) ? red(v.w) : Red{0.0, 0.0};
    Enc e;
    const unsigned sg = sig_class(h.dmax, qx.dmax, qy.dmax, P.lvl[n], P);
    e.flow = sg & 1u;
    e.near = sg & 2u;
    e.par = make_double4(h.par, qx.par, qy.par, z.par);
    const unsigned sz = INIT ? sig_class_z(z.dmax, P.lvl[n], P) : 0u;
    e.zflag = sz & 1u;
    e.znear = sz & 2u;
    return e;
}

// Re-encode + threshold of levels T, T-1, T-2 of subtree j by warps (T = L-1
// at t = 0, else L-2: level L-1 was re-encoded by the previous FV1). Warp w
// owns a contiguous block of 32*ipw tile-local level-T cells (one per lane per
// iteration), their level-(T-1) parents (lanes 4k) and level-(T-2)
// grandparents (lanes 16m); values move up by shuffles, flags are prefetched
// as words. Level-(T-2) values go to sv3[tile-local index] for the CTA-level
// part. Returns the number of re-encoded cells of this thread.
template <bool INIT>
__device__ __forceinline__ unsigned encode_warp_levels(const Params& P, double4* buf, const uint8_t* sigp,
                                                       double4* sv3, uint32_t j, int T, int R, unsigned& nnear,
                                                       unsigned& ndem) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t n1 = 1u << (2 * (T - R)), n2 = n1 >> 2, n3 = n2 >> 2;  // tile cells on T, T-1, T-2
    const int ipw = (n1 >= 32u * (kThreads / 32)) ? static_cast<int>(n1 / (32u * (kThreads / 32))) : 1;
    const uint32_t b1 = 32u * ipw * w, b2 = 8u * ipw * w, b3 = 2u * ipw * w;
    if (b1 >= n1) return 0;
    const int L1 = T, L2 = T - 1, L3 = T - 2;
    const unsigned long long g1 = slo(L1) + static_cast<unsigned long long>(j) * n1;
    const unsigned long long g2 = slo(L2) + static_cast<unsigned long long>(j) * n2;
    const unsigned long long g3 = slo(L3) + static_cast<unsigned long long>(j) * n3;
    // previous-tree / DEM flags: words for level T (4 cells per lane), bytes above
    uint32_t f1w = 0, d1w = 0;
    if (b1 + 4u * lane < n1 && lane < 8 * ipw) {
        f1w = INIT ? 0x01010101u : *reinterpret_cast<const uint32_t*>(sigp + g1 + b1 + 4u * lane);
        d1w = INIT ? 0u : *reinterpret_cast<const uint32_t*>(P.dem + g1 + b1 + 4u * lane);
    }
    uint32_t f2 = 0, d2 = 0, f3 = 0, d3 = 0, f4 = 0;
    if (lane < 8 * ipw && b2 + lane < n2) {
        f2 = INIT ? 1u : sigp[g2 + b2 + lane];
        d2 = INIT ? 0u : P.dem[g2 + b2 + lane];
    }
    if (lane < 2 * ipw && b3 + lane < n3) {
        f3 = INIT ? 1u : sigp[g3 + b3 + lane];
        d3 = INIT ? 0u : P.dem[g3 + b3 + lane];
        if (L3 > R) f4 = INIT ? 1u : sigp[slo(L3 - 1) + static_cast<unsigned long long>(j) * (n3 >> 2) + ((b3 + lane) >> 2)];
    }
    const bool zero1 = 0.0 >= P.tau[L1], zero2 = 0.0 >= P.tau[L2], zero3 = 0.0 >= P.tau[L3];
    unsigned tree = 0;
#pragma unroll 1
    for (int i = 0; i < ipw; ++i) {
        if (b1 + 32u * i >= n1) break;  // warp-uniform
        const uint32_t c1 = b1 + 32u * i + lane, c2 = b2 + 8u * i + (lane >> 2), c3 = b3 + 2u * i + (lane >> 4);
        const bool ok1 = c1 < n1, ok2 = (lane & 3) == 0 && c2 < n2, ok3 = (lane & 15) == 0 && c3 < n3;
        const uint32_t gm1 = j * n1 + c1, gm2 = j * n2 + c2, gm3 = j * n3 + c3;
        const int src1 = 8 * i + (lane >> 2), src3 = 2 * i + (lane >> 4);
        const uint32_t w1 = __shfl_sync(kFull, f1w, src1), wd1 = __shfl_sync(kFull, d1w, src1);
        const bool sp1 = ok1 && byte_of(w1, lane & 3);
        const bool dm1 = byte_of(wd1, lane & 3);
        const bool sp2 = __shfl_sync(kFull, f2, src1) != 0;  // my T-1 parent (lanes 4k: my own T-1 cell)
        const bool dm2 = __shfl_sync(kFull, d2, src1) != 0;
        const bool sp3 = __shfl_sync(kFull, f3, src3) != 0;  // my T-2 ancestor (lanes 16m: my own)
        const bool dm3 = __shfl_sync(kFull, d3, src3) != 0;
        const bool sp4 = __shfl_sync(kFull, f4, src3) != 0;
        // every global read of the iteration first: children, then the values
        // of previous-tree leaves whose parent is re-encoded here
        double4 ch[4];
        if (sp1) {
            const double4* cp = buf + cbase(L1 + 1) + (static_cast<unsigned long long>(gm1) << 2);
            ch[0] = ld4_nc(cp); ch[1] = ld4_nc(cp + 1); ch[2] = ld4_nc(cp + 2); ch[3] = ld4_nc(cp + 3);
        }
        double4 v1 = make_double4(0.0, 0.0, 0.0, 0.0), v2 = v1, v3 = v1;
        if (ok1 && !sp1 && sp2) v1 = ld4(buf + cbase(L1) + gm1);
        if (ok2 && !sp2 && sp3) v2 = ld4(buf + cbase(L2) + gm2);
        if (ok3 && !sp3 && sp4 && L3 > R) v3 = ld4(buf + cbase(L3) + gm3);
        // level T
        {
            bool flow = zero1, zf = false;
            if (sp1) {
                const Enc e = encode_children<INIT>(ch, P, L1);
                v1 = e.par;
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                zf = e.zflag;
                ndem += e.znear ? 1u : 0u;
                st4(buf + cbase(L1) + gm1, v1);
                ++tree;
            }
            if (ok1) {
                const bool d = INIT ? zf : dm1;
                if (INIT) P.dem[g1 + c1] = d ? 1 : 0;
                P.pre[g1 + c1] = (flow || d) ? 1 : 0;
            }
        }
        // level T-1: lane 4k gathers lanes 4k..4k+3
        {
            const Enc e = encode_lanes<INIT>(v1, 1, P, L2);
            if (ok2) {
                bool flow = zero2, zf = false;
                if (sp2) {
                    v2 = e.par;
                    flow = e.flow;
                    nnear += e.near ? 1u : 0u;
                    zf = e.zflag;
                    ndem += e.znear ? 1u : 0u;
                    st4(buf + cbase(L2) + gm2, v2);
                    ++tree;
                }
                const bool d = INIT ? zf : dm2;
                if (INIT) P.dem[g2 + c2] = d ? 1 : 0;
                P.pre[g2 + c2] = (flow || d) ? 1 : 0;
            }
        }
        // level T-2: lane 16m gathers lanes 16m, +4, +8, +12
        {
            const Enc e = encode_lanes<INIT>(v2, 4, P, L3);
            if (ok3) {
                bool flow = zero3, zf = false;
                if (sp3) {
                    v3 = e.par;
                    flow = e.flow;
                    nnear += e.near ? 1u : 0u;
                    zf = e.zflag;
                    ndem += e.znear ? 1u : 0u;
                    st4(buf + cbase(L3) + gm3, v3);
                    ++tree;
                }
                const bool d = INIT ? zf : dm3;
                if (INIT) P.dem[g3 + c3] = d ? 1 : 0;
                P.pre[g3 + c3] = (flow || d) ? 1 : 0;
                sv3[c3] = v3;
            }
        }
    }
    return tree;
}

// =========================================================================== K1
// zero_details_and_reencode + significance
// over the level-R subtree `blockIdx.x`; restricted to the previous tree (sig
// prev), so off-tree cells only cost a flag read. INIT = full encode at t=0
// (sig prev is all ones) and also derives the static DEM mask.
template <bool INIT>
__global__ void __launch_bounds__(kThreads, 2) k_encode(Params P, Ctl* ctl) {
    pdl_wait();
    pdl_trigger();
    const Head hd = cta_head(ctl, P, INIT);
    if (!hd.active) return;
    tl_start(ctl, hd.buf, 0);
    extern __shared__ double4 sv[];
    __shared__ unsigned s_red[32];
    __shared__ int s_last;
    const int p = hd.parity;
    double4* buf = P.cells[p];
    const uint8_t* sigp = P.sig[p];
    const int L = P.L, R = P.R, K = P.K;
    const uint32_t j = P.tile_lo + blockIdx.x;
    const uint32_t ncell = ((1u << (2 * K)) - 1u) / 3u;  // subtree cells on levels R..L-1
    uint8_t* sfl = reinterpret_cast<uint8_t*>(sv + ncell);  // previous-tree flags of the subtree
    unsigned tree = 0, nnear = 0, ndem = 0;

    // Warp part: levels T, T-1, T-2 with shuffles and no CTA barrier, where
    // T = L-1 at t = 0 and T = L-2 afterwards (the previous step's FV1 already
    // re-encoded level L-1 of the previous tree, see k_fv1). The CTA then
    // finishes levels top_n .. R from shared memory. Small trees use the
    // per-thread path for level L-1 (re-encoding it again is bit-identical).
    const int T = INIT ? L - 1 : L - 2;
    const bool warp_path = T - 2 >= R;
    const int top_n = warp_path ? T - 3 : L - 2;

    // ---- flags of the CTA-level part and the values of previous-tree leaves
    //      whose parent gets re-encoded there, issued up front
    for (int n = R; n <= top_n + (warp_path ? 0 : 1); ++n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads)
            sfl[lo(n, R) + pi] = INIT ? 1 : sigp[slo(n) + j * cnt + pi];
    }
    __syncthreads();
    if (!INIT) {
        for (int n = R + 1; n <= top_n + (warp_path ? 0 : 1); ++n) {
            const uint32_t cnt = 1u << (2 * (n - R));
            for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
                const uint32_t li = lo(n, R) + pi;
                if (!sfl[li] && sfl[lo(n - 1, R) + (pi >> 2)]) sv[li] = ld4(buf + cbase(n) + j * cnt + pi);
            }
        }
    }

    if (warp_path) {
        if (!INIT) {
            // level L-1: previous-tree cells were re-encoded (and flagged) by
            // the previous FV1; the others only get pre = DEM | (eps == 0)
            const int n = L - 1;
            const uint32_t cnt = 1u << (2 * (n - R));
            const bool zero = 0.0 >= P.tau[n];
            const unsigned long long g = slo(n) + static_cast<unsigned long long>(j) * cnt;
            for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads) {
                const uint32_t f = *reinterpret_cast<const uint32_t*>(sigp + g + q);
                const uint32_t d = *reinterpret_cast<const uint32_t*>(P.dem + g + q);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (!byte_of(f, k)) P.pre[g + q + k] = (zero || byte_of(d, k)) ? 1 : 0;
            }
        }
        tree += encode_warp_levels<INIT>(P, buf, sigp, sv + lo(T - 2, R), j, T, R, nnear, ndem);
    } else {
        // small trees: one thread per level-(L-1) parent
        const int n = L - 1;
        const uint32_t npar = 1u << (2 * (K - 1));
        const uint32_t pbase = j * npar;
        for (uint32_t pi = threadIdx.x; pi < npar; pi += kThreads) {
            const uint32_t pm = pbase + pi;
            const bool sp = sfl[lo(n, R) + pi] != 0;
            const uint8_t d0 = INIT ? 0 : P.dem[slo(n) + pm];
            bool flow, zf = false;
            if (sp) {
                const double4* cp = buf + cbase(L) + (static_cast<unsigned long long>(pm) << 2);
                const double4 c[4] = {ld4_nc(cp), ld4_nc(cp + 1), ld4_nc(cp + 2), ld4_nc(cp + 3)};
                const Enc e = encode_children<INIT>(c, P, n);
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                zf = e.zflag;
                ndem += e.znear ? 1u : 0u;
                st4(buf + cbase(n) + pm, e.par);
                if (n > R) sv[lo(n, R) + pi] = e.par;
                ++tree;
            } else {
                flow = 0.0 >= P.tau[n];
            }
            uint8_t d = d0;
            if (INIT) {
                d = zf ? 1 : 0;
                P.dem[slo(n) + pm] = d;
            }
            P.pre[slo(n) + pm] = (flow || d) ? 1 : 0;
        }
    }
    __syncthreads();

    // ---- CTA-level part: levels top_n .. R from shared memory
    for (int n = top_n; n >= R; --n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        const uint32_t pb = j * cnt;
        for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
            const uint32_t pm = pb + pi;
            const bool sp = sfl[lo(n, R) + pi] != 0;
            const uint8_t d0 = INIT ? 0 : P.dem[slo(n) + pm];
            bool flow, zf = false;
            if (sp) {
                const uint32_t c0 = lo(n + 1, R) + 4u * pi;
                const double4 c[4] = {sv[c0], sv[c0 + 1], sv[c0 + 2], sv[c0 + 3]};
                const Enc e = encode_children<INIT>(c, P, n);
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                zf = e.zflag;
                ndem += e.znear ? 1u : 0u;
                st4(buf + cbase(n) + pm, e.par);
                if (n > R) sv[lo(n, R) + pi] = e.par;
                ++tree;
            } else {
                flow = 0.0 >= P.tau[n];
            }
            uint8_t d = d0;
            if (INIT) {
                d = zf ? 1 : 0;
                P.dem[slo(n) + pm] = d;
            }
            P.pre[slo(n) + pm] = (flow || d) ? 1 : 0;
        }
        __syncthreads();
    }

    const unsigned tsum = block_sum(tree, s_red);
    if (threadIdx.x == 0 && tsum) atomicAdd(&ctl->cnt_tree, (unsigned long long)tsum);
    add_near(ctl, INIT, hd.buf, block_sum(nnear | (ndem << 16), s_red));
    if (P.G > 1) return;  // partitioned: k_encode_top runs after all partitions' subtrees
    if (!last_block(&ctl->done_k1, &s_last)) return;
    encode_top<INIT>(P, ctl, sv, s_red);
    tl_end(ctl, hd.buf, 0);
}

template <bool INIT>
__global__ void __launch_bounds__(kThreads) k_encode_top(Params P, Ctl* ctl) {
    pdl_wait();
    if (!INIT && !active(ctl, P)) return;
    extern __shared__ double4 sv_top[];
    __shared__ unsigned s_red[32];
    encode_top<INIT>(P, ctl, sv_top, s_red);
}

// Levels R-1 .. 0 of the re-encode (one CTA). Level-R children come from
// global memory (every subtree's CTA / partition wrote them); above that the
// block keeps its results in shared memory when levels 0..R-1 fit (R <= K).
template <bool INIT>
__device__ void encode_top(const Params& P, Ctl* ctl, double4* sv, unsigned* s_red) {
    const int p = ctl->parity;
    double4* buf = P.cells[p];
    const uint8_t* sigp = P.sig[p];
    const int R = P.R, K = P.K;

    unsigned ttop = 0, nnear = 0, ndem = 0;
    const bool top_smem = ((1u << (2 * R)) - 1u) / 3u <= ((1u << (2 * K)) - 1u) / 3u;
    for (int n = R - 1; n >= 0; --n) {
        const uint32_t cnt = 1u << (2 * n);
        const bool kids_in_smem = top_smem && n < R - 1;
        for (uint32_t pm = threadIdx.x; pm < cnt; pm += kThreads) {
            const bool sp = INIT || sigp[slo(n) + pm];
            bool flow, zf = false;
            if (sp) {
                double4 c[4];
                if (kids_in_smem) {
                    const uint32_t c0 = lo(n + 1, 0) + 4u * pm;
                    c[0] = sv[c0]; c[1] = sv[c0 + 1]; c[2] = sv[c0 + 2]; c[3] = sv[c0 + 3];
                } else {
                    const uint32_t c0 = pm << 2;  // the children's partition(s) hold them
                    c[0] = ld4_cg(cell_ptr(P, p, n + 1, c0)); c[1] = ld4_cg(cell_ptr(P, p, n + 1, c0 + 1));
                    c[2] = ld4_cg(cell_ptr(P, p, n + 1, c0 + 2)); c[3] = ld4_cg(cell_ptr(P, p, n + 1, c0 + 3));
                }
                const Enc e = encode_children<INIT>(c, P, n);
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                zf = e.zflag;
                ndem += e.znear ? 1u : 0u;
                st4(buf + cbase(n) + pm, e.par);
                if (top_smem) sv[lo(n, 0) + pm] = e.par;
                ++ttop;
            } else {
                flow = 0.0 >= P.tau[n];
                if (top_smem && n > 0 && sigp[slo(n - 1) + (pm >> 2)]) sv[lo(n, 0) + pm] = ld4_cg(cell_ptr(P, p, n, pm));
            }
            uint8_t d;
            if (INIT) {
                d = zf ? 1 : 0;
                P.dem[slo(n) + pm] = d;
            } else {
                d = P.dem[slo(n) + pm];
            }
            P.pre[slo(n) + pm] = (flow || d) ? 1 : 0;
        }
        __threadfence_block();
        __syncthreads();
    }
    const unsigned tt = block_sum(ttop, s_red);
    if (threadIdx.x == 0) {
        if (tt) atomicAdd(&ctl->cnt_tree, (unsigned long long)tt);
        ctl->done_k1 = 0;
    }
    const unsigned nsum = block_sum(nnear | (ndem << 16), s_red);  // (replicated levels: partition 0 counts)
    if (P.part == 0) add_near(ctl, INIT, static_cast<int>(*((volatile const long long*)&ctl->step) & 1), nsum);
}



// encode_children_t of the four values in lanes l, l+s, l+2s, l+3s (valid in
// the lanes that own a parent; every lane of the warp must call it)
__device__ __forceinline__ Enc encode_lanes_s(double4 v, int s, const double* thr4, const Params& P) {
    const int lane = threadIdx.x & 31;
    const int l1 = (lane + s) & 31, l2 = (lane + 2 * s) & 31, l3 = (lane + 3 * s) & 31;
    auto red = [&](double x) {
        return red4(x, __shfl_sync(kFull, x, l1), __shfl_sync(kFull, x, l2), __shfl_sync(kFull, x, l3));
    };
    const Red h = red(v.x);
    const Red qx = red(v.y);
    const Red qy = red(v.z);
    const double w1 = __shfl_sync(kFull, v.w, l1), w2 = __shfl_sync(kFull, v.w, l2), w3 = __shfl_sync(kFull, v.w, l3);
    const double a = v.w + w1, b = w2 + w3;
    Enc e;
    const unsigned sg = sig_class(h.dmax, qx.dmax, qy.dmax, thr4, P);
    e.flow = sg & 1u;
    e.near = sg & 2u;
    e.par = make_double4(h.par, qx.par, qy.par, 0.25 * (a + b));
    e.zflag = e.znear = false;
    return e;
}

// K1 after t = 0 (level L-1 was re-encoded and flagged by the previous
// FV1): re-encode + threshold of levels L-2 .. R of subtree j. Everything the
// CTA reads is issued at once: the previous-tree and DEM flags of levels
// R..L-1 and the values of levels R+1..L-2 (inputs where a previous-tree
// leaf's parent is re-encoded) are staged into shared memory by cp.async;
// thread t loads the four level-(L-1) children of level-(L-2) cell t straight
// into registers when that cell is on the previous tree. Levels L-3..R are
// then encoded from shared memory. No last-CTA tail: levels < R are encoded
// by an extra CTA of K2 (encode_top_staged).
template <int KT>
__global__ void __launch_bounds__(kThreads, 5) k_encode_step(Params P, Ctl* ctl) {
    // Before the wait for the previous FV1, everything that does not depend
    // on it: the previous-tree flags of BOTH copies (FV1 writes neither, and
    // which one is current is only known once FV1's last CTA has flipped the
    // parity), the DEM flags and this thread's level-(L-2) flag in both
    // copies. A CTA resident on an SM that FV1 left early has them in place
    // when the wait returns; after it only the values remain to be fetched.
    __shared__ __align__(8) unsigned long long mbar[2];  // [0] flags, [1] values
    extern __shared__ __align__(16) uint8_t sm1[];
    __shared__ unsigned s_red[32];
    __shared__ double s_thr[kMaxL][4];
    const int L = P.L, R = P.R;
    const int K = KT ? KT : P.K;
    if (P.rep_ring && blockIdx.x == gridDim.x - 1) {
        // (advance_reports' graphs: one extra CTA) the report of the step the
        // FV1 just waited for completed, into the ring slot of its number
        pdl_wait();
        const Head hd = cta_head(ctl, P, true);
        if (threadIdx.x < 32 && hd.step > 0)
            report_to(ctl, P.rep_ring + (static_cast<unsigned long long>(hd.step) & P.rep_ring_mask), hd.buf ^ 1);
        return;
    }
    const uint32_t j = P.tile_lo + blockIdx.x;
    if (P.qskip && P.qstate[j] >= 2) {
        // stable quiet subtree (K3's top of the step that FV1 just finished
        // skipped it): its re-encoded values, pre flags and counts in this
        // buffer are this kernel's of two steps ago from the same children
        // (Params::qskip); only the counts it would add
        pdl_wait();
        pdl_trigger();
        const Head hd = cta_head(ctl, P, false);
        if (hd.active && threadIdx.x == 0) {
            const unsigned tr = P.qnk1[2 * j], nn = P.qnk1[2 * j + 1];
            if (tr) atomicAdd(&ctl->cnt_tree, (unsigned long long)tr);
            if (nn) atomicAdd(&ctl->near_step[hd.buf], (unsigned long long)nn);
            if (tr) atomicAdd(&ctl->cnt_k1skip, (unsigned long long)tr);
        }
        return;
    }
    const uint32_t nv = lo(K - 1, 0);  // cells on levels R..L-2
    double4* sv = reinterpret_cast<double4*>(sm1);
    uint8_t* sf2 = sm1 + 32u * nv;     // previous-tree flags of copy 0 and copy 1, slo layout
    uint8_t* sd = sf2 + 2 * slo(K);    // DEM flags, slo layout
    uint8_t* so = sd + slo(K);         // new pre flags of levels R..L-2, slo layout
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
    }
    __syncthreads();
    // ---- the critical-path load first: this thread's level-(L-2) flag
    const int k2 = K - 2;              // tile level of L-2
    const uint32_t c2 = (k2 >= 0) ? (1u << (2 * k2)) : 0u;
    const bool has2 = threadIdx.x < c2;
    const uint32_t m2 = j * c2 + threadIdx.x;
    uint8_t f2a = 0, f2b = 0;
    if (has2) {
        f2a = P.sig[0][slo(L - 2) + m2];
        f2b = P.sig[1][slo(L - 2) + m2];
    }
    // ---- bulk copies (TMA, one thread): flags of levels R+2..L-1; the two
    //      smallest flag levels by plain loads
    if (threadIdx.x == 0) {
        unsigned bytes = 0;
        for (int k = 2; k < K; ++k) bytes += 3u << (2 * k);
        mbar_expect_tx(&mbar[0], bytes);
        for (int k = 2; k < K; ++k) {
            const uint32_t cnt = 1u << (2 * k);
            const unsigned long long g = slo(R + k) + static_cast<unsigned long long>(j) * cnt;
            bulk_g2s(sf2 + slo(k), P.sig[0] + g, cnt, &mbar[0]);
            bulk_g2s(sf2 + slo(K) + slo(k), P.sig[1] + g, cnt, &mbar[0]);
            bulk_g2s(sd + slo(k), P.dem + g, cnt, &mbar[0]);
        }
    }
    uint32_t fsa = 0, fsb = 0, dsmall = 0;
    if (threadIdx.x == 32 && K > 1) {
        fsa = *reinterpret_cast<const uint32_t*>(P.sig[0] + slo(R + 1) + 4ull * j);
        fsb = *reinterpret_cast<const uint32_t*>(P.sig[1] + slo(R + 1) + 4ull * j);
        dsmall = *reinterpret_cast<const uint32_t*>(P.dem + slo(R + 1) + 4ull * j);
    }
    uint8_t f0a = 0, f0b = 0, d0 = 0;
    if (threadIdx.x == 64) {
        f0a = P.sig[0][slo(R) + j];
        f0b = P.sig[1][slo(R) + j];
        d0 = P.dem[slo(R) + j];
    }
    stage_thresholds(P, s_thr);

    pdl_wait();
    const unsigned long long t_entry = gtimer();
    const Head hd = cta_head(ctl, P, false);
    if (!hd.active) {
        mbar_wait(&mbar[0], 0);  // no bulk copy may outlive the CTA
        return;
    }
    tl_start(ctl, hd.buf, 0);
    const Probe stamp(ctl, 0);
    stamp(7, t_entry);
    const int p = hd.parity;
    double4* buf = P.cells[p];
    uint8_t* sf = sf2 + (p ? slo(K) : 0u);  // previous-tree flags of the current copy
    const bool sp2 = has2 && (p ? f2b : f2a) != 0;
    // ---- values of levels R+1..L-2 (TMA; K = 6: R+1..L-3) and this thread's
    //      four level-(L-1) children (registers), written by the FV1 just
    //      waited for. K = 6: a level-(L-2) cell off the previous tree is
    //      loaded into ch[0] only when its parent is re-encoded (it is then
    //      a previous-tree leaf whose value the parent needs)
    const int kv = (KT == 6) ? K - 3 : K - 2;  // highest tile level staged by TMA
    if (threadIdx.x == 0) {
        unsigned bytes = 0;
        for (int k = 1; k <= kv; ++k) bytes += 32u << (2 * k);
        mbar_expect_tx(&mbar[1], bytes);
        for (int k = 1; k <= kv; ++k) {
            const uint32_t cnt = 1u << (2 * k);
            bulk_g2s(sv + lo(k, 0), buf + cbase(R + k) + static_cast<unsigned long long>(j) * cnt, 32u * cnt, &mbar[1]);
        }
    }
    double4 ch[4];
    if (sp2) {
        const double4* cp = buf + cbase(L - 1) + (static_cast<unsigned long long>(m2) << 2);
        ch[0] = ld4_nc(cp); ch[1] = ld4_nc(cp + 1); ch[2] = ld4_nc(cp + 2); ch[3] = ld4_nc(cp + 3);
    } else if (KT == 6 && has2) {
        mbar_wait(&mbar[0], 0);  // (the flags were staged before the wait for FV1)
        if (sf[slo(k2 - 1) + (threadIdx.x >> 2)]) ch[0] = ld4_nc(buf + cbase(L - 2) + m2);
    }
    stamp(0);
    if (threadIdx.x == 32 && K > 1) {
        *reinterpret_cast<uint32_t*>(sf + slo(1)) = p ? fsb : fsa;
        *reinterpret_cast<uint32_t*>(sd + slo(1)) = dsmall;
    }
    if (threadIdx.x == 64) {
        sf[0] = p ? f0b : f0a;
        sd[0] = d0;
    }
    mbar_wait(&mbar[0], 0);
    mbar_wait(&mbar[1], 0);
    __syncthreads();
    stamp(1);

    // ---- level L-1: cells off the previous tree only get pre = DEM | (eps == 0)
    {
        const int k = K - 1;
        const uint32_t cnt = 1u << (2 * k);
        const uint32_t zero = (0.0 >= s_thr[L - 1][3]) ? 0x01010101u : 0u;
        const unsigned long long g = slo(L - 1) + static_cast<unsigned long long>(j) * cnt;
        if (cnt >= 4) {
            for (uint32_t c = 4u * threadIdx.x; c < cnt; c += 4u * kThreads) {
                const uint32_t f = *reinterpret_cast<const uint32_t*>(sf + slo(k) + c);
                if (f == 0x01010101u) continue;
                const uint32_t v = zero | *reinterpret_cast<const uint32_t*>(sd + slo(k) + c);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (!byte_of(f, q)) P.pre[g + c + q] = byte_of(v, q) ? 1 : 0;
            }
        } else if (threadIdx.x == 0 && !sf[0]) {
            P.pre[g] = (zero || sd[0]) ? 1 : 0;
        }
    }
    unsigned tree = 0, nnear = 0, ndem = 0;
    stamp(2);
    if constexpr (KT == 6) {
        // K = 6: levels L-2 .. R without a CTA barrier per level — L-2 in
        // registers (one cell per thread), L-3 and L-4 by shuffles inside the
        // warp, the 16 level-(L-4) values through shared memory to warp 0 for
        // R+1 and R. A cell on the previous tree is re-encoded and stored at
        // once; the others keep their staged value (same arithmetic and
        // results as the per-level loop below).
        const int tid = threadIdx.x, lane = tid & 31;
        double4 v;
        {
            bool flow = 0.0 >= s_thr[L - 2][3];
            if (sp2) {
                const Enc e = encode_children_t(ch, s_thr[L - 2], P);
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                v = e.par;
                st4(buf + cbase(L - 2) + m2, v);
                ++tree;
            } else {
                v = ch[0];  // (only used when the parent is re-encoded: then loaded above)
            }
            so[slo(4) + tid] = (flow || sd[slo(4) + tid]) ? 1 : 0;
        }
        auto level = [&](int k, uint32_t pi, const Enc& e) {  // cell pi of tile level k, k < 4
            const int n = R + k;
            bool flow = 0.0 >= s_thr[n][3];
            if (sf[slo(k) + pi]) {
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                v = e.par;
                st4(buf + cbase(n) + static_cast<unsigned long long>(j) * (1u << (2 * k)) + pi, v);
                ++tree;
            } else if (k > 0) {
                v = sv[lo(k, 0) + pi];
            }
            so[slo(k) + pi] = (flow || sd[slo(k) + pi]) ? 1 : 0;
        };
        {
            const Enc e = encode_lanes_s(v, 1, s_thr[L - 3], P);
            if ((lane & 3) == 0) level(3, static_cast<uint32_t>(tid) >> 2, e);
        }
        {
            const Enc e = encode_lanes_s(v, 4, s_thr[L - 4], P);
            if ((lane & 15) == 0) {
                const uint32_t pi = static_cast<uint32_t>(tid) >> 4;
                level(2, pi, e);
                sv[lo(2, 0) + pi] = v;
            }
        }
        __syncthreads();
        if (tid < 32) {
            v = sv[lo(2, 0) + (lane & 15)];
            {
                const Enc e = encode_lanes_s(v, 1, s_thr[R + 1], P);
                if ((lane & 3) == 0 && lane < 16) level(1, static_cast<uint32_t>(lane) >> 2, e);
            }
            {
                const Enc e = encode_lanes_s(v, 4, s_thr[R], P);
                if (lane == 0) level(0, 0u, e);
            }
        }
        __syncthreads();
        stamp(4);
        for (int k = 0; k <= 4; ++k) {  // pre-band flags of levels R..L-2 (words where a level has >= 4)
            const uint32_t cnt = 1u << (2 * k);
            const unsigned long long jb = static_cast<unsigned long long>(j) * cnt;
            if (cnt >= 4) {
                for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads)
                    *reinterpret_cast<uint32_t*>(P.pre + slo(R + k) + jb + q) = *reinterpret_cast<const uint32_t*>(so + slo(k) + q);
            } else if (threadIdx.x == 0) {
                P.pre[slo(R) + jb] = so[0];
            }
        }
    } else {
        if (has2) {
            bool flow = 0.0 >= s_thr[L - 2][3];
            if (sp2) {
                const Enc e = encode_children_t(ch, s_thr[L - 2], P);
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                sv[lo(k2, 0) + threadIdx.x] = e.par;
                ++tree;
            }
            so[slo(k2) + threadIdx.x] = (flow || sd[slo(k2) + threadIdx.x]) ? 1 : 0;
        }
        __syncthreads();
        stamp(3);
        // ---- levels L-3 .. R in shared memory
#pragma unroll
        for (int k = (KT ? KT : kMaxL) - 3; k >= 0; --k) {
            if (!KT && k > K - 3) continue;
            const int n = R + k;
            const uint32_t cnt = 1u << (2 * k);
            for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
                bool flow = 0.0 >= s_thr[n][3];
                if (sf[slo(k) + pi]) {
                    const uint32_t c0 = lo(k + 1, 0) + 4u * pi;
                    const double4 c[4] = {sv[c0], sv[c0 + 1], sv[c0 + 2], sv[c0 + 3]};
                    const Enc e = encode_children_t(c, s_thr[n], P);
                    flow = e.flow;
                    nnear += e.near ? 1u : 0u;
                    sv[lo(k, 0) + pi] = e.par;
                    ++tree;
                }
                so[slo(k) + pi] = (flow || sd[slo(k) + pi]) ? 1 : 0;
            }
            __syncthreads();
        }
        stamp(4);
        // ---- one burst of stores: re-encoded values (previous-tree cells) and
        //      the pre-band flags of levels R..L-2 (words where a level has >= 4)
        for (int k = 0; k <= K - 2; ++k) {
            const uint32_t cnt = 1u << (2 * k);
            const unsigned long long jb = static_cast<unsigned long long>(j) * cnt;
            for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads)
                if (sf[slo(k) + pi]) st4(buf + cbase(R + k) + jb + pi, sv[lo(k, 0) + pi]);
            if (cnt >= 4) {
                for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads)
                    *reinterpret_cast<uint32_t*>(P.pre + slo(R + k) + jb + q) = *reinterpret_cast<const uint32_t*>(so + slo(k) + q);
            } else if (threadIdx.x == 0) {
                P.pre[slo(R) + jb] = so[0];
            }
        }

    }
    pdl_trigger();  // K2 may launch (late: measured ~0.5 us better than at entry)
    const unsigned tsum = block_sum(tree | (nnear << 16), s_red);  // (both < 2^16 per subtree)
    if (threadIdx.x == 0 && (tsum & 0xFFFFu)) atomicAdd(&ctl->cnt_tree, (unsigned long long)(tsum & 0xFFFFu));
    add_near(ctl, false, hd.buf, tsum >> 16);
    if (P.qskip && threadIdx.x == 0) {  // (cached for the steps this subtree is skipped)
        P.qnk1[2 * j] = tsum & 0xFFFFu;
        P.qnk1[2 * j + 1] = tsum >> 16;
    }
    tl_end(ctl, hd.buf, 0);
    stamp(5);
}

// band (D3) of cell (n, m) from the pre-band flags (flow | DEM);
// `pre_at(level, morton)` reads a pre flag (global or shared memory)
template <class PreAt>
__device__ __forceinline__ uint8_t band_flag(int mode, int L, int n, uint32_t m, PreAt&& pre_at) {
    uint8_t b = pre_at(n, m);
    if (mode == 2) {
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const uint32_t nb = zo::neighbour_dev(n, m, static_cast<zo::Direction>(d));
            if (nb != zo::kNone) b |= pre_at(n, nb);
        }
    } else if (mode == 1 && n + 1 < L) {
        for (int k = 0; k < 4; ++k) {
            const uint32_t c = 4u * m + static_cast<uint32_t>(k);
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const uint32_t nb = zo::neighbour_dev(n + 1, c, static_cast<zo::Direction>(d));
                if (nb != zo::kNone) b |= pre_at(n + 1, nb);
            }
        }
    }
    return b ? 1 : 0;
}

// Levels R-1 .. 0 of the re-encode after t = 0, one CTA (run as the extra
// CTA of K2, concurrently with the subtree CTAs). Round trip 1 stages the
// previous-tree and DEM flags of levels 0..R-1; round trip 2 loads the
// level-R children of re-encoded level-(R-1) cells into registers and stages
// the values of previous-tree leaves whose parent is re-encoded. Needs
// 32 * lo(R, 0) + 2 * fbase[R] bytes of shared memory (host: R <= 6).
// the part of encode_top_staged's staging that does not depend on K1 (the
// previous-tree and DEM flags of levels 0..R-1): issued before the PDL wait
__device__ __forceinline__ void encode_top_prestage(const Params& P, int p, uint8_t* sm) {
    const int R = P.R;
    if (R == 0) return;
    const uint32_t fb = static_cast<uint32_t>(slo(R));
    uint8_t* sf = sm + 32u * lo(R, 0);
    stage16(sf, P.sig[p], fb);
    stage16(sf + fb, P.dem, fb);
}
__device__ void encode_top_staged(const Params& P, Ctl* ctl, int p, int slot, uint8_t* sm, bool prestaged = false) {
    double4* buf = P.cells[p];
    const int R = P.R;
    if (R == 0) return;
    __shared__ unsigned s_red[32];
    __shared__ double s_thr[kMaxL][4];
    stage_thresholds(P, s_thr);
    const uint32_t fb = static_cast<uint32_t>(slo(R));  // flag bytes of levels 0..R-1 (fbase[0] = 0)
    double4* sv = reinterpret_cast<double4*>(sm);          // levels 0..R-1, compact lo(n, 0)
    uint8_t* sf = sm + 32u * lo(R, 0);                     // previous-tree flags at fbase[n]
    uint8_t* sd = sf + fb;                                 // DEM flags at fbase[n]
    uint8_t* sq = sd + fb;                                 // (top_band) new pre flags at fbase[n]
    if (!prestaged) encode_top_prestage(P, p, sm);
    cp_async_wait_all();
    __syncthreads();
    // values of previous-tree leaves (levels 1..R-2) under a re-encoded parent
    for (int n = 1; n <= R - 2; ++n) {
        const uint32_t cnt = 1u << (2 * n);
        for (uint32_t m = threadIdx.x; m < cnt; m += kThreads)
            if (!sf[slo(n) + m] && sf[slo(n - 1) + (m >> 2)]) {
                const double4* g = cell_ptr(P, p, n, m);
                cp_async16(sv + lo(n, 0) + m, g);
                cp_async16(reinterpret_cast<uint8_t*>(sv + lo(n, 0) + m) + 16, reinterpret_cast<const uint8_t*>(g) + 16);
            }
    }
    unsigned tree = 0, nnear = 0, ndem = 0;
    {
        // level R-1: children from every subtree's partition
        const int n = R - 1;
        const uint32_t cnt = 1u << (2 * n);
        for (uint32_t m0 = 0; m0 < cnt; m0 += kThreads) {
            const uint32_t m = m0 + threadIdx.x;
            if (m >= cnt) break;
            const bool sp = sf[slo(n) + m] != 0;
            const bool need = !sp && n > 0 && sf[slo(n - 1) + (m >> 2)];
            double4 c[4], v = make_double4(0.0, 0.0, 0.0, 0.0);
            if (sp) {
                c[0] = ld4_cg(cell_ptr(P, p, n + 1, 4u * m)); c[1] = ld4_cg(cell_ptr(P, p, n + 1, 4u * m + 1));
                c[2] = ld4_cg(cell_ptr(P, p, n + 1, 4u * m + 2)); c[3] = ld4_cg(cell_ptr(P, p, n + 1, 4u * m + 3));
            } else if (need) {
                v = ld4_cg(cell_ptr(P, p, n, m));
            }
            bool flow = 0.0 >= s_thr[n][3];
            if (sp) {
                const Enc e = encode_children_t(c, s_thr[n], P);
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                v = e.par;
                st4(buf + cbase(n) + m, v);
                ++tree;
            }
            if (sp || need) sv[lo(n, 0) + m] = v;
            const uint8_t pr = (flow || sd[slo(n) + m]) ? 1 : 0;
            P.pre[slo(n) + m] = pr;
            if (P.top_band) sq[slo(n) + m] = pr;
        }
    }
    cp_async_wait_all();
    __syncthreads();
    for (int n = R - 2; n >= 0; --n) {
        const uint32_t cnt = 1u << (2 * n);
        for (uint32_t m = threadIdx.x; m < cnt; m += kThreads) {
            bool flow = 0.0 >= s_thr[n][3];
            if (sf[slo(n) + m]) {
                const uint32_t c0 = lo(n + 1, 0) + 4u * m;
                const double4 c[4] = {sv[c0], sv[c0 + 1], sv[c0 + 2], sv[c0 + 3]};
                const Enc e = encode_children_t(c, s_thr[n], P);
                flow = e.flow;
                nnear += e.near ? 1u : 0u;
                st4(buf + cbase(n) + m, e.par);
                sv[lo(n, 0) + m] = e.par;
                ++tree;
            }
            const uint8_t pr = (flow || sd[slo(n) + m]) ? 1 : 0;
            P.pre[slo(n) + m] = pr;
            if (P.top_band) sq[slo(n) + m] = pr;
        }
        __syncthreads();
    }
    const unsigned tt = block_sum(tree | (nnear << 16), s_red);  // (both < 2^16: R <= 6)
    if (threadIdx.x == 0 && (tt & 0xFFFFu)) atomicAdd(&ctl->cnt_tree, (unsigned long long)(tt & 0xFFFFu));
    if (P.part == 0) add_near(ctl, false, slot, tt >> 16);  // (replicated levels: partition 0 counts)
    if (P.top_band) {
        // band (D3) of every top cell, off K3's critical path: K3's top CTA
        // stages these and goes straight to the closure (level-R pre flags of
        // the neighbours come from K1, complete before K2 started)
        uint8_t* sigc = P.sig[p ^ 1];
        for (uint32_t q = threadIdx.x; q < lo(R, 0); q += kThreads) {
            const int n = (31 - __clz(3u * q + 1u)) >> 1;  // level of compact index q
            const uint32_t m = q - lo(n, 0);
            sigc[slo(n) + m] = band_flag(P.band_mode, P.L, n, m, [&](int k, uint32_t mm) -> uint8_t {
                return k < R ? sq[slo(k) + mm] : P.pre[slo(k) + mm];
            });
        }
    }
}


// ----------------------------------------------------------- decode helper
// decode_tree under D4 + PTT (Alg. 5) +
// compact_leaves. In physical units a zero-detail decode is
// a copy of the parent's (h, qx, qy) to its children, so a cell
// below a chain of newly significant cells takes the value of the chain's top.
// The bed elevation z of every cell is static — both copies hold the full
// hierarchy from initialise, FV1 writes a leaf's own z back and re-encoding
// averages unchanged children — so a projection writes h, qx, qy only and
// never reads the destination.
__device__ __forceinline__ double4 projection_source(const double4* buf, const Params& P, uint32_t src) {
    const int ns = zo::level_of(src);
    const int p = static_cast<int>(buf == P.cells[1]);
    return ld4_cg(cell_ptr(P, p, ns, src - zo::level_offset(ns)));
}
__device__ __forceinline__ void store_hqq(double4* dst, const double4& v) {
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(dst), "d"(v.x), "d"(v.y) : "memory");
    asm volatile("st.global.f64 [%0], %1;" ::"l"(reinterpret_cast<double*>(dst) + 2), "d"(v.z) : "memory");
}
__device__ __forceinline__ void write_projection(double4* buf, const Params& P, int n, uint32_t m, uint32_t src) {
    store_hqq(buf + cbase(n) + m, projection_source(buf, P, src));
}

// =========================================================================== K2
// band + ancestor closure of subtree j and its leaf
// counts, on 32-bit words: the word at slo(k) + 4b holds the flag bytes of
// the 2x2 block b of tile level k (Morton children 0..3 = SW, SE, NW, NE), so
// same-level face neighbours inside a block are byte swaps and the ones
// outside come from the four neighbouring blocks (neighbour_dev on the block
// index, or the halo word of the adjacent subtree). The subtree's pre-band
// flags and the halo (edge blocks of the four adjacent subtrees at every
// level, read from the owning partition) are staged up front. Counts follow
// from popcounts: a reached subtree with S significant cells (S_{L-1} on
// level L-1) has 4 S_{L-1} level-L leaves and 1 + 3 S - 4 S_{L-1} coarser
// ones. No last-CTA tail: levels < R are closed by every K3 CTA
// (traverse_tile); with do_top, block 0 is an extra CTA that re-encodes
// levels R-1..0 (encode_top_staged) concurrently.
//
// halo: direction d (W, E, N, S), level k >= 1, block position pos < 2^(k-1)
// along the edge at word hw(d, k, pos) = d (2^(K-1) - 1) + 2^(k-1) - 1 + pos;
// the adjacent subtrees' roots (level R) are bytes hr[d].
template <int KT>
__device__ void k2_tile(const Params& P, Ctl* ctl, const Head& hd, uint32_t j, uint8_t* smem2);

template <int KT>
__global__ void __launch_bounds__(kThreads, 8) k_band(Params P, Ctl* ctl, int force, int do_top) {
    // t, parity and step were written by the previous step's finalize, which
    // completed before K1 passed its wait: read them while K1 still runs
    // do_top: 1 = block 0 is the top encode (an extra CTA); 2 = the top
    // encode is k_band_top, launched just before: this grid was launched
    // once it passed its wait for K1 (K1's results are visible) and waits
    // for it at the end, so K3 sees both
    const Head hd = cta_head(ctl, P, force != 0);
    extern __shared__ __align__(16) uint8_t smem2[];
    const bool top = do_top == 1 && blockIdx.x == 0;
    if (top && hd.active) encode_top_prestage(P, hd.parity, smem2);  // (the top encode is K2's longest chain)
    if (do_top != 2) pdl_wait();
    pdl_trigger();
    if (!hd.active) {
        if (top) cp_async_wait_all();
        if (do_top == 2) pdl_wait();
        return;
    }
    tl_start(ctl, hd.buf, 1);
    if (top) {
        encode_top_staged(P, ctl, hd.parity, hd.buf, smem2, true);
        return;
    }
    k2_tile<KT>(P, ctl, hd, P.tile_lo + blockIdx.x - (do_top == 1 ? 1u : 0u), smem2);
    if (do_top == 2) pdl_wait();
}

// K2's top encode (levels R-1..0 re-encoded and banded) as its own launch in
// front of the subtree grid, with a shared-memory request that keeps other
// CTAs off its SM: as block 0 of K2 it shared an SM with seven subtree CTAs
// and its chain (~8.6 us at L = 11) bounded K2's end. It triggers the
// subtree grid right after its wait for K1 (measured: the subtree grid
// first, then this kernel, started K3 1.5 us later)
__global__ void __launch_bounds__(kThreads, 1) k_band_top(Params P, Ctl* ctl) {
    const Head hd = cta_head(ctl, P, false);
    extern __shared__ __align__(16) uint8_t smem2t[];
    if (hd.active) encode_top_prestage(P, hd.parity, smem2t);
    pdl_wait();
    pdl_trigger();
    if (!hd.active) {
        cp_async_wait_all();
        return;
    }
    encode_top_staged(P, ctl, hd.parity, hd.buf, smem2t, true);
}

// the subtree part of K2 (band, closure, counts, stores); leaves the final
// flags of the subtree in smem2 + slo(K) (slo layout)
template <int KT>
__device__ void k2_tile(const Params& P, Ctl* ctl, const Head& hd, uint32_t j, uint8_t* smem2) {
    __shared__ unsigned s_red[32];
    __shared__ uint8_t hr[4];
    const int p = hd.parity;
    uint8_t* sigc = P.sig[p ^ 1];
    const int R = P.R;
    const int K = KT ? KT : P.K;
    const uint32_t hwd = (1u << (K - 1)) - 1u;          // halo words per direction
    uint8_t* spre = smem2;                              // pre-band flags, slo layout
    uint8_t* sf = spre + slo(K);                        // band, then final flags, slo layout
    __shared__ uint32_t halo[4 * 31];                   // 4 * hwd words (K <= 6)
    const int mode = P.band_mode;

    // ---- one round trip: own pre flags (async) + halo words (one per thread)
    //      (+ qskip: the previous tree's flags of the subtree, for the change test)
    const uint8_t f0 = stage_tile_flags<KT>(spre, P.pre, P, j);
    uint8_t* sprev = spre + 2 * slo(K);
    const uint8_t o0 = P.qskip ? stage_tile_flags<KT>(sprev, P.sig[p], P, j) : 0;
    const uint32_t hi = threadIdx.x;
    uint32_t hv = 0;
    if (mode != 0 && hi < 4u * hwd) {
        const int d = static_cast<int>(hi / hwd);
        const uint32_t r = hi - static_cast<uint32_t>(d) * hwd;
        const int k = 32 - __clz(r + 1u);               // level k >= 1 of this halo word
        const uint32_t pos = r + 1u - (1u << (k - 1)), sb = 1u << (k - 1);
        const uint32_t jn = zo::neighbour_dev(R, j, static_cast<zo::Direction>(d));
        if (jn != zo::kNone) {
            // the adjacent subtree's edge blocks: W -> its east column, E -> its
            // west column, N -> its south row, S -> its north row
            const uint32_t bx = (d == 0) ? sb - 1u : (d == 1) ? 0u : pos;
            const uint32_t by = (d == 2) ? 0u : (d == 3) ? sb - 1u : pos;
            const unsigned long long g =
                slo(R + k) + (static_cast<unsigned long long>(jn) << (2 * k)) + 4ull * zo::interleave(bx, by);
            hv = *reinterpret_cast<const uint32_t*>(P.ppre[owner_of(P, R, jn)] + g);
        }
    } else if (mode != 0 && hi >= 128 && hi < 132) {
        const int d = static_cast<int>(hi - 128);
        const uint32_t jn = zo::neighbour_dev(R, j, static_cast<zo::Direction>(d));
        hv = (jn != zo::kNone) ? P.ppre[owner_of(P, R, jn)][slo(R) + jn] : 0u;
    }
    cp_async_wait_all();
    if (threadIdx.x == 0) spre[0] = f0;
    if (mode != 0 && hi < 4u * hwd) halo[hi] = hv;
    if (mode != 0 && hi >= 128 && hi < 132) hr[hi - 128] = static_cast<uint8_t>(hv);
    __syncthreads();

    // pre flag of the level-k cell at local (x, y) (possibly one step outside)
    auto pre_cell = [&](int k, int x, int y) -> uint32_t {
        const int s = 1 << k;
        int d = -1;
        if (x < 0) d = 0; else if (x >= s) d = 1; else if (y >= s) d = 2; else if (y < 0) d = 3;
        if (d < 0) return spre[slo(k) + zo::interleave(x, y)];
        if (k == 0) return hr[d];
        const int xo = (x + s) & (s - 1), yo = (y + s) & (s - 1);  // cell inside the adjacent subtree
        const uint32_t pos = (d < 2) ? static_cast<uint32_t>(yo >> 1) : static_cast<uint32_t>(xo >> 1);
        const uint32_t w = halo[static_cast<uint32_t>(d) * hwd + (1u << (k - 1)) - 1u + pos];
        return (w >> (8 * (((yo & 1) << 1) | (xo & 1)))) & 0xFFu;
    };

    // ---- band (D3)
    if (mode == 2) {
        if (threadIdx.x == 0) sf[0] = (spre[0] | hr[0] | hr[1] | hr[2] | hr[3]) ? 1 : 0;
#pragma unroll
        for (int k = 1; k < (KT ? KT : kMaxL); ++k) {
            if (!KT && k >= K) break;
            const uint32_t nw = 1u << (2 * (k - 1));
            const uint32_t sb = 1u << (k - 1);                        // blocks per side
            const uint32_t* wk = reinterpret_cast<const uint32_t*>(spre + slo(k));
            const uint32_t* hk = halo + (sb - 1u);                    // + d * hwd + pos
            for (uint32_t b = threadIdx.x; b < nw; b += kThreads) {
                const uint32_t w = wk[b];
                // neighbouring blocks by dilated-integer steps on the Morton
                // index (x bits even, y bits odd); the de-interleaved
                // coordinates only for the halo words on the subtree's edge
                constexpr uint32_t xm = 0x55555555u, ym = 0xAAAAAAAAu;
                const uint32_t bxm = b & xm, bym = b & ym, top = nw - 1u;
                const bool hw = bxm == 0u, he = bxm == (xm & top), hs = bym == 0u, hn = bym == (ym & top);
                const uint32_t bx = (hs || hn) ? zo::compact_bits(b) : 0u;
                const uint32_t by = (hw || he) ? zo::compact_bits(b >> 1) : 0u;
                const uint32_t ww = !hw ? wk[((bxm - 1u) & xm) | bym] : hk[by];
                const uint32_t we = !he ? wk[(((b | ym) + 1u) & xm) | bym] : hk[hwd + by];
                const uint32_t wn = !hn ? wk[(((b | xm) + 1u) & ym) | bxm] : hk[2u * hwd + bx];
                const uint32_t ws = !hs ? wk[((bym - 1u) & ym) | bxm] : hk[3u * hwd + bx];
                uint32_t o = w | ((w >> 8) & 0x00FF00FFu) | ((w << 8) & 0xFF00FF00u) | (w >> 16) | (w << 16);
                o |= (ww >> 8) & 0x00FF00FFu;   // W block: its SE, NE
                o |= (we << 8) & 0xFF00FF00u;   // E block: its SW, NW
                o |= wn << 16;                  // N block: its SW, SE
                o |= ws >> 16;                  // S block: its NW, NE
                *reinterpret_cast<uint32_t*>(sf + slo(k) + 4u * b) = o;
            }
        }
    } else {
        for (int k = 0; k < K; ++k) {
            const uint32_t cnt = 1u << (2 * k);
            for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
                uint32_t b = spre[slo(k) + pi];
                if (mode == 1 && k + 1 < K) {
                    const int x = static_cast<int>(zo::compact_bits(pi)), y = static_cast<int>(zo::compact_bits(pi >> 1));
                    for (int q = 0; q < 4; ++q) {
                        const int cx = 2 * x + (q & 1), cy = 2 * y + (q >> 1);
                        b |= pre_cell(k + 1, cx - 1, cy) | pre_cell(k + 1, cx + 1, cy) | pre_cell(k + 1, cx, cy + 1) |
                             pre_cell(k + 1, cx, cy - 1);
                    }
                }
                sf[slo(k) + pi] = b ? 1 : 0;
            }
        }
    }
    __syncthreads();
    // ---- ancestor closure bottom-up: a cell is significant if its band flag
    //      or any child is; byte-per-cell words of level k from level k + 1
    auto nz = [](uint32_t w) -> uint32_t { return w ? 1u : 0u; };
    // levels with more than 32 words: every thread, CTA barrier per level;
    // the rest (<= 32 words, k <= 3) by warp 0 with warp barriers
#pragma unroll
    for (int k = (KT ? KT : kMaxL) - 2; k >= 0; --k) {
        if (!KT && k > K - 2) continue;
        const bool wide = k >= 4;  // 4^(k-1) > 32 words
        if (!wide && threadIdx.x >= 32) continue;
        if (k == 0) {
            if (threadIdx.x == 0) sf[0] = (sf[0] | nz(*reinterpret_cast<const uint32_t*>(sf + slo(1)))) ? 1 : 0;
        } else {
            const uint32_t nw = 1u << (2 * (k - 1));
            for (uint32_t b = threadIdx.x; b < nw; b += kThreads) {
                const uint4 c = *reinterpret_cast<const uint4*>(sf + slo(k + 1) + 16u * b);
                uint32_t* w = reinterpret_cast<uint32_t*>(sf + slo(k) + 4u * b);
                *w |= nz(c.x) | (nz(c.y) << 8) | (nz(c.z) << 16) | (nz(c.w) << 24);
            }
        }
        if (wide) __syncthreads();
        else __syncwarp();
    }
    __syncthreads();
    // ---- final flags (word stores), leaf counts from popcounts
    unsigned S = 0, S1 = 0;
    int chg = 0;  // (qskip) the subtree's final flags differ from the previous tree's
    if (threadIdx.x == 0) {
        sigc[slo(R) + j] = sf[0];
        S = sf[0];
        if (K == 1) S1 = sf[0];
        if (P.qskip) chg = sf[0] != o0;
    }
#pragma unroll
    for (int k = 1; k < (KT ? KT : kMaxL); ++k) {
        if (!KT && k >= K) break;
        const uint32_t nw = 1u << (2 * (k - 1));
        const unsigned long long g = slo(R + k) + (static_cast<unsigned long long>(j) << (2 * k));
        for (uint32_t b = threadIdx.x; b < nw; b += kThreads) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(sf + slo(k) + 4u * b);
            *reinterpret_cast<uint32_t*>(sigc + g + 4u * b) = w;
            if (P.qskip) chg |= (w != *reinterpret_cast<const uint32_t*>(sprev + slo(k) + 4u * b)) ? 1 : 0;
            const unsigned c = __popc(w);
            S += c;
            if (k == K - 1) S1 += c;
        }
    }
    if (P.qskip) {
        chg = __syncthreads_or(chg);
        if (threadIdx.x == 0) P.tchg[j] = chg ? 1 : 0;
    }
    // one block sum of both counts (S <= 4^K / 3 < 2^16)
    const unsigned SS = block_sum(S | (S1 << 16), s_red);
    const unsigned St = SS & 0xFFFFu, S1t = SS >> 16;
    if (threadIdx.x == 0) {
        P.tile_cnt[j] = 4u * S1t;
        P.tile_cnt[P.n_tiles + j] = 1u + 3u * St - 4u * S1t;
    }
    tl_end(ctl, hd.buf, 1);
}

// K3 = decode (projection, D4) + PTT (Alg. 5) + compaction
// (SPEC.md:236-244). Block 0 is the top CTA: it builds the top of the tree
// once (band + closure of levels < R from the pre-band flags, on-tree flags,
// every subtree's leaf counts, their scans into list offsets, each
// subtree's traversal depth and decode source, the projection of top
// cells) and publishes it with a release flag. The subtree CTAs meanwhile
// stage their own flags and count their leaves, then wait only for their
// offsets. Block 0 is dispatched first, so the wait cannot deadlock.
//
// Per-subtree results: tile_off[t] / [nt + t] = list A / B offsets (hot path),
// [2 nt + t] = Morton export offset; tile_lvl[t] = depth (R: reached) | 0x100
// if t is the first subtree under its covering top-level leaf; tile_src[t] =
// decode source of a reached root (kNoSrc: none).
constexpr uint32_t kEmit = 0x100u;
constexpr uint32_t kTileSub = 0x200u;  // the subtree is on FV1's tile path: no list-A leaves emitted
constexpr uint32_t kSkipSub = 0x400u;  // a stable quiet subtree FV1 skips: no leaves emitted

__device__ __forceinline__ void k3_publish(Ctl* ctl, unsigned long long epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release_u64(&ctl->k3_ready, epoch);
    }
}
__device__ __forceinline__ void k3_wait(const Ctl* ctl, unsigned long long epoch) {
    if (threadIdx.x == 0) {
        while (ld_acquire_u64(&ctl->k3_ready) != epoch) __nanosleep(64);
    }
    __syncthreads();
}

// top of the tree (block 0 of K3); top flags at the padded offsets slo(n)
// activity of subtree t from any-wet marks w[] and quadrant marks qw[]
// (qact): t itself wet, an inflow edge, or — per face neighbour — its two
// quadrants facing t wet (t's root refined) / any of it wet (root not refined)
__device__ __forceinline__ uint8_t activity_q(const Params& P, uint32_t t, const uint8_t* w, const uint8_t* qw,
                                              bool root_refined) {
    uint8_t act = w[t];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        const uint32_t nb = zo::neighbour_dev(P.R, t, static_cast<zo::Direction>(d));
        if (nb == zo::kNone) {
            act |= (P.bc[d] == 2) ? 1 : 0;
        } else if (!root_refined) {
            act |= w[nb];
        } else {
            // the neighbour's quadrants facing t: W neighbour -> its SE, NE
            // (1, 3); E -> SW, NW (0, 2); N -> SW, SE (0, 1); S -> NW, NE (2, 3)
            const uint32_t qa = (d == 0) ? 1u : (d == 1) ? 0u : (d == 2) ? 0u : 2u;
            const uint32_t qb = (d == 0) ? 3u : (d == 1) ? 2u : (d == 2) ? 1u : 3u;
            act |= qw[4u * nb + qa] | qw[4u * nb + qb];
        }
    }
    return act ? 1 : 0;
}
// shared-memory offsets of k3_top's staged arrays (also used by the split
// top's pre-wait staging)
struct K3TopLayout {
    uint32_t tv, swet, qst, sqw, sqn;  // previous top flags, wet marks, quiet-skip state, quadrant wet marks,
                                       // skipped subtrees' cached FV1 near counts
};
__host__ __device__ __forceinline__ K3TopLayout k3_top_layout(int R, uint32_t nt) {
    const uint32_t fb = slo(R), ftop = (fb + nt + 15u) & ~15u, pnt = (nt + 15u) & ~15u;
    const uint32_t tv = 2 * ftop + pnt + fb;
    const uint32_t swet = tv + fb;
    const uint32_t scnt = swet + pnt;
    const uint32_t sres = scnt + 4u * 2u * nt;
    const uint32_t nr1 = R >= 1 ? (1u << (2 * (R - 1))) : 1u;
    const uint32_t sdep = sres + 4u * 4u * nt + 4u * nr1;
    const uint32_t stl = sdep + ((nr1 + 15u) & ~15u);
    return {tv, swet, stl + 3u * pnt, stl + 4u * pnt, stl + 8u * pnt};
}
// the split top's staging that does not depend on K1 / K2 (previous top flags,
// the previous FV1's wet marks, the quiet-skip state), issued before the PDL
// wait while K2 runs (one partition, staged top)
template <int NT>
__device__ __forceinline__ void k3_top_prestage(const Params& P, int p, int tbuf, uint8_t* sm) {
    const uint32_t nt = static_cast<uint32_t>(P.n_tiles);
    const K3TopLayout ly = k3_top_layout(P.R, nt);
    stage16<NT>(sm + ly.tv, P.sig[p], slo(P.R));
    stage16<NT>(sm + ly.swet, P.wet[tbuf], nt);
    if (P.qskip) stage16<NT>(sm + ly.qst, P.qstate, nt);
    if (P.qact) stage16<NT>(sm + ly.sqw, P.qwet[tbuf], 4u * nt);
    if (P.qskip) stage16<NT>(sm + ly.sqn, reinterpret_cast<const uint8_t*>(P.qnfv), 4u * nt);
}
template <bool EXPORT, int NT = kThreads>
__device__ void k3_top(const Params& P, Ctl* ctl, int p, int tbuf, unsigned long long epoch, uint8_t* sm,
                       const Probe& stamp, bool band_done = false, bool staged_out = false, bool prestaged = false,
                       bool tact_by_subtrees = false) {
    __shared__ unsigned s_red[32];
    __shared__ unsigned s_off[6];
    const uint8_t* sigc = EXPORT ? P.sig[p] : P.sig[p ^ 1];
    const uint8_t* sigp = EXPORT ? P.sig[p ^ 1] : P.sig[p];
    const int L = P.L, R = P.R;
    const uint32_t nt = static_cast<uint32_t>(P.n_tiles);
    const uint32_t fb = slo(R);  // top flag bytes of levels 0..R-1
    const uint32_t ftop = (fb + nt + 15u) & ~15u;
    uint8_t* ts = sm;             // flags of levels 0..R
    uint8_t* ti = ts + ftop;      // on the tree, levels 0..R
    uint8_t* cbf = ti + ftop;     // first subtree under a top-level leaf
    uint8_t* tp = cbf + ((nt + 15u) & ~15u);
    uint8_t* tv = tp + fb;
    uint8_t* swet = tv + fb;      // wet subtrees after the previous FV1
    uint32_t* scnt = reinterpret_cast<uint32_t*>(swet + ((nt + 15u) & ~15u));
    uint32_t* sres = scnt + 2 * nt;  // staged_out: A / B offset, depth, source per subtree (caller sized it)
    // staged_out: per level-(R-1) cell (shared by its 4 subtrees) the depth a
    // non-reached subtree below it stops at and the decode source
    uint32_t* ssrc = sres + 4 * nt;
    uint8_t* sdep = reinterpret_cast<uint8_t*>(ssrc + (R >= 1 ? (1u << (2 * (R - 1))) : 1u));
    // (tiles: subtrees FV1 updates on its tile path, hot path of a staged top only)
    uint8_t* stl = sdep + (((R >= 1 ? (1u << (2 * (R - 1))) : 1u) + 15u) & ~15u);
    const bool tiles = !EXPORT && staged_out && P.tiles;
    __shared__ unsigned s_ntile;
    const bool cnt_smem = nt <= 1024u;
    const uint32_t* cnt = cnt_smem ? scnt : P.tile_cnt;
    const uint32_t al = P.G == 1 ? 16u : P.pb_align;
    const int rb = EXPORT ? p : p ^ 1;

    // ---- stage (one round trip)
    if (EXPORT || band_done) stage16<NT>(ts, sigc, fb);  // (band_done: K2's extra CTA banded the top cells)
    if (!EXPORT) {
        if (!band_done) stage16<NT>(tp, P.pre, fb);
        if (!prestaged) stage16<NT>(tv, sigp, fb);
        if (staged_out && P.qskip) {  // (quiet-skip state of every subtree, read by the quiet split)
            uint8_t* qc = stl + 2 * ((nt + 15u) & ~15u);
            if (nt >= 16u) {
                stage16<NT>(qc, P.tchg, nt);
                if (!prestaged) stage16<NT>(qc + ((nt + 15u) & ~15u), P.qstate, nt);
            } else if (threadIdx.x < nt) {
                qc[threadIdx.x] = P.tchg[threadIdx.x];
                if (!prestaged) qc[((nt + 15u) & ~15u) + threadIdx.x] = P.qstate[threadIdx.x];
            }
        }
        if (prestaged) {
        } else if (P.G > 1) {  // a partition marks every subtree under its wet leaves: OR over the partitions
            for (uint32_t t = threadIdx.x; t < nt; t += NT) {
                uint8_t v = 0;
                for (int g = 0; g < P.G; ++g) v |= P.pwet[g][tbuf][t];
                swet[t] = v;
            }
        } else if (nt >= 16u) {
            stage16<NT>(swet, P.wet[tbuf], nt);
        } else if (threadIdx.x < nt) {
            swet[threadIdx.x] = P.wet[tbuf][threadIdx.x];
        }
    }
    uint8_t r0 = 0;
    if (nt == 1u) {
        if (threadIdx.x == 64) r0 = P.psig[0][rb][slo(R)];
    } else if (al >= 16u) {
        for (uint32_t q = 16u * threadIdx.x; q < nt; q += 16u * NT)
            cp_async16(ts + fb + q, P.psig[owner_of(P, R, q)][rb] + slo(R) + q);
    } else if (al >= 4u) {
        for (uint32_t q = 4u * threadIdx.x; q < nt; q += 4u * NT)
            cp_async4(ts + fb + q, P.psig[owner_of(P, R, q)][rb] + slo(R) + q);
    } else {  // small partitioned grids (tests): plain byte copies
        for (uint32_t q = threadIdx.x; q < nt; q += NT)
            ts[fb + q] = P.psig[owner_of(P, R, q)][rb][slo(R) + q];
    }
    if (cnt_smem) {
        if (P.G == 1 && (nt & 3u) == 0u) {
            for (uint32_t q = 4u * threadIdx.x; q < 2u * nt; q += 4u * NT) cp_async16(scnt + q, P.tile_cnt + q);
        } else {
            for (uint32_t q = threadIdx.x; q < 2u * nt; q += NT) {
                const uint32_t t = q < nt ? q : q - nt;
                cp_async4(scnt + q, P.ptile_cnt[owner_of(P, R, t)] + q);
            }
        }
    }
    for (uint32_t q = threadIdx.x; q < nt; q += NT) cbf[q] = 0;
    cp_async_wait_all();
    __shared__ unsigned s_nwet;  // wet subtrees (R = 5 closure path), else ~0
    if (threadIdx.x == 0) {
        s_nwet = (!EXPORT && R == 5 && NT > 32) ? 0u : ~0u;
        s_ntile = 0u;  // (before the barrier below: the tile listing appends without one)
    }
    if (threadIdx.x == 64 && nt == 1u) ts[fb] = r0;
    __syncthreads();
    stamp(0);

    // ---- band (D3) of every top cell at once (band depends on pre flags only)
    if (!EXPORT && !band_done) {
        for (uint32_t q = threadIdx.x; q < lo(R, 0); q += NT) {
            const int n = (31 - __clz(3u * q + 1u)) >> 1;  // level of compact index q
            const uint32_t m = q - lo(n, 0);
            ts[slo(n) + m] = band_flag(P.band_mode, L, n, m, [&](int k, uint32_t mm) -> uint8_t {
                return k < R ? tp[slo(k) + mm] : P.ppre[owner_of(P, k, mm)][slo(k) + mm];
            });
        }
    }
    __syncthreads();
    stamp(1);
    unsigned tn = 0;
    const uint8_t* reach = ti + fb;
    if (!EXPORT && R == 5) {
        // L = 11 (1024 subtrees): closure, on-tree flags, first subtrees and
        // the newly significant count on bit masks in warp 0's registers
        // (level 5: 32 cells per lane; 4: 8; 3: 2; 2: one in lanes < 16; 1
        // and 0 in every lane), written back to the byte arrays once — the
        // same flags the generic pass below produces
        __shared__ unsigned s_tn;
        if (threadIdx.x >= 32) {  // meanwhile: the wet subtrees (the tile listing's density test)
            unsigned nw = 0;
            for (uint32_t t = threadIdx.x - 32; t < nt; t += NT - 32) nw += swet[t] ? 1u : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nw += __shfl_xor_sync(kFull, nw, o);
            if ((threadIdx.x & 31) == 0 && nw) atomicAdd(&s_nwet, nw);
        }
        if (threadIdx.x < 32) {
            const uint32_t l = threadIdx.x;
            auto bits4 = [](uint32_t x) { return ((x * 0x01020408u) >> 24) & 0xFu; };  // 4 bytes (0/1) -> 4 bits
            auto bytes4 = [](uint32_t b) { return (b * 0x00204081u) & 0x01010101u; };  // 4 bits -> 4 bytes
            auto any_nib = [](uint32_t w, int n) {  // bit c = nibble c of w nonzero, c < n
                const uint32_t t = w | (w >> 1) | (w >> 2) | (w >> 3);
                uint32_t r = 0;
                for (int c = 0; c < n; ++c) r |= ((t >> (4 * c)) & 1u) << c;
                return r;
            };
            // level 5 (subtree roots, K2's final flags)
            const uint4 a5 = *reinterpret_cast<const uint4*>(ts + slo(5) + 32u * l);
            const uint4 b5 = *reinterpret_cast<const uint4*>(ts + slo(5) + 32u * l + 16u);
            const uint32_t w5 = bits4(a5.x) | (bits4(a5.y) << 4) | (bits4(a5.z) << 8) | (bits4(a5.w) << 12) |
                                (bits4(b5.x) << 16) | (bits4(b5.y) << 20) | (bits4(b5.z) << 24) | (bits4(b5.w) << 28);
            // closure bottom-up: band | any child
            const uint2 q4 = *reinterpret_cast<const uint2*>(ts + slo(4) + 8u * l);
            const uint32_t s4 = (bits4(q4.x) | (bits4(q4.y) << 4)) | any_nib(w5, 8);
            const uint32_t s3 = (ts[slo(3) + 2u * l] | (ts[slo(3) + 2u * l + 1u] << 1)) | any_nib(s4, 2);
            const uint32_t x3 = s3 | (__shfl_down_sync(kFull, s3, 1) << 2);  // lane 2c: level-3 cells 4c..4c+3
            const uint32_t x3c = __shfl_sync(kFull, x3, (2u * l) & 31u);  // (every lane shuffles)
            const uint32_t s2l = (l < 16u) ? (ts[slo(2) + l] | (x3c ? 1u : 0u)) : 0u;
            const uint32_t m2 = __ballot_sync(kFull, s2l != 0u) & 0xFFFFu;                   // level 2, 16 bits
            const uint32_t b1 = ts[slo(1)] | (ts[slo(1) + 1] << 1) | (ts[slo(1) + 2] << 2) | (ts[slo(1) + 3] << 3);
            const uint32_t s1 = b1 | any_nib(m2, 4);
            const uint32_t s0 = (ts[0] | (s1 ? 1u : 0u)) & 1u;
            // on-tree top-down: a child is on the tree iff its parent is on it and significant
            const uint32_t in1 = s0 ? 0xFu : 0u;
            uint32_t in2 = 0;
            for (int c = 0; c < 16; ++c) in2 |= (((in1 & s1) >> (c >> 2)) & 1u) << c;
            const uint32_t par3 = l >> 1;  // this lane's level-3 cells 2l, 2l+1 share a parent
            const uint32_t in3 = (((in2 & m2) >> par3) & 1u) ? 3u : 0u;
            const uint32_t on3 = in3 & s3;
            const uint32_t in4 = ((on3 & 1u) ? 0xFu : 0u) | ((on3 & 2u) ? 0xF0u : 0u);
            const uint32_t on4 = in4 & s4;
            uint32_t in5 = 0;
            for (int j = 0; j < 8; ++j) in5 |= ((on4 >> j) & 1u) ? (0xFu << (4 * j)) : 0u;
            // write back: closure (ts) and on-tree (ti) bytes, first subtrees (cbf)
            *reinterpret_cast<uint2*>(ts + slo(4) + 8u * l) = make_uint2(bytes4(s4 & 0xFu), bytes4(s4 >> 4));
            *reinterpret_cast<uint2*>(ti + slo(4) + 8u * l) = make_uint2(bytes4(in4 & 0xFu), bytes4(in4 >> 4));
            uint32_t* t5 = reinterpret_cast<uint32_t*>(ti + slo(5) + 32u * l);
#pragma unroll
            for (int k = 0; k < 8; ++k) t5[k] = bytes4((in5 >> (4 * k)) & 0xFu);
            ts[slo(3) + 2u * l] = s3 & 1u;
            ts[slo(3) + 2u * l + 1u] = (s3 >> 1) & 1u;
            ti[slo(3) + 2u * l] = in3 & 1u;
            ti[slo(3) + 2u * l + 1u] = (in3 >> 1) & 1u;
            if (l < 16u) {
                ts[slo(2) + l] = (m2 >> l) & 1u;
                ti[slo(2) + l] = (in2 >> l) & 1u;
                if ((in2 >> l) & 1u && !((m2 >> l) & 1u)) cbf[l << 6] = 1;
            }
            if (l < 4u) {
                ts[slo(1) + l] = (s1 >> l) & 1u;
                ti[slo(1) + l] = (in1 >> l) & 1u;
                if ((in1 >> l) & 1u && !((s1 >> l) & 1u)) cbf[l << 8] = 1;
            }
            if (l == 0u) {
                ts[0] = static_cast<uint8_t>(s0);
                ti[0] = 1;
                if (!s0) cbf[0] = 1;
            }
            for (int k = 0; k < 2; ++k)
                if (((in3 >> k) & 1u) && !((s3 >> k) & 1u)) cbf[(2u * l + k) << 4] = 1;
            for (int j = 0; j < 8; ++j)
                if (((in4 >> j) & 1u) && !((s4 >> j) & 1u)) cbf[(8u * l + j) << 2] = 1;
            // newly significant top cells (significant now, not in the previous tree)
            const uint2 v4 = *reinterpret_cast<const uint2*>(tv + slo(4) + 8u * l);
            const uint32_t t4 = bits4(v4.x) | (bits4(v4.y) << 4);
            const uint32_t t3 = tv[slo(3) + 2u * l] | (tv[slo(3) + 2u * l + 1u] << 1);
            unsigned nn = __popc(s4 & ~t4) + __popc(s3 & ~t3);
            if (l < 16u) nn += ((m2 >> l) & 1u) && !tv[slo(2) + l] ? 1u : 0u;
            if (l < 4u) nn += ((s1 >> l) & 1u) && !tv[slo(1) + l] ? 1u : 0u;
            if (l == 0u) nn += s0 && !tv[0] ? 1u : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(kFull, nn, o);
            if (l == 0u) s_tn = nn;
        }
        __syncthreads();
        tn = s_tn;
    } else {
        // ---- one warp: closure bottom-up (hot path), then the on-tree flags
        //      top-down and the first subtree under each top-level leaf (closure
        //      makes significance upward-closed: a cell is on the tree iff its
        //      parent is significant and on it); the other warps clear cbf
        // closure of level R-1 (the largest) by every thread, the rest by warp 0
        if (!EXPORT && R >= 1) {
            for (uint32_t m = threadIdx.x; m < (1u << (2 * (R - 1))); m += NT)
                if (*reinterpret_cast<const uint32_t*>(ts + slo(R) + 4u * m)) ts[slo(R - 1) + m] = 1;
            __syncthreads();
        }
        auto ontree = [&](int n, uint32_t m) {
            const bool in = ti[slo(n) + m] != 0, sg = ts[slo(n) + m] != 0;
            *reinterpret_cast<uint32_t*>(ti + slo(n + 1) + 4u * m) = (in && sg) ? 0x01010101u : 0u;
            if (in && !sg) cbf[m << (2 * (R - n))] = 1;
        };
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            if (!EXPORT)
                for (int n = R - 2; n >= 0; --n) {
                    for (uint32_t m = lane; m < (1u << (2 * n)); m += 32)
                        if (*reinterpret_cast<const uint32_t*>(ts + slo(n + 1) + 4u * m)) ts[slo(n) + m] = 1;
                    __syncwarp();
                }
            if (lane == 0) ti[0] = 1;
            __syncwarp();
            for (int n = 0; n < R - 1; ++n) {
                for (uint32_t m = lane; m < (1u << (2 * n)); m += 32) ontree(n, m);
                __syncwarp();
            }
        }
        __syncthreads();
        // on-tree flags of level R (subtree roots) from level R-1, every thread
        if (R >= 1) {
            for (uint32_t m = threadIdx.x; m < (1u << (2 * (R - 1))); m += NT) ontree(R - 1, m);
            __syncthreads();
        } else if (threadIdx.x == 0) {
            ti[0] = 1;
        }
        if (R == 0) __syncthreads();
        // newly significant top cells (decode sources exist only below them)
        unsigned nnew = 0;
        if (!EXPORT)
            for (uint32_t q = threadIdx.x; q < lo(R, 0); q += NT) {
                const int n = (31 - __clz(3u * q + 1u)) >> 1;
                const uint32_t a = slo(n) + (q - lo(n, 0));
                nnew += (ts[a] && !tv[a]) ? 1u : 0u;
            }
        tn = EXPORT ? 0u : block_sum<NT>(nnew, s_red);
    }

    stamp(2);

    // ---- per-subtree counts, scans, depth and decode source
    const uint32_t per = (nt + NT - 1) / NT;
    const uint32_t a = threadIdx.x * per;
    const uint32_t b = min(nt, a + per);
    // FV1 tile path (k_fv1 fv1_tile_strip): a reached subtree whose 4^K
    // level-L cells are all leaves and whose neighbourhood holds a wet cell
    // (or touches an inflow edge) is updated as a 64 x 64 block; its leaves
    // leave list A (counted in n_leaves all the same) and it joins P.stile
    bool dense = false;
    if (tiles) {
        // which fully refined subtrees take the tile path: when most subtrees
        // hold wet cells (a wet-dominated domain), every active one (it or a
        // face neighbour wet, or an inflow edge); otherwise only those inside
        // the wet region (it and all its face neighbours wet) — where the wet
        // cells are sparse the per-leaf path's per-cell dry shortcut is
        // cheaper than a strip's rows (measured: config 5 91 vs 104 us/step
        // with every active subtree tiled; the Monai-like runup 139 vs 157).
        // Decided per subtree in the counts pass below.
        if (s_nwet != ~0u) {  // (counted by warps 1.. during warp 0's closure)
            dense = 2u * s_nwet > nt;
        } else {
            unsigned nw = 0;
            for (uint32_t t = a; t < b; ++t) nw += swet[t] ? 1u : 0u;
            dense = 2u * block_sum<NT>(nw, s_red) > nt;
        }
    }
    // FV1 tile path (k_fv1 fv1_tile_strip): a reached subtree whose 4^K
    // level-L cells are all leaves and whose neighbourhood holds a wet cell
    // (or touches an inflow edge) is updated as a 64 x 64 block; its leaves
    // leave list A (counted in n_leaves all the same) and it joins P.stile
    // (appended warp-aggregated, any order: each strip job writes its own cells)
    auto tile_of = [&](uint32_t t) {
        bool tl = false;
        if (tiles) {
            bool inner;
            if (dense) {
                inner = swet[t] != 0;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const uint32_t nb = zo::neighbour_dev(R, t, static_cast<zo::Direction>(d));
                    if (nb == zo::kNone) inner = inner || P.bc[d] == 2;
                    else inner = inner || swet[nb] != 0;
                }
            } else {
                inner = swet[t] != 0;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const uint32_t nb = zo::neighbour_dev(R, t, static_cast<zo::Direction>(d));
                    inner = inner && (nb == zo::kNone || swet[nb] != 0);
                }
            }
            tl = inner && reach[t] && cnt[t] == (1u << (2 * P.K));
            stl[t] = tl ? 1 : 0;
            const unsigned am = __activemask();
            const unsigned bal = __ballot_sync(am, tl);
            if (bal) {
                const int lane = threadIdx.x & 31, lead = __ffs(am) - 1;
                unsigned base = 0;
                if (lane == lead) base = atomicAdd(&s_ntile, static_cast<unsigned>(__popc(bal)));
                base = __shfl_sync(am, base, lead);
                if (tl) P.stile[base + __popc(bal & ((1u << lane) - 1u))] = t;
            }
        }
        return tl;
    };
    // quiet split: a reached subtree whose neighbourhood held no wet cell
    // (the dry-shortcut activity, computed again for P.tact below) and that
    // is not on the tile path lists its leaves after the active ones
    const bool qs = !EXPORT && staged_out && P.qsplit;
    uint8_t* sq = stl + ((nt + 15u) & ~15u);
    const uint8_t* qchg = sq + ((nt + 15u) & ~15u);  // (staged with the wet marks)
    const uint8_t* qst = qchg + ((nt + 15u) & ~15u);
    const uint8_t* sqw = qst + ((nt + 15u) & ~15u);  // quadrant wet marks (qact; staged before the wait)
    const uint32_t* sqn = reinterpret_cast<const uint32_t*>(sqw + 4u * ((nt + 15u) & ~15u));  // (qskip, prestaged)
    const bool use_q = qs && P.qact && prestaged;
    auto counts = [&](uint32_t t, unsigned& ca, unsigned& cb) {
        const bool r = reach[t] != 0;
        ca = (r && !(tiles && stl[t])) ? cnt[t] : 0u;
        cb = r ? cnt[nt + t] : cbf[t];
    };
    // one pass per subtree: its counts, and (quiet split) its class — active,
    // quiet (sq = 1), or stable quiet and skipped (sq = 2)
    unsigned la = 0, lb = 0, lqa = 0, lqb = 0, lsk = 0, lska = 0, lskn = 0;
    for (uint32_t t = a; t < b; ++t) {
        const uint32_t qf = (qs && P.qskip) ? (prestaged ? sqn[t] : P.qnfv[t]) : 0u;
        tile_of(t);
        unsigned ca, cb;
        counts(t, ca, cb);
        uint8_t q = 0;
        if (qs) {
            uint8_t act;
            if (use_q) {
                act = activity_q(P, t, swet, sqw, ts[fb + t] != 0);
            } else {
                act = swet[t];
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const uint32_t nb = zo::neighbour_dev(R, t, static_cast<zo::Direction>(d));
                    if (nb == zo::kNone) act |= (P.bc[d] == 2) ? 1 : 0;
                    else act |= swet[nb];
                }
            }
            q = (reach[t] && !act && !(tiles && stl[t])) ? 1 : 0;
            if (P.qskip) {
                // consecutive steps quiet and unchanged; from the second one
                // on FV1 and the next K1 skip the subtree (sq = 2)
                const uint8_t qn = (q && !qchg[t]) ? static_cast<uint8_t>(min(qst[t] + 1, 3)) : 0;
                if (qn != qst[t]) P.qstate[t] = qn;
                if (qn >= 2) q = 2;
                else if (q) P.qnfv[t] = 0u;  // (the quiet pass counts this step's near cells afresh)
            }
            sq[t] = q;
        }
        if (q == 2) {  // skipped: on no list; its cached counts below
            lsk += ca + cb;
            lska += ca;
            lskn += qf;
        } else if (q) {
            lqa += ca;
            lqb += cb;
        } else {
            la += ca;
            lb += cb;
        }
    }
#ifdef SWAMP_EXP_K3X
    if (threadIdx.x == 0 && stamp.slot == 16) ctl->dbg[32 + 1] = gtimer();
#endif
    // per level-(R-1) cell (shared by its 4 subtrees): the depth a non-reached
    // subtree below it stops at and the decode source (read by the records
    // pass after the scan, whose barriers order them)
    if (staged_out && R >= 1) {
        for (uint32_t c = threadIdx.x; c < (1u << (2 * (R - 1))); c += NT) {
            int n = 0;
            while (n < R && ts[slo(n) + (c >> (2 * (R - 1 - n)))]) ++n;
            sdep[c] = static_cast<uint8_t>(n);
            uint32_t src = kNoSrc;
            if (!EXPORT && tn)
                for (int k = 0; k < R; ++k) {
                    const uint32_t q = slo(k) + (c >> (2 * (R - 1 - k)));
                    if (ts[q] && !tv[q]) {
                        src = zo::z_of(k, c >> (2 * (R - 1 - k)));
                        break;
                    }
                }
            ssrc[c] = src;
        }
    }
    __shared__ unsigned long long s_red64[3 * (NT / 32)];
    unsigned long long tot64, qtot64 = 0, o64, q64 = 0, sk64 = 0;
    if (qs) {  // active / quiet / skipped counts in one scan
        const unsigned long long v3[3] = {(static_cast<unsigned long long>(la) << 32) | lb,
                                          (static_cast<unsigned long long>(lqa) << 32) | lqb,
                                          (static_cast<unsigned long long>(lsk) << 32) | lska};
        unsigned long long o3[3], t3[3];
        block_exscan64x3<NT>(v3, s_red64, o3, t3);
        o64 = o3[0];
        tot64 = t3[0];
        q64 = o3[1];
        qtot64 = t3[1];
        sk64 = t3[2];
#ifdef SWAMP_EXP_K3X
    if (threadIdx.x == 0 && stamp.slot == 16) ctl->dbg[32 + 2] = gtimer();
#endif
    } else {
        o64 = block_exscan64<NT>((static_cast<unsigned long long>(la) << 32) | lb, s_red64, &tot64);
    }
    unsigned sk_leaves = 0;
    if (qs && P.qskip) {  // skipped subtrees' leaves and the counts FV1 would have added
        const unsigned s0 = static_cast<unsigned>(sk64 >> 32), s1 = static_cast<unsigned>(sk64);
        sk_leaves = s0;
        if (lskn) atomicAdd(&ctl->near_step[tbuf ^ 1], (unsigned long long)lskn);  // (rare)
        if (threadIdx.x == 0 && s0) {
            atomicAdd(&ctl->cnt_skip, (unsigned long long)s0);
            atomicAdd(&ctl->cnt_quiet, (unsigned long long)s0);
            atomicAdd(&ctl->cnt_fused, (unsigned long long)(s1 >> 2));
        }
    }
    // list layout: [A active | A quiet | B active | B quiet]
    const unsigned taa = static_cast<unsigned>(tot64 >> 32), tba = static_cast<unsigned>(tot64);
    const unsigned tqa = static_cast<unsigned>(qtot64 >> 32), tqb = static_cast<unsigned>(qtot64);
    const unsigned ta = taa + tqa, tb = tba + tqb;
    unsigned oa = static_cast<unsigned>(o64 >> 32), ob = static_cast<unsigned>(o64);
    unsigned oqa = taa + static_cast<unsigned>(q64 >> 32), oqb = tba + static_cast<unsigned>(q64);
    stamp(3);
    for (uint32_t t = a; t < b; ++t) {
        unsigned ca, cb;
        counts(t, ca, cb);
        const bool tsk = qs && sq[t] == 2;
        const bool tq = qs && sq[t] == 1;
        const unsigned xa = tq ? oqa : oa, xb = tq ? oqb : ob;  // this subtree's A / B offsets
        uint32_t src = kNoSrc;
        int n = R;
        if (staged_out && R >= 1) {  // (from the per-parent table above)
            if (!reach[t]) n = sdep[t >> 2];
            else src = ssrc[t >> 2];
        } else if (!reach[t]) {
            n = 0;
            while (ts[slo(n) + (t >> (2 * (R - n)))]) ++n;
        } else if (!EXPORT && tn) {
            for (int k = 0; k < R; ++k) {
                const uint32_t q = slo(k) + (t >> (2 * (R - k)));
                if (ts[q] && !tv[q]) {
                    src = zo::z_of(k, t >> (2 * (R - k)));
                    break;
                }
            }
        }
        if (!staged_out) {
            P.tile_lvl[t] = static_cast<uint32_t>(n) | (cbf[t] ? kEmit : 0u);
            P.tile_off[2 * nt + t] = oa + ob;
        }
        if (!EXPORT) {
            if (!staged_out) {
                P.tile_off[t] = oa;
                P.tile_off[nt + t] = ta + ob;
                P.tile_src[t] = src;
            }
            if (staged_out) {  // (staged in shared memory, written out coalesced below)
                sres[t] = xa;
                sres[nt + t] = ta + xb;
                sres[2 * nt + t] = static_cast<uint32_t>(n) | (cbf[t] ? kEmit : 0u) | ((tiles && stl[t]) ? kTileSub : 0u) |
                                   (tsk ? kSkipSub : 0u);
                sres[3 * nt + t] = src;
            } else {
                const unsigned long long tag = (epoch & 0xFFFFFFFFull) << 32;
                unsigned long long* rec = P.k3_rec + 4ull * t;
                st_relaxed_u64(rec + 0, tag | oa);
                st_relaxed_u64(rec + 1, tag | (ta + ob));
                st_relaxed_u64(rec + 2, tag | (static_cast<uint32_t>(n) | (cbf[t] ? kEmit : 0u)));
                st_relaxed_u64(rec + 3, tag | src);
            }
            if (t == P.tile_lo) {
                s_off[0] = oa;
                s_off[1] = ta + ob;
            }
            if (t == P.tile_hi) {
                s_off[2] = oa;
                s_off[3] = ta + ob;
            }
        }
        if (tsk) {
        } else if (tq) {
            oqa += ca;
            oqb += cb;
        } else {
            oa += ca;
            ob += cb;
        }
    }
    if (staged_out) {
        // one 32-B vector store per subtree record (each 8-B word carries the
        // tag, so the record needs no ordering)
        __syncthreads();
        const unsigned long long tag = (epoch & 0xFFFFFFFFull) << 32;
        for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
            const uint32_t A = sres[t], B = sres[nt + t], V = sres[2 * nt + t], S = sres[3 * nt + t];
            asm volatile("st.relaxed.gpu.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(P.k3_rec + 4ull * t),
                         "l"(tag | A), "l"(tag | B), "l"(tag | V), "l"(tag | S)
                         : "memory");
        }  // (tile_off / tile_lvl / tile_src: read only by partitioned engines and exports, which run their own top)
    }
    stamp(4);
    // the subtree CTAs need only the offsets, depths and decode sources:
    // publish now; FV1's inputs (activity, list slices, final top flags,
    // top-cell projection) follow while the subtree CTAs decode and emit
    k3_publish(ctl, epoch);
    if (EXPORT) return;
    if (threadIdx.x == 0 && P.tile_hi >= nt) {
        s_off[2] = ta;
        s_off[3] = ta + tb;
    }
    for (uint32_t t = a; t < b && !tact_by_subtrees; ++t) {
        // FV1 dry shortcut: subtree t is active if it or a face-adjacent
        // subtree holds a wet cell, or it touches an inflow edge; clear the
        // flags FV1 sets next (the split K3's subtree CTAs do it for their own)
        uint8_t act = swet[t];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const uint32_t nb = zo::neighbour_dev(R, t, static_cast<zo::Direction>(d));
            if (nb == zo::kNone) act |= (P.bc[d] == 2) ? 1 : 0;
            else act |= swet[nb];
        }
        P.tact[t] = act;
        P.wet[tbuf ^ 1][t] = 0;
    }
    __syncthreads();  // s_off complete
    // ---- final flags of levels < R, projection (D4) of top cells on the tree
    //      below a newly significant ancestor
    for (uint32_t q = threadIdx.x; q < lo(R, 0); q += NT) {
        const int n = (31 - __clz(3u * q + 1u)) >> 1;
        const uint32_t a2 = slo(n) + (q - lo(n, 0));
        P.sig[p ^ 1][a2] = ts[a2];
    }
    if (threadIdx.x == 0) {  // (block_exscan above: s_off complete)
        if (tn && P.part == 0) atomicAdd(&ctl->cnt_new, (unsigned long long)tn);
        const uint32_t ntl = tiles ? s_ntile : 0u;
        ctl->n_leaves = ta + tb + (ntl << (2 * P.K)) + sk_leaves;  // (tiled and skipped subtrees' leaves are off the lists)
        ctl->n_leaves_A = ta;
        ctl->n_stile = ntl;
        ctl->cnt_tiled += static_cast<unsigned long long>(ntl) << (2 * P.K);
        // this partition's slices of the A and B lists
        ctl->a_lo = s_off[0];
        ctl->a_hi = s_off[2];
        ctl->b_lo = s_off[1];
        ctl->b_hi = s_off[3];
        if (qs) {  // (one partition: the active parts, then the quiet lists)
            ctl->a_lo = 0u;
            ctl->a_hi = taa;
            ctl->b_lo = ta;
            ctl->b_hi = ta + tba;
            ctl->qa_lo = taa;
            ctl->qa_n = tqa;
            ctl->qb_lo = ta + tba;
            ctl->qb_n = tqb;
        } else {
            ctl->qa_n = ctl->qb_n = 0u;
        }
    }
    stamp(5);
    if (tn) {
        double4* buf = P.cells[p];
        for (int n = 1; n <= R; ++n)
            for (uint32_t m = threadIdx.x; m < (1u << (2 * n)); m += NT) {
                if (!ti[slo(n) + m] || owner_of(P, n, m) != P.part) continue;
                for (int k = 0; k < n; ++k) {
                    const uint32_t q = slo(k) + (m >> (2 * (n - k)));
                    if (ts[q] && !tv[q]) {
                        write_projection(buf, P, n, m, zo::z_of(k, m >> (2 * (n - k))));
                        break;
                    }
                }
            }
    }
    stamp(6);
}

// subtree CTA of K3: stage own flags, count own leaves (independent of the
// top), wait for the top's offsets, then decode and emit
template <bool EXPORT, int KT>
__device__ void k3_tile(const Params& P, Ctl* ctl, int p, int tbuf, unsigned long long epoch, uint32_t j, uint8_t* sm,
                        const Probe& stamp, bool sc_ready = false) {
    __shared__ unsigned s_red[32];
    __shared__ uint32_t s_top[4];
    double4* buf = P.cells[p];
    const uint8_t* sigc = EXPORT ? P.sig[p] : P.sig[p ^ 1];
    const uint8_t* sigp = EXPORT ? P.sig[p ^ 1] : P.sig[p];
    const int L = P.L, R = P.R;
    const int K = KT ? KT : P.K;
    const uint32_t nt = static_cast<uint32_t>(P.n_tiles);
    const uint32_t ncell = lo(L, R);
    uint8_t* sc = sm;                                      // own current flags, slo layout
    uint8_t* sp = sc + slo(K);                             // own previous flags
    uint32_t* src = reinterpret_cast<uint32_t*>(sp + slo(K));  // [ncell] projection sources
    (void)ncell;

    {   // (sc_ready: the fused K2 left this subtree's final flags in sc)
        const uint8_t c0 = sc_ready ? 0 : stage_tile_flags(sc, sigc, P, j);
        const uint8_t q0 = EXPORT ? 0 : stage_tile_flags(sp, sigp, P, j);
        cp_async_wait_all();
        if (threadIdx.x == 0) {
            if (!sc_ready) sc[0] = c0;
            if (!EXPORT) sp[0] = q0;
        }
    }
    __syncthreads();
    stamp(0);

    // ---- anything newly significant inside the subtree (hot path)
    int any_new = 0;
    if (!EXPORT) {
        if (sc[0] && !sp[0]) any_new = 1;
#pragma unroll
        for (int k = 1; k < (KT ? KT : kMaxL); ++k) {
            if (!KT && k >= K) break;
            for (uint32_t q = 4u * threadIdx.x; q < (1u << (2 * k)); q += 4u * kThreads)
                any_new |= (*reinterpret_cast<const uint32_t*>(sc + slo(k) + q) &
                            ~*reinterpret_cast<const uint32_t*>(sp + slo(k) + q))
                               ? 1
                               : 0;
        }
    }
    // ---- PTT counts of the subtree, assuming its root is reached: one walk
    //      per level-(L-2) cell (its 4 level-(L-1) children share the path);
    //      K = 1 (L = 1) walks the level-(L-1) cells directly
    const int Gk = (K >= 2) ? K - 2 : K - 1;               // walked tile level
    const int G = R + Gk;
    const uint32_t ng = 1u << (2 * Gk);
    const uint32_t per = (ng + kThreads - 1) / kThreads;
    const uint32_t a = threadIdx.x * per;
    const uint32_t b = min(ng, a + per);
    const uint8_t* sL1 = sc + slo(K - 1);
    auto walk = [&](uint32_t t) -> int {  // first tile level <= Gk whose cell is not significant, or Gk + 1
        int k = 0;
#pragma unroll
        for (int kk = 0; kk < (KT ? KT : kMaxL); ++kk) {
            if (kk > Gk || !sc[slo(kk) + (t >> (2 * (Gk - kk)))]) break;
            k = kk + 1;
        }
        return k;
    };
    unsigned ca = 0, cb = 0;
    for (uint32_t t = a; t < b; ++t) {
        const int k = walk(t);
        if (k <= Gk) {
            cb += ((t & ((1u << (2 * (Gk - k))) - 1u)) == 0u) ? 1u : 0u;
        } else if (G == L - 1) {
            ca += 4;
        } else {
            const unsigned s4 = __popc(*reinterpret_cast<const uint32_t*>(sL1 + 4u * t));
            ca += 4 * s4;
            cb += 4 - s4;
        }
    }
    unsigned total;
    unsigned xa, xb;
    if (EXPORT) {
        xa = block_exscan(ca + cb, s_red, &total);
        xb = 0;
    } else {
        xa = block_exscan(ca, s_red, &total);
        xb = block_exscan(cb, s_red, &total);
    }
    any_new = __syncthreads_or(any_new);
    stamp(1);

    // ---- the top's results for this subtree
    if (EXPORT) {
        k3_wait(ctl, epoch);
        stamp(2);
        if (threadIdx.x == 0) {
            s_top[0] = ldcg_u32(P.tile_off + 2 * nt + j);
            s_top[1] = 0u;
            s_top[2] = ldcg_u32(P.tile_lvl + j);
            s_top[3] = kNoSrc;
        }
    } else {
        // poll this subtree's own record until all four words carry this
        // step's tag (each word is written atomically with its tag)
        if (threadIdx.x == 0) {
            const unsigned tag = static_cast<unsigned>(epoch);
            const unsigned long long* rec = P.k3_rec + 4ull * j;
            unsigned long long v0, v1, v2, v3;
            for (;;) {
                v0 = ld_relaxed_u64(rec + 0);
                v1 = ld_relaxed_u64(rec + 1);
                v2 = ld_relaxed_u64(rec + 2);
                v3 = ld_relaxed_u64(rec + 3);
                if (static_cast<unsigned>(v0 >> 32) == tag && static_cast<unsigned>(v1 >> 32) == tag &&
                    static_cast<unsigned>(v2 >> 32) == tag && static_cast<unsigned>(v3 >> 32) == tag)
                    break;
                __nanosleep(32);
            }
            s_top[0] = static_cast<uint32_t>(v0);
            s_top[1] = static_cast<uint32_t>(v1);
            s_top[2] = static_cast<uint32_t>(v2);
            s_top[3] = static_cast<uint32_t>(v3);
        }
        stamp(2);
    }
    __syncthreads();
    stamp(3);
    uint32_t oa = s_top[0], ob = s_top[1];
    const uint32_t lvl = s_top[2], rootsrc = s_top[3];
    uint32_t* outA = EXPORT ? P.leaves_x : P.leaves;
    const bool reached = (lvl & 0xFFu) == static_cast<uint32_t>(R);
    if (!reached) {
        if (threadIdx.x == 0 && (lvl & kEmit)) {
            const int n = static_cast<int>(lvl & 0xFFu);
            (EXPORT ? outA[oa] : P.leaves[ob]) = zo::z_of(n, j >> (2 * (R - n)));
        }
        if (!EXPORT) tl_end(ctl, tbuf, 2);
        stamp(6);
        return;
    }

    // ---- projection inside the subtree, top-down (the root itself was
    //      projected by the top CTA)
    unsigned nnew = 0;
    if (!EXPORT && (any_new || rootsrc != kNoSrc)) {
        if (threadIdx.x == 0) src[0] = rootsrc;
        __syncthreads();
        for (int n = R; n < L; ++n) {
            const int k = n - R;
            const uint32_t cnt_k = 1u << (2 * k);
            for (uint32_t pi = threadIdx.x; pi < cnt_k; pi += kThreads) {
                const uint32_t li = lo(n, R) + pi;
                const uint32_t pm = j * cnt_k + pi;
                const bool isnew = sc[slo(k) + pi] && !sp[slo(k) + pi];
                nnew += isnew ? 1u : 0u;
                uint32_t cs = kNoSrc;
                if (sc[slo(k) + pi]) cs = (src[li] != kNoSrc) ? src[li] : (isnew ? zo::z_of(n, pm) : kNoSrc);
                if (n + 1 < L) {
                    const uint32_t lc = lo(n + 1, R) + 4u * pi;
                    src[lc] = cs; src[lc + 1] = cs; src[lc + 2] = cs; src[lc + 3] = cs;
                }
                if (cs != kNoSrc) {
                    const double4 v = projection_source(buf, P, cs);
                    double4* dst = buf + cbase(n + 1) + 4ull * pm;
                    for (uint32_t q = 0; q < 4; ++q) store_hqq(dst + q, v);
                }
            }
            __syncthreads();
        }
        const unsigned tn = block_sum(nnew, s_red);
        if (threadIdx.x == 0 && tn) atomicAdd(&ctl->cnt_new, (unsigned long long)tn);
    }
    stamp(4);

    // ---- emit: hot path level-L leaves to list A, coarser ones to list B;
    //      export one Morton-ordered list
    oa += xa;
    ob += xb;
    auto emitA = [&](uint32_t m1) {  // the 4 level-L children of level-(L-1) cell m1
        const uint32_t z0 = zo::z_of(L, m1 << 2);
        if (EXPORT) {
            outA[oa] = z0; outA[oa + 1] = z0 + 1; outA[oa + 2] = z0 + 2; outA[oa + 3] = z0 + 3;
        } else {  // list A offsets are multiples of 4
            *reinterpret_cast<uint4*>(outA + oa) = make_uint4(z0, z0 + 1, z0 + 2, z0 + 3);
        }
        oa += 4;
    };
    auto emitB = [&](uint32_t z) {
        if (EXPORT) outA[oa++] = z;
        else P.leaves[ob++] = z;
    };
    const uint32_t gbase = j * ng;
    const bool tiled = !EXPORT && (lvl & kTileSub);  // (fully refined: every leaf is a level-L one, on the tile path)
    const bool skipped = !EXPORT && (lvl & kSkipSub);  // (stable quiet: FV1 skips it, its leaves on no list)
    for (uint32_t t = a; t < b && !tiled && !skipped; ++t) {
        const int k = walk(t);
        const uint32_t gm = gbase + t;
        if (k <= Gk) {
            if ((t & ((1u << (2 * (Gk - k))) - 1u)) == 0u) emitB(zo::z_of(R + k, gm >> (2 * (Gk - k))));
        } else if (G == L - 1) {
            emitA(gm);
        } else {
            for (uint32_t q = 0; q < 4; ++q) {
                const uint32_t m1 = 4u * gm + q;
                if (sL1[4u * t + q]) emitA(m1);
                else emitB(zo::z_of(L - 1, m1));
            }
        }
    }
    if (!EXPORT) tl_end(ctl, tbuf, 2);
    stamp(6);
}

// epoch: 0 = hot path (2 step + 2, unique per step; the host clears the flag
// after initialise), else the host's export sequence number
template <bool EXPORT, int KT>
__global__ void __launch_bounds__(kThreads, 8) k_traverse(Params P, Ctl* ctl, int force, unsigned long long epoch) {
    pdl_wait();
    pdl_trigger();
    const unsigned long long t_entry = gtimer();
    const Head hd = cta_head(ctl, P, EXPORT || force);
    if (!hd.active) return;
    const unsigned long long ep = epoch ? epoch : 2ull * static_cast<unsigned long long>(hd.step) + 2ull;
    extern __shared__ __align__(16) uint8_t smem3[];
    if (!EXPORT) tl_start(ctl, hd.buf, 2);
    const Probe stamp(ctl, EXPORT ? -1000 : 16);
    stamp(7, t_entry);
    if (blockIdx.x == 0) {
        k3_top<EXPORT>(P, ctl, hd.parity, hd.buf, ep, smem3, stamp, !EXPORT && !force && P.top_band);
        return;
    }
    k3_tile<EXPORT, KT>(P, ctl, hd.parity, hd.buf, ep, P.tile_lo + blockIdx.x - 1, smem3, stamp);
}

// K3 split over two launches (one partition): the top CTA alone, with a
// dynamic shared-memory request that keeps subtree CTAs off its SM, then the
// subtree CTAs (launched as soon as the top passed its wait for K2, so K2's
// results are visible to them without a wait of their own); they meet on the
// k3_ready flag as in k_traverse. Each subtree CTA waits for the top grid
// before it exits, so FV1 (launched after the subtree grid) also sees the
// top's post-publish results.
// the top CTA runs 1024 threads: its per-subtree loops (tile listing, quiet
// classification, counts, records, activity) take one subtree per thread at
// L = 11
constexpr int kTopThreads = 1024;
template <int KT>
__global__ void __launch_bounds__(kTopThreads, 1) k_traverse_top(Params P, Ctl* ctl) {
    extern __shared__ __align__(16) uint8_t smem3t[];
    // before the wait for K2: the staging that does not depend on K1 / K2
    // (this grid launches once K2 runs, so the previous FV1 has completed:
    // parity, step and its wet marks are final)
    const bool pre = P.n_tiles >= 16 && P.n_tiles <= 1024;
    const Head hd = cta_head(ctl, P, false);
    if (pre && hd.active) k3_top_prestage<kTopThreads>(P, hd.parity, hd.buf, smem3t);
    pdl_wait();
    pdl_trigger();
    const unsigned long long t_entry = gtimer();
    if (!hd.active) {
        cp_async_wait_all();
        return;
    }
    tl_start(ctl, hd.buf, 2);
    const Probe stamp(ctl, 16);
    stamp(7, t_entry);
    k3_top<false, kTopThreads>(P, ctl, hd.parity, hd.buf, 2ull * static_cast<unsigned long long>(hd.step) + 2ull, smem3t, stamp,
                  P.top_band != 0, P.n_tiles <= 1024, pre, true);
}
// FV1's dry-shortcut activity of subtree j (the or of its own and its face
// neighbours' wet marks, inflow edges active) and the clear of the mark FV1
// sets next — by the subtree's own K3 CTA (split K3), not the top
__device__ __forceinline__ void subtree_activity(const Params& P, int tbuf, int parity, uint32_t j) {
    if (threadIdx.x != 0) return;
    const uint8_t* w = P.wet[tbuf];
    if (P.qact) {
        const bool refined = P.sig[parity ^ 1][slo(P.R) + j] != 0;  // (this step's tree)
        P.tact[j] = activity_q(P, j, w, P.qwet[tbuf], refined);
        *reinterpret_cast<uint32_t*>(P.qwet[tbuf ^ 1] + 4u * j) = 0u;
    } else {
        uint8_t act = w[j];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const uint32_t nb = zo::neighbour_dev(P.R, j, static_cast<zo::Direction>(d));
            if (nb == zo::kNone) act |= (P.bc[d] == 2) ? 1 : 0;
            else act |= w[nb];
        }
        P.tact[j] = act;
    }
    P.wet[tbuf ^ 1][j] = 0;
}
template <int KT>
__global__ void __launch_bounds__(kThreads, 8) k_traverse_tiles(Params P, Ctl* ctl) {
    pdl_trigger();
    const unsigned long long t_entry = gtimer();
    const Head hd = cta_head(ctl, P, false);
    if (hd.active) {
        extern __shared__ __align__(16) uint8_t smem3s[];
        Probe stamp(ctl, 16);
        if (blockIdx.x == 0) stamp.slot = -1;  // (slots 16.. belong to the top CTA)
        stamp(7, t_entry);
        k3_tile<false, KT>(P, ctl, hd.parity, hd.buf, 2ull * static_cast<unsigned long long>(hd.step) + 2ull,
                           P.tile_lo + blockIdx.x, smem3s, stamp);
        subtree_activity(P, hd.buf, hd.parity, P.tile_lo + blockIdx.x);  // (after the emit: off the records' critical path)
    }
    pdl_wait();  // the top grid has completed before this grid does
}

// Fused K2 + K3 in ONE cooperative grid (one partition): block 0 is the top,
// blocks 1..n_tiles the subtree CTAs. The cooperative launch guarantees that
// every CTA is resident at once (the launch fails otherwise; the host checks
// the occupancy first), so the waits below cannot deadlock whatever order
// the CTAs are scheduled in, and none waits on a CTA of a later launch (a
// two-launch version hung wherever kernels are serialised: compute-sanitizer,
// ncu). The top re-encodes levels R-1..0 and bands the top cells (K2's extra
// CTA), waits until every subtree CTA has published its band / closure /
// counts (k2_done) and runs K3's top. A subtree CTA runs K2's subtree work on
// K1's pre flags, publishes it, and goes on with K3's subtree work on the
// final flags it still holds in shared memory (polling the top's records).
// One launch and one kernel boundary less than K2 -> K3.
template <int KT>
__global__ void __launch_bounds__(kThreads, 2) k_23(Params P, Ctl* ctl) {
    const Head hd = cta_head(ctl, P, false);  // (as k_band: final before K1 passed its wait)
    pdl_wait();
    const unsigned long long t_entry = gtimer();
    extern __shared__ __align__(16) uint8_t smem23[];
    const unsigned long long epoch = 2ull * static_cast<unsigned long long>(hd.step) + 2ull;
    if (blockIdx.x == 0) {
        // (FV1 may launch once every CTA has triggered: they are all resident)
        pdl_trigger();
        if (!hd.active) return;
        tl_start(ctl, hd.buf, 1);
        tl_start(ctl, hd.buf, 2);
        const Probe stamp(ctl, 16);
        stamp(7, t_entry);
        encode_top_staged(P, ctl, hd.parity, hd.buf, smem23);
        if (threadIdx.x == 0) {
            const unsigned nt = static_cast<unsigned>(P.n_tiles);
            while (ld_acquire_u32(&ctl->k2_done) < nt) __nanosleep(32);
            ctl->k2_done = 0u;  // (every subtree CTA of this step has counted)
        }
        __syncthreads();
        k3_top<false>(P, ctl, hd.parity, hd.buf, epoch, smem23, stamp, true, P.n_tiles <= 1024);
        return;
    }
    if (!hd.active) {
        pdl_trigger();
        return;
    }
    const uint32_t j = P.tile_lo + blockIdx.x - 1u;
    // K2's subtree work: pre flags at smem23, final flags left at
    // smem23 + slo(K) = K3's current-flag slot
    k2_tile<KT>(P, ctl, hd, j, smem23);
    __threadfence();  // every thread's final-flag stores, then the count
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&ctl->k2_done, 1u);
    pdl_trigger();
    const Probe stamp(ctl, 16);  // (the last subtree CTA: slots 24..)
    stamp(7, t_entry);
    k3_tile<false, KT>(P, ctl, hd.parity, hd.buf, epoch, j, smem23 + slo(KT ? KT : P.K), stamp, true);
}

// =========================================================================== K5
__device__ __forceinline__ double series_value(const Params& P, double t) {
    const int n = P.inflow_n;
    if (n <= 0) return 0.0;
    const double* ts = P.inflow_t;
    const double* vs = P.inflow_v;
    if (t <= ts[0]) return vs[0];
    if (t >= ts[n - 1]) return vs[n - 1];
    int k = 0;
    while (k + 1 < n && ts[k + 1] <= t) ++k;
    return vs[k] + ((vs[k + 1] - vs[k]) * ((t - ts[k]) / (ts[k + 1] - ts[k])));
}

// next dt from the CFL maximum rate (D13), clipped to the
// next output time / t_end; `advance` also commits the step (t, parity, counters).
__device__ void finalize_dt(const Params& P, Ctl* ctl, double maxrate, bool advance) {
    const double t_new = advance ? ctl->t_next : ctl->t;
    const double dtc = (maxrate == 0.0) ? P.dt_fallback : P.cfl / maxrate;
    double stop = P.t_end;
    for (int k = 0; k < P.n_out; ++k) {
        const double o = P.out_times[k];
        if (o > t_new && o < stop) stop = o;
    }
    double dt, tn;
    if (t_new + dtc >= stop) {
        dt = stop - t_new;
        tn = stop;
    } else {
        dt = dtc;
        tn = t_new + dtc;
    }
    if (t_new < P.t_end && !(dt > 0.0 && isfinite(dt))) report_error(ctl, kErrDt, 0, 0, kStageDt);
    if (advance) {
        ctl->dt_used = ctl->dt;
        ctl->t = t_new;
        ctl->step += 1;
        ctl->parity ^= 1;
        ctl->n_leaves_used = ctl->n_leaves;
        ctl->cnt_updates += ctl->n_leaves;
    }
    ctl->dt = dt;
    ctl->t_next = tn;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(kFull, v, o);
        v = y > v ? y : v;
    }
    return v;
}

// reduce the per-thread CFL rates (exact max on the bits of non-negative
// doubles) into this step's slot; with one partition the last CTA finishes
// the step, with several k_finalize does (after every partition's FV1)
__device__ __forceinline__ void cfl_reduce_and_finalize(const Params& P, Ctl* ctl, double rate, bool advance,
                                                        int slot) {
    __shared__ unsigned long long s_max[kThreads / 32];
    __shared__ int s_last;
    unsigned long long b = warp_max_u64(static_cast<unsigned long long>(__double_as_longlong(rate)));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = s_max[0];
        for (int w = 1; w < kThreads / 32; ++w) m = s_max[w] > m ? s_max[w] : m;
        atomicMax(&ctl->rate_bits[slot], m);
    }
    if (P.G > 1) return;  // partitioned: k_finalize combines every partition's slot
    if (!last_block(&ctl->done_k5, &s_last)) return;
    if (threadIdx.x == 0) {
        const unsigned long long m = atomicAdd(&ctl->rate_bits[slot], 0ull);
        finalize_dt(P, ctl, __longlong_as_double(static_cast<long long>(m)), advance);
        ctl->rate_bits[slot] = 0ull;
        ctl->done_k5 = 0;
        ctl->fv1_tail = 0u;
        ctl->fv1_tjob = 0u;
        if (advance) {  // this step's near-threshold count is complete (K1, K2 and the previous FV1 are done)
            const unsigned long long nn = ctl->near_step[slot];
            ctl->near_last = nn;
            ctl->cnt_near += nn;
            ctl->near_step[slot] = 0ull;
        }
        ctl->tl[slot][3][2] = gtimer();
        if (advance) {  // next step's buffer; its [0][1] = this step's end (the gap in front of the next K1)
            for (int k = 0; k < 4; ++k) ctl->tl[slot ^ 1][k][0] = ctl->tl[slot ^ 1][k][2] = 0ull;
            ctl->tl[slot ^ 1][0][1] = ctl->tl[slot][3][2];
        }
    }
    // the step's report straight into the host's pinned mirror (saves the
    // host a device-to-host copy and a stream synchronisation per step;
    // step_adaptive's graph). advance_reports' graphs have the next step's K1
    // write it into the ring instead (off this kernel's tail)
    if (advance && P.ctl_mirror && threadIdx.x < 32) report_to(ctl, P.ctl_mirror, slot);
}

// ctl->parity = v on the stream (a pageable host copy would block the host
// until the stream drains — fatal in front of a cross-partition barrier)
__global__ void k_set_parity(Ctl* ctl, int v) {
    if (threadIdx.x == 0 && blockIdx.x == 0) ctl->parity = v;
}

// Cross-partition barrier on the device (one thread per partition, launched
// between the phases of a partitioned step on every partition's stream): the
// kernel before it on this stream has completed, so its writes are in this
// GPU's memory; publish this partition's barrier count with a system-scope
// release (peers read it over NVLink, or from other processes through CUDA
// IPC mappings), then acquire every peer's count. Every partition runs the
// same phase sequence, so counts match. A peer that never arrives (10 s) is
// reported instead of hanging the GPU.
__global__ void k_part_barrier(Params P, Ctl* ctl) {
    pdl_wait();  // (launched with PDL behind the phase kernel: its writes first)
    if (threadIdx.x != 0) return;
    const unsigned long long seq = ctl->bar_seq + 1ull;
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&ctl->bar_seq), "l"(seq) : "memory");
    const unsigned long long t0 = gtimer();
    for (int g = 0; g < P.G; ++g) {
        if (g == P.part) continue;
        const unsigned long long* peer = &P.pctl[g]->bar_seq;
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(peer) : "memory");
            if (v >= seq) break;
            if (gtimer() - t0 > 10000000000ull) {
                report_error(ctl, kErrBarrier, static_cast<uint32_t>(g), 0, kStageBarrier);
                return;
            }
            __nanosleep(100);
        }
    }
}

// partitioned step end: global max of every partition's CFL rate (exact, so
// every partition computes the same dt), then commit the step locally. The
// slot of the next step is cleared; this step's slot stays readable by the
// other partitions until the next step's barrier chain has passed.
__global__ void k_finalize(Params P, Ctl* ctl, int advance) {
    pdl_wait();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (advance && !active(ctl, P)) return;
    const int slot = static_cast<int>(ctl->step & 1);
    unsigned long long m = 0ull;
    for (int g = 0; g < P.G; ++g) {
        const unsigned long long v = *((volatile const unsigned long long*)&P.pctl[g]->rate_bits[slot]);
        m = v > m ? v : m;
    }
    finalize_dt(P, ctl, __longlong_as_double(static_cast<long long>(m)), advance != 0);
    if (!advance) return;  // initialise: the host clears the slots afterwards
    {
        const unsigned long long nn = ctl->near_step[slot];
        ctl->near_last = nn;
        ctl->cnt_near += nn;
        ctl->near_step[slot] = 0ull;
    }
    ctl->rate_bits[slot ^ 1] = 0ull;
    ctl->fv1_tail = 0u;  // (FV1's tail counter: partitioned FV1 has no finalizing CTA)
    ctl->tl[slot][3][2] = gtimer();
    for (int k = 0; k < 4; ++k) ctl->tl[slot ^ 1][k][0] = ctl->tl[slot ^ 1][k][2] = 0ull;
}

// covering cell of a same-level neighbour region whose parent (k, mm) is NOT
// significant: walk up until the parent is significant (SPEC.md:248 — the
// coarser covering leaf); the fast path (parent significant -> the same-level
// cell itself) is tested by the caller for all four faces at once
__device__ __forceinline__ const double4* covering_local(const Params& P, const double4* cur, const uint8_t* sigc, int k,
                                                        uint32_t mm) {
    while (k > 0 && !sigc[slo(k - 1) + (mm >> 2)]) {
        mm >>= 2;
        --k;
    }
    return cur + cbase(k) + mm;
}
// covering_local that also reports the covering cell (level k, code mm)
__device__ __forceinline__ const double4* covering_at(const Params& P, const double4* cur, const uint8_t* sigc, int& k,
                                                     uint32_t& mm) {
    while (k > 0 && !sigc[slo(k - 1) + (mm >> 2)]) {
        mm >>= 2;
        --k;
    }
    return cur + cbase(k) + mm;
}
__device__ __forceinline__ double4* covering(const Params& P, int cur, int k, uint32_t mm) {
    while (k > 0 && !sig_at(P, cur ^ 1, k - 1, mm >> 2)) {
        mm >>= 2;
        --k;
    }
    return cell_ptr(P, cur, k, mm);
}

// ------------------------------------------------------------ FV1 tile path
// A face's result as both of its cells use it: the HLL flux and the two
// reconstructed depths (the west / south cell takes hL for its bed
// correction, the east / north cell hR; D12).
struct FaceR {
    double F0, F1, F2, hL, hR;
};
__device__ __forceinline__ FaceR face_r(const CellV& Lc, const CellV& Rc, bool xface, const PhysParams& p) {
    FaceR r;
    double F[3];
    face(Lc, Rc, xface, p, F, r.hL, r.hR);
    r.F0 = F[0];
    r.F1 = F[1];
    r.F2 = F[2];
    return r;
}
__device__ __forceinline__ FaceR shfl_face(const FaceR& f, int src) {
    return {__shfl_sync(kFull, f.F0, src), __shfl_sync(kFull, f.F1, src), __shfl_sync(kFull, f.F2, src),
            __shfl_sync(kFull, f.hL, src), __shfl_sync(kFull, f.hR, src)};
}
// (only what face() reads: h, z, ux, uy, c — qx, qy left 0)
__device__ __forceinline__ CellV shfl_cell(const CellV& c, int src) {
    CellV o;
    o.h = __shfl_sync(kFull, c.h, src);
    o.qx = 0.0;
    o.qy = 0.0;
    o.z = __shfl_sync(kFull, c.z, src);
    o.ux = __shfl_sync(kFull, c.ux, src);
    o.uy = __shfl_sync(kFull, c.uy, src);
    o.c = __shfl_sync(kFull, c.c, src);
    return o;
}
// the direction-d neighbour of level-L leaf m as the per-leaf path sees it:
// the same-level cell, the coarser covering leaf or the
// boundary ghost (no inactive cells on the tile path)
__device__ __forceinline__ CellV nb_cell(const Params& P, const double4* cur, const uint8_t* sigc, uint32_t m,
                                         const CellV& own, int d, double inflow) {
    const int L = P.L;
    const uint32_t nm = zo::neighbour_dev(L, m, static_cast<zo::Direction>(d));
    if (nm == zo::kNone) return boundary_cell(own, P.bc[d], d, inflow, P.inflow_mode, P.phys);
    const double4* s = sigc[slo(L - 1) + (nm >> 2)] ? cur + cbase(L) + nm : covering_local(P, cur, sigc, L - 1, nm >> 2);
    return make_cell(ld4_nc(s), P.phys);
}
// L_c + Euler + friction of a cell from its four faces: the expressions and
// their order are fv1_cell_seq's, so the bits are the per-leaf path's
__device__ __forceinline__ void cell_update(const CellV& own, const FaceR& fE, const FaceR& fW, const FaceR& fN,
                                            const FaceR& fS, double idx, double dt, const PhysParams& p, double& hn,
                                            double& qxn, double& qyn, double& rh) {
    const double hh = own.h * own.h;
    const double FE1 = fE.F1 + (p.half_g * (hh - (fE.hL * fE.hL)));
    const double FW1 = fW.F1 + (p.half_g * (hh - (fW.hR * fW.hR)));
    const double GN1 = fN.F1 + (p.half_g * (hh - (fN.hL * fN.hL)));
    const double GS1 = fS.F1 + (p.half_g * (hh - (fS.hR * fS.hR)));
    fv1_finish(own, fE.F0 - fW.F0, FE1 - FW1, fE.F2 - fW.F2, fN.F0 - fS.F0, GN1 - GS1, fN.F2 - fS.F2, idx, dt, p, hn,
               qxn, qyn, rh);
}

// the direction-d neighbour of level-L leaf m outside the strip's subtree:
// its source cell (same-level or coarser covering leaf), or null
// for the domain edge (boundary ghost); `f` = the parent-level flag of the
// same-level cell, loaded early by the caller
__device__ __forceinline__ const double4* nb_src(const Params& P, const double4* cur, const uint8_t* sigc, uint32_t nm,
                                                 uint8_t f) {
    if (nm == zo::kNone) return nullptr;
    return f ? cur + cbase(P.L) + nm : covering_local(P, cur, sigc, P.L - 1, nm >> 2);
}

// One 32 x 4 strip (job: bits 0-3 row band, bit 4 column half) of a fully
// refined active subtree `tile` (K = 6: 64 x 64 level-L leaves), one warp,
// lane = column. Every face is computed once for both of its cells — x-faces
// by the east cell (its west face, handed to the west cell by a shuffle),
// y-faces by the south cell (carried up the rows) — and every cell's
// velocities / celerity once, instead of 4 faces and 5 make_cell per leaf.
// The strip's edge faces (8 x-faces, one row of y-faces below it) come from
// the neighbours the per-leaf path would use. Every load of the strip (its
// 4 rows, the rows below and above, the edge columns; outside the subtree
// the neighbours' parent-level flags first) is issued before any
// arithmetic. Also the next step's level-(L-1) re-encode of the strip's
// quads (rows 2k, 2k+1), the CFL rates, the wet mark.
//
// Code size matters (the per-leaf k_fv1 is instruction-cache bound once it
// grows: the strip inlined into it quadrupled the kernel and cost more than
// it saved), so the strips run in their own kernel, k_fv1_tiles, and their
// rounds go through ONE copy of face() — per round a y-face and an x-face —
// with the row loop not unrolled.
struct TileOut {
    double mx;
    unsigned tree, nnear;
};
// `rows`: this warp's shared-memory slab of 6 x 32 cells (rows r0-1 .. r0+4
// of the strip's columns), filled by cp.async when the job starts
__device__ __forceinline__ TileOut fv1_tile_strip(const Params& P, Ctl* ctl, const double4* __restrict__ cur,
                                                  double4* __restrict__ nxt, const uint8_t* __restrict__ sigc,
                                                  uint32_t tile, uint32_t job, double dt, double inflow, int tbuf,
                                                  double4* rows) {
    TileOut out = {0.0, 0u, 0u};
    const int L = P.L, lane = threadIdx.x & 31;
    const int xoff = (job & 16u) ? 32 : 0, r0 = 4 * static_cast<int>(job & 15u);
    const uint32_t mb = tile << 12;
    const double4* cl = cur + cbase(L);
    const PhysParams& ph = P.phys;
    const double idx = inv_dx_of(P, L);
    // Morton code of (x, y) inside the subtree: 6-bit dilations (3 shift +
    // lop3 steps instead of zorder's 4-step 14-bit spread), own column once
    auto spread6 = [](uint32_t v) {
        v = (v ^ (v << 4)) & 0x0F0Fu;
        v = (v ^ (v << 2)) & 0x3333u;
        return (v ^ (v << 1)) & 0x5555u;
    };
    auto mc = [&](int x, int y) { return mb | spread6(static_cast<uint32_t>(x)) | (spread6(static_cast<uint32_t>(y)) << 1); };
    const int x = xoff + lane;
    const uint32_t mbx = mb | spread6(static_cast<uint32_t>(x));
    auto mcol = [&](int y) { return mbx | (spread6(static_cast<uint32_t>(y)) << 1); };
    double4* my = rows + lane;  // row i at my[32 i]
    // ---- loads, all issued before any arithmetic: this column's rows inside
    //      the subtree by cp.async into the slab; at the subtree's edges the
    //      outside neighbours' parent-level flags, then their cells
    for (int i = 0; i < 6; ++i) {
        const int y = r0 - 1 + i;
        if (y >= 0 && y < 64) {
            const double4* g = cl + mcol(y);
            cp_async16(my + 32 * i, g);
            cp_async16(reinterpret_cast<uint8_t*>(my + 32 * i) + 16, reinterpret_cast<const uint8_t*>(g) + 16);
        }
    }
    // edge lanes: 0-3 the east edge of row r0 + lane, 4-7 the west edge of
    // row r0 + lane - 4 — the strip's own edge cell and its neighbour
    const bool east = lane < 4;
    const int ex = east ? xoff + 31 : xoff, er = r0 + (lane & 3);
    const uint32_t em = mc(ex, er);
    const int nx = east ? ex + 1 : ex - 1;
    const bool e_in = nx >= 0 && nx < 64;
    double4 eo = make_double4(0.0, 0.0, 0.0, 0.0), en = eo;
    uint32_t enm = zo::kNone;
    uint8_t ef = 1;
    if (lane < 8) {
        eo = ld4_nc(cl + em);
        if (e_in) {
            en = ld4_nc(cl + mc(nx, er));
        } else {
            enm = zo::neighbour_dev(L, em, east ? zo::Direction::East : zo::Direction::West);
            if (enm != zo::kNone) ef = sigc[slo(L - 1) + (enm >> 2)];
        }
    }
    const bool s_out = r0 == 0, n_out = r0 + 4 >= 64;
    uint32_t onm = zo::kNone;  // the outside row's same-level cell (south / north)
    uint8_t of = 1;
    if (s_out || n_out) {
        onm = zo::neighbour_dev(L, s_out ? mcol(r0) : mcol(r0 + 3), s_out ? zo::Direction::South : zo::Direction::North);
        if (onm != zo::kNone) of = sigc[slo(L - 1) + (onm >> 2)];
    }
    bool e_wall = false, o_wall = false;  // domain edge: boundary ghost
    if (lane < 8 && !e_in) {
        const double4* s = nb_src(P, cur, sigc, enm, ef);
        if (s) en = ld4_nc(s);
        else e_wall = true;
    }
    if (s_out || n_out) {
        const double4* s = nb_src(P, cur, sigc, onm, of);
        if (s) my[s_out ? 0 : 160] = ld4_nc(s);
        else o_wall = true;
    }
    cp_async_wait_all();
    __syncwarp();
    // a strip whose cells, rows above / below and edge neighbours are all dry
    // (and no inflow ghost): every cell takes the per-leaf path's
    // dry-neighbourhood result (h kept, q = 0), without faces
    bool dry = true;
#pragma unroll
    for (int i = 0; i < 6; ++i)  // (a row beyond the domain edge is a ghost of the row next to it)
        if (!(o_wall && ((i == 0 && s_out) || (i == 5 && n_out)))) dry = dry && my[32 * i].x < ph.hdry;
    if (lane < 8) dry = dry && eo.x < ph.hdry && (e_wall ? P.bc[east ? 1 : 0] != 2 : en.x < ph.hdry);
    if ((s_out || n_out) && o_wall) dry = dry && P.bc[s_out ? 3 : 2] != 2;
    if (__all_sync(kFull, dry)) {
        double ph0 = 0.0, pz0 = 0.0;
        uint32_t pm0 = 0;
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
            const uint32_t m = mcol(r0 + k);
            const double4 o4 = my[32 * (k + 1)];
            const double hn = (o4.x < 0.0) ? 0.0 : o4.x;
            st4(nxt + cbase(L) + m, make_double4(hn, 0.0, 0.0, o4.w));
            if (k & 1) {
                const int o = lane | 1;
                double4 ch[4];
                ch[0] = make_double4(ph0, 0.0, 0.0, pz0);
                ch[1] = make_double4(__shfl_sync(kFull, ph0, o), 0.0, 0.0, __shfl_sync(kFull, pz0, o));
                ch[2] = make_double4(hn, 0.0, 0.0, o4.w);
                ch[3] = make_double4(__shfl_sync(kFull, hn, o), 0.0, 0.0, __shfl_sync(kFull, o4.w, o));
                if (!(lane & 1)) {
                    const Enc e = encode_children<false>(ch, P, L - 1);
                    const uint32_t pm = pm0 >> 2;
                    st4(nxt + cbase(L - 1) + pm, e.par);
                    const unsigned long long fi = slo(L - 1) + pm;
                    P.pre[fi] = (e.flow || P.dem[fi]) ? 1 : 0;
                    ++out.tree;
                    out.nnear += e.near ? 1u : 0u;
                }
            } else {
                ph0 = hn;
                pz0 = o4.w;
                pm0 = m;
            }
        }
        __syncwarp();
        return out;
    }

    // ---- prologue: the edge x-faces (lanes 0-7) and the y-faces below row r0
    FaceR fb = {0.0, 0.0, 0.0, 0.0, 0.0}, fS;
    CellV C = make_cell(my[32], ph);
    {
        const CellV own = make_cell(eo, ph);
        const CellV nb = e_wall ? boundary_cell(own, P.bc[east ? 1 : 0], east ? 1 : 0, inflow, P.inflow_mode, ph)
                                : make_cell(en, ph);
        if (lane < 8) fb = east ? face_r(own, nb, true, ph) : face_r(nb, own, true, ph);
        const CellV S = (s_out && o_wall) ? boundary_cell(C, P.bc[3], 3, inflow, P.inflow_mode, ph) : make_cell(my[0], ph);
        fS = face_r(S, C, false, ph);
    }
    double ph0 = 0.0, pq0 = 0.0, pr0 = 0.0, pz0 = 0.0;  // the even row's new state (quad re-encode)
    uint32_t pm0 = 0;
    bool wet = false;
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
        const uint32_t m = mcol(r0 + k);
        const CellV N = (k == 3 && n_out && o_wall) ? boundary_cell(C, P.bc[2], 2, inflow, P.inflow_mode, ph)
                                                    : make_cell(my[32 * (k + 2)], ph);
        const FaceR fN = face_r(C, N, false, ph);
        FaceR fW = face_r(shfl_cell(C, (lane + 31) & 31), C, true, ph);  // (lane 0: replaced by the edge face)
        {
            const FaceR bw = shfl_face(fb, 4 + k);
            if (lane == 0) fW = bw;
        }
        FaceR fE = shfl_face(fW, (lane + 1) & 31);
        {
            const FaceR be = shfl_face(fb, k);
            if (lane == 31) fE = be;
        }
        double hn, qxn, qyn, rhn;
        cell_update(C, fE, fW, fN, fS, idx, dt, ph, hn, qxn, qyn, rhn);
        if (!(isfinite(hn) && isfinite(qxn) && isfinite(qyn)))
            report_error(ctl, kErrNonFinite, zo::z_of(L, m), !isfinite(hn) ? 0 : (!isfinite(qxn) ? 1 : 2), kStageFV1);
        st4(nxt + cbase(L) + m, make_double4(hn, qxn, qyn, C.z));
        const double c = cfl_rate_rh(hn, qxn, qyn, rhn, idx, ph);
        out.mx = c > out.mx ? c : out.mx;
        wet = wet || !(hn < ph.hdry);
        // next step's zero_details_and_reencode of level L-1 (the per-leaf
        // path's fused re-encode): quad (2i, r-1), (2i+1, r-1), (2i, r), (2i+1, r)
        if (k & 1) {
            const int o = lane | 1;
            double4 ch[4];
            ch[0] = make_double4(ph0, pq0, pr0, pz0);
            ch[1] = make_double4(__shfl_sync(kFull, ph0, o), __shfl_sync(kFull, pq0, o), __shfl_sync(kFull, pr0, o),
                                 __shfl_sync(kFull, pz0, o));
            ch[2] = make_double4(hn, qxn, qyn, C.z);
            ch[3] = make_double4(__shfl_sync(kFull, hn, o), __shfl_sync(kFull, qxn, o), __shfl_sync(kFull, qyn, o),
                                 __shfl_sync(kFull, C.z, o));
            if (!(lane & 1)) {
                const Enc e = encode_children<false>(ch, P, L - 1);
                const uint32_t pm = pm0 >> 2;
                st4(nxt + cbase(L - 1) + pm, e.par);
                const unsigned long long fi = slo(L - 1) + pm;
                P.pre[fi] = (e.flow || P.dem[fi]) ? 1 : 0;
                ++out.tree;
                out.nnear += e.near ? 1u : 0u;
            }
        } else {
            ph0 = hn;
            pq0 = qxn;
            pr0 = qyn;
            pz0 = C.z;
            pm0 = m;
        }
        fS = fN;
        C = N;
    }
    if (__any_sync(kFull, wet) && lane == 0) {
        P.wet[tbuf ^ 1][tile] = 1;
        if (P.qact) P.qwet[tbuf ^ 1][4u * tile + ((r0 >> 5) << 1) + (xoff >> 5)] = 1;  // (the strip lies in one quadrant)
    }
    __syncwarp();  // (the slab is refilled by the next job)
    return out;
}

// FV1 tile phase: the strips of the active fully refined subtrees K3's top
// listed (P.stile, ctl->n_stile), run by every k_fv1 CTA before its share of
// the leaf list (the per-leaf windows' tail balancing absorbs the tile
// phase's imbalance; a separate tile kernel ran its own tail and a launch
// gap before the per-leaf kernel). Each CTA takes a contiguous range of the
// jobs (neighbouring strips share rows through L2) and hands them to its
// warps by a shared-memory counter (a grid-wide counter measured slower:
// thousands of same-address atomics queue at one L2 slice). Not inlined: the
// strip code stays out of the per-leaf loop's instruction footprint.
constexpr size_t kTileSlab = sizeof(double4) * 6 * 32 * (kThreads / 32);  // k_fv1 dynamic shared memory with tiles
__device__ __forceinline__ TileOut fv1_tile_phase(const Params& P, Ctl* ctl, const double4* __restrict__ cur,
                                               double4* __restrict__ nxt, const uint8_t* __restrict__ sigc,
                                               uint32_t ntile, double dt, double inflow, int tbuf) {
    __shared__ unsigned s_tj;
    TileOut acc = {0.0, 0u, 0u};
    const uint32_t njobs = 32u * ntile;
    const uint32_t j1 = static_cast<uint32_t>((static_cast<unsigned long long>(njobs) * (blockIdx.x + 1)) / gridDim.x);
    if (threadIdx.x == 0)
        s_tj = static_cast<uint32_t>((static_cast<unsigned long long>(njobs) * blockIdx.x) / gridDim.x);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    extern __shared__ __align__(16) double4 s_rows[];  // kTileSlab bytes: one 6 x 32-cell slab per warp
    for (;;) {
        uint32_t jb = 0;
        if (lane == 0) jb = atomicAdd(&s_tj, 1u);
        jb = __shfl_sync(kFull, jb, 0);
        if (jb >= j1) break;
        const TileOut to = fv1_tile_strip(P, ctl, cur, nxt, sigc, P.stile[jb >> 5], jb & 31u, dt, inflow, tbuf,
                                          s_rows + (threadIdx.x >> 5) * (6 * 32));
        acc.mx = to.mx > acc.mx ? to.mx : acc.mx;
        acc.tree += to.tree;
        acc.nnear += to.nnear;
    }
    return acc;
}

// FV1's quiet lists (K3's top: reached subtrees whose neighbourhood held no
// wet cell, Params::qsplit): every leaf and neighbour is dry, so each leaf
// takes the per-leaf path's quiet result h = max(h, 0), q = 0 (no CFL rate,
// no wet mark); level-L quads one per thread — four contiguous cells, no
// gathers, no shuffles — with the next step's re-encode of their parent in
// registers (encode_lanes' arithmetic on the same four children), coarser
// leaves one per thread. Grid-stride over both lists.
__device__ __forceinline__ void fv1_quiet_pass(const Params& P, const double4* __restrict__ cur,
                                               double4* __restrict__ nxt, uint32_t qa_lo, uint32_t qa_n,
                                               uint32_t qb_lo, uint32_t qb_n, unsigned& tree, unsigned& nnear,
                                               unsigned& nquiet) {
    const uint32_t nthr = gridDim.x * kThreads, tid = blockIdx.x * kThreads + threadIdx.x;
    const uint32_t nq = qa_n >> 2;
    const uint32_t* qa = P.leaves + qa_lo;
    const double4* cl = cur + cbase(P.L);
    double4* nl = nxt + cbase(P.L);
    for (uint32_t k = tid; k < nq; k += nthr) {
        const uint32_t m0 = qa[4u * k] - zo::level_offset(P.L);  // first child of the quad
        double4 v[4] = {ld4_nc(cl + m0), ld4_nc(cl + m0 + 1), ld4_nc(cl + m0 + 2), ld4_nc(cl + m0 + 3)};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[q] = make_double4((v[q].x < 0.0) ? 0.0 : v[q].x, 0.0, 0.0, v[q].w);
            st4(nl + m0 + q, v[q]);
        }
        const Enc e = encode_children<false>(v, P, P.L - 1);
        const uint32_t pm = m0 >> 2;
        st4(nxt + cbase(P.L - 1) + pm, e.par);
        const unsigned long long fi = slo(P.L - 1) + pm;
        P.pre[fi] = (e.flow || P.dem[fi]) ? 1 : 0;
        ++tree;
        nnear += e.near ? 1u : 0u;
        nquiet += 4u;
        if (P.qskip && e.near) atomicAdd(&P.qnfv[m0 >> (2 * (P.L - P.R))], 1u);  // (cached for skipped steps)
    }
    const uint32_t* qb = P.leaves + qb_lo;
    for (uint32_t k = tid; k < qb_n; k += nthr) {
        const uint32_t z = qb[k];
        const int n = zo::level_of(z);
        const uint32_t m = z - zo::level_offset(n);
        const double4 v = ld4_nc(cur + cbase(n) + m);
        st4(nxt + cbase(n) + m, make_double4((v.x < 0.0) ? 0.0 : v.x, 0.0, 0.0, v.w));
        ++nquiet;
    }
}

// FV1 per-leaf pass for short leaf lists (small L): LPL = 4 or 2 lanes per
// leaf, so one warp-iteration's dependent chain holds one face (LPL = 4: the
// W, E, N, S face of lane q = 0..3) or one face pair (LPL = 2: the x faces in
// lane 0, the y faces in lane 1) instead of four; lane 0 of each group
// combines them by shuffles and finishes the cell. A short list fits in one
// grid-stride window, so the per-leaf path's latency is the iteration's
// dependent chain (~7-9 us on pseudo-2D L8 / humps L9 for four serial faces).
// Every face is the same face() call with the same argument order and the
// same adjustment expression as fv1_cell_seq, and the differences are formed
// in the same order: the bits are those of the one-lane path.
template <int LPL>
__device__ __forceinline__ void fv1_fp_loop(const Params& P, Ctl* ctl, const double4* __restrict__ cur,
                                            double4* __restrict__ nxt, const uint8_t* __restrict__ sigc,
                                            uint32_t a_lo, uint32_t NA, uint32_t b_lo, uint32_t N, double dt,
                                            double inflow, int tbuf, double& mx, unsigned& tree, unsigned& nnear,
                                            unsigned& nquiet) {
    constexpr int ND = 4 / LPL;  // faces per lane
    const int lane = threadIdx.x & 31, q = lane % LPL;
    const uint32_t gmask = ((1u << LPL) - 1u) << (lane - q);
    const uint32_t stride = gridDim.x * (kThreads / LPL);
    for (uint32_t wb = (blockIdx.x * kThreads + (threadIdx.x & ~31u)) / LPL; wb < N; wb += stride) {
        const uint32_t i = wb + static_cast<uint32_t>(lane / LPL);
        const bool valid = i < N;
        const uint32_t z = valid ? P.leaves[i < NA ? a_lo + i : b_lo + (i - NA)] : zo::level_offset(P.L);
        const int n = zo::level_of(z);
        const uint32_t m = z - zo::level_offset(n);
        const uint8_t ta = (valid && n >= P.R) ? P.tact[m >> (2 * (n - P.R))] : 1;
        const double4 o4 = ld4_nc(cur + cbase(n) + m);
        const bool quiet = valid && ta == 0;
        const bool needs = valid && !quiet;
        uint32_t nm[ND];
        double4 r4[ND];
        bool dry = true;
#pragma unroll
        for (int k = 0; k < ND; ++k) {
            const int d = q * ND + k;
            nm[k] = needs ? zo::neighbour_dev(n, m, static_cast<zo::Direction>(d)) : zo::kNone;
            r4[k] = make_double4(0.0, 0.0, 0.0, 0.0);
            if (nm[k] != zo::kNone) {
                const double4* src = sigc[slo(n - 1) + (nm[k] >> 2)] ? cur + cbase(n) + nm[k]
                                                                      : covering_local(P, cur, sigc, n - 1, nm[k] >> 2);
                r4[k] = ld4_nc(src);
            }
        }
#pragma unroll
        for (int k = 0; k < ND; ++k) {
            if (nm[k] != zo::kNone) dry = dry && r4[k].x < P.phys.hdry;
            else if (needs && P.bc[q * ND + k] == 2) dry = false;  // inflow ghosts can be wet
        }
        // dry neighbourhood (the one-lane path's all_dry): own and every face of the group
        const bool gdry = (__ballot_sync(kFull, dry) & gmask) == gmask;
        const bool phys = needs && !(o4.x < P.phys.hdry && gdry);
        double hn = (o4.x < 0.0) ? 0.0 : o4.x, qxn = 0.0, qyn = 0.0;
        if (__any_sync(kFull, phys)) {
            const CellV own = make_cell(o4, P.phys);
            const double hh = own.h * own.h;
            auto nb_of = [&](uint32_t nmk, const double4& rk, int d) -> CellV {
                if (nmk == zo::kNone) return boundary_cell(own, P.bc[d], d, inflow, P.inflow_mode, P.phys);
                return make_cell(rk, P.phys);
            };
            double v0, v1, v2;
            double hLs, hRs, F[3];
            if (LPL == 4) {
                // face d = q: own on the left of the E (1) and N (2) faces
                const bool left = q == 1 || q == 2;
                const CellV nb = nb_of(nm[0], r4[0], q);
                face(left ? own : nb, left ? nb : own, q < 2, P.phys, F, hLs, hRs);
                const double sd = left ? hLs : hRs;
                v0 = F[0];
                v1 = F[1] + (P.phys.half_g * (hh - (sd * sd)));
                v2 = F[2];
            } else {
                // faces 2q, 2q + 1 (x: W, E; y: N, S) as fv1_cell_seq's blocks
                // (selects, not a lane-dependent index: no local memory)
                const CellV e = nb_of(q ? nm[0] : nm[ND - 1], q ? r4[0] : r4[ND - 1], q ? 2 : 1);  // E (q = 0) / N (q = 1)
                face(own, e, q == 0, P.phys, F, hLs, hRs);
                const double FE0 = F[0], FE1 = F[1] + (P.phys.half_g * (hh - (hLs * hLs))), FE2 = F[2];
                const CellV w = nb_of(q ? nm[ND - 1] : nm[0], q ? r4[ND - 1] : r4[0], q ? 3 : 0);  // W (q = 0) / S (q = 1)
                face(w, own, q == 0, P.phys, F, hLs, hRs);
                const double FW1 = F[1] + (P.phys.half_g * (hh - (hRs * hRs)));
                v0 = FE0 - F[0];
                v1 = FE1 - FW1;
                v2 = FE2 - F[2];
            }
            double dFx0, dFx1, dFx2, dGy0, dGy1, dGy2;
            if (LPL == 4) {
                const int b = lane - q;
                const double e0 = __shfl_sync(kFull, v0, b + 1), e1 = __shfl_sync(kFull, v1, b + 1),
                             e2 = __shfl_sync(kFull, v2, b + 1);
                const double n0 = __shfl_sync(kFull, v0, b + 2), n1 = __shfl_sync(kFull, v1, b + 2),
                             n2 = __shfl_sync(kFull, v2, b + 2);
                const double s0 = __shfl_sync(kFull, v0, b + 3), s1 = __shfl_sync(kFull, v1, b + 3),
                             s2 = __shfl_sync(kFull, v2, b + 3);
                dFx0 = e0 - v0;
                dFx1 = e1 - v1;
                dFx2 = e2 - v2;
                dGy0 = n0 - s0;
                dGy1 = n1 - s1;
                dGy2 = n2 - s2;
            } else {
                dFx0 = v0;
                dFx1 = v1;
                dFx2 = v2;
                dGy0 = __shfl_down_sync(kFull, v0, 1);
                dGy1 = __shfl_down_sync(kFull, v1, 1);
                dGy2 = __shfl_down_sync(kFull, v2, 1);
            }
            if (phys && q == 0) {
                double rhn;
                fv1_finish(own, dFx0, dFx1, dFx2, dGy0, dGy1, dGy2, inv_dx_of(P, n), dt, P.phys, hn, qxn, qyn, rhn);
                const double c = cfl_rate_rh(hn, qxn, qyn, rhn, inv_dx_of(P, n), P.phys);
                mx = c > mx ? c : mx;
            }
        }
        if (valid && q == 0) {
            nquiet += quiet ? 1u : 0u;
            if (!(hn < P.phys.hdry)) {  // wet marks (as the one-lane path)
                uint8_t* wn = P.wet[tbuf ^ 1];
                if (n >= P.R) {
                    wn[m >> (2 * (n - P.R))] = 1;
                } else {
                    const uint32_t t0 = m << (2 * (P.R - n)), t1 = (m + 1u) << (2 * (P.R - n));
                    for (uint32_t t = t0; t < t1; ++t) wn[t] = 1;
                }
                if (P.qact) {
                    uint8_t* qn = P.qwet[tbuf ^ 1];
                    if (n > P.R) {
                        qn[m >> (2 * (n - P.R - 1))] = 1;
                    } else {
                        const uint32_t t0 = m << (2 * (P.R - n)), t1 = (m + 1u) << (2 * (P.R - n));
                        for (uint32_t t = t0; t < t1; ++t) *reinterpret_cast<uint32_t*>(qn + 4u * t) = 0x01010101u;
                    }
                }
            }
            if (!(isfinite(hn) && isfinite(qxn) && isfinite(qyn)))
                report_error(ctl, kErrNonFinite, zo::z_of(n, m), !isfinite(hn) ? 0 : (!isfinite(qxn) ? 1 : 2),
                             kStageFV1);
            st4(nxt + cbase(n) + m, make_double4(hn, qxn, qyn, o4.w));
        }
        // the next step's level-(L-1) re-encode (as the one-lane path; the
        // four children sit in lanes 4 LPL k + {0, LPL, 2 LPL, 3 LPL})
        if (wb < NA) {
            const Enc e = encode_lanes<false, false>(make_double4(hn, qxn, qyn, o4.w), LPL, P, P.L - 1);
            if (lane % (4 * LPL) == 0 && i < NA && valid) {
                const uint32_t pm = m >> 2;
                store_hqq(nxt + cbase(P.L - 1) + pm, e.par);  // (z is static, ZPAR)
                const unsigned long long fi = slo(P.L - 1) + pm;
                P.pre[fi] = (e.flow || P.dem[fi]) ? 1 : 0;
                ++tree;
                nnear += e.near ? 1u : 0u;
            }
        }
    }
}

// FV1 over the leaf list: persistent grid-stride, one thread per
// leaf; reads the current buffer, writes leaf slots of the other (D15).
// STAGE 0: next iteration's own cell prefetched into L2; 2: loaded into
// registers an iteration ahead with its subtree activity; 3: also the
// neighbours' parent-level flags; 5: 3 + tail balancing.
#ifndef SWAMP_FV1_MINB
#define SWAMP_FV1_MINB 2  // resident CTAs per SM the register budget is sized for (3: DESIGN.md §8)
#endif
template <bool UNIFORM, bool PART = false, bool INA = false, int STAGE = 0>
__global__ void __launch_bounds__(kThreads, SWAMP_FV1_MINB) k_fv1(Params P, Ctl* ctl) {
    pdl_wait();
    // control words, read once per CTA (line 0 of Ctl)
    __shared__ double s_td[2];
    __shared__ uint32_t s_u[11];
    if (threadIdx.x == 0) {
        const volatile Ctl* vc = ctl;
        s_td[0] = vc->t;
        s_td[1] = vc->dt;
        s_u[0] = static_cast<uint32_t>(vc->parity);
        s_u[1] = static_cast<uint32_t>(vc->step & 1);
        s_u[2] = vc->a_lo; s_u[3] = vc->a_hi; s_u[4] = vc->b_lo; s_u[5] = vc->b_hi;
        s_u[6] = vc->n_stile;
        s_u[7] = vc->qa_lo; s_u[8] = vc->qa_n; s_u[9] = vc->qb_lo; s_u[10] = vc->qb_n;
    }
    __syncthreads();
    const double t = s_td[0], dt = s_td[1];
    if (!(t < P.t_end)) return;
    const int tbuf = static_cast<int>(s_u[1]);
    tl_start(ctl, tbuf, 3);
    const int p = static_cast<int>(s_u[0]);
    const double4* __restrict__ cur = P.cells[p];
    double4* __restrict__ nxt = P.cells[p ^ 1];
    const uint8_t* __restrict__ sigc = P.sig[p ^ 1];
    // this partition's leaves: its slice of the level-L list A (sibling
    // quadruples at indices 4g..4g+3) followed by its slice of list B
    const uint32_t a_lo = UNIFORM ? 0u : s_u[2], b_lo = UNIFORM ? 0u : s_u[4];
    const uint32_t NA = UNIFORM ? 0u : s_u[3] - a_lo;
    const uint32_t N = UNIFORM ? (1u << (2 * P.L)) : NA + (s_u[5] - b_lo);
    auto leaf_at = [&](uint32_t k) { return P.leaves[k < NA ? a_lo + k : b_lo + (k - NA)]; };
    const double inflow = series_value(P, t);
    const int lane = threadIdx.x & 31;
    double mx = 0.0;
    unsigned tree = 0, nnear = 0, ndem = 0, nquiet = 0;
    (void)ndem;
#if defined(SWAMP_EXP_PHASET) || defined(SWAMP_EXP_WHIST)
    unsigned long long ph_t[4];
    ph_t[0] = gtimer();
    unsigned ngrab = 0;
#endif
    if constexpr (!UNIFORM && !PART && !INA) {
        if (P.tiles && s_u[6]) {  // the tile path first (its leaves are off list A)
            const TileOut to = fv1_tile_phase(P, ctl, cur, nxt, sigc, s_u[6], dt, inflow, tbuf);
            mx = to.mx;
            tree = to.tree;
            nnear = to.nnear;
        }
    }
    if constexpr (!UNIFORM && !PART && !INA) {  // (before the per-leaf windows: measured 3.5 us better than after)
#if defined(SWAMP_EXP_PHASET) || defined(SWAMP_EXP_WHIST)
        ph_t[1] = gtimer();
#endif
        if (P.qsplit) fv1_quiet_pass(P, cur, nxt, s_u[7], s_u[8], s_u[9], s_u[10], tree, nnear, nquiet);
    }
#if defined(SWAMP_EXP_PHASET) || defined(SWAMP_EXP_WHIST)
    ph_t[2] = gtimer();
#endif
    // short lists at small L: several lanes per leaf (fv1_fp_loop); the
    // one-lane windows below then see an empty list
    uint32_t NL = N;
    if constexpr (!UNIFORM && !PART && !INA && STAGE == 3) {
        const unsigned long long cap = static_cast<unsigned long long>(gridDim.x) * kThreads * P.fv1_fp_cap16;
        if (64ull * N <= cap) {
            fv1_fp_loop<4>(P, ctl, cur, nxt, sigc, a_lo, NA, b_lo, N, dt, inflow, tbuf, mx, tree, nnear, nquiet);
            NL = 0;
        } else if (32ull * N <= cap) {
            fv1_fp_loop<2>(P, ctl, cur, nxt, sigc, a_lo, NA, b_lo, N, dt, inflow, tbuf, mx, tree, nnear, nquiet);
            NL = 0;
        }
    }
    const uint32_t stride = gridDim.x * kThreads;
    // warp-uniform trip count: every lane runs every iteration (shuffles below)
    uint32_t wbase = blockIdx.x * kThreads + (threadIdx.x & ~31u);
    // STAGE 5 (= 3 + tail balancing): the last fv1_tail16 / 16 of the windows
    // are taken one warp-iteration (32 leaves) at a time from a per-step
    // counter by whichever warps finish their static windows first; the
    // bases of the next two iterations are kept in b1, b2 (the finalizing
    // CTA resets the counter)
    constexpr bool TAIL = STAGE == 5;
    const uint32_t nwin = NL / stride, ntail = (nwin * P.fv1_tail16 + 8u) >> 4;
    const uint32_t nstat = (TAIL && ntail > 0u && nwin > ntail) ? (nwin - ntail) * stride : NL;  // (small lists: static)
    // one warp-iteration per grab (2 or 4 per grab measured slower at L = 11)
    // a grab uses the counter value fetched one grab earlier and fetches the
    // next one, so the atomic's round trip (long under contention: every warp
    // of the grid hits this address) overlaps an iteration instead of
    // stalling the warp; the last fetched value is never used
    uint32_t pend = 0;
    if (TAIL && lane == 0 && nstat < NL) pend = atomicAdd(&ctl->fv1_tail, 1u);
    auto grab = [&]() -> uint32_t {
        const uint32_t c = __shfl_sync(kFull, pend, 0);
        if (lane == 0) pend = atomicAdd(&ctl->fv1_tail, 1u);
#ifdef SWAMP_EXP_WHIST
        ++ngrab;
#endif
        const uint32_t b = nstat + 32u * c;
        return b < NL ? b : NL;
    };
    // the static windows as a per-CTA pool: the CTA's 8 warp-slots of every
    // static window, taken in order by whichever of its warps asks next
    // (shared-memory counter), so warps that ran a tile strip take fewer
    // (config 5 -1 us, wet point -2.8 us against a fixed slot per warp)
    __shared__ unsigned s_slot;
    if (threadIdx.x == 0) s_slot = 0u;
    __syncthreads();
    const uint32_t nslots = TAIL ? ((nstat + stride - 1u) / stride) * (kThreads / 32) : 0u;  // (partial last window: nstat = NL)
    auto slot_base = [&]() -> uint32_t {
        uint32_t sl = 0;
        if (lane == 0) sl = atomicAdd(&s_slot, 1u);
        sl = __shfl_sync(kFull, sl, 0);
        if (sl >= nslots) return ~0u;
        return (sl / (kThreads / 32)) * stride + blockIdx.x * kThreads + 32u * (sl % (kThreads / 32));
    };
    auto next_of = [&](uint32_t b) -> uint32_t {
        if (b >= NL) return NL;
        const uint32_t sb = slot_base();
        return sb != ~0u ? sb : grab();
    };
    uint32_t b1 = 0, b2 = 0;
    if (TAIL) {
        const uint32_t sb = slot_base();
        wbase = sb != ~0u ? sb : grab();
        b1 = next_of(wbase);
        b2 = next_of(b1);
    }
    // STAGE 2: the next iteration's own cell and subtree activity are loaded
    // into registers one iteration ahead (instead of an L2 prefetch)
    constexpr int pf = 1;
    // leaf ids two iterations ahead; the next iteration's own cell is
    // prefetched (no registers held) while this one computes: the leaf
    // cells were written a step ago and come from DRAM
    uint32_t z_next = (!UNIFORM && wbase + lane < NL) ? leaf_at(wbase + lane) : 0u;
    const uint32_t nb1_0 = TAIL ? b1 : wbase + stride;
    uint32_t z_nn = (!UNIFORM && pf && nb1_0 + lane < NL) ? leaf_at(nb1_0 + lane) : 0u;
    double4 o4_pre = make_double4(0.0, 0.0, 0.0, 0.0);
    uint8_t ta_pre = 1;
    uint8_t fl_pre[4] = {1, 1, 1, 1};  // STAGE 3: the neighbours' parent-level flags too
    auto pre_load = [&](uint32_t zz) {
        const int n1 = zo::level_of(zz);
        const uint32_t m1 = zz - zo::level_offset(n1);
        o4_pre = ld4_nc(cur + cbase(n1) + m1);
        ta_pre = (n1 >= P.R) ? P.tact[m1 >> (2 * (n1 - P.R))] : 1;
        if ((STAGE == 3 || STAGE == 5) && !PART && n1 > 0) {  // (PART: flags through the peer tables below)
            // a sibling neighbour (W of an east child, E of a west child, S of
            // a north child, N of a south child) shares this leaf's parent,
            // which is significant: only the other two flags are loaded
            const uint32_t c = m1 & 3u;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const bool sib = (d == 0) ? (c & 1u) != 0u : (d == 1) ? (c & 1u) == 0u : (d == 2) ? (c & 2u) == 0u : (c & 2u) != 0u;
                if (sib) {
                    fl_pre[d] = 1;
                } else {
                    const uint32_t q = zo::neighbour_dev(n1, m1, static_cast<zo::Direction>(d));
                    fl_pre[d] = (q != zo::kNone) ? sigc[slo(n1 - 1) + (q >> 2)] : 1;
                }
            }
        }
    };
    if (STAGE >= 2 && !UNIFORM && wbase + lane < NL) pre_load(z_next);
    auto advance_base = [&]() {
        if (TAIL) {
            wbase = b1;
            b1 = b2;
            b2 = next_of(b1);
        } else {
            wbase += stride;
        }
    };
    for (; wbase < NL; advance_base()) {
        const uint32_t i = wbase + lane;
        const uint32_t nb1 = TAIL ? b1 : wbase + stride, nb2 = TAIL ? b2 : wbase + 2 * stride;  // next two bases
        bool valid = i < NL;
        int n;
        uint32_t m;
        const double4 o4_k = o4_pre;
        const uint8_t ta_k = ta_pre;
        const uint8_t fl_k[4] = {fl_pre[0], fl_pre[1], fl_pre[2], fl_pre[3]};
        if (UNIFORM) {
            n = P.L;
            m = valid ? i : 0u;
            if (pf && nb1 + lane < NL) {
                const double4* q = cur + cbase(n) + nb1 + lane;
                prefetch_l2(q);
            }
        } else {
            const uint32_t z = valid ? z_next : zo::level_offset(P.L);  // leaf ids prefetched one iteration ahead
            if (pf) {
                z_next = z_nn;
                if (nb2 + lane < NL) z_nn = leaf_at(nb2 + lane);
                if (nb1 + lane < NL) {
                    if (STAGE >= 2) {
                        pre_load(z_next);
                    } else {
                        const int n1 = zo::level_of(z_next);
                        const double4* q = cur + cbase(n1) + (z_next - zo::level_offset(n1));
                        prefetch_l2(q);
                    }
                }
            } else if (nb1 + lane < NL) {
                z_next = leaf_at(nb1 + lane);
            }
            n = zo::level_of(z);
            m = z - zo::level_offset(n);
        }
        // subtree activity (bit 0: wet neighbourhood)
        const uint8_t ta = (STAGE >= 2 && !UNIFORM) ? (valid ? ta_k : 1)
                           : ((!UNIFORM && valid && n >= P.R) ? P.tact[m >> (2 * (n - P.R))] : 1);
        double hn = 0.0, qxn = 0.0, qyn = 0.0, zown = 0.0;
        if (valid) {
            // every global read of this leaf is issued before any arithmetic:
            // own cell, the neighbours' parent-level flags, the neighbours
            const double4 o4 = (STAGE >= 2 && !UNIFORM) ? o4_k : ld4_nc(cur + cbase(n) + m);
            // dry shortcut: in a subtree whose neighbourhood holds no wet cell
            // (K3's tact) the leaf and all its neighbours are dry, so the
            // dry-neighbourhood result below follows without the gathers
            const bool quiet = ta == 0;
            nquiet += quiet ? 1u : 0u;
            const bool dead = INA && (P.ina[slo(n) + m] & 1u);  // D16: an inactive leaf keeps its state
            if (dead) {
                hn = o4.x;
                qxn = o4.y;
                qyn = o4.z;
            } else if (quiet) {
                hn = (o4.x < 0.0) ? 0.0 : o4.x;
                qxn = 0.0;
                qyn = 0.0;
            } else {
            uint32_t nm[4];
            const double4* src[4];
            bool wall[4] = {false, false, false, false};  // D16: inactive neighbour = reflective wall
#pragma unroll
            for (int d = 0; d < 4; ++d) nm[d] = zo::neighbour_dev(n, m, static_cast<zo::Direction>(d));
            if (UNIFORM) {
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    src[d] = cur + cbase(n) + nm[d];
                    if (INA && nm[d] != zo::kNone) wall[d] = (P.ina[slo(n) + nm[d]] & 1u) != 0;
                }
            } else if (!PART && INA) {
                uint8_t f[4];
#pragma unroll
                for (int d = 0; d < 4; ++d) f[d] = (nm[d] != zo::kNone) ? sigc[slo(n - 1) + (nm[d] >> 2)] : 1;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    int k = n;
                    uint32_t mm = nm[d];
                    if (nm[d] == zo::kNone) {
                        src[d] = cur;
                        continue;
                    }
                    if (f[d]) src[d] = cur + cbase(n) + nm[d];
                    else {
                        k = n - 1;
                        mm = nm[d] >> 2;
                        src[d] = covering_at(P, cur, sigc, k, mm);
                    }
                    wall[d] = (P.ina[slo(k) + mm] & 1u) != 0;
                }
            } else {
                uint8_t f[4];
                if (PART) {  // cross-partition reads through the peer tables
#pragma unroll
                    for (int d = 0; d < 4; ++d) f[d] = (nm[d] != zo::kNone) ? sig_at(P, p ^ 1, n - 1, nm[d] >> 2) : 1;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        if (nm[d] == zo::kNone) {
                            src[d] = cur;
                            continue;
                        }
                        int k = n;
                        uint32_t mm = nm[d];
                        if (!f[d]) {  // the coarser covering leaf
                            k = n - 1;
                            mm = nm[d] >> 2;
                            while (k > 0 && !sig_at(P, p ^ 1, k - 1, mm >> 2)) {
                                mm >>= 2;
                                --k;
                            }
                        }
                        src[d] = cell_ptr(P, p, k, mm);
                        if (INA) wall[d] = (P.ina[slo(k) + mm] & 1u) != 0;  // replicated (static)
                    }
                } else {
#pragma unroll
                    for (int d = 0; d < 4; ++d)
                        f[d] = (STAGE >= 3) ? fl_k[d] : ((nm[d] != zo::kNone) ? sigc[slo(n - 1) + (nm[d] >> 2)] : 1);
#pragma unroll
                    for (int d = 0; d < 4; ++d)
                        src[d] = f[d] ? cur + cbase(n) + nm[d] : covering_local(P, cur, sigc, n - 1, nm[d] >> 2);
                }
            }
            double4 r4s[4];
#pragma unroll
            for (int d = 0; d < 4; ++d)
                if (nm[d] != zo::kNone) r4s[d] = ld4_nc(src[d]);
            auto nbv = [&](int d) -> double4 { return r4s[d]; };
            // dry neighbourhood: own cell and every neighbour / ghost below
            // h_dry => every reconstructed depth is 0, every flux 0, the bed
            // corrections cancel pairwise: h stays, q = 0 (the general path
            // gives the same bits)
            bool all_dry = o4.x < P.phys.hdry;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                if (nm[d] != zo::kNone) all_dry = all_dry && (wall[d] || nbv(d).x < P.phys.hdry);
                else if (P.bc[d] == 2) all_dry = false;  // inflow ghosts can be wet
            }
            if (all_dry) {
                hn = (o4.x < 0.0) ? 0.0 : o4.x;
                qxn = 0.0;
                qyn = 0.0;
            } else {
                const CellV own = make_cell(o4, P.phys);
                // the W, E, N, S neighbour as seen by its face (ghost on the boundary)
                auto neighbour = [&](int d) -> CellV {
                    if (nm[d] == zo::kNone) return boundary_cell(own, P.bc[d], d, inflow, P.inflow_mode, P.phys);
                    if (wall[d]) return boundary_cell(own, 0, d, inflow, P.inflow_mode, P.phys);
                    return make_cell(nbv(d), P.phys);
                };
                double rhn;
                fv1_cell_seq(own, neighbour, inv_dx_of(P, n), dt, P.phys, hn, qxn, qyn, rhn);
                // the CFL rate here, with friction's reciprocal depth (every
                // result with h >= h_dry comes from this path; dry results
                // and inactive leaves have rate 0)
                const double c = cfl_rate_rh(hn, qxn, qyn, rhn, inv_dx_of(P, n), P.phys);
                mx = c > mx ? c : mx;
            }
            }  // !quiet
            zown = o4.w;
        }
        if (valid) {
            // mark the subtree(s) of a leaf that ends wet (a leaf above level R
            // marks every subtree under it)
            if (!UNIFORM && !(hn < P.phys.hdry)) {
                uint8_t* wn = P.wet[tbuf ^ 1];
                if (n >= P.R) {
                    wn[m >> (2 * (n - P.R))] = 1;
                } else {
                    const uint32_t t0 = m << (2 * (P.R - n)), t1 = (m + 1u) << (2 * (P.R - n));
                    for (uint32_t t = t0; t < t1; ++t) wn[t] = 1;
                }
                if (!UNIFORM && !PART && P.qact) {  // quadrant marks (level R + 1; coarser leaves: all quadrants under them)
                    uint8_t* qn = P.qwet[tbuf ^ 1];
                    if (n > P.R) {
                        qn[m >> (2 * (n - P.R - 1))] = 1;
                    } else {
                        const uint32_t t0 = m << (2 * (P.R - n)), t1 = (m + 1u) << (2 * (P.R - n));
                        for (uint32_t t = t0; t < t1; ++t) *reinterpret_cast<uint32_t*>(qn + 4u * t) = 0x01010101u;
                    }
                }
            }
            if (!(isfinite(hn) && isfinite(qxn) && isfinite(qyn)))
                report_error(ctl, kErrNonFinite, zo::z_of(n, m), !isfinite(hn) ? 0 : (!isfinite(qxn) ? 1 : 2),
                             kStageFV1);
            st4(nxt + cbase(n) + m, make_double4(hn, qxn, qyn, zown));

        }
        // Next step's zero_details_and_reencode of level L-1, fused here: the
        // four updated children of a previous-tree level-(L-1) cell sit in
        // lanes 4k..4k+3; lane 4k forms the parent and its significance
        // (identical arithmetic to k_encode; the next K1 starts at L-2).
        if (!UNIFORM && wbase < NA) {
            const Enc e = encode_lanes<false, false>(make_double4(hn, qxn, qyn, zown), 1, P, P.L - 1);
            if ((lane & 3) == 0 && i < NA && valid) {
                const uint32_t pm = m >> 2;
                store_hqq(nxt + cbase(P.L - 1) + pm, e.par);  // (z is static, ZPAR)
                const unsigned long long fi = slo(P.L - 1) + pm;
                P.pre[fi] = (e.flow || P.dem[fi]) ? 1 : 0;
                ++tree;
                nnear += e.near ? 1u : 0u;
            }
        }
    }
#ifdef SWAMP_EXP_WHIST
    if (lane == 0) {  // (diagnostics) per-warp histograms, 4 us bins: tile phase, per-leaf loop, work end; grabs
        const unsigned long long te = gtimer(), t0 = ~ctl->tl[tbuf][3][0];
        auto bin = [](unsigned long long d, unsigned long long off) {
            return d > off ? static_cast<unsigned>(min(7ull, (d - off) / 4000ull)) : 0u;
        };
        atomicAdd(&ctl->dbg[32 + bin(ph_t[1] - ph_t[0], 0)], 1ull);
        atomicAdd(&ctl->dbg[40 + bin(te - ph_t[2], 0)], 1ull);
        atomicAdd(&ctl->dbg[48 + bin(te > t0 ? te - t0 : 0, 20000ull)], 1ull);
        atomicAdd(&ctl->dbg[56 + min(7u, ngrab)], 1ull);
    }
#endif
    if (!UNIFORM) {
        // work counters (bench.py's per-class byte accounting) and the
        // near-threshold level-(L-1) cells, which belong to the NEXT step's count
        __shared__ unsigned s_red5[3][kThreads / 32];
        unsigned v[3] = {tree, nquiet, nnear};
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(kFull, v[k], o);
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 3; ++k) s_red5[k][threadIdx.x >> 5] = v[k];
        __syncthreads();
        if (threadIdx.x < 3) {
            unsigned long long s = 0;
            for (int w = 0; w < kThreads / 32; ++w) s += s_red5[threadIdx.x][w];
            unsigned long long* dst = threadIdx.x == 0 ? &ctl->cnt_fused
                                      : threadIdx.x == 1 ? &ctl->cnt_quiet : &ctl->near_step[tbuf ^ 1];
            if (s) atomicAdd(dst, s);
        }
    }
#ifdef SWAMP_EXP_PHASET
    ph_t[3] = gtimer();
    if (lane == 0) {  // per warp: durations of tile phase, quiet pass, per-leaf loop (sum, max) + kernel span
        for (int k = 0; k < 3; ++k) {
            atomicAdd(&ctl->dbg[40 + k], ph_t[k + 1] - ph_t[k]);
            atomicMax(&ctl->dbg[44 + k], ph_t[k + 1] - ph_t[k]);
        }
        atomicAdd(&ctl->dbg[47], 1ull);
        atomicMin(&ctl->dbg[48], ph_t[0]);
        atomicMax(&ctl->dbg[49], ph_t[3]);
    }
#endif
#ifdef SWAMP_EXP_WEND
    if (lane == 0) {  // (diagnostics) histogram of CTA end times after the kernel's first start, 4 us bins
        const unsigned long long t0 = ~ctl->tl[tbuf][3][0];
        const unsigned long long te = gtimer();
        const unsigned bin = te > t0 ? static_cast<unsigned>(min(13ull, (te - t0) / 4000ull)) : 0u;
        atomicAdd(&ctl->dbg[50 + bin], 1ull);
    }
#endif
    // the next step's K1 may launch once every CTA is here: K1 CTAs made
    // resident early (trigger at entry) land on the SMs the FV1 tail frees
    // first and ran K1 5-7 us slower
    pdl_trigger();
    cfl_reduce_and_finalize(P, ctl, mx, true, tbuf);
}

// initialise: the near-threshold count of the first step's level-(L-1)
// cells. On later steps the previous FV1 re-encodes and classifies them (the
// fused level-(L-1) re-encode above); before the first step that is
// initialise's tree: its level-(L-1) cells re-encoded from their level-L
// children (unchanged since initialise), this partition's subtrees only.
__global__ void __launch_bounds__(kThreads) k_near_l1(Params P, Ctl* ctl) {
    const int p = ctl->parity;
    const uint8_t* sg = P.sig[p];
    const double4* buf = P.cells[p];
    const int n = P.L - 1;
    const uint32_t m0 = P.tile_lo << (2 * (n - P.R)), m1 = P.tile_hi << (2 * (n - P.R));
    unsigned nn = 0;
    for (uint32_t m = m0 + blockIdx.x * kThreads + threadIdx.x; m < m1; m += gridDim.x * kThreads) {
        if (!sg[slo(n) + m]) continue;
        const double4* c = buf + cbase(P.L) + 4ull * m;
        const double4 ch[4] = {ld4(c), ld4(c + 1), ld4(c + 2), ld4(c + 3)};
        nn += encode_children<false>(ch, P, n).near ? 1u : 0u;
    }
    __shared__ unsigned s_red[32];
    const unsigned t = block_sum(nn, s_red);
    if (threadIdx.x == 0 && t) atomicAdd(&ctl->near_step[0], (unsigned long long)t);
}

// dt at initialise: CFL over the initial leaves, no update.
__global__ void __launch_bounds__(kThreads) k_cfl_init(Params P, Ctl* ctl, int uniform) {
    const int p = ctl->parity;
    const double4* cur = P.cells[p];
    const uint32_t a_lo = uniform ? 0u : ctl->a_lo, b_lo = uniform ? 0u : ctl->b_lo;
    const uint32_t NA = uniform ? 0u : ctl->a_hi - a_lo;
    const uint32_t N = uniform ? (1u << (2 * P.L)) : NA + (ctl->b_hi - b_lo);
    double mx = 0.0;
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < N; i += gridDim.x * kThreads) {
        int n;
        uint32_t m;
        if (uniform) {
            n = P.L;
            m = i;
        } else {
            const uint32_t z = P.leaves[i < NA ? a_lo + i : b_lo + (i - NA)];
            n = zo::level_of(z);
            m = z - zo::level_offset(n);
        }
        const double4 v = ld4(cur + cbase(n) + m);
        const double c = (P.has_ina && (P.ina[slo(n) + m] & 1u)) ? 0.0 : cfl_rate(v.x, v.y, v.z, inv_dx_of(P, n), P.phys);
        mx = c > mx ? c : mx;
    }
    cfl_reduce_and_finalize(P, ctl, mx, false, static_cast<int>(ctl->step & 1));
}

// =========================================================== import / export
// initial discretisation: row-major (south row first) finest
// fields -> Morton slots of level L; s_max per quantity.
__global__ void __launch_bounds__(kThreads) k_import(Params P, Ctl* ctl, const double* h, const double* qx,
                                                     const double* qy, const double* z, const uint8_t* mask,
                                                     int buffer) {
    const uint32_t side = 1u << P.L;
    const uint64_t total = static_cast<uint64_t>(side) * side;
    double mx[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint64_t r = blockIdx.x * (uint64_t)kThreads + threadIdx.x; r < total; r += (uint64_t)gridDim.x * kThreads) {
        const uint32_t i = static_cast<uint32_t>(r & (side - 1)), jj = static_cast<uint32_t>(r >> P.L);
        const uint32_t m = zo::interleave(i, jj);
        const double4 v = make_double4(h[r], qx[r], qy[r], z[r]);
        if (!(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w)))
            report_error(ctl, kErrNonFinite, zo::z_of(P.L, m), 0, kStageImport);
        st4(P.cells[buffer] + cbase(P.L) + m, v);
        if (mask) {  // D16: finest inactive flags (bits 0 and 1), excluded from s_max
            const uint8_t b = mask[r] ? 3 : 0;
            P.ina[slo(P.L) + m] = b;
            if (b) continue;
        }
        mx[0] = max2(mx[0], absd(v.x));
        mx[1] = max2(mx[1], absd(v.y));
        mx[2] = max2(mx[2], absd(v.z));
        mx[3] = max2(mx[3], absd(v.w));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(mx[q]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(kFull, b, o);
            b = y > b ? y : b;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&ctl->smax_bits[q], b);
    }
}

// s_max from the import's maxima (the bits of non-negative doubles) and its
// reciprocal (IEEE division, as the host computed it before)
__global__ void k_smax_table(const Ctl* ctl, double* smx) {
    const int q = threadIdx.x;
    if (q < 4) {
        const double s = __longlong_as_double(static_cast<long long>(ctl->smax_bits[q]));
        smx[q] = s;
        smx[4 + q] = (s < 1e-12) ? 0.0 : 1.0 / s;
    }
}

// hierarchy export in z-index order, s-units (s = p * 2^(L-n)); leaves from
// the current buffer, significant cells from the other; off-tree cells NaN.
__global__ void k_export_tree(Params P, const Ctl* ctl, double* h, double* qx, double* qy, double* z, uint8_t* sig) {
    const int p = ctl->parity;
    const uint8_t* sigc = P.sig[p];
    const uint32_t total = zo::level_offset(P.L + 1);
    for (uint32_t zi = blockIdx.x * kThreads + threadIdx.x; zi < total; zi += gridDim.x * kThreads) {
        const int n = zo::level_of(zi);
        const uint32_t m = zi - zo::level_offset(n);
        if (n < P.L) sig[zi] = sig_at(P, p, n, m);
        const bool in_tree = (n == 0) || sig_at(P, p, n - 1, m >> 2);
        const bool is_sig = (n < P.L) && sig_at(P, p, n, m);
        const double nan = __longlong_as_double(0x7FF8000000000000ll);
        double4 v = make_double4(nan, nan, nan, nan);
        if (in_tree) v = ld4(cell_ptr(P, is_sig ? (p ^ 1) : p, n, m));
        const double sc = ldexp(1.0, P.L - n);
        h[zi] = v.x * sc;
        qx[zi] = v.y * sc;
        qy[zi] = v.z * sc;
        z[zi] = v.w * sc;
    }
}

// neighbour descriptors of the current leaf list
__global__ void k_descriptors(Params P, const Ctl* ctl, uint32_t* nbr, uint32_t N) {
    const int p = ctl->parity;
    const uint8_t* sigc = P.sig[p];
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < N; i += gridDim.x * kThreads) {
        const uint32_t z = P.leaves_x[i];
        const int n = zo::level_of(z);
        const uint32_t m = z - zo::level_offset(n);
        for (int d = 0; d < 4; ++d) {
            const uint32_t nm = zo::neighbour_dev(n, m, static_cast<zo::Direction>(d));
            uint32_t desc;
            if (nm == zo::kNone) {
                desc = 0xFFFFFFF0u + static_cast<uint32_t>(P.bc[d]);
            } else {
                int k = n;
                uint32_t mm = nm;
                while (k > 0 && !sig_at(P, p, k - 1, mm >> 2)) {
                    mm >>= 2;
                    --k;
                }
                desc = zo::z_of(k, mm);
            }
            nbr[static_cast<uint64_t>(d) * N + i] = desc;
        }
    }
}

// zero-detail expansion to the finest grid: physical,
// row-major south row first
__global__ void k_export_finest(Params P, const Ctl* ctl, double* h, double* qx, double* qy) {
    const int p = ctl->parity;
    const uint8_t* sigc = P.sig[p];
    const uint32_t side = 1u << P.L;
    const uint64_t total = static_cast<uint64_t>(side) * side;
    for (uint64_t r = blockIdx.x * (uint64_t)kThreads + threadIdx.x; r < total; r += (uint64_t)gridDim.x * kThreads) {
        const uint32_t i = static_cast<uint32_t>(r & (side - 1)), jj = static_cast<uint32_t>(r >> P.L);
        const uint32_t m = zo::interleave(i, jj);
        int n = 0;
        while (n < P.L && sig_at(P, p, n, m >> (2 * (P.L - n)))) ++n;
        const double4 v = ld4(cell_ptr(P, p, n, m >> (2 * (P.L - n))));
        h[r] = v.x;
        qx[r] = v.y;
        qy[r] = v.z;
    }
}

// gauges ("point sampling the covering leaf"): the finest cell
// (i, j) under each point, then the leaf covering it by the same flag walk as
// the expansion; out = [h, qx, qy, eta = h + z] x n, physical
__global__ void k_gauges(Params P, const Ctl* ctl, const uint32_t* cells, int n, double* out) {
    const int p = ctl->parity;
    for (int k = blockIdx.x * kThreads + threadIdx.x; k < n; k += gridDim.x * kThreads) {
        const uint32_t c = cells[k];
        const uint32_t m = zo::interleave(c & 0xFFFFu, c >> 16);
        int lv = 0;
        while (lv < P.L && sig_at(P, p, lv, m >> (2 * (P.L - lv)))) ++lv;
        const double4 v = ld4(cell_ptr(P, p, lv, m >> (2 * (P.L - lv))));
        out[k] = v.x;
        out[n + k] = v.y;
        out[2 * n + k] = v.z;
        out[3 * n + k] = v.x + v.w;
    }
}

// D16: inactive flags of level n from level n + 1 (bit 0 = all, bit 1 = any)
__global__ void k_ina_level(Params P, int n) {
    const uint32_t cnt = 1u << (2 * n);
    for (uint32_t m = blockIdx.x * kThreads + threadIdx.x; m < cnt; m += gridDim.x * kThreads) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(P.ina + slo(n + 1) + 4u * m);
        const uint32_t all = (w & 0x01010101u) == 0x01010101u ? 1u : 0u;
        const uint32_t any = (w & 0x02020202u) ? 2u : 0u;
        P.ina[slo(n) + m] = static_cast<uint8_t>(all | any);
    }
}
// D16: mixed active / inactive cells join the static DEM mask (and the
// pre-band flags of initialise), so every leaf is wholly active or inactive
__global__ void k_ina_mix(Params P) {
    const uint32_t nd = lo(P.L, 0);
    for (uint32_t q = blockIdx.x * kThreads + threadIdx.x; q < nd; q += gridDim.x * kThreads) {
        const int n = (31 - __clz(3u * q + 1u)) >> 1;
        const uint32_t a = slo(n) + (q - lo(n, 0));
        if (P.ina[a] == 2u) {
            P.dem[a] = 1;
            P.pre[a] = 1;
        }
    }
}

// Dynamic repartitioning: with the NEW boundaries in P and
// the old ones in `old`, CTA b of the new range pulls subtree tile_lo + b
// from its old owner when that owner is another partition: the subtree's
// cells of levels R..L (both buffers), its flags of levels R..L-1 (both
// copies, pre-band, DEM), its leaf counts and wet marks. Block 0 also pulls
// the top cells (levels < R) whose first subtree changed owner. Peers are
// idle (between steps); every partition pulls only what it gains.
__global__ void __launch_bounds__(kThreads) k_rebalance_pull(Params P, Params old) {
    const int R = P.R, L = P.L;
    const uint32_t t = P.tile_lo + blockIdx.x;
    const int from = owner_of(old, R, t);
    if (blockIdx.x == 0) {  // top cells: their value lives in the partition of their first subtree
        for (uint32_t q = threadIdx.x; q < lo(R, 0); q += kThreads) {
            const int n = (31 - __clz(3u * q + 1u)) >> 1;
            const uint32_t m = q - lo(n, 0);
            const int src = owner_of(old, n, m);
            if (owner_of(P, n, m) != P.part || src == P.part) continue;
            for (int b = 0; b < 2; ++b) P.cells[b][cbase(n) + m] = old.pcells[src][b][cbase(n) + m];
        }
    }
    if (from == P.part) return;
    for (int n = R; n <= L; ++n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        const unsigned long long base = cbase(n) + static_cast<unsigned long long>(t) * cnt;
        for (uint32_t c = threadIdx.x; c < cnt; c += kThreads)
            for (int b = 0; b < 2; ++b) P.cells[b][base + c] = old.pcells[from][b][base + c];
        if (n < L) {
            const unsigned long long fb = slo(n) + static_cast<unsigned long long>(t) * cnt;
            for (uint32_t c = threadIdx.x; c < cnt; c += kThreads) {
                P.sig[0][fb + c] = old.psig[from][0][fb + c];
                P.sig[1][fb + c] = old.psig[from][1][fb + c];
                P.pre[fb + c] = old.ppre[from][fb + c];
                P.dem[fb + c] = old.pdem[from][fb + c];
            }
        }
    }
    if (threadIdx.x == 0) {
        P.tile_cnt[t] = old.ptile_cnt[from][t];
        P.tile_cnt[P.n_tiles + t] = old.ptile_cnt[from][P.n_tiles + t];
        P.wet[0][t] = old.pwet[from][0][t];
        P.wet[1][t] = old.pwet[from][1][t];
    }
}

// compare: per-block partial sums and maxima of |hA - hB|
// over the finest expansions (fixed grid, so the host's in-order sum of the
// partials is deterministic)
__global__ void k_compare(const double* a, const double* b, uint64_t n, double* part_sum, double* part_max) {
    __shared__ double ss[kThreads / 32], sm[kThreads / 32];
    double s = 0.0, mx = 0.0;
    for (uint64_t k = blockIdx.x * (uint64_t)kThreads + threadIdx.x; k < n; k += (uint64_t)gridDim.x * kThreads) {
        const double d = absd(a[k] - b[k]);
        s += d;
        mx = max2(mx, d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(kFull, s, o);
        mx = max2(mx, __shfl_xor_sync(kFull, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        ss[threadIdx.x >> 5] = s;
        sm[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, m = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) {
            t += ss[w];
            m = max2(m, sm[w]);
        }
        part_sum[blockIdx.x] = t;
        part_max[blockIdx.x] = m;
    }
}

}  // namespace hwfv1
