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
enum ErrCode : int { kErrNone = 0, kErrNonFinite = -3, kErrDt = -4 };

struct Ctl {
    double t;        // current simulation time
    double dt;       // dt of the next step
    double t_next;   // time after the next step (exact stop time when clipped)
    double dt_used;  // dt of the last step taken
    unsigned long long rate_bits[2];  // CFL max-rate accumulators (bits of a non-negative double), by step parity
    unsigned long long smax_bits[4];
    long long step;
    unsigned long long cnt_tree;    // cells re-encoded by the last K1
    unsigned long long cnt_new;     // newly significant cells decoded by the last K3
    uint32_t n_leaves;              // leaves of the grid built by the last K2/K3
    uint32_t n_leaves_A;            // of which level-L leaves (listed first, in sibling quadruples)
    uint32_t a_lo, a_hi, b_lo, b_hi; // this partition's slices of the A (level-L) and B lists
    uint32_t n_leaves_used;         // leaves the last FV1 updated
    int parity;                     // current cell buffer / previous-tree flags
    int err_code;
    uint32_t err_z;
    int err_q;
    int err_stage;
    unsigned int done_k1, done_k2, done_k5;
    unsigned long long k2_ready;    // step + 1 once K2's last CTA published the traversal offsets
    unsigned long long dbg[16];     // per-phase globaltimer stamps of probe CTAs (diagnostics)
    // stage timeline (globaltimer ns), double-buffered by step parity: for
    // kernel k (K1, K2, K3, K5) [3k] = ~(first CTA start), [3k+1] = last CTA
    // elected, [3k+2] = last CTA done (atomicMax; K5 zeroes the next buffer)
    unsigned long long tl[2][12];
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
__device__ __forceinline__ int tl_buf(const Ctl* c) { return static_cast<int>(c->step & 1); }
__device__ __forceinline__ void tl_start(Ctl* c, int k) {
    if (threadIdx.x == 0) atomicMax(&c->tl[tl_buf(c)][3 * k], ~gtimer());
}
__device__ __forceinline__ void tl_mark(Ctl* c, int slot) {
    if (threadIdx.x == 0) atomicMax(&c->tl[tl_buf(c)][slot], gtimer());
}

struct Params {
    int L, R, K, n_tiles;
    int band_mode;
    int bc[4];
    int inflow_mode, inflow_n, n_out;
    double W, cfl, t_end, dt_fallback;
    double tau[kMaxL + 1];    // 0 >= tau[n]: significance of a zero-detail cell (eps == 0)
    double thr[4][kMaxL + 1]; // per quantity and level: max |D| >= thr (D7)
    double dx[kMaxL + 1];     // W * 2^-n
    double inv_dx[kMaxL + 1]; // 1.0 / dx[n] (IEEE division, as the oracle)
    double smax[4];
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
    uint32_t* tile_lvl;   // traversal depth of each level-R subtree root (R = reached)
    uint32_t* tile_src;   // z of the root's decode source, or kNoSrc
    // Morton-subtree partitions: this partition owns level-R
    // subtrees [tile_lo, tile_hi); cells on levels >= R belong to their
    // subtree's partition, cells above R are replicated except that a leaf's
    // value is current only in the partition of its first subtree. pcells /
    // psig / ppre / ptile_cnt / pctl are every partition's arrays (peer
    // pointers across GPUs; index 0 = self when G = 1).
    int G, part;
    int fuse_k3;          // K3 runs inside K2 (every K2 CTA is resident; host-checked)
    uint32_t tile_lo, tile_hi, tiles_per_part;
    double4* pcells[kMaxParts][2];
    uint8_t* psig[kMaxParts][2];
    uint8_t* ppre[kMaxParts];
    uint32_t* ptile_cnt[kMaxParts];
    Ctl* pctl[kMaxParts];
};

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
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
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
__device__ __forceinline__ int owner_of(const Params& P, int n, uint32_t m) {
    if (P.G == 1) return 0;
    const uint32_t t = (n >= P.R) ? (m >> (2 * (n - P.R))) : (m << (2 * (P.R - n)));
    return static_cast<int>(t / P.tiles_per_part);
}
__device__ __forceinline__ double4* cell_ptr(const Params& P, int buf, int n, uint32_t m) {
    return P.pcells[owner_of(P, n, m)][buf] + P.base[n] + m;
}
// significance byte of (n, m) in copy `which`; levels above R are replicated
__device__ __forceinline__ uint8_t sig_at(const Params& P, int which, int n, uint32_t m) {
    const int g = (n < P.R) ? P.part : owner_of(P, n, m);
    return P.psig[g][which][P.fbase[n] + m];
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
// significance of one quantity (D6, D7), division-free:
// thr = ldexp(eps * s_max, 2n - 2L + 2) in physical units (+inf / 0 when
// s_max < 1e-12, i.e. d_norm = 0)
__device__ __forceinline__ bool sig_q(double dmax, double thr) { return dmax >= thr; }

struct Enc {
    double4 par;
    bool flow, zflag;
};
// WITH_Z: also threshold z's details (the static DEM mask, t = 0 only)
template <bool WITH_Z = true>
__device__ __forceinline__ Enc encode_children(const double4 c[4], const Params& P, int n) {
    const Red h = red4(c[0].x, c[1].x, c[2].x, c[3].x);
    const Red qx = red4(c[0].y, c[1].y, c[2].y, c[3].y);
    const Red qy = red4(c[0].z, c[1].z, c[2].z, c[3].z);
    Enc e;
    e.flow = sig_q(h.dmax, P.thr[0][n]) || sig_q(qx.dmax, P.thr[1][n]) || sig_q(qy.dmax, P.thr[2][n]);
    if (WITH_Z) {
        const Red z = red4(c[0].w, c[1].w, c[2].w, c[3].w);
        e.par = make_double4(h.par, qx.par, qy.par, z.par);
        e.zflag = sig_q(z.dmax, P.thr[3][n]);
    } else {
        const double a = c[0].w + c[1].w, b = c[2].w + c[3].w;
        e.par = make_double4(h.par, qx.par, qy.par, 0.25 * (a + b));
        e.zflag = false;
    }
    return e;
}

__device__ __forceinline__ bool active(const Ctl* c, const Params& P) {
    return *((volatile const double*)&c->t) < P.t_end;
}

// Block-wide sum of unsigned values (256 threads).
__device__ __forceinline__ unsigned block_sum(unsigned v, unsigned* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    unsigned s = 0;
    if (threadIdx.x < 32) {
        s = (l < kThreads / 32) ? scratch[l] : 0u;
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
        unsigned s = (l < kThreads / 32) ? scratch[l] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFull, s, o);
            if (l >= o) s += y;
        }
        if (l < kThreads / 32) scratch[l] = s;  // inclusive warp totals
    }
    __syncthreads();
    const unsigned warp_prefix = (w == 0) ? 0u : scratch[w - 1];
    *total = scratch[kThreads / 32 - 1];
    __syncthreads();
    return warp_prefix + x - v;
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

// ---------------------------------------------------------------- K1 warp part
__device__ __forceinline__ double4 shfl4(double4 v, int src) {
    return make_double4(__shfl_sync(kFull, v.x, src), __shfl_sync(kFull, v.y, src), __shfl_sync(kFull, v.z, src),
                        __shfl_sync(kFull, v.w, src));
}
__device__ __forceinline__ bool byte_of(uint32_t w, int k) { return ((w >> (8 * k)) & 0xFFu) != 0u; }

// Encode of 4 children held by lanes lane, lane+s, lane+2s, lane+3s (result
// meaningful at the gathering lane); one component at a time to keep few
// values live. Same arithmetic as encode_children.
template <bool INIT>
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
    const Red z = red(v.w);
    Enc e;
    e.flow = sig_q(h.dmax, P.thr[0][n]) || sig_q(qx.dmax, P.thr[1][n]) || sig_q(qy.dmax, P.thr[2][n]);
    e.par = make_double4(h.par, qx.par, qy.par, z.par);
    e.zflag = INIT && sig_q(z.dmax, P.thr[3][n]);
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
                                                       double4* sv3, uint32_t j, int T, int R) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t n1 = 1u << (2 * (T - R)), n2 = n1 >> 2, n3 = n2 >> 2;  // tile cells on T, T-1, T-2
    const int ipw = (n1 >= 32u * (kThreads / 32)) ? static_cast<int>(n1 / (32u * (kThreads / 32))) : 1;
    const uint32_t b1 = 32u * ipw * w, b2 = 8u * ipw * w, b3 = 2u * ipw * w;
    if (b1 >= n1) return 0;
    const int L1 = T, L2 = T - 1, L3 = T - 2;
    const unsigned long long g1 = P.fbase[L1] + static_cast<unsigned long long>(j) * n1;
    const unsigned long long g2 = P.fbase[L2] + static_cast<unsigned long long>(j) * n2;
    const unsigned long long g3 = P.fbase[L3] + static_cast<unsigned long long>(j) * n3;
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
        if (L3 > R) f4 = INIT ? 1u : sigp[P.fbase[L3 - 1] + static_cast<unsigned long long>(j) * (n3 >> 2) + ((b3 + lane) >> 2)];
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
            const double4* cp = buf + P.base[L1 + 1] + (static_cast<unsigned long long>(gm1) << 2);
            ch[0] = ld4_nc(cp); ch[1] = ld4_nc(cp + 1); ch[2] = ld4_nc(cp + 2); ch[3] = ld4_nc(cp + 3);
        }
        double4 v1 = make_double4(0.0, 0.0, 0.0, 0.0), v2 = v1, v3 = v1;
        if (ok1 && !sp1 && sp2) v1 = ld4(buf + P.base[L1] + gm1);
        if (ok2 && !sp2 && sp3) v2 = ld4(buf + P.base[L2] + gm2);
        if (ok3 && !sp3 && sp4 && L3 > R) v3 = ld4(buf + P.base[L3] + gm3);
        // level T
        {
            bool flow = zero1, zf = false;
            if (sp1) {
                const Enc e = encode_children<INIT>(ch, P, L1);
                v1 = e.par;
                flow = e.flow;
                zf = e.zflag;
                st4(buf + P.base[L1] + gm1, v1);
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
                    zf = e.zflag;
                    st4(buf + P.base[L2] + gm2, v2);
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
                    zf = e.zflag;
                    st4(buf + P.base[L3] + gm3, v3);
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
    if (!INIT && !active(ctl, P)) return;
    tl_start(ctl, 0);
    extern __shared__ double4 sv[];
    __shared__ unsigned s_red[32];
    __shared__ int s_last;
    const int p = ctl->parity;
    double4* buf = P.cells[p];
    const uint8_t* sigp = P.sig[p];
    const int L = P.L, R = P.R, K = P.K;
    const uint32_t j = P.tile_lo + blockIdx.x;
    const uint32_t ncell = ((1u << (2 * K)) - 1u) / 3u;  // subtree cells on levels R..L-1
    uint8_t* sfl = reinterpret_cast<uint8_t*>(sv + ncell);  // previous-tree flags of the subtree
    unsigned tree = 0;

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
            sfl[lo(n, R) + pi] = INIT ? 1 : sigp[P.fbase[n] + j * cnt + pi];
    }
    __syncthreads();
    if (!INIT) {
        for (int n = R + 1; n <= top_n + (warp_path ? 0 : 1); ++n) {
            const uint32_t cnt = 1u << (2 * (n - R));
            for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
                const uint32_t li = lo(n, R) + pi;
                if (!sfl[li] && sfl[lo(n - 1, R) + (pi >> 2)]) sv[li] = ld4(buf + P.base[n] + j * cnt + pi);
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
            const unsigned long long g = P.fbase[n] + static_cast<unsigned long long>(j) * cnt;
            for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads) {
                const uint32_t f = *reinterpret_cast<const uint32_t*>(sigp + g + q);
                const uint32_t d = *reinterpret_cast<const uint32_t*>(P.dem + g + q);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (!byte_of(f, k)) P.pre[g + q + k] = (zero || byte_of(d, k)) ? 1 : 0;
            }
        }
        tree += encode_warp_levels<INIT>(P, buf, sigp, sv + lo(T - 2, R), j, T, R);
    } else {
        // small trees: one thread per level-(L-1) parent
        const int n = L - 1;
        const uint32_t npar = 1u << (2 * (K - 1));
        const uint32_t pbase = j * npar;
        for (uint32_t pi = threadIdx.x; pi < npar; pi += kThreads) {
            const uint32_t pm = pbase + pi;
            const bool sp = sfl[lo(n, R) + pi] != 0;
            const uint8_t d0 = INIT ? 0 : P.dem[P.fbase[n] + pm];
            bool flow, zf = false;
            if (sp) {
                const double4* cp = buf + P.base[L] + (static_cast<unsigned long long>(pm) << 2);
                const double4 c[4] = {ld4_nc(cp), ld4_nc(cp + 1), ld4_nc(cp + 2), ld4_nc(cp + 3)};
                const Enc e = encode_children<INIT>(c, P, n);
                flow = e.flow;
                zf = e.zflag;
                st4(buf + P.base[n] + pm, e.par);
                if (n > R) sv[lo(n, R) + pi] = e.par;
                ++tree;
            } else {
                flow = 0.0 >= P.tau[n];
            }
            uint8_t d = d0;
            if (INIT) {
                d = zf ? 1 : 0;
                P.dem[P.fbase[n] + pm] = d;
            }
            P.pre[P.fbase[n] + pm] = (flow || d) ? 1 : 0;
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
            const uint8_t d0 = INIT ? 0 : P.dem[P.fbase[n] + pm];
            bool flow, zf = false;
            if (sp) {
                const uint32_t c0 = lo(n + 1, R) + 4u * pi;
                const double4 c[4] = {sv[c0], sv[c0 + 1], sv[c0 + 2], sv[c0 + 3]};
                const Enc e = encode_children<INIT>(c, P, n);
                flow = e.flow;
                zf = e.zflag;
                st4(buf + P.base[n] + pm, e.par);
                if (n > R) sv[lo(n, R) + pi] = e.par;
                ++tree;
            } else {
                flow = 0.0 >= P.tau[n];
            }
            uint8_t d = d0;
            if (INIT) {
                d = zf ? 1 : 0;
                P.dem[P.fbase[n] + pm] = d;
            }
            P.pre[P.fbase[n] + pm] = (flow || d) ? 1 : 0;
        }
        __syncthreads();
    }

    const unsigned tsum = block_sum(tree, s_red);
    if (threadIdx.x == 0 && tsum) atomicAdd(&ctl->cnt_tree, (unsigned long long)tsum);
    if (P.G > 1) return;  // partitioned: k_encode_top runs after all partitions' subtrees
    if (!last_block(&ctl->done_k1, &s_last)) return;
    tl_mark(ctl, 1);
    encode_top<INIT>(P, ctl, sv, s_red);
    tl_mark(ctl, 2);
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

    unsigned ttop = 0;
    const bool top_smem = ((1u << (2 * R)) - 1u) / 3u <= ((1u << (2 * K)) - 1u) / 3u;
    for (int n = R - 1; n >= 0; --n) {
        const uint32_t cnt = 1u << (2 * n);
        const bool kids_in_smem = top_smem && n < R - 1;
        for (uint32_t pm = threadIdx.x; pm < cnt; pm += kThreads) {
            const bool sp = INIT || sigp[P.fbase[n] + pm];
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
                zf = e.zflag;
                st4(buf + P.base[n] + pm, e.par);
                if (top_smem) sv[lo(n, 0) + pm] = e.par;
                ++ttop;
            } else {
                flow = 0.0 >= P.tau[n];
                if (top_smem && n > 0 && sigp[P.fbase[n - 1] + (pm >> 2)]) sv[lo(n, 0) + pm] = ld4_cg(cell_ptr(P, p, n, pm));
            }
            uint8_t d;
            if (INIT) {
                d = zf ? 1 : 0;
                P.dem[P.fbase[n] + pm] = d;
            } else {
                d = P.dem[P.fbase[n] + pm];
            }
            P.pre[P.fbase[n] + pm] = (flow || d) ? 1 : 0;
        }
        __threadfence_block();
        __syncthreads();
    }
    const unsigned tt = block_sum(ttop, s_red);
    if (threadIdx.x == 0) {
        if (tt) atomicAdd(&ctl->cnt_tree, (unsigned long long)tt);
        ctl->done_k1 = 0;
    }
}



// K1 after t = 0 (level L-1 was re-encoded by the previous FV1): the
// subtree's level slices R..L-1 (contiguous, 32 B per cell) are brought into
// shared memory by TMA bulk copies (one per level, one mbarrier), the flags
// by word loads in parallel; levels L-2..R are then re-encoded from shared
// memory. One global round trip per CTA instead of one per level.
__global__ void __launch_bounds__(kThreads) k_encode_tma(Params P, Ctl* ctl) {
    pdl_wait();
    pdl_trigger();
    const unsigned long long t_entry = gtimer();
    if (!active(ctl, P)) return;
    tl_start(ctl, 0);
    const int probe = (blockIdx.x == 0) ? 0 : ((blockIdx.x == gridDim.x / 2) ? 8 : -1);
    auto stamp = [&](int k) {
        if (probe >= 0 && threadIdx.x == 0) ctl->dbg[probe + k] = gtimer();
    };
    stamp(0);
    if (probe >= 0 && threadIdx.x == 0) ctl->dbg[probe + 7] = t_entry;
    extern __shared__ __align__(128) double4 sv[];
    __shared__ unsigned s_red[32];
    __shared__ int s_last;
    __shared__ __align__(8) unsigned long long mbar;
    const int p = ctl->parity;
    double4* buf = P.cells[p];
    const uint8_t* sigp = P.sig[p];
    const int L = P.L, R = P.R, K = P.K;
    const uint32_t j = P.tile_lo + blockIdx.x;
    const uint32_t ncell = ((1u << (2 * K)) - 1u) / 3u;
    uint8_t* sfl = reinterpret_cast<uint8_t*>(sv + ncell);  // previous-tree flags
    uint8_t* sdm = sfl + ncell;                             // DEM flags
    if (threadIdx.x == 0) mbar_init(&mbar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&mbar, ncell * static_cast<unsigned>(sizeof(double4)));
        for (int n = R; n < L; ++n) {
            const uint32_t cnt = 1u << (2 * (n - R));
            bulk_g2s(sv + lo(n, R), buf + P.base[n] + static_cast<unsigned long long>(j) * cnt,
                     cnt * static_cast<unsigned>(sizeof(double4)), &mbar);
        }
    }
    for (int n = R; n < L; ++n) {  // flags while the bulk copies fly
        const uint32_t cnt = 1u << (2 * (n - R));
        const unsigned long long g = P.fbase[n] + static_cast<unsigned long long>(j) * cnt;
        if (cnt >= 4) {
            for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads) {
                const uint32_t wf = *reinterpret_cast<const uint32_t*>(sigp + g + q);
                const uint32_t wd = *reinterpret_cast<const uint32_t*>(P.dem + g + q);
                uint8_t* df = sfl + lo(n, R) + q;
                uint8_t* dd = sdm + lo(n, R) + q;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    df[k] = (wf >> (8 * k)) & 0xFFu;
                    dd[k] = (wd >> (8 * k)) & 0xFFu;
                }
                if (n == L - 1) {  // level L-1: the previous FV1 flagged the tree cells
                    const bool zero = 0.0 >= P.tau[n];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (!byte_of(wf, k)) P.pre[g + q + k] = (zero || byte_of(wd, k)) ? 1 : 0;
                }
            }
        } else if (threadIdx.x < cnt) {
            const uint8_t f = sigp[g + threadIdx.x], d = P.dem[g + threadIdx.x];
            sfl[lo(n, R) + threadIdx.x] = f;
            sdm[lo(n, R) + threadIdx.x] = d;
            if (n == L - 1 && !f) P.pre[g + threadIdx.x] = ((0.0 >= P.tau[n]) || d) ? 1 : 0;
        }
    }
    __syncthreads();
    stamp(1);
    mbar_wait(&mbar, 0);
    stamp(2);
    unsigned tree = 0;
    for (int n = L - 2; n >= R; --n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        const uint32_t pb = j * cnt;
        for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
            const uint32_t pm = pb + pi;
            const uint32_t li = lo(n, R) + pi;
            bool flow = 0.0 >= P.tau[n];
            if (sfl[li]) {
                const uint32_t c0 = lo(n + 1, R) + 4u * pi;
                const double4 c[4] = {sv[c0], sv[c0 + 1], sv[c0 + 2], sv[c0 + 3]};
                const Enc e = encode_children<false>(c, P, n);
                flow = e.flow;
                st4(buf + P.base[n] + pm, e.par);
                sv[li] = e.par;
                ++tree;
            }
            P.pre[P.fbase[n] + pm] = (flow || sdm[li]) ? 1 : 0;
        }
        __syncthreads();
    }
    stamp(3);
    const unsigned tsum = block_sum(tree, s_red);
    if (threadIdx.x == 0 && tsum) atomicAdd(&ctl->cnt_tree, (unsigned long long)tsum);
    stamp(4);
    if (P.G > 1) return;
    const bool lastb = last_block(&ctl->done_k1, &s_last);
    stamp(5);
    if (!lastb) return;
    tl_mark(ctl, 1);
    encode_top<false>(P, ctl, sv, s_red);
    tl_mark(ctl, 2);
}


// ----------------------------------------------------------- decode helper
// decode_tree under D4 + PTT (Alg. 5) +
// compact_leaves. In physical units a zero-detail decode is
// a copy of the parent's (h, qx, qy) to its children, so a cell
// below a chain of newly significant cells takes the value of the chain's top.
__device__ __forceinline__ void write_projection(double4* buf, const Params& P, int n, uint32_t m, uint32_t src) {
    const int ns = zo::level_of(src);
    const int p = static_cast<int>(buf == P.cells[1]);
    const double4 v = ld4_cg(cell_ptr(P, p, ns, src - zo::level_offset(ns)));
    double4* dst = buf + P.base[n] + m;
    const double4 old = ld4_cg(dst);
    st4(dst, make_double4(v.x, v.y, v.z, old.w));
}

// =========================================================================== K2
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

// band + ancestor closure per subtree; per-subtree leaf
// count; the last CTA closes levels < R and scans subtree counts into the
// leaf-list offsets (the PTT compaction's global scan, done once on 4^R
// values instead of per finest cell).
__device__ void band_top(const Params& P, Ctl* ctl, uint8_t* sfl_top, unsigned* s_red);
template <bool EXPORT>
__device__ void traverse_tile(const Params& P, Ctl* ctl, uint32_t j, uint32_t* smem3, unsigned* s_red);

__global__ void __launch_bounds__(kThreads) k_band(Params P, Ctl* ctl, int force) {
    pdl_wait();
    pdl_trigger();
    if (!force && !active(ctl, P)) return;
    tl_start(ctl, 1);
    extern __shared__ __align__(16) uint8_t smem2[];
    __shared__ unsigned s_red[32];
    __shared__ int s_last;
    const int p = ctl->parity;
    uint8_t* sigc = P.sig[p ^ 1];
    const uint8_t* pre = P.pre;
    const int L = P.L, R = P.R, K = P.K;
    const uint32_t j = P.tile_lo + blockIdx.x;
    const uint32_t ncell = ((1u << (2 * K)) - 1u) / 3u;     // subtree cells on levels R..L-1
    uint16_t* cA = reinterpret_cast<uint16_t*>(smem2);      // level-L leaves under the cell
    uint16_t* cB = cA + ncell;                              // coarser leaves under the cell
    uint8_t* sf = reinterpret_cast<uint8_t*>(cB + ncell);   // band, then final flags
    uint8_t* spre = sf + ncell;                             // pre-band flags of the subtree

    // ---- the subtree's pre-band flags, word loads where a level has >= 4 cells
    for (int n = R; n < L; ++n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        const unsigned long long g = P.fbase[n] + static_cast<unsigned long long>(j) * cnt;
        if (cnt >= 4) {
            for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads) {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(pre + g + q);
                uint8_t* d = spre + lo(n, R) + q;
                d[0] = w & 0xFFu; d[1] = (w >> 8) & 0xFFu; d[2] = (w >> 16) & 0xFFu; d[3] = w >> 24;
            }
        } else if (threadIdx.x < cnt) {
            spre[lo(n, R) + threadIdx.x] = pre[g + threadIdx.x];
        }
    }
    __syncthreads();
    // ---- band (D3). The subtree is aligned, so a neighbour inside it is the
    //      neighbour of the subtree-local Morton code on the local grid (level
    //      n - R); only edge cells look outside (global / other partitions).
    for (int n = R; n < L; ++n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        const uint32_t loN = lo(n, R), jb = j * cnt;
        auto pre_out = [&](int k, uint32_t mm) -> uint8_t {  // (k, mm) outside the subtree
            return P.ppre[owner_of(P, k, mm)][P.fbase[k] + mm];
        };
        for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
            uint8_t b = spre[loN + pi];
            if (P.band_mode == 2) {
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const uint32_t ln = zo::neighbour_dev(n - R, pi, static_cast<zo::Direction>(d));
                    if (ln != zo::kNone) {
                        b |= spre[loN + ln];
                    } else {
                        const uint32_t nb = zo::neighbour_dev(n, jb + pi, static_cast<zo::Direction>(d));
                        if (nb != zo::kNone) b |= pre_out(n, nb);
                    }
                }
            } else if (P.band_mode == 1 && n + 1 < L) {
                const uint32_t loC = lo(n + 1, R), jc = jb << 2;
                for (int k = 0; k < 4; ++k) {
                    const uint32_t lc = 4u * pi + static_cast<uint32_t>(k);
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        const uint32_t ln = zo::neighbour_dev(n + 1 - R, lc, static_cast<zo::Direction>(d));
                        if (ln != zo::kNone) {
                            b |= spre[loC + ln];
                        } else {
                            const uint32_t nb = zo::neighbour_dev(n + 1, jc + lc, static_cast<zo::Direction>(d));
                            if (nb != zo::kNone) b |= pre_out(n + 1, nb);
                        }
                    }
                }
            }
            sf[loN + pi] = b ? 1 : 0;
        }
    }
    __syncthreads();
    // ---- ancestor closure bottom-up, with the leaf counts of every subtree
    //      cell assuming it is reached (level L-1: 4 level-L leaves or itself)
    {
        const uint32_t cnt = 1u << (2 * (L - 1 - R));
        for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
            const bool sg = sf[lo(L - 1, R) + pi] != 0;
            cA[lo(L - 1, R) + pi] = sg ? 4 : 0;
            cB[lo(L - 1, R) + pi] = sg ? 0 : 1;
        }
    }
    __syncthreads();
    for (int n = L - 2; n >= R; --n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
            const uint32_t c = lo(n + 1, R) + 4u * pi;
            const bool sg = sf[lo(n, R) + pi] || sf[c] || sf[c + 1] || sf[c + 2] || sf[c + 3];
            sf[lo(n, R) + pi] = sg ? 1 : 0;
            cA[lo(n, R) + pi] = sg ? static_cast<uint16_t>(cA[c] + cA[c + 1] + cA[c + 2] + cA[c + 3]) : 0;
            cB[lo(n, R) + pi] = sg ? static_cast<uint16_t>(cB[c] + cB[c + 1] + cB[c + 2] + cB[c + 3]) : 1;
        }
        __syncthreads();
    }
    // ---- final flags of the subtree, word stores where a level has >= 4 cells
    for (int n = R; n < L; ++n) {
        const uint32_t cnt = 1u << (2 * (n - R));
        const unsigned long long g = P.fbase[n] + static_cast<unsigned long long>(j) * cnt;
        if (cnt >= 4) {
            for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads) {
                const uint8_t* d = sf + lo(n, R) + q;
                *reinterpret_cast<uint32_t*>(sigc + g + q) =
                    uint32_t(d[0]) | (uint32_t(d[1]) << 8) | (uint32_t(d[2]) << 16) | (uint32_t(d[3]) << 24);
            }
        } else if (threadIdx.x < cnt) {
            sigc[g + threadIdx.x] = sf[lo(n, R) + threadIdx.x];
        }
    }
    if (threadIdx.x == 0) {
        P.tile_cnt[j] = cA[0];
        P.tile_cnt[P.n_tiles + j] = cB[0];
    }
    if (P.G > 1) return;  // partitioned: k_band_top runs after all partitions' subtrees
    const bool fuse = P.fuse_k3 && !force;
    const unsigned long long target = static_cast<unsigned long long>(ctl->step) + 1ull;
    const bool last = last_block(&ctl->done_k2, &s_last);
    if (last) {
        tl_mark(ctl, 4);
        band_top(P, ctl, smem2, s_red);
        tl_mark(ctl, 5);
    }
    if (!fuse) return;
    // ---- K3 fused: every CTA is resident (host-checked), so the others wait
    //      for the last CTA's offsets instead of a new launch
    __syncthreads();
    if (threadIdx.x == 0) {
        if (last) {
            __threadfence();
            st_release_u64(&ctl->k2_ready, target);
        } else {
            const unsigned long long t0 = gtimer();
            while (ld_acquire_u64(&ctl->k2_ready) != target) {
                __nanosleep(200);
                if (gtimer() - t0 > 2000000000ull) {  // 2 s: never expected; fail instead of hanging
                    report_error(ctl, kErrDt, j, 0, kStageTraverse);
                    break;
                }
            }
        }
    }
    __syncthreads();
    tl_start(ctl, 2);
    traverse_tile<false>(P, ctl, j, reinterpret_cast<uint32_t*>(smem2), s_red);
}

__global__ void __launch_bounds__(kThreads) k_band_top(Params P, Ctl* ctl, int force) {
    pdl_wait();
    if (!force && !active(ctl, P)) return;
    extern __shared__ __align__(16) uint8_t smem2t[];
    __shared__ unsigned s_red[32];
    band_top(P, ctl, smem2t, s_red);
}

// Top of K2 (one CTA), all in shared memory: tpre / tprev = pre-band and
// previous flags of levels 0..R (replicated), tsig = current flags of levels
// 0..R (level R from every subtree's partition), intree = "on the current
// tree", tcnt = per-subtree counts. Band + closure of levels R-1..0, decode of
// levels 1..R, per-subtree traversal depth and the leaf-list scans.
__device__ void band_top(const Params& P, Ctl* ctl, uint8_t* sfl_top, unsigned* s_red) {
    const int p = ctl->parity;
    uint8_t* sigc = P.sig[p ^ 1];
    const uint8_t* pre = P.pre;
    const int L = P.L, R = P.R;

    uint8_t* tsig = sfl_top;                  // lo(R+1)
    uint8_t* tprev = tsig + lo(R + 1, 0);     // lo(R+1)
    uint8_t* tpre = tprev + lo(R + 1, 0);     // lo(R+1)
    uint8_t* intree = tpre + lo(R + 1, 0);    // lo(R+1)
    uint32_t* tcnt = reinterpret_cast<uint32_t*>(sfl_top + ((4u * lo(R + 1, 0) + 15u) & ~15u));  // 2 x 4^R
    const uint8_t* sigp = P.sig[p];
    for (int n = 0; n <= R; ++n) {
        const uint32_t cnt = 1u << (2 * n);
        for (uint32_t m = threadIdx.x; m < cnt; m += kThreads) {
            if (n < L) {
                tpre[lo(n, 0) + m] = pre[P.fbase[n] + m];
                tprev[lo(n, 0) + m] = sigp[P.fbase[n] + m];
            }
            if (n == R) {
                const int g = owner_of(P, R, m);  // subtree m's partition
                tsig[lo(R, 0) + m] = ldcg_u8(P.psig[g][p ^ 1] + P.fbase[R] + m);
                tcnt[m] = ldcg_u32(P.ptile_cnt[g] + m);
                tcnt[P.n_tiles + m] = ldcg_u32(P.ptile_cnt[g] + P.n_tiles + m);
            }
        }
    }
    __syncthreads();
    for (int n = R - 1; n >= 0; --n) {  // band + closure, levels R-1 .. 0
        const uint32_t cnt = 1u << (2 * n);
        for (uint32_t m = threadIdx.x; m < cnt; m += kThreads) {
            uint8_t b = band_flag(P.band_mode, L, n, m, [&](int k, uint32_t mm) { return tpre[lo(k, 0) + mm]; });
            const uint8_t* c = tsig + lo(n + 1, 0) + 4u * m;
            if (c[0] | c[1] | c[2] | c[3]) b = 1;
            sigc[P.fbase[n] + m] = b;
            tsig[lo(n, 0) + m] = b;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) intree[0] = 1;
    __syncthreads();
    for (int n = 1; n <= R; ++n) {
        const uint32_t cnt = 1u << (2 * n);
        for (uint32_t m = threadIdx.x; m < cnt; m += kThreads)
            intree[lo(n, 0) + m] = intree[lo(n - 1, 0) + (m >> 2)] & tsig[lo(n - 1, 0) + (m >> 2)];
        __syncthreads();
    }
    // decode (projection, D4) of levels 1..R: a cell on the tree below a newly
    // significant ancestor takes the value of the topmost such ancestor; the
    // level-R result is also each subtree's inherited source for K3
    {
        double4* buf = P.cells[p];
        unsigned nnew = 0;
        for (int n = 0; n < R; ++n) {
            const uint32_t cnt = 1u << (2 * n);
            for (uint32_t m = threadIdx.x; m < cnt; m += kThreads)
                nnew += (tsig[lo(n, 0) + m] && !tprev[lo(n, 0) + m]) ? 1u : 0u;
        }
        for (int n = 1; n <= R; ++n) {
            const uint32_t cnt = 1u << (2 * n);
            for (uint32_t m = threadIdx.x; m < cnt; m += kThreads) {
                uint32_t src = kNoSrc;
                if (intree[lo(n, 0) + m]) {
                    for (int k = 0; k < n; ++k) {
                        const uint32_t a = lo(k, 0) + (m >> (2 * (n - k)));
                        if (tsig[a] && !tprev[a]) {
                            src = zo::z_of(k, m >> (2 * (n - k)));
                            break;
                        }
                    }
                    if (src != kNoSrc) write_projection(buf, P, n, m, src);
                }
                if (n == R) P.tile_src[m] = src;
            }
        }
        if (R == 0 && threadIdx.x == 0) P.tile_src[0] = kNoSrc;  // the root has no ancestor
        const unsigned tn = block_sum(nnew, s_red);
        if (threadIdx.x == 0 && tn) atomicAdd(&ctl->cnt_new, (unsigned long long)tn);
    }
    // ---- per-subtree leaf counts, their exclusive scans, and each subtree's
    //      traversal depth (R = reached, else the level of its covering leaf).
    //      Hot-path list: all level-L leaves (A) first, then the coarser ones
    //      (B); export list: Morton order (A and B interleaved per subtree).
    const uint32_t nt = static_cast<uint32_t>(P.n_tiles);
    const uint32_t per = (nt + kThreads - 1) / kThreads;
    const uint32_t a = threadIdx.x * per;
    const uint32_t b = min(nt, a + per);
    unsigned la = 0, lb = 0;
    for (uint32_t t = a; t < b; ++t) {
        int n = R;
        while (!intree[lo(n, 0) + (t >> (2 * (R - n)))]) --n;
        unsigned ca = 0, cb;
        if (n == R) {
            ca = tcnt[t];
            cb = tcnt[nt + t];
        } else {
            cb = ((t & ((1u << (2 * (R - n))) - 1u)) == 0u) ? 1u : 0u;
        }
        P.tile_lvl[t] = static_cast<uint32_t>(n);
        P.tile_off[t] = ca;       // temporarily the counts
        P.tile_off[nt + t] = cb;
        la += ca;
        lb += cb;
    }
    unsigned ta, tb;
    unsigned oa = block_exscan(la, s_red, &ta);
    unsigned ob = block_exscan(lb, s_red, &tb);
    unsigned om = oa + ob;
    for (uint32_t t = a; t < b; ++t) {
        const unsigned ca = P.tile_off[t], cb = P.tile_off[nt + t];
        P.tile_off[t] = oa;               // A: level-L leaves
        P.tile_off[nt + t] = ta + ob;     // B: after all of A
        P.tile_off[2 * nt + t] = om;      // Morton-ordered export list
        oa += ca;
        ob += cb;
        om += ca + cb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ctl->n_leaves = ta + tb;
        ctl->n_leaves_A = ta;
        // this partition's slices of the A and B lists
        ctl->a_lo = P.tile_off[P.tile_lo];
        ctl->a_hi = (P.tile_hi < nt) ? P.tile_off[P.tile_hi] : ta;
        ctl->b_lo = P.tile_off[nt + P.tile_lo];
        ctl->b_hi = (P.tile_hi < nt) ? P.tile_off[nt + P.tile_hi] : ta + tb;
        ctl->done_k2 = 0;
    }
}


// decode + PTT + compaction of subtree j (K3). EXPORT = re-run the traversal
// of the current tree (after a step) into the Morton-ordered export list, with
// no side effects (no decode, no timeline).
template <bool EXPORT>
__device__ void traverse_tile(const Params& P, Ctl* ctl, uint32_t j, uint32_t* smem3, unsigned* s_red) {
    const int p = ctl->parity;
    double4* buf = P.cells[p];
    const uint8_t* sigc = EXPORT ? P.sig[p] : P.sig[p ^ 1];
    const uint8_t* sigp = EXPORT ? P.sig[p ^ 1] : P.sig[p];
    const int L = P.L, R = P.R, K = P.K;
    const uint32_t ncell = ((1u << (2 * K)) - 1u) / 3u;  // subtree cells on levels R..L-1
    uint32_t* src = smem3;                               // [ncell]
    uint8_t* sc = reinterpret_cast<uint8_t*>(src + ncell);  // [ncell]
    uint8_t* sp = sc + ncell;                               // [ncell]

    const uint32_t leafn = ldcg_u32(P.tile_lvl + j);  // written by K2's last CTA
    const uint32_t rootsrc = ldcg_u32(P.tile_src + j);
    const bool reached = leafn == static_cast<uint32_t>(R);
    int any_new = 0;
    for (int n = R; n < L; ++n) {  // current / previous flags of the subtree, word loads
        const uint32_t cnt = 1u << (2 * (n - R));
        const unsigned long long g = P.fbase[n] + static_cast<unsigned long long>(j) * cnt;
        if (cnt >= 4) {
            for (uint32_t q = 4u * threadIdx.x; q < cnt; q += 4u * kThreads) {
                const uint32_t wc = *reinterpret_cast<const uint32_t*>(sigc + g + q);
                const uint32_t wp = *reinterpret_cast<const uint32_t*>(sigp + g + q);
                uint8_t* dc = sc + lo(n, R) + q;
                uint8_t* dp = sp + lo(n, R) + q;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    dc[k] = (wc >> (8 * k)) & 0xFFu;
                    dp[k] = (wp >> (8 * k)) & 0xFFu;
                }
                any_new |= (wc & ~wp) ? 1 : 0;
            }
        } else if (threadIdx.x < cnt) {
            const uint8_t c = sigc[g + threadIdx.x], q = sigp[g + threadIdx.x];
            sc[lo(n, R) + threadIdx.x] = c;
            sp[lo(n, R) + threadIdx.x] = q;
            any_new |= (c && !q) ? 1 : 0;
        }
    }
    // decode is needed only where something became significant
    any_new = __syncthreads_or(any_new | (rootsrc != kNoSrc ? 1 : 0));
    if (EXPORT) any_new = 0;
    unsigned nnew = 0;

    if (reached && any_new) {
        // ---- projection inside the subtree, top-down
        if (threadIdx.x == 0) src[0] = rootsrc;  // the root itself was projected by K2
        __syncthreads();
        for (int n = R; n < L; ++n) {
            const uint32_t cnt = 1u << (2 * (n - R));
            for (uint32_t pi = threadIdx.x; pi < cnt; pi += kThreads) {
                const uint32_t li = lo(n, R) + pi;
                const uint32_t pm = j * cnt + pi;
                const bool isnew = sc[li] && !sp[li];
                nnew += isnew ? 1u : 0u;
                uint32_t cs = kNoSrc;
                if (sc[li]) cs = (src[li] != kNoSrc) ? src[li] : (isnew ? zo::z_of(n, pm) : kNoSrc);
                if (n + 1 < L) {
                    const uint32_t lc = lo(n + 1, R) + 4u * pi;
                    src[lc] = cs; src[lc + 1] = cs; src[lc + 2] = cs; src[lc + 3] = cs;
                }
                if (cs != kNoSrc)
                    for (uint32_t k = 0; k < 4; ++k) write_projection(buf, P, n + 1, 4u * pm + k, cs);
            }
            __syncthreads();
        }
    }
    if (!EXPORT) {
        const unsigned tn = block_sum(nnew, s_red);
        if (threadIdx.x == 0 && tn) atomicAdd(&ctl->cnt_new, (unsigned long long)tn);
    }

    // ---- PTT + compaction. Hot path: level-L leaves to list A at
    //      tile_off[j], coarser leaves to list B at tile_off[nt + j]; export:
    //      one Morton-ordered list at tile_off[2 nt + j].
    const uint32_t nt = static_cast<uint32_t>(P.n_tiles);
    uint32_t* outA = EXPORT ? P.leaves_x : P.leaves;
    uint32_t oa = ldcg_u32(P.tile_off + (EXPORT ? 2 * nt + j : j));
    uint32_t ob = EXPORT ? 0u : ldcg_u32(P.tile_off + nt + j);
    if (!reached) {
        const int n = static_cast<int>(leafn);
        if (threadIdx.x == 0 && ((j & ((1u << (2 * (R - n))) - 1u)) == 0u))
            (EXPORT ? outA[oa] : P.leaves[ob]) = zo::z_of(n, j >> (2 * (R - n)));
        if (!EXPORT) tl_mark(ctl, 8);
        return;
    }
    // one walk per level-(L-2) cell (its 4 level-(L-1) children share the
    // path); K = 1 (L = 1) walks the level-(L-1) cells directly
    const int G = (K >= 2) ? L - 2 : L - 1;              // walked level
    const uint32_t ng = 1u << (2 * (G - R));               // walked cells in the subtree
    const uint32_t per = (ng + kThreads - 1) / kThreads;
    const uint32_t a = threadIdx.x * per;
    const uint32_t b = min(ng, a + per);
    const uint32_t loL1 = lo(L - 1, R);
    // depth of the walk: first level <= G whose cell is not significant, or G + 1
    auto walk = [&](uint32_t t) -> int {
        int n = R;
        uint32_t off = 0, span = 1;
        while (n <= G && sc[off + (t >> (2 * (G - n)))]) {
            off += span;
            span <<= 2;
            ++n;
        }
        return n;
    };
    unsigned ca = 0, cb = 0;
    for (uint32_t t = a; t < b; ++t) {
        const int n = walk(t);
        if (n <= G) {
            cb += ((t & ((1u << (2 * (G - n))) - 1u)) == 0u) ? 1u : 0u;
        } else if (G == L - 1) {
            ca += 4;
        } else {
            for (uint32_t k = 0; k < 4; ++k) {
                if (sc[loL1 + 4u * t + k]) ca += 4;
                else cb += 1;
            }
        }
    }
    unsigned total;
    if (EXPORT) {
        oa += block_exscan(ca + cb, s_red, &total);
    } else {
        oa += block_exscan(ca, s_red, &total);
        ob += block_exscan(cb, s_red, &total);
    }
    auto emitA = [&](uint32_t m1) {  // the 4 level-L children of level-(L-1) cell m1
        const uint32_t z0 = zo::z_of(L, m1 << 2);
        outA[oa] = z0; outA[oa + 1] = z0 + 1; outA[oa + 2] = z0 + 2; outA[oa + 3] = z0 + 3;
        oa += 4;
    };
    auto emitB = [&](uint32_t z) {
        if (EXPORT) outA[oa++] = z;
        else P.leaves[ob++] = z;
    };
    const uint32_t gbase = j * ng;
    for (uint32_t t = a; t < b; ++t) {
        const int n = walk(t);
        const uint32_t gm = gbase + t;
        if (n <= G) {
            if ((t & ((1u << (2 * (G - n))) - 1u)) == 0u) emitB(zo::z_of(n, gm >> (2 * (G - n))));
        } else if (G == L - 1) {
            emitA(gm);
        } else {
            for (uint32_t k = 0; k < 4; ++k) {
                const uint32_t m1 = 4u * gm + k;
                if (sc[loL1 + 4u * t + k]) emitA(m1);
                else emitB(zo::z_of(L - 1, m1));
            }
        }
    }
    if (!EXPORT) {
        __syncthreads();
        tl_mark(ctl, 8);
    }
}

template <bool EXPORT>
__global__ void __launch_bounds__(kThreads) k_traverse(Params P, Ctl* ctl, int force) {
    pdl_wait();
    pdl_trigger();
    if (!EXPORT && !force && !active(ctl, P)) return;
    if (!EXPORT) tl_start(ctl, 2);
    extern __shared__ uint32_t smem3[];
    __shared__ unsigned s_red[32];
    traverse_tile<EXPORT>(P, ctl, P.tile_lo + blockIdx.x, smem3, s_red);
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
__device__ __forceinline__ void cfl_reduce_and_finalize(const Params& P, Ctl* ctl, double rate, bool advance) {
    __shared__ unsigned long long s_max[kThreads / 32];
    __shared__ int s_last;
    const int slot = static_cast<int>(ctl->step & 1);
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
    tl_mark(ctl, 10);
    if (threadIdx.x == 0) {
        const unsigned long long m = atomicAdd(&ctl->rate_bits[slot], 0ull);
        finalize_dt(P, ctl, __longlong_as_double(static_cast<long long>(m)), advance);
        ctl->rate_bits[slot] = 0ull;
        ctl->done_k5 = 0;
        const int tb = advance ? static_cast<int>((ctl->step - 1) & 1) : tl_buf(ctl);
        ctl->tl[tb][11] = gtimer();
        if (advance)
            for (int k = 0; k < 12; ++k) ctl->tl[tb ^ 1][k] = 0ull;  // next step's buffer
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
    const int tb = tl_buf(ctl);
    finalize_dt(P, ctl, __longlong_as_double(static_cast<long long>(m)), advance != 0);
    if (!advance) return;  // initialise: the host clears the slots afterwards
    ctl->rate_bits[slot ^ 1] = 0ull;
    ctl->tl[tb][11] = gtimer();
    for (int k = 0; k < 12; ++k) ctl->tl[tb ^ 1][k] = 0ull;
}

// covering cell of a same-level neighbour region whose parent (k, mm) is NOT
// significant: walk up until the parent is significant (SPEC.md:248 — the
// coarser covering leaf); the fast path (parent significant -> the same-level
// cell itself) is tested by the caller for all four faces at once
__device__ __forceinline__ const double4* covering_local(const Params& P, const double4* cur, const uint8_t* sigc, int k,
                                                        uint32_t mm) {
    while (k > 0 && !sigc[P.fbase[k - 1] + (mm >> 2)]) {
        mm >>= 2;
        --k;
    }
    return cur + P.base[k] + mm;
}
__device__ __forceinline__ double4* covering(const Params& P, int cur, int k, uint32_t mm) {
    while (k > 0 && !sig_at(P, cur ^ 1, k - 1, mm >> 2)) {
        mm >>= 2;
        --k;
    }
    return cell_ptr(P, cur, k, mm);
}

// FV1 over the leaf list: persistent grid-stride, one thread per
// leaf; reads the current buffer, writes leaf slots of the other (D15).
template <bool UNIFORM, int MINB = 2, bool PART = false>
__global__ void __launch_bounds__(kThreads, MINB) k_fv1(Params P, Ctl* ctl) {
    pdl_wait();
    pdl_trigger();
    if (!active(ctl, P)) return;
    tl_start(ctl, 3);
    const int p = ctl->parity;
    const double4* __restrict__ cur = P.cells[p];
    double4* __restrict__ nxt = P.cells[p ^ 1];
    const uint8_t* __restrict__ sigc = P.sig[p ^ 1];
    // this partition's leaves: its slice of the level-L list A (sibling
    // quadruples at indices 4g..4g+3) followed by its slice of list B
    const uint32_t a_lo = UNIFORM ? 0u : ctl->a_lo, b_lo = UNIFORM ? 0u : ctl->b_lo;
    const uint32_t NA = UNIFORM ? 0u : ctl->a_hi - a_lo;
    const uint32_t N = UNIFORM ? (1u << (2 * P.L)) : NA + (ctl->b_hi - b_lo);
    auto leaf_at = [&](uint32_t k) { return P.leaves[k < NA ? a_lo + k : b_lo + (k - NA)]; };
    const double t = ctl->t, dt = ctl->dt;
    const double inflow = series_value(P, t);
    const int lane = threadIdx.x & 31;
    double mx = 0.0;
    unsigned tree = 0;
    const uint32_t stride = gridDim.x * kThreads;
    // warp-uniform trip count: every lane runs every iteration (shuffles below)
    uint32_t wbase = blockIdx.x * kThreads + (threadIdx.x & ~31u);
    uint32_t z_next = (!UNIFORM && wbase + lane < N) ? leaf_at(wbase + lane) : 0u;
    for (; wbase < N; wbase += stride) {
        const uint32_t i = wbase + lane;
        const bool valid = i < N;
        int n;
        uint32_t m;
        if (UNIFORM) {
            n = P.L;
            m = valid ? i : 0u;
        } else {
            const uint32_t z = valid ? z_next : zo::level_offset(P.L);  // leaf ids prefetched one iteration ahead
            if (i + stride < N) z_next = leaf_at(i + stride);
            n = zo::level_of(z);
            m = z - zo::level_offset(n);
        }
        double hn = 0.0, qxn = 0.0, qyn = 0.0, zown = 0.0;
        if (valid) {
            // every global read of this leaf is issued before any arithmetic:
            // own cell, the neighbours' parent-level flags, the neighbours
            const double4 o4 = ld4_nc(cur + P.base[n] + m);
            uint32_t nm[4];
            const double4* src[4];
#pragma unroll
            for (int d = 0; d < 4; ++d) nm[d] = zo::neighbour_dev(n, m, static_cast<zo::Direction>(d));
            if (UNIFORM) {
#pragma unroll
                for (int d = 0; d < 4; ++d) src[d] = cur + P.base[n] + nm[d];
            } else {
                uint8_t f[4];
                if (PART) {  // cross-partition reads through the peer tables
#pragma unroll
                    for (int d = 0; d < 4; ++d) f[d] = (nm[d] != zo::kNone) ? sig_at(P, p ^ 1, n - 1, nm[d] >> 2) : 1;
#pragma unroll
                    for (int d = 0; d < 4; ++d)
                        src[d] = f[d] ? cell_ptr(P, p, n, nm[d]) : covering(P, p, n - 1, nm[d] >> 2);
                } else {
#pragma unroll
                    for (int d = 0; d < 4; ++d) f[d] = (nm[d] != zo::kNone) ? sigc[P.fbase[n - 1] + (nm[d] >> 2)] : 1;
#pragma unroll
                    for (int d = 0; d < 4; ++d)
                        src[d] = f[d] ? cur + P.base[n] + nm[d] : covering_local(P, cur, sigc, n - 1, nm[d] >> 2);
                }
            }
            double4 r4[4];
#pragma unroll
            for (int d = 0; d < 4; ++d)
                if (nm[d] != zo::kNone) r4[d] = ld4_nc(src[d]);
            // dry neighbourhood: own cell and every neighbour / ghost below
            // h_dry => every reconstructed depth is 0, every flux 0, the bed
            // corrections cancel pairwise: h stays, q = 0 (the general path
            // gives the same bits)
            bool all_dry = o4.x < P.phys.hdry;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                if (nm[d] != zo::kNone) all_dry = all_dry && r4[d].x < P.phys.hdry;
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
                    return make_cell(r4[d], P.phys);
                };
                fv1_cell_seq(own, neighbour, P.inv_dx[n], dt, P.phys, hn, qxn, qyn);
            }
            zown = o4.w;
            if (!(isfinite(hn) && isfinite(qxn) && isfinite(qyn)))
                report_error(ctl, kErrNonFinite, zo::z_of(n, m), !isfinite(hn) ? 0 : (!isfinite(qxn) ? 1 : 2),
                             kStageFV1);
            st4(nxt + P.base[n] + m, make_double4(hn, qxn, qyn, zown));
            const double c = cfl_rate(hn, qxn, qyn, P.inv_dx[n], P.phys);
            mx = c > mx ? c : mx;
        }
        // Next step's zero_details_and_reencode of level L-1, fused here: the
        // four updated children of a previous-tree level-(L-1) cell sit in
        // lanes 4k..4k+3; lane 4k forms the parent and its significance
        // (identical arithmetic to k_encode; the next K1 starts at L-2).
        if (!UNIFORM && wbase < NA) {
            const Enc e = encode_lanes<false>(make_double4(hn, qxn, qyn, zown), 1, P, P.L - 1);
            if ((lane & 3) == 0 && i < NA) {
                const uint32_t pm = m >> 2;
                st4(nxt + P.base[P.L - 1] + pm, e.par);
                const unsigned long long fi = P.fbase[P.L - 1] + pm;
                P.pre[fi] = (e.flow || P.dem[fi]) ? 1 : 0;
                ++tree;
            }
        }
    }
    if (!UNIFORM) {
        __shared__ unsigned s_red5[32];
        const unsigned tt = block_sum(tree, s_red5);
        if (threadIdx.x == 0 && tt) atomicAdd(&ctl->cnt_tree, (unsigned long long)tt);
    }
    cfl_reduce_and_finalize(P, ctl, mx, true);
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
        const double4 v = ld4(cur + P.base[n] + m);
        const double c = cfl_rate(v.x, v.y, v.z, P.inv_dx[n], P.phys);
        mx = c > mx ? c : mx;
    }
    cfl_reduce_and_finalize(P, ctl, mx, false);
}

// =========================================================== import / export
// initial discretisation: row-major (south row first) finest
// fields -> Morton slots of level L; s_max per quantity.
__global__ void __launch_bounds__(kThreads) k_import(Params P, Ctl* ctl, const double* h, const double* qx,
                                                     const double* qy, const double* z, int buffer) {
    const uint32_t side = 1u << P.L;
    const uint64_t total = static_cast<uint64_t>(side) * side;
    double mx[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint64_t r = blockIdx.x * (uint64_t)kThreads + threadIdx.x; r < total; r += (uint64_t)gridDim.x * kThreads) {
        const uint32_t i = static_cast<uint32_t>(r & (side - 1)), jj = static_cast<uint32_t>(r >> P.L);
        const uint32_t m = zo::interleave(i, jj);
        const double4 v = make_double4(h[r], qx[r], qy[r], z[r]);
        if (!(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w)))
            report_error(ctl, kErrNonFinite, zo::z_of(P.L, m), 0, kStageImport);
        st4(P.cells[buffer] + P.base[P.L] + m, v);
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

}  // namespace hwfv1
