/* swamp_gpu.h — C-ABI of the B200-native GPU-HWFV1 adaptive time-step loop.
 *
 * This is the drop-in boundary for the reference's adaptive solver path
 * (SPEC.md "engine" module) built on the
 * reference's Z-order index algebra (/root/reference/proj/include/swamp/
 * zorder.hpp:9-133). The reference ships no compiled engine; its interface is
 * the spec's  SimConfig, SimState,
 * StepReport, initialise, step_adaptive
 * (SPEC.md:399), step_uniform, run. Each entry
 * point below names the operation it replaces.
 *
 * ABI rules: plain C types only; every function returns a status (0 = ok,
 * <0 = error, see SWAMP_E_*); no exceptions cross; the handle owns all device
 * memory, the caller owns every host buffer; one handle per engine, driven
 * from one control thread. The include/swamp/engine.hpp facade
 * rethrows errors as std::runtime_error / std::out_of_range.
 *
 * Conventions shared with the reference:
 *   - finest-level input rasters are row-major with row j = 0 the SOUTH row
 *     and column i = 0 the WEST column (j up, zorder.hpp:11-12, 123-128);
 *   - hierarchy exports are indexed by z-index z = (4^n-1)/3 + m
 *     (zorder.hpp:68-73) and hold SCALE COEFFICIENTS s (physical value =
 *     s * 2^(n-L));
 *   - neighbour descriptors are z-indices, or
 *     SWAMP_BOUNDARY_BASE + boundary kind for an edge of the domain;
 *   - leaves are listed in ascending first-covered-Morton order.
 */
#ifndef SWAMP_GPU_H
#define SWAMP_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWAMP_OK 0
#define SWAMP_E_ARG (-1)      /* invalid argument / config         */
#define SWAMP_E_CUDA (-2)     /* CUDA runtime failure                            */
#define SWAMP_E_NONFINITE (-3) /* non-finite coefficient / flux */
#define SWAMP_E_DT (-4)       /* dt <= 0 or non-finite             */
#define SWAMP_E_STATE (-5)    /* call not valid in the current state             */
#define SWAMP_E_NOMEM (-6)    /* device allocation failed                        */
#define SWAMP_E_PEER (-7)     /* a partition / rank never reached a barrier (10 s) */

/* boundary kinds */
#define SWAMP_BC_REFLECTIVE 0
#define SWAMP_BC_TRANSMISSIVE 1
#define SWAMP_BC_INFLOW 2

/* refinement safety band (D3) */
#define SWAMP_BAND_NONE 0       /* strict-paper mode              */
#define SWAMP_BAND_PARENTS 1    /* SPEC.md:195 literal: neighbours' parents     */
#define SWAMP_BAND_NEIGHBOURS 2 /* default: same-level face neighbours          */

#define SWAMP_INFLOW_DEPTH 0
#define SWAMP_INFLOW_ETA 1

#define SWAMP_BOUNDARY_BASE 0xFFFFFFF0u /* descriptor = BASE + kind            */

/* SimConfig. The hierarchy is the 2^L x 2^L square of side
 * `width` with lower-left corner (x0, y0). */
typedef struct swamp_config {
    int32_t L;             /* finest level, 1..13 (zorder.hpp:21)              */
    int32_t band_mode;     /* SWAMP_BAND_*                                      */
    double epsilon;        /* error threshold >= 0                              */
    double width;          /* side W of the square domain (m)                   */
    double x0, y0;         /* lower-left corner (m)                             */
    double cfl;            /* CFL number C (default 0.5)           */
    double g;              /* gravity (default 9.80665)            */
    double manning;        /* n_M (s m^-1/3)                                    */
    double h_dry;          /* dry threshold (default 1e-6)         */
    double t_end;          /* simulation end time (s)                           */
    double dt_fallback;    /* all-dry time step                   */
    int32_t bc[4];         /* W, E, N, S edge kinds: SWAMP_BC_*                 */
    int32_t inflow_mode;   /* SWAMP_INFLOW_DEPTH or SWAMP_INFLOW_ETA            */
    int32_t inflow_n;      /* number of (t, v) samples                          */
    int32_t n_outputs;     /* number of output times                            */
    const double* inflow_t; /* inflow series times, ascending                   */
    const double* inflow_v; /* inflow series values                             */
    const double* output_times; /* ascending; dt is clipped to hit them        */
    /* inactive finest cells (D16): 4^L bytes,
     * row-major south row first, nonzero = inactive (a reflective wall,
     * excluded from CFL and s_max; its state is kept); NULL = all active.
     * swamp_io_load_dem produces it from a DEM's nodata / outside cells. */
    const uint8_t* inactive;
} swamp_config;

/* StepReport. Stage times are device times in ms of the
 * step just taken, from the kernels' %globaltimer stamps (first CTA start to
 * last CTA end of each kernel); with swamp_gpu_set_profiling(1) they come
 * from CUDA events recorded between the kernels instead. */
typedef struct swamp_step_report {
    int64_t step;          /* steps taken so far                                */
    double t;              /* simulation time after the step                    */
    double dt;             /* dt that the NEXT step will use                    */
    double dt_used;        /* dt of the step just taken                         */
    int64_t n_leaves;      /* leaves of the grid the step was computed on       */
    int64_t n_leaves_next; /* leaves after re-adaptation (next step's grid)     */
    double ms_encode_flag; /* zero_details_and_reencode + significance          */
    double ms_band_closure;/* band + ancestor closure + leaf-count scan         */
    double ms_decode_traverse; /* decode + PTT + compaction                     */
    double ms_neighbours;  /* fused into FV1 on this build: always 0            */
    double ms_fv1;         /* FV1 + friction + write-back + CFL reduce          */
    double ms_total;
    /* near-threshold cells of the step (BASELINE north star; D8):
     * cells whose significance was evaluated in the step's re-encode (the
     * previous tree) with |d_norm - eps 2^(n-L)| <= 1e-12 eps 2^(n-L),
     * d_norm = max over h, qx, qy of max|d| / s_max */
    int64_t n_near_threshold;
} swamp_step_report;

typedef struct swamp_gpu swamp_gpu;

/* initialise: upload the finest-level fields (row-major,
 * south row first, length 4^L each), full bottom-up encode, DEM mask,
 * significance, traversal, first dt. `device` is the CUDA ordinal. */
int swamp_gpu_create(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                     const double* z, int device, swamp_gpu** out);
int swamp_gpu_destroy(swamp_gpu* g);

/* Destroyed engines return their device buffers (and pinned control mirrors)
 * to a process-wide cache that the next swamp_gpu_create of the same shape
 * reuses (cudaMalloc / cudaFree of an L = 11 engine's ~400 MB cost 3-50 ms
 * per call on B200). This releases every cached block of `device` (-1: all
 * devices). No reference counterpart (host-side allocation policy). */
int swamp_gpu_trim_cache(int device);

/* Morton-subtree partitioned engine (BASELINE north star):
 * n_parts (1, 2, 4 or 8; must divide the number of level-R subtrees 4^R)
 * contiguous ranges of level-R subtrees, partition k on CUDA device
 * devices[k] (devices may repeat: several partitions on one GPU run as
 * virtual partitions with identical results). Cross-partition data (band
 * flags, flux neighbours, level-R encode inputs, subtree counts, the CFL max)
 * is read in place through peer pointers (NVLink peer access between distinct
 * devices); results are bitwise equal to the single-partition engine. All
 * other entry points accept the returned handle (no uniform / profiling). */
int swamp_gpu_create_partitioned(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                                 const double* z, int n_parts, const int* devices, swamp_gpu** out);

/* One Morton-subtree partition per process (torchrun: one rank per GPU).
 * Three calls, in this order on every rank:
 *   swamp_gpu_rank_create  — allocate and import partition `rank` of `world`
 *     on CUDA `device`; writes this rank's SWAMP_RANK_BLOB_BYTES blob (CUDA
 *     IPC handles of the arrays peers read in place);
 *   (the caller all-gathers the blobs, rank order, e.g. torch.distributed)
 *   swamp_gpu_rank_connect — map every peer's arrays (IPC; a rank handle of
 *     the same process is used directly) and enqueue initialise; it
 *     completes once every rank has connected (device-side barriers);
 *   swamp_gpu_rank_ready   — wait for initialise, build the step graphs.
 * Then step / advance / enqueue / run / info / export_finest / export_tree
 * work as for one engine; every rank must step the same number of times
 * (the ranks synchronise on the device). copy_leaves returns the count only. */
#define SWAMP_RANK_BLOB_BYTES 1024
int swamp_gpu_rank_create(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                          const double* z, int rank, int world, int device, swamp_gpu** out, uint8_t* blob);
int swamp_gpu_rank_connect(swamp_gpu* g, const uint8_t* blobs);
int swamp_gpu_rank_ready(swamp_gpu* g);

/* Dynamic repartitioning: move the partition boundaries
 * so that every partition holds about the same number of leaves (contiguous
 * Morton subtree ranges from the current leaf-list offsets) and pull the
 * subtrees a partition gains from their old owner (peer reads). Between
 * steps; rank engines: every rank calls it at the same step (the ranks meet
 * on the device). *changed = 1 when boundaries moved. Results are unchanged
 * (bitwise). No-op for a single partition. */
int swamp_gpu_rebalance(swamp_gpu* g, int32_t* changed);

/* Host-side partition plan (no device needed; the same code the engine uses
 * at creation and in swamp_gpu_rebalance): the subtree boundaries bounds[0..G]
 * of G partitions at level L. leaves_before = NULL: equal subtree counts
 * (creation); else leaves_before[t] (t = 0..4^R, non-decreasing) = leaves in
 * subtrees [0, t): ranges with ~equal leaf counts, boundaries on multiples of
 * 16 subtrees when there are >= 64 per partition (4 when >= 16). */
int swamp_partition_plan(int32_t L, int32_t G, const uint64_t* leaves_before, uint32_t* bounds);
/* Partition owning cell (level n, Morton m) under bounds (>= 0), or < 0 on
 * bad arguments. Cells above the subtree level belong to the owner of their
 * first subtree. */
int swamp_partition_owner(const uint32_t* bounds, int32_t G, int32_t L, int32_t n, uint32_t m);

/* step_adaptive: one Alg. 3 iteration. No-op when
 * t >= t_end. Fills `rep` (may be NULL). Returns once the step is complete
 * and its report is in host memory (one partition: the step's last CTA
 * writes the report into a pinned mirror behind a system-scope fence, so
 * the call waits for that word instead of a stream synchronisation; later
 * calls are stream-ordered after the step). */
int swamp_gpu_step(swamp_gpu* g, swamp_step_report* rep);

/* Advance `n_steps` adaptive steps without host round trips (CUDA graph of
 * the step's kernels, replayed); stops early (device-side no-op) once
 * t >= t_end. Synchronises once at the end and checks the error word. */
int swamp_gpu_advance(swamp_gpu* g, int64_t n_steps, swamp_step_report* rep);

/* Advance `n_steps` adaptive steps back to back and return EVERY step's
 * report (reps[0..n_steps-1]): an extra CTA of the next step's first kernel
 * writes each step's report into a pinned ring slot and the host copies it
 * out while later steps run (at most 16 steps ahead; the last report comes
 * from a synchronising read), so there is no host round trip between steps. Steps past t_end are no-ops whose reports repeat the final
 * state. Partitioned / rank / uniform engines fall back to one
 * swamp_gpu_step per report. */
int swamp_gpu_advance_reports(swamp_gpu* g, int64_t n_steps, swamp_step_report* reps);

/* Asynchronous form of swamp_gpu_advance: enqueue `n_steps` graph replays on
 * the handle's stream and return without synchronising or checking errors
 * (the next synchronising call reports them). */
int swamp_gpu_enqueue(swamp_gpu* g, int64_t n_steps);
/* The cudaStream_t (as void*) every kernel of this handle runs on. */
int swamp_gpu_stream(swamp_gpu* g, void** stream);

/* run without outputs: step until t >= t_end. */
int swamp_gpu_run(swamp_gpu* g, swamp_step_report* rep);

/* step_uniform: the GPU-FV1 comparator on all 4^L cells,
 * no MRA. Only valid on a handle created with swamp_gpu_create_uniform. */
int swamp_gpu_create_uniform(const swamp_config* cfg, const double* h, const double* qx,
                             const double* qy, const double* z, int device, swamp_gpu** out);
int swamp_gpu_step_uniform(swamp_gpu* g, int64_t n_steps, swamp_step_report* rep);

/* Stage timing from CUDA event nodes between the kernels (a separate graph
 * with event record nodes) instead of the device timeline. */
int swamp_gpu_set_profiling(swamp_gpu* g, int enabled);

/* State queries / export (SimState). */
int swamp_gpu_info(const swamp_gpu* g, double* t, double* dt, int64_t* step, int64_t* n_leaves);
/* Leaves (ascending first-covered Morton) and W,E,N,S descriptors; arrays of
 * capacity `cap`; *n receives the leaf count. Any pointer may be NULL. */
int swamp_gpu_copy_leaves(swamp_gpu* g, uint32_t* leaves, uint32_t* nbr_w, uint32_t* nbr_e,
                          uint32_t* nbr_n, uint32_t* nbr_s, int64_t cap, int64_t* n);
/* Hierarchy scale coefficients of the CURRENT tree (length hierarchy_cells):
 * leaves hold post-step values, significant cells their re-encoded / decoded
 * values; cells off the tree are unspecified. sig: detail_cells bytes, 1 =
 * significant. Any pointer may be NULL. */
int swamp_gpu_export_tree(swamp_gpu* g, double* h, double* qx, double* qy, double* z, uint8_t* sig);
/* Zero-detail expansion to the finest grid: physical
 * values, row-major south row first, length 4^L each. */
int swamp_gpu_export_finest(swamp_gpu* g, double* h, double* qx, double* qy);

/* Gauges ("gauge time series by point sampling the covering
 * leaf"): for each of the n points (x[k], y[k]) (m, inside the domain
 * square), the leaf covering the finest cell that holds the point. out:
 * 4 n doubles, [h | qx | qy | eta = h + z] (physical). SWAMP_E_ARG for a
 * point outside the square. Synchronises the engine's stream. */
int swamp_gpu_sample_gauges(swamp_gpu* g, int32_t n, const double* x, const double* y, double* out);

/* Device error word of the last failure: code, z-index, quantity, stage. */
int swamp_gpu_last_error(const swamp_gpu* g, int32_t* code, uint32_t* z, int32_t* quantity,
                         int32_t* stage, char* msg, size_t msg_cap);

/* Counters for roofline bookkeeping: [0] leaves N of the last step, [1]
 * significant tree cells re-encoded (cumulative), [2] newly significant cells
 * decoded (cumulative), [3] 4^L, [4] leaf updates of all steps (sum of N,
 * cumulative), [5] kernels launched per adaptive step (kernel nodes of the
 * one-step graph, summed over partitions), [6] near-threshold cells of all
 * steps (cumulative), [7] near-threshold cells of the last step. */
int swamp_gpu_counters(swamp_gpu* g, int64_t* out8);

/* Work done so far, for per-kernel byte accounting (bench.py roofline):
 * [0] cells re-encoded by K1 and the top-level encodes, [1] level-(L-1)
 * cells re-encoded inside FV1 (the fused next-step re-encode), [2] newly
 * significant cells decoded, [3] leaf updates (sum of N), [4] of which took
 * FV1's dry-subtree shortcut, [5] of which FV1's tile path updated (active
 * fully refined subtrees), [6] steps, [7] detail cells. Cumulative; summed
 * over partitions. */
int swamp_gpu_work_counters(swamp_gpu* g, int64_t* out8);

/* Stable-quiet skips: [0] leaves of stable quiet subtrees
 * whose update FV1 skipped because the buffer it writes already holds the
 * result (also counted in work_counters[4]; their quads' re-encodes in
 * work_counters[1]); [1] re-encoded cells K1 skipped for the same reason
 * (also counted in work_counters[0]). Cumulative; summed over partitions. */
int swamp_gpu_skip_counters(swamp_gpu* g, int64_t* out2);

/* Near-threshold cell counts (north star: cells whose normalised detail lies
 * within FP tolerance of the threshold are counted and reported; DESIGN.md
 * D8): [0] of the last step, [1] summed over all steps, [2] initialise's
 * full encode (flow quantities, every detail cell), [3] initialise's DEM
 * mask (z details). Summed over partitions. */
int swamp_gpu_near_threshold(swamp_gpu* g, int64_t* out4);

/* Device timeline of the last step, microseconds from K1's first CTA: for
 * K1, K2, K3, K5 (k = 0..3): [3k] first CTA start, [3k+1] unused (-1; [1]: the
 * previous step's end, <= 0, in a back-to-back run),
 * [3k+2] last CTA done. */
int swamp_gpu_timeline(swamp_gpu* g, double* out12);

/* Diagnostics: raw %globaltimer phase stamps (ns) of the first and last CTA
 * of K1 ([0, 16)) and K3 ([16, 32)) of the last step; [8 * c + 7] = entry. */
int swamp_gpu_debug(swamp_gpu* g, uint64_t* out64);

/* compare: L1 = sum |h_A - h_B| dx^2 / area and L-infinity
 * of the depths of two engines on the same device and grid (finest-grid
 * expansions, both at their current times). SWAMP_E_ARG on mismatched
 * grids. Deterministic. */
int swamp_gpu_compare(swamp_gpu* a, swamp_gpu* b, double* l1, double* linf);

/* Build identification (arch, flags) for logs. */
const char* swamp_gpu_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SWAMP_GPU_H */
