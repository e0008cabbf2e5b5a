/* oracle/oracle.h — CPU-HWFV1 oracle: TEST INFRASTRUCTURE ONLY.
 *
 * A plain C++ restatement of the reference specification of the adaptive
 * time step (/root/reference/SPEC.md modules zorder, mra, traversal, swe,
 * engine) used as the parity checker for the B200 kernels and as the timed
 * CPU baseline (bench.py `cpu_baseline` and `--impl reference`). Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs may load it. The product
 * (paper_2206_05761_b200/, libswamp_gpu.so) never links or calls it.
 *
 * Parity pinning: the index algebra is checked against the reference's own
 * header compiled by oracle/Makefile into oracle/_ref/ (tests/golden/
 * zorder_ref.json); every SPEC example that has a number is a known-answer
 * test in tests/test_oracle_kats.py. The reference ships no engine, so the
 * MRA / traversal / FV1 restatement is pinned by SPEC's examples and
 * properties plus the decisions D1-D16 recorded in DESIGN.md (the reference
 * has no golden vectors for those stages — "parity pinned to SPEC examples").
 */
#ifndef SWAMP_ORACLE_H
#define SWAMP_ORACLE_H
#include <stdint.h>
#include "../include/swamp_gpu.h" /* swamp_config: the shared SimConfig layout */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_state oracle_state;

/* engine */
int oracle_create(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                  const double* z, oracle_state** out);
int oracle_destroy(oracle_state* s);
int oracle_step(oracle_state* s);
int oracle_step_uniform(oracle_state* s);
int oracle_create_uniform(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                          const double* z, oracle_state** out);
int oracle_set_threads(int n);
int oracle_info(const oracle_state* s, double* t, double* dt, int64_t* step, int64_t* n_leaves);
int oracle_copy_leaves(const oracle_state* s, uint32_t* leaves, uint32_t* w, uint32_t* e, uint32_t* n,
                       uint32_t* so, int64_t cap, int64_t* count);
int oracle_export_tree(const oracle_state* s, double* h, double* qx, double* qy, double* z, uint8_t* sig);
int oracle_export_finest(const oracle_state* s, double* h, double* qx, double* qy);
int oracle_counters(const oracle_state* s, int64_t* out4);
/* near-threshold cells (D8): [0] last step, [1] all steps, [2]
 * initialise (flow quantities), [3] initialise (z, the DEM mask) */
int oracle_near_threshold(const oracle_state* s, int64_t* out4);
const char* oracle_last_error(const oracle_state* s);
/* overwrite the current state with a hierarchy + tree (s-units, z-index
 * order) — used to run GPU and oracle from one identical mid-run state */
int oracle_import_tree(oracle_state* s, const double* h, const double* qx, const double* qy,
                       const uint8_t* sig, double t, double dt, double t_next, int64_t step);

/* per-operation known-answer entry points */
uint32_t oracle_morton_encode(uint32_t i, uint32_t j);
void oracle_morton_decode(uint32_t m, uint32_t* i, uint32_t* j);
int64_t oracle_neighbour(int n, uint32_t m, int dir); /* -1 = off-grid */
void oracle_encode4(const double c[4], double out[4]);  /* s, da, db, dg */
void oracle_decode4(const double in[4], double c[4]);
int oracle_significance(const double d[3], double smax, int n, int L, double eps);
void oracle_hll(double hL, double uL, double vL, double hR, double uR, double vR, double g, double F[3]);
void oracle_face(const double L[4], const double R[4], double g, double hdry, double F[3], double hs[2]);
void oracle_fv1_cell(const double own[4], const double nb[16], double dx, double dt, double g,
                     double hdry, double nM, double out[3]);
void oracle_friction(double h, double qx, double qy, double dt, double g, double nM, double hdry,
                     double out[2]);
double oracle_cfl_cell(double h, double qx, double qy, double dx, double g, double hdry);
double oracle_cbrt(double x);
void oracle_boundary(const double own[4], int kind, int dir, double t, const double* ts, const double* vs,
                     int n, int mode, double hdry, double out[4]);
void oracle_ptt(int L, const uint8_t* sig, uint32_t* recorded);
int64_t oracle_compact(const uint32_t* recorded, int64_t n, uint32_t* leaves);
int oracle_neighbours(int L, const uint32_t* recorded, const uint32_t* leaves, int64_t N, const int32_t bc[4],
                      uint32_t* nbr4);
int64_t oracle_dft_leaves(int L, const uint8_t* sig, uint32_t* leaves);

#ifdef __cplusplus
}
#endif
#endif
