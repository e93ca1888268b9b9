/* C ABI of the B200 leaf-box reduction engine (libhps_leaf.so).
 *
 * Plain pointers and sizes only.  All `double*` arguments of the device entry
 * points are CUDA device pointers; `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Launches of one plan are ordered after each other whatever
 * stream they are issued on (the plan's slot workspace is shared).  Every function returns 0 on success and a negative value
 * on failure; hps_last_error() then describes the failure (thread-local).
 *
 * Reference interfaces replaced (steklov, /root/reference/pkg/src/steklov):
 *
 *   hps_plan_create            <- LeafTemplate.__init__            local_ops.py:224-306
 *                                 (D1 = diff[axis], D2 = diff@diff, a_bi, a_bb), corner_mode="drop"
 *   hps_plan_create_legendre   <- the same, corner_mode="legendre"  local_ops.py:289-299,320-353
 *                                 (+ Q = _boundary_injection, cross terms local_ops.py:375-378)
 *   hps_leaf_dtn               <- build_leaf_factors, batched      local_ops.py:439-446
 *                                 as driven by condensation.build   condensation.py:220-264
 *                                 incl. factor_interior's guard     local_ops.py:422-436
 *   hps_leaf_dtn_host          <- the same, host buffers, with the
 *                                 two-level schedule (BatchSchedule) condensation.py:49-95,225-264
 *   hps_leaf_solution_operator <- LeafFactors.s = -A_ii^{-1} a_ib    local_ops.py:443
 *                                 (cache_leaf_factors path)         condensation.py:258-260,376-377
 *   hps_leaf_factors           <- build_leaf_factors: s and dtn      local_ops.py:439-446
 *                                 of the same factorization, one launch
 *   hps_leaf_reduce_load       <- reduce_load.leaf_task             condensation.py:314-323
 *   hps_leaf_interior_solve    <- solve.leaf_task (recompute path)  condensation.py:372-383
 *   hps_leaf_apply             <- explicit_rows @ full in           problems.py:473-505
 *                                 crank_nicolson_run
 *   hps_plan_release           <- (no counterpart: the reference's per-leaf workspace is
 *   hps_plan_workspace             transient; BatchSchedule.memory_budget  condensation.py:49-84)
 *
 * Data layout (row-major, C order, float64):
 *   coeffs : [n_leaves][ncoef][n]   ncoef = d (diagonal second-order a_kk)
 *                                         + d(d-1)/2 (a_ab + a_ba for (0,1),(0,2),(1,2),
 *                                           if has_cross; legendre plans only)
 *                                         + d (first order, if has_first)
 *                                         + 1 (zeroth order, if has_zeroth)
 *                                   values at the leaf's interior nodes in the
 *                                   reference's interior order (C order).
 *   dtn    : [n_leaves][m][m]       T = A_bb - A_bi A_ii^{-1} A_ib
 *   s      : [n_leaves][n][m]       S = -A_ii^{-1} A_ib
 *   f, v, u: [n_leaves][n]          interior vectors
 *   ub, flux: [n_leaves][m]         boundary vectors (template face order)
 *   stats  : [n_leaves][2]          min |pivot|, max |pivot| of the LU of A_ii;
 *                                   the caller applies the reference's
 *                                   singularity rule (min <= 1e-14 * max).
 * with n = (p-2)^d interior nodes and m = 2 d (p-2)^(d-1) boundary DOFs for
 * corner-dropping face grids, m = 2 d (p-1)^(d-1) Gauss-Legendre face DOFs
 * for legendre plans.
 */
#ifndef HPS_LEAF_H
#define HPS_LEAF_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_ABI_VERSION 2

typedef struct hps_plan_s* hps_plan_t;

int hps_abi_version(void);
const char* hps_last_error(void);
int hps_device_count(void);

/* D1, D2: [dim][p][p] scaled Chebyshev differentiation matrices and their
 * squares; a_bi: [m][n]; a_bb: [m][m] (host pointers, copied).
 * max_slots: leaves in flight (0 = one per SM); workspace_budget_bytes bounds
 * the per-slot workspace (0 = unbounded). */
int hps_plan_create(hps_plan_t* plan, int device, int dim, int p, int has_first, int has_zeroth,
                    const double* D1, const double* D2, const double* a_bi, const double* a_bb,
                    int max_slots, size_t workspace_budget_bytes);
/* Legendre face grids: Q [n_bnd][m] maps Gauss face data to the n_bnd
 * Chebyshev boundary nodes (edge/corner averaged); bpos [p^dim] maps a full
 * grid flat index (C order) to its position among those boundary nodes
 * (-1 for interior nodes); a_bi [m][n] and a_bb [m][m] are dense. */
int hps_plan_create_legendre(hps_plan_t* plan, int device, int dim, int p, int has_cross,
                             int has_first, int has_zeroth, const double* D1, const double* D2,
                             const double* a_bi, const double* a_bb, const double* Q, int n_bnd,
                             const int* bpos, int max_slots, size_t workspace_budget_bytes);
int hps_plan_destroy(hps_plan_t plan);
int hps_plan_info(hps_plan_t plan, int* n_interior, int* n_boundary, int* ncoef, int* slots,
                  size_t* dtn_slot_bytes, size_t* solve_slot_bytes);
/* Device memory the plan holds now (slot workspace, pivot tables, inverse cache,
 * streaming buffers) and the slots it is sized for.  The workspace grows on the
 * first launch of a mode (bounded by workspace_budget_bytes and ~85% of free
 * device memory) and is kept until hps_plan_release / hps_plan_destroy. */
int hps_plan_workspace(hps_plan_t plan, size_t* bytes, int* slots);
/* Free the workspace and streaming buffers after the plan's last launch has
 * finished; templates and op programs stay and the next launch re-allocates. */
int hps_plan_release(hps_plan_t plan);

/* Diagnostics: when `counters` (device, [slots][16] uint64, zeroed by the
 * caller) is set, every launch accumulates clock64 cycles per op kind
 * (0 small panel, 1 swaps, 2/3 triangular inverses, 4/5 GEMM sub/set,
 * 6 assembly, 7 output), GEMM MFLOP (8) and leaves (9) per slot.  NULL disables. */
int hps_plan_set_profile(hps_plan_t plan, unsigned long long* counters);

int hps_leaf_dtn(hps_plan_t plan, int n_leaves, const double* coeffs, double* dtn, double* stats,
                 void* stream);
int hps_leaf_dtn_host(hps_plan_t plan, int n_leaves, const double* coeffs_host, double* dtn_host,
                      double* stats_host, int chunk_leaves);
int hps_leaf_solution_operator(hps_plan_t plan, int n_leaves, const double* coeffs, double* s,
                               double* stats, void* stream);
/* dtn [n_leaves][m][m] and s [n_leaves][n][m] from one factorization per leaf. */
int hps_leaf_factors(hps_plan_t plan, int n_leaves, const double* coeffs, double* dtn, double* s,
                     double* stats, void* stream);
int hps_leaf_reduce_load(hps_plan_t plan, int n_leaves, const double* coeffs, const double* f,
                         double* v, double* flux, double* stats, void* stream);
/* w = rows(coeffs) [u_int; u_b]: the leaf's collocation operator applied to
 * interior + boundary values (drop plans; the explicit Crank-Nicolson half
 * step, reference problems.py:473-505).  u_int, w: [n_leaves][n]; u_b: [n_leaves][m]. */
int hps_leaf_apply(hps_plan_t plan, int n_leaves, const double* coeffs, const double* u_int,
                   const double* u_b, double* w, void* stream);
int hps_leaf_interior_solve(hps_plan_t plan, int n_leaves, const double* coeffs, const double* ub,
                            const double* v, double* u, double* stats, void* stream);

/* Interface assembly (reference condensation.py:230-246, the scatter of each
 * leaf's DtN map T^tau into the interface matrix T and the Dirichlet coupling):
 * blocks = device DtN maps of leaves leaf0, leaf0 + 1, ...: leaf l at
 * blocks + (l - leaf0) * block_stride, row stride ld;
 * jobs = device int64 [n_jobs][8] = {leaf l, row0, col0, rows, cols, target
 * (0: out_t, 1: out_c), base, row stride}; adds block rows into
 * target[base + a * stride + b] (the CSR value arrays, zeroed by the caller).
 * Entries with at most two contributors are bit-identical to the host COO sum. */
int hps_interface_scatter(int device, const double* blocks, long long ld, long long block_stride,
                          long long leaf0, int n_jobs, const long long* jobs, double* out_t,
                          double* out_c, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HPS_LEAF_H */
