// B200 (sm_100a) leaf-box reduction engine for the two-level HPS solver.
//
// A persistent grid of two CTAs per SM; each CTA owns one "slot" of HBM workspace and
// reduces leaf boxes one after another (next leaf from a global counter).  For each leaf
// the CTA
//   1. assembles the padded augmented collocation matrix
//          M = [ A_ii  A_ib ]      (DtN mode,  NR = NC = n_pad + m_pad)
//              [ A_bi  A_bb ]
//      or  M = [ A_ii | rhs ]      (solve mode, NR = n_pad, NC = n_pad + 16)
//      directly from the Chebyshev differentiation tables and the coefficient
//      values at interior nodes (reference: local_ops.py:362-398),
//   2. factors the first n_pad columns with partial pivoting restricted to the
//      interior rows (recursive right-looking LU; reference: local_ops.py:422-436
//      uses LAPACK getrf on A_ii),
//   3. DtN mode: forms T = A_bb - A_bi A_ii^{-1} A_ib block by block as
//      A_bb - (A_bi U^-1)(L^-1 P A_ib) (reference: local_ops.py:439-446,
//      dtn = a_bb + a_bi @ (-A_ii^{-1} a_ib));
//      solve mode: forward/back substitution of the rhs column
//      (reference: condensation.py:314-323 and 372-383).
//
// All O(n^3) work runs in one FP64 tensor-core GEMM engine (mma.sync m8n8k4 f64
// -> SASS DMMA): 64 x 128 CTA tiles of 8 warps (32 x 32 each), operands staged by
// TMA in a 2-stage ring of 32-deep k chunks with mbarriers, epilogue as f64
// reductions in L2.  Pivot search, the narrow panels and the triangular-block
// inversions run on the same CTA between GEMMs; the other CTA of the SM keeps the
// tensor pipe busy with its own leaf, so there is no grid-wide synchronisation.

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <string>
#include <vector>

#include "hps_leaf.h"

namespace {

#ifndef HPS_NT
#define HPS_NT 256
#endif
constexpr int NT = HPS_NT;       // threads per CTA; two CTAs (two leaves) per SM
constexpr int CTAS_PER_SM = 2;
constexpr int TM = 64;           // GEMM tile rows (1 x 4 warps of 64 x 32)
constexpr int TN = 128;          // GEMM tile cols
#ifndef HPS_KC
#define HPS_KC 32
#endif
constexpr int KC = HPS_KC;       // k-chunk per pipeline stage
#ifndef HPS_STAGES
#define HPS_STAGES 2
#endif
#ifndef HPS_EPI_SLOTS
#define HPS_EPI_SLOTS 1
#endif
constexpr int STAGES = HPS_STAGES;
constexpr int EPI_SLOTS = HPS_EPI_SLOTS;
// Epilogue of C -= A B.  0: -acc staged in a per-warp smem ring and added in L2 by TMA
// reduce-add (each warp waits for the previous block to be read out of smem);
// 1: fire-and-forget f64 reductions in L2 (red.global.add.f64) straight from the
// accumulators — no smem ring, no waits (the same IEEE round-to-nearest add).
#ifndef HPS_EPI_RED
#define HPS_EPI_RED 1
#endif
constexpr bool EPI_RED = HPS_EPI_RED != 0;
// Skip the DMMAs of 8 x 8 sub-blocks whose rows or columns are structurally zero over
// the whole k chunk (per-row first nonzero gpos / wf, per-8-column bounds), on top of
// the per-warp chunk skipping: exact zeros, so the results are unchanged.
#ifndef HPS_SUB_SKIP
#define HPS_SUB_SKIP 0
#endif
#ifndef HPS_WARP_SWIZZLE
#define HPS_WARP_SWIZZLE 1
#endif
// Operand boxes.  Padded boxes (A 20, B 132 doubles per row; the extra
// columns are just neighbouring data) give bank-conflict-free m8n8k4 fragment
// loads; the alternative is a 128B-swizzled 16-column A box / unpadded B box.
#ifndef HPS_A_PAD
#define HPS_A_PAD 1
#endif
#ifndef HPS_B_PAD
#define HPS_B_PAD 1
#endif
constexpr bool A_PAD = HPS_A_PAD != 0;
constexpr int A_STRIDE = A_PAD ? KC + 4 : KC;
constexpr int B_STRIDE = HPS_B_PAD ? TN + 4 : TN;
constexpr int STAGE_A = TM * A_STRIDE;
constexpr int STAGE_B = KC * B_STRIDE;
// swizzled A boxes need 1024-byte aligned stages
constexpr int STAGE_DBL = A_PAD ? STAGE_A + STAGE_B : ((STAGE_A + STAGE_B + 127) / 128) * 128;
constexpr int WARPS = NT / 32;
constexpr int WN = 4;                 // warps along N (4 x 32 = TN)
constexpr int WM = WARPS / WN;        // warps along M
constexpr int MI = TM / WM / 8;       // 8-row m-tiles per warp
constexpr int NJ = TN / WN / 8;       // 8-col n-tiles per warp (4)
static_assert(MI * 8 * WM == TM && NJ == 4, "warp tiling");
constexpr int EPI_DBL = EPI_RED ? 0 : EPI_SLOTS * 2 * 8 * 16;  // per warp: ring slots x two [8][16] blocks
constexpr int WIDE_SMEM_BYTES = (STAGES * STAGE_DBL + (NT / 32) * EPI_DBL) * 8;
constexpr int TRI_BLOCK = 64;    // triangular base block (explicit inverse + GEMM)
#ifndef HPS_SMALL_PANEL
#define HPS_SMALL_PANEL 32
#endif
constexpr int SMALL_PANEL = HPS_SMALL_PANEL;  // recursion leaf width handled by the narrow panel
constexpr int RHS_COLS = 16;     // padded rhs block in solve mode
constexpr int PANEL_SMEM_CAP = 96 * 1024;

// MODE_FACTORS: the solution-operator program, then both outputs of the leaf
// (S = -A_ii^{-1} A_ib and T = A_bb + A_bi S) from one factorization
enum { MODE_DTN = 0, MODE_REDUCE = 1, MODE_INTERIOR = 2, MODE_SOLOP = 3, MODE_FACTORS = 4 };
constexpr int N_MODES = 5;

// Endgame GEMM sharing.  Once every leaf of the launch has been claimed, a CTA
// that finds no leaf left does not exit: it joins the GEMMs of CTAs still
// reducing a leaf, claiming their output tiles through a per-slot counter.
// The owner publishes each large GEMM op (op index, tile count, sequence
// number), claims tiles itself with atomicAdd, and waits for the tile-done
// count before its next op; helpers claim with compare-and-swap on the same
// (seq, next) word so a stale helper can never take a tile of a newer op.
struct ShareSlot {
  unsigned long long claim;  // (seq << 32) | next unclaimed tile
  int op_seq, op, tiles, done;
  int pad[2];
};
constexpr int SHARE_MIN_TILES = 16;
#ifndef HPS_PIVOT_TAU
#define HPS_PIVOT_TAU 0.0
#endif
#ifndef HPS_PF
#define HPS_PF 0  // GEMM operand L2 prefetch distance in k chunks (0: off)
#endif
constexpr int PF_DIST = HPS_PF;
#ifndef HPS_PROF_GEMM
#define HPS_PROF_GEMM 0  // diagnostics build: setup / data-wait / tail / producer cycles per GEMM bucket
#endif
#ifndef HPS_WARP_PRODUCER
#define HPS_WARP_PRODUCER 1  // the producer warp's 32 lanes share the tile claims / k bounds
#endif
#ifndef HPS_SHARE_FENCE
#define HPS_SHARE_FENCE 1  // all threads' writes performed (membar.gl) before an op is published
#endif
#ifndef HPS_BOUNDS_ONEPASS
#define HPS_BOUNDS_ONEPASS 1  // all of a tile's bound-table loads issued before the reductions
#endif
#ifndef HPS_WARP_BOUNDS
#define HPS_WARP_BOUNDS 1  // each warp's own k bounds at a tile start: table loads one per lane
#endif
#ifndef HPS_PF_NEXT
#define HPS_PF_NEXT 0  // narrow / tall GEMMs: chunks of the next tile prefetched into L2
#endif
// C tile L2 prefetch issued HPS_CPF k chunks before the tile's last chunk (0: with the
// first chunk).  A long tile outlives L2 residency (K = 1376: ~180 us per tile while L2
// turns over every ~35 us), so a prefetch at the start is evicted before the epilogue's
// reductions, which then fetch C from DRAM a second time.
#ifndef HPS_CPF
#define HPS_CPF 2
#endif
// Serpentine k order: odd tiles walk their k chunks backwards, so a tile starts on the
// operand chunks its predecessor (same 64-row A panel) read last, while they are in L2.
#ifndef HPS_KREV
#define HPS_KREV 0
#endif
// The TMA producer is lane 0 of this warp.  Issuing a chunk costs the producer ~500
// cycles of its own DMMA issue; warp 5 holds the tile's last-starting 32 x 32 block (wide
// tiles: row block 1, column block 3; tall tiles: row block 3, column block 1), so in
// ragged tiles it issues while it has no DMMAs of its own.
// (round 2: warp 5 deadlocked the shared endgame ops, whose done count was added by
// thread 0 while the producer counted the skipped tiles; the producer adds its own
// count now — see the end of gemm_t.)
#ifndef HPS_PRODUCER_WARP
#define HPS_PRODUCER_WARP 0
#endif
static_assert(HPS_PRODUCER_WARP >= 0 && HPS_PRODUCER_WARP < NT / 32, "producer warp");
constexpr int PRODUCER_TID = 32 * HPS_PRODUCER_WARP;
// L2 eviction hints on the operand loads: bit 1 A evict_last, bit 2 B evict_first
#ifndef HPS_L2HINT
#define HPS_L2HINT 2
#endif
// Wide GEMMs as two independent 4-warp groups on 64 x 64 tiles (1) instead of all 8
// warps on one 64 x 128 tile (0).  The per-warp k bounds are ragged mostly across
// column blocks (a 64 x 128 tile walks its k range from its earliest column's start:
// 86% of the walked warp slots carry DMMAs at p = 16; 92% for 64 x 64 tiles that
// walk independently; tools/r03/sim_program.py).  Measured: -5% at p = 16, -7% at
// p = 20 (twice the chunks per FLOP, lower operand reuse; profiles/r02c_variant_sweep.jsonl),
// so it stays off.
#ifndef HPS_HALF
#define HPS_HALF 0
#endif
constexpr int HSTAGES = 2;  // ring depth of each group (16-deep k chunks)
// Wide GEMMs of a CTA's own op: every warp issues its slice of each chunk (A: 8 of the
// 64 rows, B: 4 of the 32 k rows) instead of warp 0 issuing whole chunks, so no warp
// carries the producer's work (the stage's full barrier then counts 8 arrivals).
// Measured -3.6% at p = 16, -0.5% at p = 20 (profiles/r02c_variant_sweep.jsonl): off.
#ifndef HPS_SLICE
#define HPS_SLICE 0
#endif
constexpr unsigned FULL_COUNT = HPS_SLICE ? NT / 32 : 1;
static_assert(!(HPS_SLICE && (HPS_HALF || HPS_KREV)), "sliced production: 8-warp tiles, forward k order");
#ifndef HPS_RW
#define HPS_RW 256  // W-trick block of sorted boundary DOFs (rows below A_ii)
#endif

struct LeafParams {
  int mode;
  int d, p, q;            // q = p - 2 interior points per axis
  int n, m;               // interior / boundary DOFs
  int n_pad, m_pad;
  int NR, NC, ld;         // rows, cols, leading dim of the slot matrix
  int wb;                 // base panel width (candidate rows live in smem)
  int has_first, has_zeroth, ncoef;
  int legendre, has_cross;  // legendre face grids; mixed second derivatives
  int nb, col_rb;           // Chebyshev boundary nodes; first column of the R_b / T region
  const double* Q;          // [nb_pad][m_pad] face injection (legendre)
  const int* bpos;          // [p^d] full-grid flat index -> Chebyshev boundary position
  int n_leaves;
  size_t slot_stride;     // doubles per slot matrix
  double* work;           // slots * slot_stride
  int* piv;               // slots * piv_stride: pivots (n_pad), then the RHS prefix table
  int piv_stride;         // n_pad + (n_pad / 16 + 16) + m_pad + RW: pivots, rhs_tab, rhs_g, wf
  int colperm;            // DtN drop mode: A_ib columns sorted by their line's first row
  int rowperm;            // drop mode: interior unknowns / equations in the engine's order
  const int* rowpos;      // [n]: slot column (unknown order) of natural interior node i
  const int* eqpos;       // [n]: slot row of node i's collocation equation (rows sorted by first nonzero)
  const int* gsorted;     // [n_pad]: first nonzero column of the equation in slot row p (padding: p)
  double pivot_tau;       // threshold partial pivoting factor for the sorted-row LU
  const int* colpos;      // [m]: slot column (after n_pad) of natural boundary DOF b
  const int* colnat;      // [m]: natural boundary DOF in slot column s
  const int* fsort;       // [m_pad]: first slot row of the line of slot column s (non-decreasing)
  int wt, RW;             // W-trick DtN (T = A_bb - (A_bi U^-1)(L^-1 P A_ib)) and its row-block size
  double* scratch;        // slots * 2 n_pad * TRI_BLOCK: cached diagonal-block inverses
  const double* D1;       // d * p * p (scaled first derivative)
  const double* D2;       // d * p * p (D1 @ D1, computed on host like the reference)
  const double* a_bi;     // m * n
  const double* a_bb;     // m * m
  const double* coeffs;   // n_leaves * ncoef * n
  const double* in0;      // REDUCE: f (n per leaf); INTERIOR: ub (m per leaf)
  const double* in1;      // INTERIOR: v (n per leaf)
  double* out0;           // DTN: T (m*m); REDUCE: v (n); INTERIOR: u (n)
  double* out1;           // REDUCE: flux (m per leaf)
  double* stats;          // n_leaves * 2 : min |pivot|, max |pivot| over real columns
  unsigned long long* prof;  // optional [slots][PROF_SLOTS] cycle counters (diagnostics)
  int* leaf_counter;         // next leaf to reduce (zeroed before each launch)
  int* done_counts;          // optional: finished leaves per output chunk (streamed D2H)
  int done_chunk;            // leaves per output chunk
  int smem_doubles;          // dynamic shared memory of the launch, in doubles
  ShareSlot* share;          // [slots] endgame GEMM sharing (nullptr: off)
  int* share_finished;       // CTAs that found no leaf left
  int debug;                 // diagnostics (env HPS_DEBUG): 1 skip the LU program, 2 old DtN output,
                             // 4 natural A_ib column order without zero-prefix skipping, 8 one CTA per SM,
                             // 16 no endgame GEMM sharing
};

#ifndef HPS_PROF_EXEC
#define HPS_PROF_EXEC 0  // diagnostics build: count the DMMAs each GEMM op executes
#endif
constexpr int PROF_SLOTS = 64;  // 0..8 op kinds, 9 leaves, 10-14 panel steps, 15 interchanges,
                                // 16-18 GEMM cycles by N (<=64, <=256, >256), 19-21 their MFLOP, 22 assemble, 23 output
                                // (HPS_PROF_EXEC) 32-34 executed DMMA flops by N bucket, 35-37 by phase,
                                // 38-40 GEMM cycles by phase

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cp_async16(void* smem_ptr, const void* gptr, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_ptr));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gptr), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}
#ifndef HPS_DMMA_NV
#define HPS_DMMA_NV 0  // 1: the DMMA asm is not volatile (the compiler may schedule around it)
#endif
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
#if HPS_DMMA_NV
  asm(
#else
  asm volatile(
#endif
"mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// mbarrier / TMA helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, unsigned cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#ifdef HPS_TRACE  // probe: per-warp chunk timeline of CTA 0 (wait start, data ready, chunk done)
__device__ long long g_trace[NT / 32][HPS_TRACE][3];
__device__ long long g_trace_prod[HPS_TRACE][4];
#endif
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// the same load with an L2 eviction-priority hint (createpolicy cache policy)
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, int c0, int c1, int c2,
                                                  const void* src) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// bulk (non-tensor) copy shared -> global through the async proxy (TMA unit)
__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// generic-proxy global writes of this thread become visible to later TMA (async-proxy) reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

constexpr unsigned STAGE_BYTES = (unsigned)((STAGE_A + STAGE_B) * 8);  // TMA transaction bytes

// ---------------------------------------------------------------------------
// Per-CTA context
// ---------------------------------------------------------------------------

struct TmaMaps {
  CUtensorMap a_work;     // box {A_STRIDE, TM, 1} over [slots][NR][NC]
  CUtensorMap b_work;     // box {B_STRIDE, KC, 1}
  CUtensorMap a_scratch;  // box {A_STRIDE, TM, 1} over [slots][2 n_pad][TRI]
  CUtensorMap c_red;      // box {16, 8, 1} over [slots][NR][NC]: epilogue reduce-add
  CUtensorMap a_abi;      // legendre: box {A_STRIDE, TM, 1} over the plan's a_bi [m_pad][n_pad]
  CUtensorMap b_q;        // legendre: box {B_STRIDE, KC, 1} over the plan's Q [nb_pad][m_pad]
  CUtensorMap b_scratch;  // box {B_STRIDE, KC, 1} over [slots][2 n_pad][TRI]: inverse as B operand
  CUtensorMap a_work_t;   // tall tiles: box {12, 128, 1} over [slots][NR][NC]
  CUtensorMap b_scratch_t;  // tall tiles: box {68, 8, 1} over the inverse cache
  CUtensorMap a_work_n;   // narrow tiles: box {12, 256, 1} over [slots][NR][NC]
  CUtensorMap b_work_n;   // narrow tiles: box {36, 8, 1}
  CUtensorMap a_work_h;   // half tiles: box {20, 64, 1} over [slots][NR][NC]
  CUtensorMap b_work_h;   // half tiles: box {68, 16, 1}
  CUtensorMap a_scratch_h;  // half tiles: box {20, 64, 1} over the inverse cache
  CUtensorMap b_scratch_h;  // half tiles: box {68, 16, 1} over the inverse cache
  CUtensorMap a_work_s;     // sliced wide chunks: box {A_STRIDE, 8, 1} (a warp's 8 A rows)
  CUtensorMap a_scratch_s;  // ... over the inverse cache
  CUtensorMap b_work_s;     // box {B_STRIDE, 4, 1} (a warp's 4 B k rows)
  CUtensorMap b_scratch_s;  // ... over the inverse cache
};

// GEMM tile configurations.  Wide: 64 x 128 tiles, 2 x 4 warps of 32 x 32, k-chunk 16
// (A box 20 / B box 132 doubles per row).  Narrow: 256 x 32 tiles, 8 x 1 warps,
// k-chunk 8 (A box 12 / B box 36: row strides = +-8 banks mod 32, conflict-free
// fragments) for the tall rank-32/64 updates at the bottom of the LU recursion,
// which use a quarter / half of a wide tile.  Both share the stage ring, the
// mbarriers and the per-warp epilogue ring.
struct GemmWide {
  static constexpr int TM_ = TM, TN_ = TN, KC_ = KC, AS = A_STRIDE, BS = B_STRIDE, WN_ = WN, KIND = 0;
  static constexpr int GROUPS = 1, ST_ = STAGES;
  static constexpr bool SWZ = !A_PAD;
};
// Half: 64 x 64 tiles, two independent groups of 4 warps (2 x 2 of 32 x 32), each with
// its own producer, 2-stage ring of 16-deep k chunks and mbarriers; tiles claimed from
// one shared counter.  A box stride 20 / B stride 68: conflict-free fragments.
struct GemmHalf {
  static constexpr int TM_ = 64, TN_ = 64, KC_ = 16, AS = 20, BS = 68, WN_ = 2, KIND = 3;
  static constexpr int GROUPS = 2, ST_ = HSTAGES;
  static constexpr bool SWZ = false;
};
struct GemmNarrow {
  // k-chunk 16 (row stride 20) with the 32-wide chunks of the wide tiles, else 8 (row
  // stride 12) with a 3-stage ring, 4 (stride 4) with deeper rings
  static constexpr int TM_ = 256, TN_ = 32, KC_ = KC >= 32 ? 16 : ((STAGES <= 3 || EPI_RED) ? 8 : 4);
  static constexpr int AS = KC_ == 16 ? 20 : (KC_ == 8 ? 12 : 4);
  static constexpr int BS = 36, WN_ = 1, KIND = 1;
  static constexpr int GROUPS = 1, ST_ = STAGES;
  static constexpr bool SWZ = false;
};
// Tall: 128 x 64 tiles (4 x 2 warps), k-chunk 8, B stride 68, for the W-block
// right inverses (N = 64, in place: one tile column, so no tile reads columns
// another tile already wrote).
struct GemmTall {
  static constexpr int TM_ = 128, TN_ = 64, KC_ = KC >= 32 ? 16 : 8, AS = KC_ == 16 ? 20 : 12, BS = 68, WN_ = 2,
                       KIND = 2;
  static constexpr int GROUPS = 1, ST_ = STAGES;
  static constexpr bool SWZ = false;
};
template <class G>
struct GemmShape {
  static constexpr int WM_ = (NT / 32) / G::GROUPS / G::WN_;
  static constexpr int MI_ = G::TM_ / WM_ / 8;
  static constexpr int NJ_ = G::TN_ / G::WN_ / 8;
  static constexpr int SA = G::TM_ * G::AS, SB = G::KC_ * G::BS;
  static constexpr int SDBL = G::SWZ ? ((SA + SB + 127) / 128) * 128 : SA + SB;
  static constexpr unsigned BYTES = (unsigned)((SA + SB) * 8);
  static_assert(MI_ == 4 && NJ_ == 4, "32 x 32 warp tiles");
};
constexpr int NARROW_SMEM_DBL = STAGES * GemmShape<GemmNarrow>::SDBL + (NT / 32) * EPI_DBL;
constexpr int TALL_SMEM_DBL = STAGES * GemmShape<GemmTall>::SDBL + (NT / 32) * EPI_DBL;
constexpr int HALF_SMEM_DBL = 2 * HSTAGES * GemmShape<GemmHalf>::SDBL;
static_assert(!HPS_HALF || EPI_RED, "half tiles reduce C in L2 (no epilogue ring)");
// dynamic shared memory of the GEMM engine: the largest of the tile shapes
constexpr int GEMM_SMEM_BYTES =
    std::max(WIDE_SMEM_BYTES, 8 * std::max(std::max(NARROW_SMEM_DBL, TALL_SMEM_DBL), HALF_SMEM_DBL));
constexpr int STAGES_MAX = STAGES > HSTAGES ? STAGES : HSTAGES;

struct Ctx {
  double* M;
  int ld, n_piv, n_real, NR, wb, slot;
  int* piv;
  int* rhs_tab;  // [n_pad / 16 + 1]: RHS columns with a nonzero above row 16 g (forward solve)
  int* rhs_g;    // [m_pad]: first row with a nonzero in RHS columns >= s (non-decreasing)
  int* wf;       // [RW]: first nonzero column of each row of the current W block
  int* gpos;     // [n_pad]: first nonzero column of the equation now in row p (sorted-row LU), or null
  int* gmin16;   // [n_pad / 16 + 1]: min of gpos over 16-row groups (refreshed by OP_GMIN16)
  double tau;    // pivot threshold (0: strict partial pivoting)
  int* gcol16;   // [n_pad / 16 + 1]: first row of U with a nonzero, per 16 columns (symmetric
                 // pattern: = gmin16 at leaf start); [-1]: first interchange step, a floor
  double* scratch;
  double* smem;
  int smem_doubles;
  unsigned long long* prof;
  const TmaMaps* maps;
  uint64_t* full;   // STAGES mbarriers: stage filled (TMA tx complete)
  uint64_t* empty;  // STAGES mbarriers: stage released by all 8 warps
  unsigned pipe;    // running stage counter, identical in every thread
  uint64_t* gfull;  // half tiles: [2 groups][HSTAGES] stage-filled mbarriers
  uint64_t* gempty; // half tiles: [2 groups][HSTAGES] stage-released mbarriers (4 warps)
  unsigned gpipe;   // half tiles: the group's running stage counter (same in its threads)
  // endgame sharing: sh = share record of the slot whose GEMM runs (own slot for
  // an owner, the helped slot for a helper); role 0 owner-capable, 2 helper
  ShareSlot* sh;
  int role;
  unsigned seq;     // owner: last published sequence (thread 0); helper: the op's sequence
  int cur_op;       // owner: index of the op being executed
  const int* leaf_counter;
  int n_leaves;
};
// per warp: first k (relative to the GEMM's k origin) of each 8-row group and each
// 8-column group of the warp's 32 x 32 block in the current tile (HPS_SUB_SKIP)
__shared__ int s_sub[NT / 32][8];
#if HPS_PROF_EXEC
__shared__ unsigned long long s_exec_dmma;  // DMMAs issued by this CTA's warps in the current op
__shared__ unsigned long long s_exec_cap;   // DMMA slots of the chunks the CTA walked (8 warps x tile)
#endif

// ---------------------------------------------------------------------------
// GEMM engine: C[MxN] = (sub ? C - A*B : A*B) with A = M[ar.., ac..] (or the
// slot's scratch block when a_scratch), B = M[br.., bc..], C = M[cr.., cc..].
// Operand chunks (A 128x16, B 16x128 doubles) arrive by TMA into padded smem
// stages (row strides 20 / 132 doubles: conflict-free m8n8k4 fragments);
// thread 0 produces, all 8 warps consume and release stages through
// mbarriers, so the mainloop has no block-wide barrier.  Out-of-range rows /
// columns are zero-filled by TMA and masked in the epilogue.
// ---------------------------------------------------------------------------

// Operand sources: a_src 0 = slot, 1 = slot scratch (triangular inverse),
// 2 = plan a_bi; b_src 0 = slot, 1 = plan Q (legendre face injection).
template <class G>
__device__ __forceinline__ void gemm_t(Ctx& c, const bool sub, const int a_src, int ar, int ac,
                                       const int b_src, int br, int bc, int cr, int cc, int M, int N,
                                       int K, const int kmode, const int tri) {
  using S = GemmShape<G>;
  constexpr int TM = G::TM_, TN = G::TN_, KC = G::KC_, A_STRIDE = G::AS, B_STRIDE = G::BS;
  constexpr int WN = G::WN_, MI = S::MI_, NJ = S::NJ_, STAGE_A = S::SA, STAGE_DBL = S::SDBL;
  constexpr bool narrow = (G::KIND == 1);
  constexpr bool half = (G::KIND == 3);
  constexpr int GR = G::GROUPS, STG = G::ST_;
  constexpr int WARPS_ = NT / 32;
  constexpr int GW = WARPS_ / GR;  // warps per group (half tiles: two groups walk their own tiles)
  if (M <= 0 || N <= 0 || K <= 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = GR == 1 ? 0 : warp / GW, gwarp = warp - grp * GW;
  const int prod_tid = PRODUCER_TID + grp * GW * 32;  // the group's TMA producer
#if HPS_PROF_GEMM
  // diagnostics (the producer thread, by the GEMM's N bucket): 48+b setup, 51+b its warp's
  // waits for stage data, 54+b tail (epilogue fences and syncs), 57+b chunks, 60+b producer
  // time (44+b of it waiting for a released stage; 47 tile claims + k bounds, 63 chunk issue)
  const int pb = N <= 64 ? 0 : (N <= 256 ? 1 : 2);
  const bool pt = c.prof != nullptr && tid == prod_tid;
  long long pt0 = pt ? clock64() : 0;
#endif
  // warp -> (row block wm, column block wn).  The warps of an SM sub-partition are
  // warp and warp + 4; with HPS_WARP_SWIZZLE the second row of warps is rotated by
  // WN / 2 columns, so each sub-partition holds an early and a late column block
  // (columns are sorted by their first nonzero row: the per-warp k bounds leave
  // late blocks idle in early chunks) instead of two warps of the same column.
  // (tall 4 x 2 warp grids: the second half of the warps takes the other column
  // block and the row blocks two further on)
  // (half tiles: group warps 2 x 2; a group's warps sit on the four sub-partitions)
  const int wm = half ? gwarp / WN
                      : ((!HPS_WARP_SWIZZLE || WN != 2) ? warp / WN : (warp < 4 ? warp : (warp - 2) % 4));
  const int wn = half ? gwarp % WN
                      : (!HPS_WARP_SWIZZLE ? warp % WN
                                           : (WN == 2 ? warp / 4 : (warp % WN + wm * (WN / 2)) % WN));
  const int lr = lane >> 2, lc = lane & 3;
  const int tiles_n = (N + TN - 1) / TN;
  const int tiles = ((M + TM - 1) / TM) * tiles_n;
  const int kchunks = (K + KC - 1) / KC;  // K is a multiple of 16; the last chunk may be partial
  double* smem = c.smem + grp * STG * STAGE_DBL;
  uint64_t* full = half ? c.gfull + grp * HSTAGES : c.full;
  uint64_t* empty = half ? c.gempty + grp * HSTAGES : c.empty;
  unsigned& pipe = half ? c.gpipe : c.pipe;
  const CUtensorMap* mapA = narrow ? &c.maps->a_work_n
                           : half ? (a_src == 0 ? &c.maps->a_work_h : &c.maps->a_scratch_h)
                           : G::KIND == 2 ? &c.maps->a_work_t
                           : (a_src == 0 ? &c.maps->a_work
                                         : (a_src == 1 ? &c.maps->a_scratch : &c.maps->a_abi));
  const CUtensorMap* mapB = narrow ? &c.maps->b_work_n
                           : half ? (b_src == 0 ? &c.maps->b_work_h : &c.maps->b_scratch_h)
                           : G::KIND == 2 ? &c.maps->b_scratch_t
                           : (b_src == 0 ? &c.maps->b_work : (b_src == 1 ? &c.maps->b_q : &c.maps->b_scratch));
  const int a_slot = a_src == 2 ? 0 : c.slot, b_slot = b_src == 1 ? 0 : c.slot;
  double* C = c.M + (size_t)cr * c.ld + cc;

  // Tile claims: mode 0 in order; mode 1 owner of a published op (atomicAdd on
  // the slot's claim word); mode 2 helper (compare-and-swap with the op's seq).
  __shared__ int s_gmode;
  __shared__ int s_tile_ring[2][STAGES_MAX];  // per group: tile id started in each stage (-1: end)
  __shared__ int s_kc0_ring[2][STAGES_MAX];   // its first k-chunk
  __shared__ int s_next_tile;                 // half tiles, in-order mode: next unclaimed tile
  // An op published for sharing is read by other CTAs' TMA loads: every thread's earlier
  // global writes (the previous ops' f64 reductions and stores, which bar.sync does not
  // wait for) must be performed GPU-wide before thread 0 publishes.
  __shared__ int s_pub;
  bool pub = false;
  if (HPS_SHARE_FENCE && c.role != 2 && c.sh && tiles >= SHARE_MIN_TILES) {
    if (tid == 0) s_pub = *reinterpret_cast<const volatile int*>(c.leaf_counter) >= c.n_leaves;
    __syncthreads();
    pub = s_pub != 0;
    if (pub) {
      __threadfence();
      fence_proxy_async_global();
      __syncthreads();
    }
  }
  if (tid == 0) {
    int m = 0;
    s_next_tile = 0;
    if (c.role == 2) {
      m = 2;
    } else if (HPS_SHARE_FENCE ? pub
                               : (c.sh && tiles >= SHARE_MIN_TILES &&
                                  *reinterpret_cast<const volatile int*>(c.leaf_counter) >= c.n_leaves)) {
      m = 1;
      ShareSlot* sh = c.sh;
      c.seq += 1;
      sh->op = c.cur_op;
      sh->tiles = tiles;
      sh->done = 0;
      sh->op_seq = (int)c.seq;
      __threadfence();
      atomicExch(&sh->claim, (unsigned long long)c.seq << 32);
    }
    s_gmode = m;
  }
  // every thread's earlier global writes must be visible to the TMA reads below
  fence_proxy_async_global();
  __syncthreads();
  const int gmode = s_gmode;
#if HPS_PROF_GEMM
  if (pt) { const long long t = clock64(); c.prof[48 + pb] += t - pt0; pt0 = t; }
#endif
  // sliced production: own-op (in-order) wide GEMMs on slot / inverse-cache operands
  const bool slice = HPS_SLICE && G::KIND == 0 && gmode == 0 && a_src != 2 && b_src != 1;
  __shared__ int s_tile_ring_w[NT / 32][STAGES_MAX];  // sliced: per warp, tile id of each stage
  __shared__ int s_kc0_ring_w[NT / 32][STAGES_MAX];
  // producer state (thread 0 only)
  int p_it = 0, p_tile = 0, p_kc = 0, p_next = 0, p_skipped = 0, p_k0 = 0, p_j = 0;
  bool p_end = false, p_in = false;
  // warp producer: the whole producer warp runs the tile claims and k bounds (the 16-row /
  // 16-column table loads one per lane, min by redux.sync) and lane 0 issues the chunks
  constexpr bool WPM = HPS_WARP_PRODUCER && GR == 1;
  const bool wp = WPM && !slice;
  auto claim_tile1 = [&]() -> int {
    if (gmode == 0) {
      if (GR == 1) return p_next < tiles ? p_next++ : -1;
      const int t = atomicAdd(&s_next_tile, 1);
      return t < tiles ? t : -1;
    }
    if (gmode == 1) {
      const unsigned long long old = atomicAdd(&c.sh->claim, 1ull);
      const int t = (int)(old & 0xffffffffull);
      return t < tiles ? t : -1;
    }
    unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(&c.sh->claim);
    for (;;) {
      if ((unsigned)(old >> 32) != c.seq || (int)(old & 0xffffffffull) >= tiles) return -1;
      const unsigned long long prev = atomicCAS(&c.sh->claim, old, old + 1);
      if (prev == old) return (int)(old & 0xffffffffull);
      old = prev;
    }
  };
  auto claim_tile = [&]() -> int {
    if (!wp || gmode == 0) return claim_tile1();  // (in-order claims: the same sequence in every lane)
    int t = 0;
    if (lane == 0) t = claim_tile1();
    return __shfl_sync(0xffffffffu, t, 0);
  };
  // the next chunk into its stage, once every warp has released the stage's last use
  auto produce = [&]() {
    if (p_end) return;
    const unsigned g = pipe + p_it;
    const unsigned s = g % STG, use = g / STG;
    if (use > 0) {
#ifdef HPS_TRACE
      if (blockIdx.x == 0 && g < HPS_TRACE) g_trace_prod[g][0] = clock64();
#endif
#if HPS_PROF_GEMM
      const long long pe = pt ? clock64() : 0;
#endif
      mbar_wait(&empty[s], (use - 1) & 1);
#if HPS_PROF_GEMM
      if (pt) c.prof[44 + pb] += clock64() - pe;  // the producer's wait for a released stage
#endif
#ifdef HPS_TRACE
      if (blockIdx.x == 0 && g < HPS_TRACE) g_trace_prod[g][1] = clock64();
#endif
    }
    const bool first_chunk = !p_in;
#if HPS_PROF_GEMM
    const long long pc = pt ? clock64() : 0;
#endif
    if (!p_in) {
      for (;;) {
        p_tile = claim_tile();
        if (p_tile < 0) break;
        p_kc = 0;
        if (!kmode) break;
        // first k with a nonzero in this tile's B columns / A rows
        int kk = 0;
        if (wp && HPS_BOUNDS_ONEPASS) {
          // every table load of the tile issued before any is consumed: one L2 round trip
          int vr = 0, vw = 0, vc1 = 0x7fffffff, vc = 0x7fffffff, vg = 0x7fffffff;
          const int cb = bc + (p_tile % tiles_n) * TN, r0 = ar + (p_tile / tiles_n) * TM;
          if (kmode & 1) vr = c.rhs_g[(p_tile % tiles_n) * TN];
          if (kmode & 2) vw = c.wf[r0 - c.n_piv];
          if (kmode & 8) {
            vc1 = c.gcol16[-1];
            if (lane < TN / 16 && cb + 16 * lane < bc + N) vc = c.gcol16[(cb + 16 * lane) >> 4];
          }
          if ((kmode & 4) && lane < TM / 16 && r0 + 16 * lane < ar + M) vg = c.gmin16[(r0 + 16 * lane) >> 4];
          if (kmode & 1) kk = max(kk, vr - br);
          if (kmode & 2) kk = max(kk, vw - ac);
          if (kmode & 8) kk = max(kk, min(vc1, __reduce_min_sync(0xffffffffu, vc)) - br);
          if (kmode & 4) {
            kk = max(kk, __reduce_min_sync(0xffffffffu, vg) - ac);
            if (kk >= K) {
              ++p_skipped;
              if (c.prof && lane == 0) c.prof[31] += ((unsigned long long)K * TM * TN * 2) >> 20;
              continue;
            }
            if (c.prof && kk > 0 && lane == 0) c.prof[31] += ((unsigned long long)(kk / KC) * KC * TM * TN * 2) >> 20;
          }
          const int k0 = kk / KC;
          p_kc = k0 > kchunks - 1 ? kchunks - 1 : k0;
          break;
        }
        if (kmode & 1) kk = max(kk, c.rhs_g[(p_tile % tiles_n) * TN] - br);
        if (kmode & 2) kk = max(kk, c.wf[ar + (p_tile / tiles_n) * TM - c.n_piv] - ac);
        if (kmode & 8) {  // columns of the tile: first row of U with a nonzero (16-column minima)
          const int cb = bc + (p_tile % tiles_n) * TN;
          int gm = c.gcol16[-1];
          if (wp) {
            const int cq = cb + 16 * lane;
            const int v = (lane < TN / 16 && cq < bc + N) ? c.gcol16[cq >> 4] : 0x7fffffff;
            gm = min(gm, __reduce_min_sync(0xffffffffu, v));
          } else {
            for (int cq = cb; cq < cb + TN && cq < bc + N; cq += 16) gm = min(gm, c.gcol16[cq >> 4]);
          }
          kk = max(kk, gm - br);
        }
        if (kmode & 4) {  // rows of the tile: first nonzero column (16-row group minima)
          const int r0 = ar + (p_tile / tiles_n) * TM;
          int gm = 0x7fffffff;
          if (wp) {
            const int r = r0 + 16 * lane;
            const int v = (lane < TM / 16 && r < ar + M) ? c.gmin16[r >> 4] : 0x7fffffff;
            gm = __reduce_min_sync(0xffffffffu, v);
          } else {
            for (int r = r0; r < r0 + TM && r < ar + M; r += 16) gm = min(gm, c.gmin16[r >> 4]);
          }
          kk = max(kk, gm - ac);
          if (kk >= K) {  // the tile's rows are zero over the whole k range: C unchanged
            ++p_skipped;
            if (c.prof && (!(slice || wp) || lane == 0) && (!slice || tid == 0))
              c.prof[31] += ((unsigned long long)K * TM * TN * 2) >> 20;
            continue;
          }
          if (c.prof && kk > 0 && (!(slice || wp) || lane == 0) && (!slice || tid == 0))
            c.prof[31] += ((unsigned long long)(kk / KC) * KC * TM * TN * 2) >> 20;
        }
        const int k0 = kk / KC;
        p_kc = k0 > kchunks - 1 ? kchunks - 1 : k0;
        break;
      }
      p_k0 = p_kc;
      p_j = 0;
      if (HPS_KREV && (p_tile & 1)) p_kc = kchunks - 1;
      if (slice) {
        if (lane == 0) s_tile_ring_w[warp][s] = p_tile;
      } else if (!wp || lane == 0) {
        s_tile_ring[grp][s] = p_tile;
      }
      if (p_tile < 0) {  // end marker: a stage with no data
        p_end = true;
        if (slice) {
          if (lane == 0) mbar_arrive(&full[s]);
        } else if (!wp || lane == 0) {
          mbar_arrive_cnt(&full[s], FULL_COUNT);
        }
        ++p_it;
        return;
      }
      if (slice) {
        if (lane == 0) s_kc0_ring_w[warp][s] = p_k0;
      } else if (!wp || lane == 0) {
        s_kc0_ring[grp][s] = p_k0;
      }
      p_in = true;
    }
#if HPS_PROF_GEMM
    long long pi = 0;
    if (pt) { pi = clock64(); c.prof[47] += pi - pc; }  // tile claim + k bounds (all buckets)
#endif
    if (wp && lane != 0) {  // lanes 1..31 of the producer warp: state only, lane 0 issues
      ++p_it;
      ++p_j;
      if (HPS_KREV && (p_tile & 1)) --p_kc;
      else ++p_kc;
      if (p_j == kchunks - p_k0) p_in = false;
      return;
    }
    const int tm = p_tile / tiles_n, tn = p_tile - tm * tiles_n;
    double* sa = smem + s * STAGE_DBL;
    double* sb = sa + STAGE_A;
#ifdef HPS_TRACE
    if (blockIdx.x == 0 && g < HPS_TRACE) g_trace_prod[g][2] = clock64();
#endif
#ifdef HPS_TEST_NOTMA  // probe: no operand transfer (stale stage data), the ring protocol alone
    (void)sa; (void)sb; (void)tm; (void)tn;
    mbar_arrive_cnt(&full[s], FULL_COUNT);
#else
    if (slice) {
      // this warp's slice: A rows [8 warp, 8 warp + 8), B k rows [4 warp, 4 warp + 4)
      if (lane == 0) {
        mbar_expect_tx(&full[s], S::BYTES / (NT / 32));
        const CUtensorMap* mA = a_src == 0 ? &c.maps->a_work_s : &c.maps->a_scratch_s;
        const CUtensorMap* mB = b_src == 0 ? &c.maps->b_work_s : &c.maps->b_scratch_s;
        tma_load_3d(sa + warp * 8 * A_STRIDE, mA, ac + p_kc * KC, ar + tm * TM + warp * 8, a_slot, &full[s]);
        if (HPS_L2HINT & 2)
          tma_load_3d_hint(sb + warp * 4 * B_STRIDE, mB, bc + tn * TN, br + p_kc * KC + warp * 4, b_slot, &full[s],
                           policy_evict_first());
        else
          tma_load_3d(sb + warp * 4 * B_STRIDE, mB, bc + tn * TN, br + p_kc * KC + warp * 4, b_slot, &full[s]);
        if (sub && p_j == max(0, kchunks - p_k0 - HPS_CPF)) {  // this warp's 8 rows of the C tile into L2
          tma_prefetch_3d(&c.maps->b_work_s, cc + tn * TN, cr + tm * TM + warp * 8, c.slot);
          tma_prefetch_3d(&c.maps->b_work_s, cc + tn * TN, cr + tm * TM + warp * 8 + 4, c.slot);
        }
      }
      ++p_it;
      ++p_j;
      ++p_kc;
      if (p_j == kchunks - p_k0) p_in = false;
      return;
    }
    mbar_expect_tx(&full[s], S::BYTES);
    if (FULL_COUNT > 1) mbar_arrive_cnt(&full[s], FULL_COUNT - 1);
#if HPS_L2HINT
    // the A panel of a tile row is read again by the row's next tile: keep it; the B
    // panel is not reused before it would be evicted anyway
    if (HPS_L2HINT & 1) tma_load_3d_hint(sa, mapA, ac + p_kc * KC, ar + tm * TM, a_slot, &full[s], policy_evict_last());
    else tma_load_3d(sa, mapA, ac + p_kc * KC, ar + tm * TM, a_slot, &full[s]);
    if (HPS_L2HINT & 2) tma_load_3d_hint(sb, mapB, bc + tn * TN, br + p_kc * KC, b_slot, &full[s], policy_evict_first());
    else tma_load_3d(sb, mapB, bc + tn * TN, br + p_kc * KC, b_slot, &full[s]);
#else
    tma_load_3d(sa, mapA, ac + p_kc * KC, ar + tm * TM, a_slot, &full[s]);
    tma_load_3d(sb, mapB, bc + tn * TN, br + p_kc * KC, b_slot, &full[s]);
#endif
#endif
    if (PF_DIST > 0 && p_kc + PF_DIST < kchunks) {  // operand chunks further ahead into L2
      tma_prefetch_3d(mapA, ac + (p_kc + PF_DIST) * KC, ar + tm * TM, a_slot);
      tma_prefetch_3d(mapB, bc + tn * TN, br + (p_kc + PF_DIST) * KC, b_slot);
    }
#if HPS_PF_NEXT
    // narrow / tall tiles (short K, latency-bound): with a tile's first chunk, the next
    // tile's A chunks (up to HPS_PF_NEXT of them, from this tile's first k) into L2
    if ((narrow || G::KIND == 2) && gmode == 0 && first_chunk) {
      const int nt = p_tile + 1;
      if (nt < tiles) {
        const int ntm = nt / tiles_n;
        for (int q = p_k0; q < kchunks && q < p_k0 + HPS_PF_NEXT; ++q)
          tma_prefetch_3d(mapA, ac + q * KC, ar + ntm * TM, a_slot);
      }
    }
#endif
    if (sub && (HPS_CPF == 0 ? first_chunk : p_j == max(0, kchunks - p_k0 - HPS_CPF))) {
      // C tile into L2 ahead of the reduce-add epilogue
      if (narrow) {
        for (int r = 0; r < TM; r += 8) tma_prefetch_3d(&c.maps->b_work_n, cc + tn * TN, cr + tm * TM + r, c.slot);
      } else if (half) {
        for (int r = 0; r < TM; r += KC) tma_prefetch_3d(&c.maps->b_work_h, cc + tn * TN, cr + tm * TM + r, c.slot);
      } else {
        for (int r = 0; r < TM; r += KC)
          tma_prefetch_3d(&c.maps->b_work, cc + tn * TN, cr + tm * TM + r, c.slot);
      }
    }
#ifdef HPS_TRACE
    if (blockIdx.x == 0 && g < HPS_TRACE) g_trace_prod[g][3] = clock64();
#endif
    ++p_it;
    ++p_j;
    if (HPS_KREV && (p_tile & 1)) --p_kc;
    else ++p_kc;
    if (p_j == kchunks - p_k0) p_in = false;
#if HPS_PROF_GEMM
    if (pt) c.prof[63] += clock64() - pi;  // TMA issue and prefetches (all buckets)
#endif
  };
  const bool is_prod = slice || (wp ? (tid >> 5) == (prod_tid >> 5) : tid == prod_tid);
  if (is_prod) {
    for (int s = 0; s < STG - 1; ++s) produce();
  }

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int tile = 0, kc = 0, it = 0, my_tiles = 0, kj = 0, kn = 0;
  bool in_tile = false, krev = false;
#if HPS_PROF_EXEC
  unsigned long long my_dmma = 0;
#endif
  // 8x8 sub-tiles of this warp that lie inside the GEMM extent (warp-uniform):
  // edge tiles skip the DMMAs on zero-filled rows / columns.
  int mv = MI, nv = NJ;
  // first k this warp's part of the tile needs: the kmode bounds of the tile,
  // taken over the warp's own rows (A) and columns (B)
  int wk = 0;
  // 8 x 8 sub-blocks (i * NJ + j) with work in the current chunk; the starts only
  // grow with k, so once every in-range sub-block is active the mask is final for the tile
  unsigned sub_mask = 0xffffu, sub_final = 0xffffu;
  bool sub_done = false;
  auto set_valid = [&](int t) {
    const int tm = t / tiles_n, tn = t - tm * tiles_n;
    const int rows = M - (tm * TM + wm * (MI * 8)), cols = N - (tn * TN + wn * (NJ * 8));
    mv = rows <= 0 ? 0 : (rows >= MI * 8 ? MI : (rows + 7) / 8);
    nv = cols <= 0 ? 0 : (cols >= NJ * 8 ? NJ : (cols + 7) / 8);
    wk = 0;
    if (kmode && mv > 0 && nv > 0) {
      const int r0 = ar + tm * TM + wm * (MI * 8), r1 = min(r0 + MI * 8, ar + M);
      const int c0w = tn * TN + wn * (NJ * 8), c1w = min(c0w + NJ * 8, N);
      if (HPS_WARP_BOUNDS && HPS_BOUNDS_ONEPASS) {
        // every table load of the warp's block issued before any is consumed
        int vr = 0, vw = 0x7fffffff, vg = 0x7fffffff, vc1 = 0x7fffffff, vc = 0x7fffffff;
        if (kmode & 1) vr = c.rhs_g[c0w];
        if ((kmode & 2) && r0 + lane < r1) vw = c.wf[r0 + lane - c.n_piv];
        if ((kmode & 4) && lane < MI * 8 / 16 + 1 && r0 + 16 * lane < r1) vg = c.gmin16[(r0 + 16 * lane) >> 4];
        if (kmode & 8) {
          vc1 = c.gcol16[-1];
          if (lane < NJ * 8 / 16 + 1 && c0w + 16 * lane < c1w) vc = c.gcol16[(bc + c0w + 16 * lane) >> 4];
        }
        if (kmode & 1) wk = max(wk, vr - br);
        if (kmode & 2) wk = max(wk, __reduce_min_sync(0xffffffffu, vw) - ac);
        if (kmode & 4) wk = max(wk, __reduce_min_sync(0xffffffffu, vg) - ac);
        if (kmode & 8) wk = max(wk, min(vc1, __reduce_min_sync(0xffffffffu, vc)) - br);
      } else {
        if (kmode & 1) wk = max(wk, c.rhs_g[c0w] - br);  // suffix minima: first column is the min
        if (kmode & 2) {  // W rows: per-row first nonzero, warp-reduced
          int f = 0x7fffffff;
          for (int r = r0 + lane; r < r1; r += 32) f = min(f, c.wf[r - c.n_piv]);
          if (HPS_WARP_BOUNDS) {
            f = __reduce_min_sync(0xffffffffu, f);
          } else {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) f = min(f, __shfl_xor_sync(0xffffffffu, f, off));
          }
          wk = max(wk, f - ac);
        }
        if (kmode & 4) {
          int gm = 0x7fffffff;
          if (HPS_WARP_BOUNDS) {  // the 16-row groups of the warp's rows, one per lane
            const int r = r0 + 16 * lane;
            gm = __reduce_min_sync(0xffffffffu, (lane < MI * 8 / 16 + 1 && r < r1) ? c.gmin16[r >> 4] : 0x7fffffff);
          } else {
            for (int r = r0; r < r1; r += 16) gm = min(gm, c.gmin16[r >> 4]);
          }
          wk = max(wk, gm - ac);
        }
        if (kmode & 8) {
          int gm = c.gcol16[-1];
          if (HPS_WARP_BOUNDS) {
            const int cq = bc + c0w + 16 * lane;
            gm = min(gm, __reduce_min_sync(0xffffffffu,
                                           (lane < NJ * 8 / 16 + 1 && c0w + 16 * lane < c1w) ? c.gcol16[cq >> 4] : 0x7fffffff));
          } else {
            for (int cq = bc + c0w; cq < bc + c1w; cq += 16) gm = min(gm, c.gcol16[cq >> 4]);
          }
          wk = max(wk, gm - br);
        }
      }
    }
    sub_final = 0;
#pragma unroll
    for (int i = 0; i < MI; ++i)
      if (i < mv) sub_final |= ((1u << nv) - 1u) << (i * NJ);
    sub_done = !HPS_SUB_SKIP;
    sub_mask = sub_final;
    if (HPS_SUB_SKIP) {
      // rows: lane l holds row r0 + l's first k, min over each 8-row group
      const int r0 = ar + tm * TM + wm * (MI * 8);
      const int r = r0 + lane;
      int f = 0;
      if (r >= ar + M) {
        f = 0x7fffffff;
      } else {
        if (kmode & 2) f = max(f, c.wf[r - c.n_piv] - ac);
        if (kmode & 4) f = max(f, c.gpos[r] - ac);
      }
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) f = min(f, __shfl_xor_sync(0xffffffffu, f, off));
      if (lane < MI * 8 && (lane & 7) == 0) s_sub[warp][lane >> 3] = f;
      if (lane < NJ) {  // columns: 8-column groups
        const int cw = tn * TN + wn * (NJ * 8) + lane * 8;
        int g = 0;
        if (cw >= N) {
          g = 0x7fffffff;
        } else {
          if (kmode & 1) g = max(g, c.rhs_g[cw] - br);
          if (kmode & 8) g = max(g, min(c.gcol16[-1], c.gcol16[(bc + cw) >> 4]) - br);
        }
        s_sub[warp][4 + lane] = g;
      }
      __syncwarp();
    }
  };
  for (;; ++it) {
#if HPS_PROF_GEMM
    long long pq = pt ? clock64() : 0;
#endif
    if (is_prod) produce();
#if HPS_PROF_GEMM
    if (pt) { const long long t = clock64(); c.prof[60 + pb] += t - pq; pq = t; }
#endif
    const unsigned g = pipe + it;
    const unsigned s = g % STG;
#ifdef HPS_TRACE
    const long long tr0 = clock64();
#endif
    mbar_wait(&full[s], (g / STG) & 1);
#if HPS_PROF_GEMM
    if (pt) { c.prof[51 + pb] += clock64() - pq; c.prof[57 + pb] += 1; }
#endif
#ifdef HPS_TRACE
    if (blockIdx.x == 0 && lane == 0 && g < HPS_TRACE) { g_trace[warp][g][0] = tr0; g_trace[warp][g][1] = clock64(); }
#endif
    if (!in_tile) {
      tile = slice ? reinterpret_cast<volatile int*>(s_tile_ring_w[warp])[s]
                   : reinterpret_cast<volatile int*>(s_tile_ring[grp])[s];
      if (tile < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        ++it;
        break;
      }
      kc = slice ? reinterpret_cast<volatile int*>(s_kc0_ring_w[warp])[s]
                 : reinterpret_cast<volatile int*>(s_kc0_ring[grp])[s];
      kn = kchunks - kc;  // chunks of this tile
      kj = 0;
      krev = HPS_KREV && (tile & 1);
      if (krev) kc = kchunks - 1;
      in_tile = true;
      set_valid(tile);
    }
#if HPS_PROF_EXEC
    if (c.prof && tid == prod_tid) atomicAdd(&s_exec_cap, (unsigned long long)(GW * MI * NJ * (KC / 4)));
#endif
    const double* sa = smem + s * STAGE_DBL;
    const double* sb = sa + STAGE_A;
    auto load_frags = [&](int ks, double (&af)[MI], double (&bf)[NJ]) {
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = wm * (MI * 8) + i * 8 + lr, k = ks + lc;
        if (!G::SWZ) {
          af[i] = sa[row * A_STRIDE + k];
        } else {
          // 128B swizzle: 16-byte chunk index ^= row % 8  (row % 8 == lr here)
          af[i] = sa[row * A_STRIDE + ((((k >> 1) ^ lr) << 1) | (k & 1))];
        }
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) bf[j] = sb[(ks + lc) * B_STRIDE + wn * (NJ * 8) + j * 8 + lr];
    };
    // k-steps (4 k each) of this chunk the warp executes: [klo, khi).  The last chunk
    // of a K that is not a multiple of KC is partial; steps whose rows / columns of
    // this warp are zero (first nonzero wk, explicit-inverse triangles) are skipped.
    constexpr int KS = KC / 4;
    const int kbase = kc * KC;
    int khi = min(KS, (K - kbase) >> 2);
    int klo = wk > kbase ? (wk - kbase) >> 2 : 0;
    if (tri) {
      const int tm = tile / tiles_n, tn = tile - tm * tiles_n;
      const int r_lo = tm * TM + wm * (MI * 8), r_hi = r_lo + MI * 8 - 1;
      const int c_hi = tn * TN + wn * (NJ * 8) + NJ * 8 - 1;
      if (tri == 1) khi = min(khi, r_hi >= kbase ? ((r_hi - kbase) >> 2) + 1 : 0);  // A lower: k <= row
      else if (tri == 3) klo = max(klo, r_lo > kbase ? (r_lo - kbase) >> 2 : 0);    // A upper: k >= row
      else if (tri == 2) khi = min(khi, c_hi >= kbase ? ((c_hi - kbase) >> 2) + 1 : 0);  // B upper: k <= col
    }
#ifdef HPS_TEST_IDLE  // probe: warps of the given mask do no DMMAs (is a lone warp per SMSP DMMA-limited?)
    if ((HPS_TEST_IDLE >> warp) & 1) khi = 0;
#endif
    auto mainloop = [&](auto edge) {
#pragma unroll
      for (int t = 0; t < KS; ++t) {
        if (t < klo || t >= khi) continue;
        double af[MI], bf[NJ];
        load_frags(4 * t, af, bf);
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (!decltype(edge)::value || ((sub_mask >> (i * NJ + j)) & 1u)) dmma(acc[i][j], af[i], bf[j]);
      }
    };
    if (klo < khi && mv > 0 && nv > 0) {
      if (!sub_done) {
        const int kend = kbase + KC;
        unsigned ra = 0, ca = 0;
#pragma unroll
        for (int i = 0; i < MI; ++i) ra |= (kend > s_sub[warp][i] ? 1u : 0u) << i;
#pragma unroll
        for (int j = 0; j < NJ; ++j) ca |= (kend > s_sub[warp][4 + j] ? 1u : 0u) << j;
        sub_mask = 0;
#pragma unroll
        for (int i = 0; i < MI; ++i)
          if ((ra >> i) & 1u) sub_mask |= ca << (i * NJ);
        sub_mask &= sub_final;
        sub_done = sub_mask == sub_final;
      }
      if (sub_mask == 0xffffu) mainloop(std::false_type{});
      else if (sub_mask) mainloop(std::true_type{});
#if HPS_PROF_EXEC
      my_dmma += (unsigned long long)(__popc(sub_mask) * (khi - klo));
#endif
    }
    __syncwarp();
#ifdef HPS_TRACE
    if (blockIdx.x == 0 && lane == 0 && g < HPS_TRACE) g_trace[warp][g][2] = clock64();
#endif
    if (lane == 0) mbar_arrive(&empty[s]);
    kc += krev ? -1 : 1;
    if (++kj == kn) {
      in_tile = false;
      const int tm = tile / tiles_n, tn = tile - tm * tiles_n;
      ++my_tiles;
      if (sub && EPI_RED) {
        // C -= acc as f64 reductions in L2, issued straight from the accumulators
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int row = tm * TM + wm * (MI * 8) + i * 8 + lr;
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const int col = tn * TN + wn * (NJ * 8) + j * 8 + 2 * lc;
            if (row < M && col < N) {
              double* cp = C + (size_t)row * c.ld + col;
              red_add_f64(cp, -acc[i][j][0]);
              red_add_f64(cp + 1, -acc[i][j][1]);
            }
            acc[i][j][0] = acc[i][j][1] = 0.0;
          }
        }
        continue;
      }
      if (sub) {
        // C -= acc through TMA reduce-add in L2: -acc goes to a per-warp smem ring
        // (two [8][16] blocks per m-tile) and drains asynchronously.
        double* ring = smem + STAGES * STAGE_DBL + warp * EPI_DBL;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int row0 = tm * TM + wm * (MI * 8) + i * 8;
          if (row0 < M) {
            double* buf = ring + (EPI_SLOTS == 1 ? 0 : (i & 1)) * 256;
            if (lane == 0) {
              if (EPI_SLOTS == 1) bulk_wait_read0();
              else bulk_wait_read1();
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<double2*>(buf + (j >> 1) * 128 + lr * 16 + (j & 1) * 8 + 2 * lc) =
                  make_double2(-acc[i][j][0], -acc[i][j][1]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              const int col0 = tn * TN + wn * (NJ * 8);
              if (col0 < N) tma_reduce_add_3d(&c.maps->c_red, cc + col0, cr + row0, c.slot, buf);
              if (col0 + 16 < N) tma_reduce_add_3d(&c.maps->c_red, cc + col0 + 16, cr + row0, c.slot, buf + 128);
              bulk_commit();
            }
          }
#pragma unroll
          for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = tm * TM + wm * (MI * 8) + i * 8 + lr;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int col = tn * TN + wn * (NJ * 8) + j * 8 + 2 * lc;
          if (row < M && col < N) {
            double2* cp = reinterpret_cast<double2*>(C + (size_t)row * c.ld + col);
            double2 v;
            if (sub) {
              const double2 old = *cp;
              v.x = old.x - acc[i][j][0];
              v.y = old.y - acc[i][j][1];
            } else {
              v.x = acc[i][j][0];
              v.y = acc[i][j][1];
            }
            *cp = v;
          }
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      }
    }
  }
  pipe += it;
#if HPS_PROF_GEMM
  if (pt) pt0 = clock64();
#endif
#if HPS_PROF_EXEC
  if (c.prof && lane == 0) atomicAdd(&s_exec_dmma, my_dmma);
#endif
  if (sub && !EPI_RED && lane == 0) {
    bulk_wait_all();
    fence_proxy_async_global();
  }
  if (sub && EPI_RED) fence_proxy_async_global();  // this thread's reductions before later TMA reads
  if (gmode != 0) {  // shared op: count the tiles done here; the owner waits for all
    __threadfence();
    __syncthreads();
    // each group's producer counts its group's tiles; thread 0 (owner) waits for all
    if (tid == prod_tid && my_tiles + p_skipped > 0) atomicAdd(&c.sh->done, my_tiles + p_skipped);
    if (tid == 0) {
      if (gmode == 1) {
        while (*reinterpret_cast<volatile int*>(&c.sh->done) < tiles) __nanosleep(200);
        __threadfence();
      }
    }
  }
  __syncthreads();
#if HPS_PROF_GEMM
  if (pt) c.prof[54 + pb] += clock64() - pt0;
#endif
}

// kmode: per-tile k offsets where an operand has structural zero prefixes —
// bit 1: B = the sorted RHS (bc = first RHS column), rows above the first
// nonzero of the tile's columns are zero (rhs_g); bit 2: A = W-block rows
// (ar >= n_pad), columns left of the tile's first nonzero are zero (wf);
// bit 4: A = LU rows, zero left of their first nonzero column (gmin16, 16-row
// minima; tiles whose rows are zero over all of K are skipped); bit 8: B = U
// rows of LU columns, zero above each column's first nonzero row (gcol16,
// floored at the first interchange).
// The k origin is br (A column ac + k pairs with B row br + k).
// tri: 1 A lower-triangular, 3 A upper-triangular, 2 B upper-triangular (the
// explicit inverses of the TRSM base blocks), 0 dense.
__device__ __forceinline__ void gemm(Ctx& c, const bool sub, const int a_src, int ar, int ac,
                                     const int b_src, int br, int bc, int cr, int cc, int M, int N,
                                     int K, const int kmode = 0, const int tri = 0) {
  // tall, narrow slot-only updates (the rank-32/64 steps of the LU recursion) on 256 x 32 tiles
  if (sub && a_src == 0 && b_src == 0 && N <= 64 && M >= 256 && K % 8 == 0)
    gemm_t<GemmNarrow>(c, sub, a_src, ar, ac, b_src, br, bc, cr, cc, M, N, K, kmode, tri);
  else if (!sub && a_src == 0 && b_src == 2 && N <= 64 && K % 8 == 0)  // W-block right inverse
    gemm_t<GemmTall>(c, sub, a_src, ar, ac, b_src, br, bc, cr, cc, M, N, K, kmode, tri);
#if HPS_HALF
  else if (a_src != 2 && b_src != 1)  // (legendre's plan-level operands stay wide)
    gemm_t<GemmHalf>(c, sub, a_src, ar, ac, b_src, br, bc, cr, cc, M, N, K, kmode, tri);
#endif
  else
    gemm_t<GemmWide>(c, sub, a_src, ar, ac, b_src, br, bc, cr, cc, M, N, K, kmode, tri);
}

__shared__ double s_pmin, s_pmax;
__shared__ double s_redv[NT / 32];
__shared__ int s_redi[NT / 32];
__shared__ int s_pivot;


// Row interchanges j in [j0, j0+cnt) applied, in order, to columns [c_lo, c_hi).
// Row interchanges j in [j0, j0+cnt) applied, in order, to columns [c_lo, c_hi).
// Most pivots are on the diagonal (partial pivoting rarely swaps on these
// operators), so the interchange list is first compacted into shared memory;
// then every thread applies the list to its columns, all of a swap's column
// loads in flight at once.
__shared__ int s_cnt, s_wcnt[NT / 32];

__device__ void apply_swaps(const Ctx& c, int j0, int cnt, int c_lo, int c_hi) {
  if (c_hi <= c_lo || cnt <= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* list = reinterpret_cast<int*>(c.smem);
  __syncthreads();
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (int base = j0; base < j0 + cnt; base += NT) {
    const int j = base + tid;
    const int pr = (j < j0 + cnt) ? c.piv[j] : j;
    const bool flag = pr != j;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) s_wcnt[warp] = __popc(bal);
    __syncthreads();
    int off = s_cnt;
    for (int w = 0; w < warp; ++w) off += s_wcnt[w];
    if (flag) {
      const int k = off + __popc(bal & ((1u << lane) - 1u));
      list[2 * k] = j;
      list[2 * k + 1] = pr;
    }
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < NT / 32; ++w) t += s_wcnt[w];
      s_cnt += t;
    }
    __syncthreads();
  }
  const int n = s_cnt;
  constexpr int CW = 4;  // columns in flight per thread
  for (int col0 = c_lo + tid; col0 < c_hi; col0 += NT * CW) {
    for (int k = 0; k < n; ++k) {
      const int j = list[2 * k], pr = list[2 * k + 1];
      double* ra = c.M + (size_t)j * c.ld;
      double* rb = c.M + (size_t)pr * c.ld;
      double va[CW], vb[CW];
#pragma unroll
      for (int u = 0; u < CW; ++u) {
        const int col = col0 + u * NT;
        if (col < c_hi) { va[u] = ra[col]; vb[u] = rb[col]; }
      }
#pragma unroll
      for (int u = 0; u < CW; ++u) {
        const int col = col0 + u * NT;
        if (col < c_hi) { ra[col] = vb[u]; rb[col] = va[u]; }
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Narrow panel (<= SMALL_PANEL columns), left-looking in blocks of WB columns.
// For block [b0, b0+WB) of the panel [c0, c0+w):
//   1. the U rows above the block (rows [c0, b0)) by forward substitution with
//      the panel's unit-lower L (staged in smem, warp-parallel dot products);
//   2. one coalesced warp-per-row pass over rows [b0, NR) reading the contiguous
//      segment [c0, b0+WB) and applying every earlier block's update at once
//      (partial products + warp reduce-scatter); candidate rows land in smem;
//   3. partial pivoting on the smem block (max |a|, lowest index on ties, as
//      LAPACK's idamax);
//   4. write-back, and L = A U^{-1} for the non-candidate rows;
//   5. the block's row interchanges applied to the rest of the panel segment
//      as one permutation gather.
// ---------------------------------------------------------------------------

__shared__ int s_swp_dst[16], s_swp_src[16], s_swp_cnt;
__shared__ int s_swp_rows[16], s_swp_cont[16];  // thread 0's scratch (no local-memory arrays)
// pivot search state, parity-buffered by column: per-warp best |a| / row / row values,
// and row j's values at the start of step j
// Pivot search keys: |a| compared as an integer (the bit pattern of a non-negative
// double orders like its value), +1 so that 0 means "no candidate" and NaN never
// wins — the same choice as the double compares (max |a|, lowest index on ties),
// made with integer compares and warp reductions (redux.sync) instead of FP64
// compares, which queue behind the co-resident CTA's DMMAs on the FP64 pipe.
#ifndef HPS_PROF_PIVOT
#define HPS_PROF_PIVOT 0  // diagnostics build: per-column pivot-step timers (prof 44-47)
#endif
#ifndef HPS_PIVOT_IKEY
#define HPS_PIVOT_IKEY 1
#endif
#if HPS_PIVOT_IKEY
typedef unsigned long long PivKey;
__device__ __forceinline__ PivKey piv_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
  return b > 0x7ff0000000000000ull ? 0ull : b + 1ull;
}
__device__ __forceinline__ double piv_val(PivKey k) { return k ? __longlong_as_double((long long)(k - 1ull)) : -1.0; }
#define PIV_NONE 0ull
#else
typedef double PivKey;
__device__ __forceinline__ PivKey piv_key(double v) { return fabs(v); }
__device__ __forceinline__ double piv_val(PivKey k) { return k; }
#define PIV_NONE (-1.0)
#endif
__shared__ PivKey s_pv[2][NT / 32];
__shared__ int s_pi[2][NT / 32];
__shared__ double s_cand[2][NT / 32][8];
__shared__ double s_rowj[2][8];
// compacted pivot candidates: the 16-row groups after the block's own group that
// have a structural nonzero in the panel
constexpr int MAXG = 768;
#ifndef HPS_PANEL_COMPACT_WB
#define HPS_PANEL_COMPACT_WB 1  // panel block width from the compacted candidate count
#endif
__shared__ int s_glist[MAXG];
__shared__ int s_ng;

// candidate index -> slot row: the head (rows b0 .. end of b0's 16-row group), then
// the listed groups
__device__ __forceinline__ int cand_row(int i, int b0, int head, bool compact) {
  if (!compact || i < head) return b0 + i;
  const int k = i - head;
  return (s_glist[k >> 4] << 4) + (k & 15);
}

// Pivot of column b0 + j chosen (candidate index bi, pivot value pv): the pivot row in
// c.piv, the equations' first-nonzero tables follow an interchange, pivot statistics.
#ifndef HPS_PIVOT_DEFER
#define HPS_PIVOT_DEFER 1
#endif
__shared__ int s_jbi[8];
__shared__ double s_jpv[8];
__device__ __forceinline__ void pivot_bookkeeping(Ctx& c, int b0, int j, int bi, int head, bool compact, double pv) {
  const int prow = cand_row(bi, b0, head, compact);
  c.piv[b0 + j] = prow;
  if (c.prof && bi != j) c.prof[15] += 1;
  if (c.gpos && bi != j) {  // the equations' first-nonzero table follows the interchange
    const int ta = c.gpos[b0 + j], tb = c.gpos[prow];
    c.gpos[b0 + j] = tb;
    c.gpos[prow] = ta;
    // 16-row minima stay lower bounds (a group may only gain a smaller g)
    int* ga = c.gmin16 + ((b0 + j) >> 4);
    int* gb = c.gmin16 + (prow >> 4);
    *ga = min(*ga, tb);
    *gb = min(*gb, ta);
    // column bounds hold only up to the first interchange (the swapped-in row
    // brings its own columns): floor every column's bound at this step
    if (c.gcol16[-1] > b0 + j) c.gcol16[-1] = b0 + j;
  }
  if (b0 + j < c.n_real) {
    const double ap = fabs(pv);
    s_pmin = fmin(s_pmin, ap);
    s_pmax = fmax(s_pmax, ap);
  }
}

template <int WB>
__device__ void panel_block(Ctx& c, int c0, int w, int b0) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int n_full = c.n_piv - b0;
  // rows whose 16-row group is zero over the whole panel (gmin16 >= c0 + w: a lower
  // bound on the group's first nonzero column) are neither pivot candidates nor
  // updated — their panel entries stay exact zeros — so they are left out
  const int head = min(16 - (b0 & 15), n_full);
  const bool compact = c.gpos != nullptr && ((c.n_piv + 15) >> 4) - (b0 >> 4) <= MAXG;
  int n_cand = n_full;
  if (compact) {
    __syncthreads();  // s_glist of the previous block is no longer read
    if (warp == 0) {
      const int g_end = (c.n_piv + 15) >> 4;
      int cnt = 0;
      for (int g0 = (b0 >> 4) + 1; g0 < g_end; g0 += 32) {
        const int g = g0 + lane;
        const bool act = g < g_end && c.gmin16[g] < c0 + w;
        const unsigned bal = __ballot_sync(0xffffffffu, act);
        if (act) s_glist[cnt + __popc(bal & ((1u << lane) - 1u))] = g;
        cnt += __popc(bal);
      }
      if (lane == 0) s_ng = cnt;
    }
    __syncthreads();
    const int ng = s_ng;
    n_cand = head + 16 * ng;
    // a listed last group that crosses n_piv (clipped row range) is partial
    if (ng > 0 && (c.n_piv & 15) && s_glist[ng - 1] == ((c.n_piv - 1) >> 4)) n_cand -= 16 - (c.n_piv & 15);
  }
  const int done = b0 - c0, len = done + WB;
  double* S = c.smem;                          // column-major [WB][n_cand]: S[j * NS + r]
  const int NS = n_cand;
  // staging T (<= 32 x 32) and Q (<= 16 x 32) alias S; Ut sits after all of them
  double* Ut = c.smem + (size_t)max(n_cand * WB, 1024);  // WB x 32, Ut[j*32 + kk]
  unsigned long long* prof = c.prof;
  long long tp = (prof && tid == 0) ? clock64() : 0;
#define PANEL_TICK(slot)                                   \
  if (prof && tid == 0) {                                  \
    const long long now = clock64();                       \
    prof[slot] += now - tp;                                \
    tp = now;                                              \
  }
  __syncthreads();
  if (done > 0) {
    // 1. U rows above the block
    double* T = c.smem;  // done x 32 staging of rows [c0, b0), cols [c0, b0+WB)
    for (int e = tid; e < done * len; e += NT) {
      const int kk = e / len, q = e - kk * len;
      T[kk * 32 + q] = c.M[(size_t)(c0 + kk) * c.ld + c0 + q];
    }
    __syncthreads();
    // warp j solves column j of the block by right-looking substitution with the
    // panel's unit-lower L: lane i holds x_i; one broadcast + one FMA per step
    if (warp < WB) {
      const int jj = warp;
      double x = (lane < done) ? T[lane * 32 + done + jj] : 0.0;
      for (int kk = 0; kk + 1 < done; ++kk) {
        const double xk = __shfl_sync(0xffffffffu, x, kk);
        if (lane > kk && lane < done) x -= T[lane * 32 + kk] * xk;
      }
      if (lane < done) {
        Ut[jj * 32 + lane] = x;
        c.M[(size_t)(c0 + lane) * c.ld + b0 + jj] = x;
      }
    }
    __syncthreads();
    PANEL_TICK(10)
    // 2. fused update + gather as a thin DMMA GEMM:
    //    V[rows x WB] = A_blk - L_seg[rows x done] * Ut^T[done x WB]
    //    8-row groups per warp (m8n8k4: A fragments straight from global,
    //    B fragments = Ut held in registers), G groups in flight.
    constexpr int G = 4;
    // k order permuted so each lane's A operands of a DMMA pair are adjacent:
    // DMMA kq uses k = 8 (kq / 2) + 2 lc + (kq & 1), one 16-byte load per pair
    const int nkp = (done + 7) >> 3;  // DMMA pairs
    const int lr = lane >> 2, lc = lane & 3;
    double bfr[8];
#pragma unroll
    for (int kq = 0; kq < 8; ++kq) {
      const int k = 8 * (kq >> 1) + 2 * lc + (kq & 1);
      bfr[kq] = ((kq >> 1) < nkp && lr < WB && k < done) ? Ut[lr * 32 + k] : 0.0;
    }
    const bool owns = 2 * lc < WB;  // lane holds output columns 2lc, 2lc+1
    // candidate rows by compacted index, then the non-candidate rows [n_piv, NR)
    const int n_ext = n_cand + (c.NR - c.n_piv);
    for (int i0 = warp * 8 * G; i0 < n_ext; i0 += NW * 8 * G) {
      double af[G][8], av[G][2];
      int rg[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int i = i0 + g * 8 + lr;
        const int r = i < n_cand ? cand_row(i, b0, head, compact) : c.n_piv + (i - n_cand);
        rg[g] = i < n_cand ? i : -1 - r;  // candidate index, or -1 - row
        const bool ok = i < n_ext;
        const double* row = c.M + (size_t)(r < c.NR ? r : c.NR - 1) * c.ld;
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {
          double2 v2 = make_double2(0.0, 0.0);
          if (ok && pq < nkp) v2 = *reinterpret_cast<const double2*>(row + c0 + 8 * pq + 2 * lc);
          af[g][2 * pq] = v2.x;
          af[g][2 * pq + 1] = v2.y;
        }
        if (WB >= 2) {
          double2 v2 = make_double2(0.0, 0.0);
          if (ok && owns) v2 = *reinterpret_cast<const double2*>(row + b0 + 2 * lc);
          av[g][0] = v2.x;
          av[g][1] = v2.y;
        } else {
          av[g][0] = (ok && owns) ? row[b0 + 2 * lc] : 0.0;
          av[g][1] = 0.0;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          if ((kq >> 1) < nkp) dmma(acc, af[g][kq], bfr[kq]);
        const int i = i0 + g * 8 + lr;
        if (i < n_ext && owns) {
          const double v0 = av[g][0] - acc[0], v1 = av[g][1] - acc[1];
          if (rg[g] >= 0) {
            S[(2 * lc) * NS + rg[g]] = v0;
            if (2 * lc + 1 < WB) S[(2 * lc + 1) * NS + rg[g]] = v1;
          } else {
            const int r = -1 - rg[g];
            c.M[(size_t)r * c.ld + b0 + 2 * lc] = v0;
            if (2 * lc + 1 < WB) c.M[(size_t)r * c.ld + b0 + 2 * lc + 1] = v1;
          }
        }
      }
    }
  } else {
    for (int e = tid; e < n_cand * WB; e += NT) {
      const int r = e / WB, j = e - r * WB;
      const int row = cand_row(r, b0, head, compact);
      const bool nz = c.gpos == nullptr || c.gmin16[row >> 4] < c0 + w;
      S[j * NS + r] = nz ? c.M[(size_t)row * c.ld + b0 + j] : 0.0;
    }
  }
  __syncthreads();
  PANEL_TICK(11)
  // 3. partial pivoting on the block, one barrier per column.  The search for
  //    column j+1 is fused into the rank-1 update of column j (each thread scans
  //    the rows it just updated).  Before the barrier each warp stashes its
  //    candidate row and thread 0 (owner of row j+1) stashes row j+1, so after
  //    it every thread picks the pivot itself and the interchange happens in
  //    flight: row j takes the pivot row, the pivot row's owner takes old row j.
  {
    auto warp_argmax = [&](PivKey best, int bidx, int par) {
#if HPS_PIVOT_IKEY
      const unsigned hi = (unsigned)(best >> 32), lo = (unsigned)best;
      const unsigned hmax = __reduce_max_sync(0xffffffffu, hi);
      const unsigned lmax = __reduce_max_sync(0xffffffffu, hi == hmax ? lo : 0u);
      bidx = __reduce_min_sync(0xffffffffu, (hi == hmax && lo == lmax) ? bidx : 0x7fffffff);
      best = ((PivKey)hmax << 32) | lmax;
#else
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
      }
#endif
      __syncwarp();  // the winner row's owner lane wrote it before the shuffles
      if (lane == 0) {
        s_pv[par][warp] = best;
        s_pi[par][warp] = bidx;
        if (bidx != 0x7fffffff) {
#pragma unroll
          for (int t = 0; t < WB; ++t) s_cand[par][warp][t] = S[t * NS + bidx];
        }
      }
    };
    {
      PivKey best = PIV_NONE;
      int bidx = 0x7fffffff;
      for (int r = tid; r < n_cand; r += NT) {
        const PivKey v = piv_key(S[r]);
        if (v > best) { best = v; bidx = r; }
      }
      warp_argmax(best, bidx, 0);
      if (tid == 0) {
#pragma unroll
        for (int t = 0; t < WB; ++t) s_rowj[0][t] = S[t * NS];
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < WB; ++j) {  // unrolled: register arrays indexed by j
      const int par = j & 1;
#if HPS_PROF_PIVOT  // diagnostics (thread 0): 44 selection + bookkeeping + 1/pivot, 45 row
                    // loop, 46 warp argmax + candidate stash, 47 the column barrier
      long long pq0 = (prof && tid == 0) ? clock64() : 0;
#endif
      PivKey bk = s_pv[par][0];
      int bi = s_pi[par][0], bw = 0;
#pragma unroll
      for (int q = 1; q < NT / 32; ++q) {
        const PivKey v = s_pv[par][q];
        const int i = s_pi[par][q];
        if (v > bk || (v == bk && i < bi)) { bk = v; bi = i; bw = q; }
      }
      if (bi == 0x7fffffff) bi = j;
      double urow[WB], rowj[WB];
#pragma unroll
      for (int t = 0; t < WB; ++t) rowj[t] = s_rowj[par][t];
      // threshold partial pivoting (sorted-row LU): keep the row in place when its
      // entry is within a factor c.tau of the column maximum — fewer interchanges
      // keep the equations' first-nonzero order, which the trailing updates use
      if (c.tau > 0.0 && bi != j && fabs(rowj[j]) >= c.tau * piv_val(bk)) bi = j;
#pragma unroll
      for (int t = 0; t < WB; ++t) urow[t] = (bi == j) ? rowj[t] : s_cand[par][bw][t];
      if (tid == 0) {
        if (HPS_PIVOT_DEFER) {
          // the column's bookkeeping waits for the end of the block (nothing in the
          // block reads it): thread 0 stays off the column's critical path
          s_jbi[j] = bi;
          s_jpv[j] = urow[j];
        } else {
          pivot_bookkeeping(c, b0, j, bi, head, compact, urow[j]);
        }
#pragma unroll
        for (int t = 0; t < WB; ++t) S[t * NS + j] = urow[t];
      }
      const double pivot = urow[j];
      const double inv = (pivot != 0.0) ? 1.0 / pivot : 1.0;
      PivKey best = PIV_NONE;
      int bidx = 0x7fffffff;
#if HPS_PROF_PIVOT
      if (prof && tid == 0) { const long long t = clock64(); prof[44] += t - pq0; pq0 = t; }
#endif
      constexpr int RU = WB >= 8 ? 2 : 4;  // rows in flight per thread
      for (int r0 = j + 1 + tid; r0 < n_cand; r0 += NT * RU) {
        double v[RU][WB];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int r = r0 + u * NT;
#pragma unroll
          for (int t = 0; t < WB; ++t)
            v[u][t] = (r >= n_cand || t < j) ? 0.0 : (r == bi ? rowj[t] : S[t * NS + r]);
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int r = r0 + u * NT;
          if (r < n_cand) {
            const double l = v[u][j] * inv;
            v[u][j] = l;
#pragma unroll
            for (int t = 0; t < WB; ++t)
              if (t > j) v[u][t] -= l * urow[t];
#pragma unroll
            for (int t = 0; t < WB; ++t) {
              if (t >= j) S[t * NS + r] = v[u][t];
              else if (r == bi) S[t * NS + r] = rowj[t];
            }
            if (j + 1 < WB) {
              const PivKey a = piv_key(v[u][j + 1]);
              if (a > best) { best = a; bidx = r; }
              if (r == j + 1) {  // thread 0: stash row j+1 for the next step
#pragma unroll
                for (int t = 0; t < WB; ++t)
                  s_rowj[par ^ 1][t] = (t >= j) ? v[u][t] : (r == bi ? rowj[t] : S[t * NS + r]);
              }
            }
          }
        }
      }
      if (j + 1 < WB) {
#if HPS_PROF_PIVOT
        if (prof && tid == 0) { const long long t = clock64(); prof[45] += t - pq0; pq0 = t; }
#endif
        if (j + 1 >= n_cand && tid == 0) {
#pragma unroll
          for (int t = 0; t < WB; ++t) s_rowj[par ^ 1][t] = 0.0;
        }
        warp_argmax(best, bidx, par ^ 1);
#if HPS_PROF_PIVOT
        if (prof && tid == 0) { const long long t = clock64(); prof[46] += t - pq0; pq0 = t; }
#endif
      }
      __syncthreads();
#if HPS_PROF_PIVOT
      if (prof && tid == 0) prof[47] += clock64() - pq0;
#endif
    }
  }
  if (HPS_PIVOT_DEFER && tid == 0)
    for (int j = 0; j < WB; ++j) pivot_bookkeeping(c, b0, j, s_jbi[j], head, compact, s_jpv[j]);
  PANEL_TICK(12)
  // 4. write-back; non-candidate rows L = A U^{-1}
  for (int e = tid; e < n_cand * WB; e += NT) {
    const int r = e / WB, j = e - r * WB;
    c.M[(size_t)cand_row(r, b0, head, compact) * c.ld + b0 + j] = S[j * NS + r];
  }
  {
    // 8 rows per thread in flight: loads first, then the WB x WB substitution
    constexpr int RR = 2;
    for (int r0 = c.n_piv + tid; r0 < c.NR; r0 += NT * RR) {
      double x[RR][WB];
#pragma unroll
      for (int t = 0; t < RR; ++t) {
        const int r = r0 + t * NT;
#pragma unroll
        for (int j = 0; j < WB; ++j) x[t][j] = (r < c.NR) ? c.M[(size_t)r * c.ld + b0 + j] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < RR; ++t) {
#pragma unroll
        for (int j = 0; j < WB; ++j) {
          double v = x[t][j];
#pragma unroll
          for (int i = 0; i < j; ++i) v -= x[t][i] * S[j * NS + i];
          const double pv = S[j * NS + j];
          x[t][j] = v * ((pv != 0.0) ? 1.0 / pv : 1.0);
        }
        const int r = r0 + t * NT;
        if (r < c.NR) {
#pragma unroll
          for (int j = 0; j < WB; ++j) c.M[(size_t)r * c.ld + b0 + j] = x[t][j];
        }
      }
    }
  }
  __syncthreads();
  PANEL_TICK(13)
  // 5. the block's interchanges on the rest of the panel segment [c0, c0+w)
  bool any_swap = false;  // most blocks have no interchange at all
  for (int j = 0; j < WB; ++j) any_swap |= c.piv[b0 + j] != b0 + j;
  if (tid == 0 && !any_swap) s_swp_cnt = 0;
  if (tid == 0 && any_swap) {
    int* rows = s_swp_rows;
    int* cont = s_swp_cont;
    int cnt = 0;
    for (int j = 0; j < WB; ++j) {
      const int cand[2] = {b0 + j, c.piv[b0 + j]};
      for (int t = 0; t < 2; ++t) {
        bool seen = false;
        for (int q = 0; q < cnt; ++q) seen |= (rows[q] == cand[t]);
        if (!seen) { rows[cnt] = cand[t]; cont[cnt] = cand[t]; ++cnt; }
      }
    }
    for (int j = 0; j < WB; ++j) {
      int ia = 0, ib = 0;
      for (int q = 0; q < cnt; ++q) {
        if (rows[q] == b0 + j) ia = q;
        if (rows[q] == c.piv[b0 + j]) ib = q;
      }
      const int t = cont[ia];
      cont[ia] = cont[ib];
      cont[ib] = t;
    }
    int n = 0;
    for (int q = 0; q < cnt; ++q)
      if (cont[q] != rows[q]) { s_swp_dst[n] = rows[q]; s_swp_src[n] = cont[q]; ++n; }
    s_swp_cnt = n;
  }
  __syncthreads();
  const int nsw = s_swp_cnt;
  const int ncol = w - WB;  // panel columns outside the block
  if (nsw > 0 && ncol > 0) {
    double* Q = c.smem;  // nsw x 32 staging (S already written back)
    for (int e = tid; e < nsw * ncol; e += NT) {
      const int q = e / ncol, k = e - q * ncol;
      const int col = (k < done) ? c0 + k : b0 + WB + (k - done);
      Q[q * 32 + k] = c.M[(size_t)s_swp_src[q] * c.ld + col];
    }
    __syncthreads();
    for (int e = tid; e < nsw * ncol; e += NT) {
      const int q = e / ncol, k = e - q * ncol;
      const int col = (k < done) ? c0 + k : b0 + WB + (k - done);
      c.M[(size_t)s_swp_dst[q] * c.ld + col] = Q[q * 32 + k];
    }
  }
  __syncthreads();
  PANEL_TICK(14)
#undef PANEL_TICK
}

// Columns [c0, c0+w), w <= SMALL_PANEL.  The block width grows as the
// candidate set shrinks (the smem block holds n_cand x WB doubles).
__device__ void lu_small(Ctx& c, int c0, int w) {
  int wb = c.wb;
  // candidate rows of the panel's first block (the most of any block: later blocks see
  // a subset of these groups — an interchange only lowers the bound of a group that
  // already holds a candidate, or of the head group): the compacted count of
  // panel_block, so panels whose rows are mostly structurally zero get wider blocks
  int n_cand = c.n_piv - c0;
  if (HPS_PANEL_COMPACT_WB && c.gpos != nullptr && ((c.n_piv + 15) >> 4) - (c0 >> 4) <= MAXG) {
    __shared__ int s_ncg;
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x, g_end = (c.n_piv + 15) >> 4;
      int cnt = 0, last = -1;
      for (int g0 = (c0 >> 4) + 1; g0 < g_end; g0 += 32) {
        const int g = g0 + lane;
        const bool act = g < g_end && c.gmin16[g] < c0 + w;
        const unsigned bal = __ballot_sync(0xffffffffu, act);
        cnt += __popc(bal);
        if (bal) last = g0 + 31 - __clz(bal);
      }
      if (lane == 0) {
        int nc = min(16 - (c0 & 15), c.n_piv - c0) + 16 * cnt;
        if (cnt > 0 && (c.n_piv & 15) && last == ((c.n_piv - 1) >> 4)) nc -= 16 - (c.n_piv & 15);
        s_ncg = nc;
      }
    }
    __syncthreads();
    // + 16: a later block's head group (rows b0 .. the end of b0's group) is counted
    // whole even when that group held no candidate for the first block
    n_cand = min(s_ncg + 16, c.n_piv - c0);
  }
  // panel block smem: max(n_cand * WB, 1024) doubles (S and the staging it hosts) + 32 * WB (Ut)
  auto fits = [&](int W) {
    const int sz = n_cand * W;
    return (sz > 1024 ? sz : 1024) + 32 * W <= c.smem_doubles;
  };
  while (wb < 8 && w % (2 * wb) == 0 && fits(2 * wb)) wb *= 2;
  for (int b0 = c0; b0 < c0 + w; b0 += wb) {
    switch (wb) {
      case 8: panel_block<8>(c, c0, w, b0); break;
      case 4: panel_block<4>(c, c0, w, b0); break;
      case 2: panel_block<2>(c, c0, w, b0); break;
      default: panel_block<1>(c, c0, w, b0); break;
    }
  }
}

// Explicit inverse of the unit-lower block M[r0.., r0..] (h <= TRI_BLOCK) into scratch (ld TRI_BLOCK).
// Explicit inverses of the h x h (h <= TRI_BLOCK) diagonal block of M at r0
// into the slot's scratch (ld TRI_BLOCK).  The block is staged in shared
// memory with coalesced loads; thread j then owns column j of the inverse.
constexpr int TRI_LD = TRI_BLOCK + 1;

__device__ void stage_tri(const Ctx& c, int r0, int h, double* Ls) {
  __syncthreads();
  for (int e0 = threadIdx.x; e0 < h * h; e0 += NT * 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * NT;
      v[u] = (e < h * h) ? c.M[(size_t)(r0 + e / h) * c.ld + r0 + e % h] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * NT;
      if (e < h * h) Ls[(e / h) * TRI_LD + e % h] = v[u];
    }
  }
  __syncthreads();
}

// Explicit inverse of a staged triangular block by recursive doubling: the
// 8 x 8 diagonal blocks are inverted by substitution (thread per column), then
// pairs of inverted s x s blocks are merged, s = 8, 16, 32:
//   lower  [A 0; B C]^-1 = [A^-1 0; -C^-1 (B A^-1)  C^-1]
//   upper  [A B; 0 C]^-1 = [A^-1  -A^-1 (B C^-1); 0 C^-1]
// with every product of a level spread over all threads (no 64-long serial
// chain).  Rows / columns h..63 are padded with the identity.
__device__ void tri_inverse(double* T, double* X, double* W, int h, bool upper) {
  const int tid = threadIdx.x;
  // pad + zero X
  for (int e = tid; e < TRI_BLOCK * TRI_BLOCK; e += NT) {
    const int i = e / TRI_BLOCK, j = e - i * TRI_BLOCK;
    if (i >= h || j >= h) T[i * TRI_LD + j] = (i == j) ? 1.0 : 0.0;
    X[i * TRI_LD + j] = 0.0;
  }
  __syncthreads();
  // level 0: 8 x 8 diagonal blocks, thread per (block, column)
  if (tid < TRI_BLOCK) {
    const int b = tid >> 3, j = tid & 7, o = b * 8;
    const int cj = o + j;
    if (!upper) {  // unit lower
      X[cj * TRI_LD + cj] = 1.0;
      for (int i = j + 1; i < 8; ++i) {
        double v = 0.0;
        for (int k = j; k < i; ++k) v -= T[(o + i) * TRI_LD + o + k] * X[(o + k) * TRI_LD + cj];
        X[(o + i) * TRI_LD + cj] = v;
      }
    } else {
      X[cj * TRI_LD + cj] = 1.0 / T[cj * TRI_LD + cj];
      for (int i = j - 1; i >= 0; --i) {
        double v = 0.0;
        for (int k = i + 1; k <= j; ++k) v -= T[(o + i) * TRI_LD + o + k] * X[(o + k) * TRI_LD + cj];
        X[(o + i) * TRI_LD + cj] = v / T[(o + i) * TRI_LD + o + i];
      }
    }
  }
  __syncthreads();
  for (int sz = 8; sz < TRI_BLOCK; sz *= 2) {
    const int pairs = TRI_BLOCK / (2 * sz), items = pairs * sz * sz;
    // W = B A^-1 (lower) / B C^-1 (upper); W stored per pair as sz x sz
    for (int e = tid; e < items; e += NT) {
      const int pr = e / (sz * sz), r = (e / sz) % sz, cc = e % sz;
      const int o = pr * 2 * sz;
      double v = 0.0;
      if (!upper) {  // B = T[o+sz+r][o+k], A^-1 = X[o+k][o+cc] (lower: k >= cc)
        for (int k = cc; k < sz; ++k) v += T[(o + sz + r) * TRI_LD + o + k] * X[(o + k) * TRI_LD + o + cc];
      } else {       // B = T[o+r][o+sz+k], C^-1 = X[o+sz+k][o+sz+cc] (upper: k <= cc)
        for (int k = 0; k <= cc; ++k)
          v += T[(o + r) * TRI_LD + o + sz + k] * X[(o + sz + k) * TRI_LD + o + sz + cc];
      }
      W[e] = v;
    }
    __syncthreads();
    for (int e = tid; e < items; e += NT) {
      const int pr = e / (sz * sz), r = (e / sz) % sz, cc = e % sz;
      const int o = pr * 2 * sz;
      const double* Wp = W + pr * sz * sz;
      double v = 0.0;
      if (!upper) {  // X21 = -C^-1 W: C^-1 = X[o+sz+r][o+sz+k] (k <= r)
        for (int k = 0; k <= r; ++k) v -= X[(o + sz + r) * TRI_LD + o + sz + k] * Wp[k * sz + cc];
        X[(o + sz + r) * TRI_LD + o + cc] = v;
      } else {       // X12 = -A^-1 W: A^-1 = X[o+r][o+k] (k >= r)
        for (int k = r; k < sz; ++k) v -= X[(o + r) * TRI_LD + o + k] * Wp[k * sz + cc];
        X[(o + r) * TRI_LD + o + sz + cc] = v;
      }
    }
    __syncthreads();
  }
}

__device__ void invert_unit_lower(const Ctx& c, int r0, int h) {
  double* Ls = c.smem;
  double* X = c.smem + TRI_BLOCK * TRI_LD;
  double* W = X + TRI_BLOCK * TRI_LD;
  stage_tri(c, r0, h, Ls);
  tri_inverse(Ls, X, W, h, false);
  double* dst = c.scratch + (size_t)r0 * TRI_BLOCK;
  for (int e = threadIdx.x; e < h * TRI_BLOCK; e += NT) dst[e] = X[(e / TRI_BLOCK) * TRI_LD + e % TRI_BLOCK];
  __syncthreads();
}

__device__ void invert_upper(const Ctx& c, int r0, int h) {
  double* Us = c.smem;
  double* X = c.smem + TRI_BLOCK * TRI_LD;
  double* W = X + TRI_BLOCK * TRI_LD;
  stage_tri(c, r0, h, Us);
  tri_inverse(Us, X, W, h, true);
  double* dst = c.scratch + (size_t)(c.n_piv + r0) * TRI_BLOCK;
  for (int e = threadIdx.x; e < h * TRI_BLOCK; e += NT) dst[e] = X[(e / TRI_BLOCK) * TRI_LD + e % TRI_BLOCK];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Op program.  The recursive LU / TRSM structure is unrolled on the host into a
// flat list of ops; the persistent CTA interprets it, so the GEMM engine is
// inlined once and nothing recurses on the device.
// ---------------------------------------------------------------------------

enum OpKind : int {
  OP_SMALL = 0,      // lu_small(c0=a, w=b)
  OP_SWAP = 1,       // apply_swaps(j0=a, cnt=b, c_lo=c, c_hi=d)
  OP_INV_LOWER = 2,  // scratch[a..a+b, :] := inv(unit lower M[a..a+b, a..a+b])
  OP_INV_UPPER = 3,  // scratch[n_pad+a.., :] := inv(upper M[a..a+b, a..a+b])
  OP_GEMM_SUB = 4,   // M[c_r.., c_c..] -= M[a_r.., a_c..] * M[b_r.., b_c..]  (Mdim, Ndim, Kdim)
  OP_GEMM_SET = 5,   // M[c_r.., c_c..]  = scratch[a_r.., 0..] * M[b_r.., b_c..]
  OP_GEMM_SET_Q = 6, // legendre: A_ib = R_b (slot) * Q (plan)
  OP_GEMM_SUB_ABI = 7,  // legendre: T -= a_bi (plan) * X (slot)
  OP_COPY_ABB = 8,   // legendre: T region := a_bb (rows [0,m), cols [a, a+m))
  OP_RHS_PROFILE = 9,  // rhs_tab from the pivots (zero prefixes of P A_ib's columns)
  OP_WBLOCK_INIT = 10, // W-trick: rows [n_pad, n_pad+RW) := A_bi / A_bb rows of sorted DOFs [a, a+b)
  OP_WBLOCK_OUT = 11,  // W-trick: T rows of sorted DOFs [a, a+b) -> DtN output (natural order)
  OP_GEMM_SET_R = 12,  // M[c_r.., c_c..] = M[a_r.., a_c..] * scratch[b_r.., 0..]  (right inverse)
  OP_GMIN16 = 13,      // gmin16 over rows [a, b) from gpos
};

struct Op {
  int kind;
  int a, b, c, d;          // generic small-op arguments
  int ar, ac, br, bc, cr, cc, Mdim, Ndim, Kdim;  // GEMM operands (row, col offsets)
  int dyn;  // forward solve against the RHS: B rows above `dyn` are zero beyond rhs_tab[dyn/16] columns
  int kmode;  // per-tile k offset: 1 from the tile's RHS columns (rhs_g), 2 from its W rows (wf)
};

// ---------------------------------------------------------------------------
// Operator assembly (reference: local_ops.py:362-398, sum order x,y,z second
// order; first order x,y,z; zeroth).  Explicit _rn intrinsics forbid FMA
// contraction so entries match scipy's sparse arithmetic bit for bit.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void interior_multi(const LeafParams& P, int r, int* I) {
  const int q = P.q;
  if (P.d == 3) {
    I[0] = r / (q * q) + 1;
    I[1] = (r / q) % q + 1;
    I[2] = r % q + 1;
  } else {
    I[0] = r / q + 1;
    I[1] = r % q + 1;
    I[2] = 0;
  }
}

// Boundary DOF index of the endpoint of the axis-`a` line through interior node I
// (face order -x,+x,-y,+y[,-z,+z]; lexicographic over the tangential indices,
// reference geometry convention local_ops.py:249-262).
// Multi-indices live in 3 registers: every access below uses a compile-time
// index (unrolled over 3 axes) so the arrays never go to local memory.
__device__ __forceinline__ int pick3(const int* v, int a) {
  return a == 0 ? v[0] : (a == 1 ? v[1] : v[2]);
}
__device__ __forceinline__ int boundary_index(const LeafParams& P, int a, int side, const int* I) {
  const int q = P.q;
  int t, fd;
  if (P.d == 3) {
    const int i0 = (a == 0) ? I[1] : I[0], i1 = (a == 2) ? I[1] : I[2];
    t = (i0 - 1) * q + (i1 - 1);
    fd = q * q;
  } else {
    t = (a == 0 ? I[1] : I[0]) - 1;
    fd = q;
  }
  return (2 * a + side) * fd + t;
}

// DtN drop mode: interior node i sits in slot row rowpos[i] and boundary DOF b
// in A_ib slot column colpos[b] (host-built orderings, build_orderings): the
// columns are sorted by the first slot row of their line, so the forward solve
// L^{-1} P A_ib skips each column's zero prefix (rhs_tab / rhs_g).
__device__ __forceinline__ int rhs_col(const LeafParams& P, int b) { return P.colperm ? P.colpos[b] : b; }
__device__ __forceinline__ int rhs_nat(const LeafParams& P, int s) { return P.colperm ? P.colnat[s] : s; }
__device__ __forceinline__ int slot_row(const LeafParams& P, int i) { return P.rowperm ? P.rowpos[i] : i; }
__device__ __forceinline__ int eq_row(const LeafParams& P, int i) { return P.rowperm ? P.eqpos[i] : i; }
// interior rows of the axis-a line of face DOF t: base + i * stride, i < q
__device__ __forceinline__ void line_rows(const LeafParams& P, int a, int t, int& base, int& stride) {
  const int q = P.q;
  if (P.d == 3) {
    if (a == 0) { base = t; stride = q * q; }
    else if (a == 1) { base = (t / q) * q * q + t % q; stride = q; }
    else { base = t * q; stride = 1; }
  } else {
    if (a == 0) { base = t; stride = q; }
    else { base = t * q; stride = 1; }
  }
}

// rhs_tab[g] = number of leading RHS columns that contain every column with a
// nonzero of P A_ib above row 16 g (P = the LU's row interchanges).  Computed
// once per leaf after the factorization; the forward-solve GEMMs clip N to it.
__device__ void rhs_profile(const LeafParams& P, Ctx& c) {
  const int n_pad = c.n_piv, m = P.m, m_pad = P.m_pad;
  const int groups = n_pad / 16 + 1;
  int* perm = reinterpret_cast<int*>(c.smem);
  int* pinv = perm + n_pad;
  int* g = pinv + n_pad;
  __syncthreads();
  if (2 * n_pad + m_pad > 2 * c.smem_doubles) {  // no room: no skipping
    for (int e = threadIdx.x; e < groups; e += NT) c.rhs_tab[e] = m_pad;
    for (int e = threadIdx.x; e < m_pad; e += NT) c.rhs_g[e] = 0;
    __syncthreads();
    return;
  }
  for (int r = threadIdx.x; r < n_pad; r += NT) { perm[r] = r; pinv[r] = c.piv[r]; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < n_pad; ++j) {
      const int pj = pinv[j];
      if (pj != j) { const int t = perm[j]; perm[j] = perm[pj]; perm[pj] = t; }
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < n_pad; r += NT) pinv[perm[r]] = r;
  __syncthreads();
  const int fd = P.d == 3 ? P.q * P.q : P.q;
  for (int sc = threadIdx.x; sc < m_pad; sc += NT) {
    int f = 0x7fffffff;
    if (sc < m) {
      const int b = rhs_nat(P, sc), face = b / fd;
      int base, stride;
      line_rows(P, face >> 1, b - face * fd, base, stride);
      for (int i = 0; i < P.q; ++i) f = min(f, pinv[eq_row(P, base + i * stride)]);
    }
    g[sc] = f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // suffix minimum: g non-decreasing
    int run = 0x7fffffff;
    for (int sc = m_pad - 1; sc >= 0; --sc) { run = min(run, g[sc]); g[sc] = run; }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m_pad; e += NT) c.rhs_g[e] = g[e];
  for (int e = threadIdx.x; e < groups; e += NT) {
    const int R = 16 * e;
    int lo = 0, hi = m_pad;  // first column with g >= R
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (g[mid] < R) lo = mid + 1; else hi = mid; }
    c.rhs_tab[e] = lo;
  }
  __syncthreads();
}

// A[row r][col with multi-index J]; coefficient pointer layout (ncoef, n):
// [a_kk (d) | a_ab + a_ba for (0,1),(0,2),(1,2) (if cross) | b_k (d) | c].
// Sum order follows collocation_rows (local_ops.py:370-387): second order
// x, y, z; cross pairs; first order x, y, z; zeroth.
// One row's coefficients, loaded once per row (warp-uniform) instead of per entry.
struct RowCoef {
  double a[3];  // a_kk
  double x[3];  // a_ab + a_ba for (0,1), (0,2), (1,2)
  double b[3];  // b_k
  double c;     // zeroth order
};
__device__ __forceinline__ RowCoef row_coef(const LeafParams& P, const double* cf, int r) {
  RowCoef rc;
  const int d = P.d, n = P.n;
  int k = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) rc.a[a] = (a < d) ? cf[(k + a) * n + r] : 0.0;
  k += d;
  const int npair = d * (d - 1) / 2;
#pragma unroll
  for (int a = 0; a < 3; ++a) rc.x[a] = (P.has_cross && a < npair) ? cf[(k + a) * n + r] : 0.0;
  if (P.has_cross) k += npair;
#pragma unroll
  for (int a = 0; a < 3; ++a) rc.b[a] = (P.has_first && a < d) ? cf[(k + a) * n + r] : 0.0;
  if (P.has_first) k += d;
  rc.c = P.has_zeroth ? cf[k * n + r] : 0.0;
  return rc;
}

// D1 / D2 are the plan's d x p x p tables (global) or their shared-memory copies.
__device__ double op_entry(const LeafParams& P, const RowCoef& rc, const double* D1, const double* D2,
                           const int* I, const int* J) {
  const int p = P.p, d = P.d;
  double v = 0.0;
  int ndiff = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) ndiff += (k < d && I[k] != J[k]);
  bool line[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) line[a] = (a < d) && (ndiff == 0 || (ndiff == 1 && I[a] != J[a]));
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (line[a]) v = __dadd_rn(v, __dmul_rn(-rc.a[a], D2[(a * p + I[a]) * p + J[a]]));
  if (P.has_cross) {
    // pairs (0,1), (0,2), (1,2); d = 2 has only (0,1)
#pragma unroll
    for (int pair = 0; pair < 3; ++pair) {
      const int a = pair == 2 ? 1 : 0, b = pair == 0 ? 1 : 2, o = 3 - a - b;
      if (b < d) {
        const bool in_plane = (d < 3) || I[o] == J[o];  // J differs from I at most in a, b
        if (in_plane) {
          const double kr = __dmul_rn(D1[(a * p + I[a]) * p + J[a]], D1[(b * p + I[b]) * p + J[b]]);
          v = __dadd_rn(v, __dmul_rn(-rc.x[pair], kr));
        }
      }
    }
  }
  if (P.has_first) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (line[a]) v = __dadd_rn(v, __dmul_rn(rc.b[a], D1[(a * p + I[a]) * p + J[a]]));
  }
  if (P.has_zeroth && ndiff == 0) v = __dadd_rn(v, rc.c);
  return v;
}

// Nonzero pattern of row I: the d grid lines through I (d*p positions, the
// diagonal once) and, with cross terms, the strict interiors of the coordinate
// planes through I ((p-1)^2 each).  Returns the multi-index J of item e.
__device__ __forceinline__ int pattern_size(const LeafParams& P) {
  return P.d * P.p + (P.has_cross ? (P.d * (P.d - 1) / 2) * (P.p - 1) * (P.p - 1) : 0);
}
__device__ __forceinline__ bool pattern_item(const LeafParams& P, const int* I, int e, int* J) {
  const int p = P.p, d = P.d;
  if (e < d * p) {
    const int a = e / p, pos = e - a * p;
    if (pos == pick3(I, a) && a > 0) return false;
#pragma unroll
    for (int t = 0; t < 3; ++t) J[t] = (t == a) ? pos : I[t];
    return true;
  }
  e -= d * p;
  const int per = (p - 1) * (p - 1);
  const int pair = e / per, w = e - pair * per;
  const int a = (d == 3 && pair == 2) ? 1 : 0, b = (d == 2) ? 1 : (pair == 0 ? 1 : 2);
  int ja = w / (p - 1), jb = w - ja * (p - 1);
  ja += (ja >= pick3(I, a));  // skip I[a] / I[b]: strict plane interior
  jb += (jb >= pick3(I, b));
#pragma unroll
  for (int t = 0; t < 3; ++t) J[t] = (t == a) ? ja : ((t == b) ? jb : I[t]);
  return true;
}

__device__ __forceinline__ bool is_interior(const LeafParams& P, const int* J) {
  bool in = true;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if (k < P.d && (J[k] == 0 || J[k] == P.p - 1)) in = false;
  return in;
}

__device__ __forceinline__ int full_flat(const LeafParams& P, const int* J) {
  int f = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if (k < P.d) f = f * P.p + J[k];
  return f;
}

// Fill the slot matrix.  Warp per row: zero the row, then scatter structural nonzeros.
// Drop mode: boundary endpoints are the face DOF columns of A_ib.  Legendre
// mode: boundary nodes are Chebyshev boundary nodes; their entries R_b go to
// the slot's R_b region (A_ib = R_b Q is a GEMM op) or, for interior solves,
// are contracted with Q u_b directly.
__device__ void assemble(const LeafParams& P, double* M, int leaf, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* cf = P.coeffs + (size_t)leaf * P.ncoef * P.n;
  const int d = P.d;
  const bool solve_mode = (P.mode == MODE_REDUCE || P.mode == MODE_INTERIOR);
  double* qub = smem;  // legendre interior solve: (Q u_b)[g], g over Chebyshev boundary nodes
  if (P.legendre && P.mode == MODE_INTERIOR) {
    const double* ub = P.in0 + (size_t)leaf * P.m;
    for (int g = warp; g < P.nb; g += NT / 32) {
      double acc = 0.0;
      for (int c = lane; c < P.m; c += 32) acc += P.Q[(size_t)g * P.m_pad + c] * ub[c];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) qub[g] = acc;
    }
  }
  // derivative tables in shared memory (after the qub vector)
  double* D1s = smem + (P.legendre ? ((P.nb + 1) & ~1) : 0);
  const int dpp = d * P.p * P.p;
  double* D2s = D1s + dpp;
  for (int e = threadIdx.x; e < dpp; e += NT) { D1s[e] = P.D1[e]; D2s[e] = P.D2[e]; }
  __syncthreads();
  const int npat = pattern_size(P);
  // permuted rows (DtN drop orderings): zero the whole slot before any row is filled
  const bool two_pass = P.rowperm != 0;
  if (two_pass && P.smem_doubles < 1024 + 2 * dpp) {
    for (int r = warp; r < P.NR; r += NT / 32) {
      double2* row2 = reinterpret_cast<double2*>(M + (size_t)r * P.ld);
      for (int c2 = lane; c2 < P.NC / 2; c2 += 32) row2[c2] = make_double2(0.0, 0.0);
    }
    __syncthreads();
  } else if (two_pass) {
    // bulk stores from a zeroed smem block at the end of the dynamic smem (past the
    // derivative tables): the TMA unit writes the slot, the LSUs stay free for the
    // co-resident CTA
    constexpr int ZB = 1024;  // doubles per bulk store (8 KB)
    double* zb = smem + (P.smem_doubles - ZB);
    for (int e = threadIdx.x; e < ZB; e += NT) zb[e] = 0.0;
    fence_proxy_async_smem();
    __syncthreads();
    if (lane == 0) {
      const size_t row_bytes = (size_t)P.NC * 8;
      for (int r = warp; r < P.NR; r += NT / 32) {
        char* row = reinterpret_cast<char*>(M + (size_t)r * P.ld);
        for (size_t o = 0; o < row_bytes; o += ZB * 8)
          bulk_store_s2g(row + o, zb, (unsigned)min((size_t)ZB * 8, row_bytes - o));
      }
      bulk_commit();
      bulk_wait_all();
      fence_proxy_async_global();
    }
    __syncthreads();
  }
  for (int r = warp; r < P.NR; r += NT / 32) {
    double* row = M + (size_t)(r < P.n ? eq_row(P, r) : r) * P.ld;
    if (!two_pass) {
      double2* row2 = reinterpret_cast<double2*>(row);
      for (int c2 = lane; c2 < P.NC / 2; c2 += 32) row2[c2] = make_double2(0.0, 0.0);
      __syncwarp();
    }
    if (r < P.n) {
      int I[3];
      interior_multi(P, r, I);
      const RowCoef rc = row_coef(P, cf, r);
      double rhs = 0.0;  // interior solve: A_ib u_b accumulated over the pattern
      for (int e = lane; e < npat; e += 32) {
        int J[3];
        if (!pattern_item(P, I, e, J)) continue;
        if (is_interior(P, J)) {
          int flat = 0;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (k < d) flat = flat * P.q + (J[k] - 1);
          row[slot_row(P, flat)] = op_entry(P, rc, D1s, D2s, I, J);
        } else if (P.legendre) {
          if (P.mode == MODE_INTERIOR) rhs += op_entry(P, rc, D1s, D2s, I, J) * qub[P.bpos[full_flat(P, J)]];
          else if (!solve_mode) row[P.col_rb + P.bpos[full_flat(P, J)]] = op_entry(P, rc, D1s, D2s, I, J);
        } else if (!solve_mode) {
          // drop mode: line endpoints are face-interior DOFs
          int a = 0;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (k < d && J[k] != I[k]) a = k;
          row[P.n_pad + rhs_col(P, boundary_index(P, a, pick3(J, a) == P.p - 1 ? 1 : 0, I))] =
              op_entry(P, rc, D1s, D2s, I, J);
        }
      }
      if (P.mode == MODE_REDUCE && lane == 0) {
        row[P.n_pad] = P.in0[(size_t)leaf * P.n + r];
      } else if (P.mode == MODE_INTERIOR) {
        if (P.legendre) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) rhs += __shfl_xor_sync(0xffffffffu, rhs, off);
          if (lane == 0) row[P.n_pad] = rhs;
        } else if (lane == 0) {
          // rhs = A_ib u_b over its 2d structural nonzeros, in column (face) order
          const double* ub = P.in0 + (size_t)leaf * P.m;
          double sacc = 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (a >= d) continue;
#pragma unroll
            for (int side = 0; side < 2; ++side) {
              int J[3];
#pragma unroll
              for (int t = 0; t < 3; ++t) J[t] = (t == a) ? (side ? P.p - 1 : 0) : I[t];
              sacc += op_entry(P, rc, D1s, D2s, I, J) * ub[boundary_index(P, a, side, I)];
            }
          }
          row[P.n_pad] = sacc;
        }
      }
    } else if (r < P.n_pad) {
      if (lane == 0) row[r] = 1.0;  // dummy pivot keeps padding inert
    }
  }
  __syncthreads();
}

// Legendre DtN: T region (rows [0, m), cols [col, col + m_pad)) := a_bb, zero padded.
__device__ void copy_abb(const LeafParams& P, Ctx& c, int col) {
  __syncthreads();
  for (int e = threadIdx.x; e < P.m_pad * P.m_pad; e += NT) {
    const int i = e / P.m_pad, j = e - i * P.m_pad;
    c.M[(size_t)i * c.ld + col + j] = (i < P.m && j < P.m) ? P.a_bb[(size_t)i * P.m + j] : 0.0;
  }
  __syncthreads();
}

// rows x cols block of M (ld) -> dense out (ld_out), 16-byte vectors, 8 in flight
// per thread; cols and both row strides even.
__device__ void copy_block(const double* src, int ld, double* out, int ld_out, int rows, int cols,
                           bool negate, const int* rmap = nullptr) {
  const int c2 = cols / 2;
  const int total = rows * c2;
  for (int e0 = threadIdx.x; e0 < total; e0 += NT * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * NT;
      if (e < total) {
        const int i = e / c2, j = e - i * c2;
        v[u] = reinterpret_cast<const double2*>(src + (size_t)(rmap ? rmap[i] : i) * ld)[j];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * NT;
      if (e < total) {
        const int i = e / c2, j = e - i * c2;
        double2 w = v[u];
        if (negate) { w.x = -w.x; w.y = -w.y; }
        reinterpret_cast<double2*>(out + (size_t)i * ld_out)[j] = w;
      }
    }
  }
}

// DtN from the solution block: with X = A_ii^{-1} A_ib in columns [n_pad, n_pad+m)
// of M, T = A_bb - A_bi X.  A_bi is structurally sparse: boundary DOF b reads
// only the q = p-2 interior nodes on its normal grid line, with weights
// -D1[a][0][.] (low face) / +D1[a][p-1][.] (high face) (local_ops.py:310-315).
// Each interior line serves the two opposite face DOFs, so X is read once per
// line: 2 q m^2 flops instead of the dense 2 n m^2.
// Streamed variant: X is read exactly once.  X's rows are walked in slabs of
// fixed first index i (S = q^(d-1) rows): the lines along the last d-1 axes
// lie inside one slab and finish there; the lines along axis 0 take their i-th
// point from slab i and accumulate in shared memory.  Columns go in chunks of
// CW through an NBUF-deep cp.async ring.  A_bb (two structural nonzeros per
// row, the line endpoints: a_bb[b, b_lo] = sign D1[a][edge][0], a_bb[b, b_hi] =
// sign D1[a][edge][p-1]) is added in registers instead of read from HBM.
// Returns false when the slab ring does not fit; the caller then uses dtn_lines.
constexpr int LINE_NBUF = 4;
#ifndef HPS_LINE_CW
#define HPS_LINE_CW 16
#endif
static_assert(HPS_LINE_CW <= 16, "line-output column chunk within m_pad");
__device__ bool dtn_lines_stream(const LeafParams& P, Ctx& c, const double* M, int ld, double* T) {
  __shared__ double s_w[3][2][32];
  __shared__ double s_e[3][2][2];
  const int q = P.q, p = P.p, d = P.d, m = P.m;
  const int S = (d == 3) ? q * q : q;
  // int tables in shared memory: slot column -> DtN column, interior node -> slot row
  const int tab_d = P.rowperm ? (m + 1) / 2 + (P.n + 1) / 2 : 0;
  // column chunk: 16 columns (128-byte row segments of X) when the ring fits (p <= 12),
  // else 8 or fewer (m_pad is a multiple of 16, so a chunk never leaves the row)
  int CW = HPS_LINE_CW;
  while (CW >= 2 && (2 + LINE_NBUF) * S * CW + tab_d > c.smem_doubles) CW >>= 1;
  if (CW < 2 || q > 32) return false;
  __syncthreads();  // smem is free (previous op finished with it)
  for (int e = threadIdx.x; e < d * 2 * q; e += NT) {
    const int a = e / (2 * q), side = (e / q) & 1, i = e % q;
    s_w[a][side][i] = P.D1[(a * p + (side ? p - 1 : 0)) * p + i + 1];
  }
  if (threadIdx.x < d * 4) {
    const int a = threadIdx.x >> 2, side = (threadIdx.x >> 1) & 1, end = threadIdx.x & 1;
    const double sgn = side ? 1.0 : -1.0;
    s_e[a][side][end] = sgn * P.D1[(a * p + (side ? p - 1 : 0)) * p + (end ? p - 1 : 0)];
  }
  double* acc = c.smem;              // [2][S*CW]: axis-0 lines, low / high face
  double* ring = c.smem + 2 * S * CW;  // [NBUF][S*CW]
  int* nat_tab = reinterpret_cast<int*>(ring + LINE_NBUF * S * CW);
  int* row_tab = nat_tab + m;
  if (P.rowperm) {
    for (int e = threadIdx.x; e < m; e += NT) nat_tab[e] = rhs_nat(P, e);
    for (int e = threadIdx.x; e < P.n; e += NT) row_tab[e] = P.rowpos[e];
  }
  __syncthreads();
  const double* X = M + P.n_pad;
  const int fd = S;
  const int SC = S * CW;
  const int vec = CW / 2;  // 16-byte pieces per row chunk
  // in-slab line directions: d = 3 -> axis 1 (q lines, stride q) and axis 2 (q lines,
  // stride 1); d = 2 -> axis 1 (1 line, stride 1)
  const int nl = (d == 3) ? q : 1;
  const int n_dir = d - 1;
  auto load_slab = [&](int i, int c0) {
    if (i < q) {
      double* buf = ring + (i % LINE_NBUF) * SC;
      for (int e = threadIdx.x; e < S * vec; e += NT) {
        const int r = e / vec, v = e - r * vec;
        const double* src = X + (size_t)(P.rowperm ? row_tab[i * S + r] : i * S + r) * ld + c0;
        cp_async16(buf + r * CW + 2 * v, src + 2 * v, 16);
      }
    }
    cp_async_commit();
  };
  auto put = [&](int b, int col0, int b_lo, int b_hi, const double* e2, double v0, double v1, bool neg) {
    // T[b, nat(col0 + {0,1})] = a_bb + (neg ? -v : v); col0 is a slot column
    double o[2] = {v0, v1};
    int nat[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      nat[u] = (col0 + u >= m) ? -1 : (P.rowperm ? nat_tab[col0 + u] : col0 + u);
      const int col = nat[u];
      const double abb = col == b_lo ? e2[0] : (col == b_hi ? e2[1] : 0.0);
      o[u] = neg ? abb - o[u] : abb + o[u];
    }
    if (col0 + 1 < m && nat[1] == nat[0] + 1 && (nat[0] & 1) == 0) {
      *reinterpret_cast<double2*>(T + (size_t)b * m + nat[0]) = make_double2(o[0], o[1]);
    } else {
      if (col0 < m) T[(size_t)b * m + nat[0]] = o[0];
      if (col0 + 1 < m) T[(size_t)b * m + nat[1]] = o[1];
    }
  };
  for (int c0 = 0; c0 < m; c0 += CW) {
    for (int e = threadIdx.x; e < 2 * SC; e += NT) acc[e] = 0.0;
#pragma unroll 1
    for (int s = 0; s < LINE_NBUF - 1; ++s) load_slab(s, c0);
    for (int i = 0; i < q; ++i) {
      cp_async_wait<LINE_NBUF - 2>();
      __syncthreads();
      load_slab(i + LINE_NBUF - 1, c0);
      const double* buf = ring + (i % LINE_NBUF) * SC;
      // axis-0 lines: slab row t is point i of line t
      const double wl = s_w[0][0][i], wh = s_w[0][1][i];
      for (int e = threadIdx.x; e < SC; e += NT) {
        const double x = buf[e];
        acc[e] += wl * x;
        acc[SC + e] += wh * x;
      }
      // in-slab lines, two adjacent columns per item
      const int items = n_dir * nl * vec;
      for (int e = threadIdx.x; e < items; e += NT) {
        const int v = e % vec, l = (e / vec) % nl, dir = e / (vec * nl);
        const int a = dir + 1;
        const int s0 = (d == 3 && a == 1) ? l : l * q;
        const int st = (d == 3 && a == 1) ? q : 1;
        double lo0 = 0.0, lo1 = 0.0, hi0 = 0.0, hi1 = 0.0;
        for (int k = 0; k < q; ++k) {
          const double2 x = *reinterpret_cast<const double2*>(buf + (s0 + k * st) * CW + 2 * v);
          const double w0 = s_w[a][0][k], w1 = s_w[a][1][k];
          lo0 += w0 * x.x; lo1 += w0 * x.y;
          hi0 += w1 * x.x; hi1 += w1 * x.y;
        }
        const int t = i * nl + l;
        const int b_lo = 2 * a * fd + t, b_hi = b_lo + fd;
        const int col0 = c0 + 2 * v;
        put(b_lo, col0, b_lo, b_hi, s_e[a][0], lo0, lo1, false);
        put(b_hi, col0, b_lo, b_hi, s_e[a][1], hi0, hi1, true);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int e = threadIdx.x; e < S * vec; e += NT) {
      const int t = e / vec, v = e - t * vec;
      const int b_lo = t, b_hi = fd + t;
      const int col0 = c0 + 2 * v;
      put(b_lo, col0, b_lo, b_hi, s_e[0][0], acc[t * CW + 2 * v], acc[t * CW + 2 * v + 1], false);
      put(b_hi, col0, b_lo, b_hi, s_e[0][1], acc[SC + t * CW + 2 * v], acc[SC + t * CW + 2 * v + 1],
          true);
    }
    __syncthreads();
  }
  return true;
}

__device__ void dtn_lines(const LeafParams& P, const double* M, int ld, double* T) {
  __shared__ double s_w[3][2][32];
  const int q = P.q, p = P.p, d = P.d, m = P.m;
  for (int e = threadIdx.x; e < d * 2 * q; e += NT) {
    const int a = e / (2 * q), side = (e / q) & 1, i = e % q;
    s_w[a][side][i] = P.D1[(a * p + (side ? p - 1 : 0)) * p + i + 1];
  }
  __syncthreads();
  const int fd = (d == 3) ? q * q : q;
  const int lines = d * fd;
  const double* X = M + P.n_pad;
  constexpr int U = 2;  // independent (line, column) items per thread iteration
  for (int e0 = threadIdx.x; e0 < lines * m; e0 += NT * U) {
    double lo[U], hi[U];
    int a_[U], t_[U], col_[U], xcol_[U], base_[U], stride_[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      const int line = (e < lines * m) ? e / m : 0;
      col_[u] = (e < lines * m) ? e - line * m : 0;
      xcol_[u] = rhs_col(P, col_[u]);
      a_[u] = line / fd;
      t_[u] = line - a_[u] * fd;
      const int a = a_[u], t = t_[u];
      if (d == 3) {
        if (a == 0) { base_[u] = t; stride_[u] = q * q; }
        else if (a == 1) { base_[u] = (t / q) * q * q + t % q; stride_[u] = q; }
        else { base_[u] = t * q; stride_[u] = 1; }
      } else {
        if (a == 0) { base_[u] = t; stride_[u] = q; }
        else { base_[u] = t * q; stride_[u] = 1; }
      }
      lo[u] = hi[u] = 0.0;
    }
    for (int i = 0; i < q; ++i) {
      double x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = X[(size_t)slot_row(P, base_[u] + i * stride_[u]) * ld + xcol_[u]];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        lo[u] += s_w[a_[u]][0][i] * x[u];
        hi[u] += s_w[a_[u]][1][i] * x[u];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      if (e < lines * m) {
        const int b_lo = 2 * a_[u] * fd + t_[u], b_hi = b_lo + fd;
        T[(size_t)b_lo * m + col_[u]] = P.a_bb[(size_t)b_lo * m + col_[u]] + lo[u];
        T[(size_t)b_hi * m + col_[u]] = P.a_bb[(size_t)b_hi * m + col_[u]] - hi[u];
      }
    }
  }
}

// W-trick DtN (drop mode).  T = A_bb - W Y with W = A_bi U^-1 (m x n) and
// Y = L^-1 P A_ib (n x m): both triangular solves start at the first nonzero of
// each line (W row b is zero left of f_b in the slot's interior order, Y
// column c above the pivoted f_c), and so does the k range of W Y.  W is
// formed in blocks of RW sorted boundary DOFs in the slot rows below A_ii;
// the same rows hold the block's T rows in the A_ib columns.
//   wblock_init: rows [n_pad, n_pad + RW) := [A_bi rows | A_bb rows] of the
//   sorted DOFs s0 .. s0+R (zero elsewhere from column zc on); wf = their f.
__device__ void wblock_init(const LeafParams& P, Ctx& c, int s0, int R, int zc) {
  const int q = P.q, p = P.p, d = P.d, m = P.m;
  const int fd = (d == 3) ? q * q : q;
  __syncthreads();
  for (int r = threadIdx.x >> 5; r < P.RW; r += NT / 32) {
    double* row = c.M + (size_t)(c.n_piv + r) * c.ld;
    for (int col = zc + (threadIdx.x & 31) * 2; col < P.NC; col += 64)
      *reinterpret_cast<double2*>(row + col) = make_double2(0.0, 0.0);
  }
  for (int r = threadIdx.x; r < P.RW; r += NT) c.wf[r] = (r < R) ? P.fsort[s0 + r] : 0x7fffffff;
  __syncthreads();
  // warp per DOF: lanes over the q line nodes (+ 2 endpoints)
  for (int r = threadIdx.x >> 5; r < R; r += NT / 32) {
    const int lane = threadIdx.x & 31;
    const int b = P.colnat[s0 + r];
    const int face = b / fd, t = b - face * fd, a = face >> 1, side = face & 1;
    int base, stride;
    line_rows(P, a, t, base, stride);
    const double sgn = side ? 1.0 : -1.0;
    const double* Drow = P.D1 + (size_t)(a * p + (side ? p - 1 : 0)) * p;
    double* row = c.M + (size_t)(c.n_piv + r) * c.ld;
    for (int k = lane; k < q; k += 32) row[P.rowpos[base + k * stride]] = sgn * Drow[k + 1];
    if (lane == 0) {
      const int b_lo = (2 * a) * fd + t, b_hi = b_lo + fd;
      row[c.n_piv + P.colpos[b_lo]] = sgn * Drow[0];
      row[c.n_piv + P.colpos[b_hi]] = sgn * Drow[p - 1];
    }
  }
  (void)m;
  __syncthreads();
}

// T rows of sorted DOFs s0 .. s0+R -> DtN output rows colnat[s], columns in
// natural order (staged through shared memory, coalesced both ways).
__device__ void wblock_out(const LeafParams& P, Ctx& c, int s0, int R, int leaf) {
  const int m = P.m;
  double* T = P.out0 + (size_t)leaf * m * m;
  const int rows_per = max(1, c.smem_doubles / P.m_pad);
  __syncthreads();
  for (int r0 = 0; r0 < R; r0 += rows_per) {
    const int nr = min(rows_per, R - r0);
    for (int e = threadIdx.x; e < nr * (m / 2); e += NT) {
      const int r = e / (m / 2), j = e - r * (m / 2);
      reinterpret_cast<double2*>(c.smem + r * P.m_pad)[j] =
          reinterpret_cast<const double2*>(c.M + (size_t)(c.n_piv + r0 + r) * c.ld + c.n_piv)[j];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * m; e += NT) {
      const int r = e / m, j = e - r * m;
      T[(size_t)P.colnat[s0 + r0 + r] * m + j] = c.smem[r * P.m_pad + P.colpos[j]];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    hps_leaf_kernel(LeafParams P, const Op* __restrict__ ops, int n_ops, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(1024) double smem[];
  __shared__ __align__(8) uint64_t bars[2 * STAGES];
  __shared__ __align__(8) uint64_t gbars[2 * 2 * HSTAGES];  // half tiles: [full | empty][group][stage]
  const int slot = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bars[s], FULL_COUNT);
      mbar_init(&bars[STAGES + s], NT / 32);
    }
    for (int s = 0; s < 2 * HSTAGES; ++s) {
      mbar_init(&gbars[s], 1);
      mbar_init(&gbars[2 * HSTAGES + s], NT / 32 / 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#if HPS_PROF_EXEC
    s_exec_dmma = 0;
    s_exec_cap = 0;
#endif
  }
  __syncthreads();
  Ctx c;
  c.slot = slot;
  c.maps = &maps;
  c.full = bars;
  c.empty = bars + STAGES;
  c.pipe = 0;
  c.gfull = gbars;
  c.gempty = gbars + 2 * HSTAGES;
  c.gpipe = 0;
  c.M = P.work + (size_t)slot * P.slot_stride;
  c.ld = P.ld;
  c.n_piv = P.n_pad;
  c.n_real = P.n;
  c.NR = P.NR;
  c.wb = P.wb;
  c.piv = P.piv + (size_t)slot * P.piv_stride;
  c.rhs_tab = c.piv + P.n_pad;
  c.rhs_g = c.rhs_tab + P.n_pad / 16 + 16;
  c.wf = c.rhs_g + P.m_pad;
  c.gpos = P.rowperm ? c.wf + P.RW : nullptr;
  c.tau = P.rowperm ? P.pivot_tau : 0.0;
  c.gmin16 = c.wf + P.RW + P.n_pad;
  c.gcol16 = c.gmin16 + P.n_pad / 16 + 17;
  c.scratch = P.scratch + (size_t)slot * 2 * P.n_pad * TRI_BLOCK;
  c.smem = smem;
  c.smem_doubles = P.smem_doubles;
  c.sh = P.share ? P.share + slot : nullptr;
  c.role = 0;
  c.seq = 0;
  c.cur_op = 0;
  c.leaf_counter = P.leaf_counter;
  c.n_leaves = P.n_leaves;

  unsigned long long* prof = P.prof ? P.prof + (size_t)slot * PROF_SLOTS : nullptr;
  c.prof = prof;
  if (prof && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    prof[25] = smid;
  }
  // dynamic leaf scheduling: the two CTAs sharing an SM do not progress at the
  // same rate (warp arbitration), so slots grab the next leaf when done
  __shared__ int s_leaf;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_leaf = atomicAdd(P.leaf_counter, 1);
    __syncthreads();
    const int leaf = s_leaf;
    if (leaf >= P.n_leaves) break;
    long long t0 = clock64();
    if (c.gpos) {
      for (int r = threadIdx.x; r < P.n_pad; r += NT) c.gpos[r] = P.gsorted[r];
      for (int g = threadIdx.x; g < P.n_pad / 16; g += NT) {
        int mn = 0x7fffffff;
        for (int r = 16 * g; r < 16 * g + 16; ++r) mn = min(mn, P.gsorted[r]);
        c.gmin16[g] = mn;
        c.gcol16[g] = mn;
      }
      if (threadIdx.x == 0) c.gcol16[-1] = P.n_pad;
    }
    assemble(P, c.M, leaf, c.smem);
    if (threadIdx.x == 0) { s_pmin = INFINITY; s_pmax = 0.0; }
    __syncthreads();
    if (prof && threadIdx.x == 0) { prof[22] += clock64() - t0; prof[9] += 1; }
    int phase = 0;  // profile: 0 LU, 1 forward solve, 2 W blocks / backward solve
    for (int k = 0; k < ((P.debug & 1) ? 0 : n_ops); ++k) {
      Op op = ops[k];
      c.cur_op = k;
      if (op.kind == OP_RHS_PROFILE) phase = 1;
      if (op.kind == OP_WBLOCK_INIT || (phase == 1 && op.kind == OP_INV_UPPER)) phase = 2;
      if (prof) t0 = clock64();
      switch (op.kind) {
        case OP_SMALL: {
          // rows at or beyond op.c are structurally zero in these columns (sorted equations)
          const int np = c.n_piv, nr = c.NR;
          if (op.c > 0) { c.n_piv = min(np, op.c); c.NR = min(nr, op.c); }
          lu_small(c, op.a, op.b);
          c.n_piv = np; c.NR = nr;
          break;
        }
        case OP_SWAP: apply_swaps(c, op.a, op.b, op.c, op.d); break;
        case OP_INV_LOWER: invert_unit_lower(c, op.a, op.b); break;
        case OP_INV_UPPER: invert_upper(c, op.a, op.b); break;
        case OP_COPY_ABB: copy_abb(P, c, op.a); break;
        case OP_RHS_PROFILE: rhs_profile(P, c); break;
        case OP_WBLOCK_INIT: wblock_init(P, c, op.a, op.b, op.c); break;
        case OP_WBLOCK_OUT: wblock_out(P, c, op.a, op.b, leaf); break;
        case OP_GMIN16: {
          __syncthreads();
          for (int g = (op.a >> 4) + (int)threadIdx.x; g < ((op.b + 15) >> 4); g += NT) {
            int mn = 0x7fffffff;
            for (int r = g * 16; r < g * 16 + 16 && r < P.n_pad; ++r) mn = min(mn, c.gpos[r]);
            c.gmin16[g] = mn;
          }
          __syncthreads();
          break;
        }
        default: {
          const bool sub = (op.kind == OP_GEMM_SUB || op.kind == OP_GEMM_SUB_ABI);
          const int a_src = op.kind == OP_GEMM_SET ? 1 : (op.kind == OP_GEMM_SUB_ABI ? 2 : 0);
          const int b_src = op.kind == OP_GEMM_SET_Q ? 1 : (op.kind == OP_GEMM_SET_R ? 2 : 0);
          const int N = op.dyn ? min(op.Ndim, c.rhs_tab[op.dyn >> 4]) : op.Ndim;
          const int tri = op.kind == OP_GEMM_SET ? (op.ar < P.n_pad ? 1 : 3)
                          : (op.kind == OP_GEMM_SET_R ? 2 : 0);
          gemm(c, sub, a_src, op.ar, op.ac, b_src, op.br, op.bc, op.cr, op.cc, op.Mdim, N, op.Kdim,
               op.kmode, tri);
          op.Ndim = N;  // profile counters below count the work done
        }
      }
      if (prof && threadIdx.x == 0) {
        const long long dt = clock64() - t0;
        prof[28 + phase] += dt;
#if HPS_PROF_EXEC
        if (op.kind == OP_GEMM_SUB || op.kind == OP_GEMM_SET || op.kind == OP_GEMM_SET_Q ||
            op.kind == OP_GEMM_SUB_ABI || op.kind == OP_GEMM_SET_R) {
          const unsigned long long f = s_exec_dmma * 512ull;  // flops per m8n8k4 DMMA
          const int bk = op.Ndim <= 64 ? 0 : (op.Ndim <= 256 ? 1 : 2);
          prof[32 + bk] += f;
          prof[35 + phase] += f;
          prof[38 + phase] += dt;
          prof[41 + bk] += s_exec_cap * 512ull;  // capacity of the walked chunks
        }
        s_exec_dmma = 0;
        s_exec_cap = 0;
#endif
        const int pk = op.kind < OP_RHS_PROFILE ? op.kind
                       : (op.kind == OP_RHS_PROFILE ? 24
                          : (op.kind == OP_GEMM_SET_R ? OP_GEMM_SET : (op.kind == OP_GMIN16 ? 22 : 27)));
        prof[pk] += dt;
        if (op.kind == OP_GEMM_SUB || op.kind == OP_GEMM_SET || op.kind == OP_GEMM_SET_Q ||
            op.kind == OP_GEMM_SUB_ABI || op.kind == OP_GEMM_SET_R) {
          const int bucket = op.Ndim <= 64 ? 0 : (op.Ndim <= 256 ? 1 : 2);
          prof[16 + bucket] += dt;
          prof[19 + bucket] += (2ull * op.Mdim * op.Ndim * op.Kdim) >> 20;
        }
      }
    }
    if (prof) t0 = clock64();
    if (P.mode == MODE_DTN && P.legendre) {
      copy_block(c.M + P.col_rb, c.ld, P.out0 + (size_t)leaf * P.m * P.m, P.m, P.m, P.m, false);
    } else if (P.mode == MODE_DTN && P.wt) {
      // written block by block by OP_WBLOCK_OUT
    } else if (P.mode == MODE_DTN) {
      double* T = P.out0 + (size_t)leaf * P.m * P.m;
      if ((P.debug & 2) || !dtn_lines_stream(P, c, c.M, c.ld, T)) dtn_lines(P, c.M, c.ld, T);
    } else if (P.mode == MODE_SOLOP) {
      copy_block(c.M + P.n_pad, c.ld, P.out0 + (size_t)leaf * P.n * P.m, P.m, P.n, P.m, true,
                 P.rowperm ? P.rowpos : nullptr);
    } else if (P.mode == MODE_FACTORS) {
      // S = -X, then T from the same X: a_bb - a_bi X (legendre: already formed in the
      // R_b region by the program; drop: the line-sparse A_bi applied here)
      copy_block(c.M + P.n_pad, c.ld, P.out1 + (size_t)leaf * P.n * P.m, P.m, P.n, P.m, true,
                 P.rowperm ? P.rowpos : nullptr);
      __syncthreads();
      double* T = P.out0 + (size_t)leaf * P.m * P.m;
      if (P.legendre) {
        copy_block(c.M + P.col_rb, c.ld, T, P.m, P.m, P.m, false);
      } else if (!dtn_lines_stream(P, c, c.M, c.ld, T)) {
        dtn_lines(P, c.M, c.ld, T);
      }
    } else {
      double* out = P.out0 + (size_t)leaf * P.n;
      if (P.mode == MODE_REDUCE) {
        for (int i = threadIdx.x; i < P.n; i += NT) out[i] = c.M[(size_t)slot_row(P, i) * c.ld + P.n_pad];
        __syncthreads();
        // flux = A_bi v : warp per boundary row, lanes stride the interior
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        double* flux = P.out1 + (size_t)leaf * P.m;
        for (int b = warp; b < P.m; b += NT / 32) {
          const double* abi = P.a_bi + (size_t)b * P.n;
          double s = 0.0;
          for (int k = lane; k < P.n; k += 32) s += abi[k] * out[k];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
          if (lane == 0) flux[b] = s;
        }
      } else {
        const double* v = P.in1 + (size_t)leaf * P.n;
        for (int i = threadIdx.x; i < P.n; i += NT)
          out[i] = v[i] - c.M[(size_t)slot_row(P, i) * c.ld + P.n_pad];
      }
    }
    if (threadIdx.x == 0) {
      P.stats[2 * leaf] = s_pmin;
      P.stats[2 * leaf + 1] = s_pmax;
    }
    if (P.done_counts) {
      // outputs of this leaf complete and visible device-wide before the count
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(P.done_counts + leaf / P.done_chunk, 1);
    }
    __syncthreads();
    if (prof && threadIdx.x == 0) prof[23] += clock64() - t0;
  }
  // Endgame: no leaf left for this CTA.  Help the CTAs still reducing a leaf
  // with the tiles of their published GEMMs until every CTA is done.
  if (P.share) {
    __shared__ int s_tgt, s_top;
    __shared__ unsigned s_tseq;
    const int nslots = (int)gridDim.x;
    long long th = prof ? clock64() : 0;
    if (threadIdx.x == 0) atomicAdd(P.share_finished, 1);
    for (int round = 0;; ++round) {
      if (threadIdx.x == 0) {
        int tgt = -1;
        if (*reinterpret_cast<volatile int*>(P.share_finished) >= nslots) {
          tgt = -2;
        } else {
          for (int k = 1; k < nslots && tgt < 0; ++k) {
            const int s2 = (slot + k) % nslots;
            ShareSlot* sh = P.share + s2;
            const unsigned long long w = *reinterpret_cast<volatile unsigned long long*>(&sh->claim);
            const unsigned seq = (unsigned)(w >> 32);
            if (seq == 0) continue;
            __threadfence();
            const int oseq = *reinterpret_cast<volatile int*>(&sh->op_seq);
            const int tiles = *reinterpret_cast<volatile int*>(&sh->tiles);
            const int op = *reinterpret_cast<volatile int*>(&sh->op);
            if ((unsigned)oseq == seq && (int)(w & 0xffffffffull) < tiles) {
              tgt = s2;
              s_tseq = seq;
              s_top = op;
            }
          }
          if (tgt < 0) __nanosleep(1000);
        }
        s_tgt = tgt;
      }
      __syncthreads();
      const int tgt = s_tgt;
      if (tgt == -2) break;
      if (tgt >= 0) {
        Ctx h = c;
        h.slot = tgt;
        h.M = P.work + (size_t)tgt * P.slot_stride;
        h.piv = P.piv + (size_t)tgt * P.piv_stride;
        h.rhs_tab = h.piv + P.n_pad;
        h.rhs_g = h.rhs_tab + P.n_pad / 16 + 16;
        h.wf = h.rhs_g + P.m_pad;
        h.gpos = P.rowperm ? h.wf + P.RW : nullptr;
        h.gmin16 = h.wf + P.RW + P.n_pad;
        h.gcol16 = h.gmin16 + P.n_pad / 16 + 17;
        h.scratch = P.scratch + (size_t)tgt * 2 * P.n_pad * TRI_BLOCK;
        h.sh = P.share + tgt;
        h.role = 2;
        h.seq = s_tseq;
        const Op op = ops[s_top];
        const bool sub = (op.kind == OP_GEMM_SUB || op.kind == OP_GEMM_SUB_ABI);
        const int a_src = op.kind == OP_GEMM_SET ? 1 : (op.kind == OP_GEMM_SUB_ABI ? 2 : 0);
        const int b_src = op.kind == OP_GEMM_SET_Q ? 1 : (op.kind == OP_GEMM_SET_R ? 2 : 0);
        const int N = op.dyn ? min(op.Ndim, h.rhs_tab[op.dyn >> 4]) : op.Ndim;
        const int tri = op.kind == OP_GEMM_SET ? (op.ar < P.n_pad ? 1 : 3)
                        : (op.kind == OP_GEMM_SET_R ? 2 : 0);
        gemm(h, sub, a_src, op.ar, op.ac, b_src, op.br, op.bc, op.cr, op.cc, op.Mdim, N, op.Kdim,
             op.kmode, tri);
        c.pipe = h.pipe;
        c.gpipe = h.gpipe;
      }
      __syncthreads();
    }
    if (prof && threadIdx.x == 0) prof[26] += clock64() - th;
  }
}

// ---------------------------------------------------------------------------
// Host-side program builder: the recursion of the blocked algorithm, unrolled.
// ---------------------------------------------------------------------------

// Left part of a recursive split: multiples of TN (128) above 256 columns so the
// big GEMMs see tile-aligned N/M extents (p=16: tile utilisation 0.85 -> 0.91),
// multiples of 16 (the TMA/K-chunk granule) below.
// Tuning knobs (diagnostics): HPS_SPLIT_ALIGN (default TN), HPS_SPLIT_PCT (left
// part in percent of w, default 50).
static int g_split_align = TN, g_split_pct = 50;
int split16_host(int w) {
  const int A = g_split_align;
  const int half = (int)((long long)w * g_split_pct / 100);
  if (w > 2 * A) {
    const int h = half / A * A;
    return h < A ? A : (h >= w ? w - A : h);
  }
  const int h = ((half + 15) / 16) * 16;
  return h < 16 ? 16 : (h >= w ? w - 16 : h);
}

struct ProgramBuilder {
  std::vector<Op> ops;
  int n_pad = 0;
  // diagonal blocks are final once factored (later interchanges only touch rows
  // below them), so each block's inverse is computed once and reused by every
  // recursion level that solves against it
  // owner[g] = (r0, h) of the inverse whose rows currently occupy cache rows
  // [16g, 16g + 16); a block is reusable while it still owns all its rows
  std::vector<std::pair<int, int>> owner[2];
  std::vector<int> rowlim;  // equations with a nonzero left of column k (sorted rows), else empty
  bool tilek = false;       // per-tile k offsets in the LU trailing updates (row first-nonzero table)
  bool colk = true;         // ... and the columns' first-nonzero rows of U (kmode 8)
  int small_panel = SMALL_PANEL;  // recursion leaf width (<= 32)
  int rlim(int k) const { return rowlim.empty() ? n_pad : rowlim[k]; }
  void small(int c0, int w) {
    Op o{}; o.kind = OP_SMALL; o.a = c0; o.b = w; o.c = rowlim.empty() ? 0 : rowlim[c0 + w];
    ops.push_back(o);
  }
  void swaps(int j0, int cnt, int lo, int hi) {
    if (hi <= lo || cnt <= 0) return;
    Op o{}; o.kind = OP_SWAP; o.a = j0; o.b = cnt; o.c = lo; o.d = hi; ops.push_back(o);
  }
  void inv(int kind, int r0, int h) { Op o{}; o.kind = kind; o.a = r0; o.b = h; ops.push_back(o); }
  void gemm(int kind, int ar, int ac, int br, int bc, int cr, int cc, int M, int N, int K,
            int dyn = 0, int kmode = -1) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    Op o{}; o.kind = kind; o.ar = ar; o.ac = ac; o.br = br; o.bc = bc; o.cr = cr; o.cc = cc;
    o.Mdim = M; o.Ndim = N; o.Kdim = K; o.dyn = dyn; o.kmode = kmode < 0 ? (dyn ? 1 : 0) : kmode;
    ops.push_back(o);
  }
  // W-trick right solve W U = B on the W-block rows (slot rows n_pad.., M of them),
  // columns [c0, c0+h) of the upper-triangular recursion tree; W is zero left of
  // column cst, so subtrees left of it are skipped and k ranges start there.
  void trsm_right(int c0, int h, int cst, int M) {
    if (c0 + h <= cst) return;
    if (h <= TRI_BLOCK) {
      inv_cached(OP_INV_UPPER, c0, h);
      gemm(OP_GEMM_SET_R, n_pad, c0, n_pad + c0, 0, n_pad, c0, M, h, h, 0, 2);
      return;
    }
    const int h1 = split16_host(h);
    trsm_right(c0, h1, cst, M);
    const int k0 = c0 > cst ? c0 : cst;
    if (c0 + h1 > k0)
      gemm(OP_GEMM_SUB, n_pad, k0, k0, c0 + h1, n_pad, c0 + h1, M, h - h1, c0 + h1 - k0, 0,
           2 | (tilek && colk ? 8 : 0));
    trsm_right(c0 + h1, h - h1, cst, M);
  }
  bool dyn_rhs = false;  // forward solve against the slab-ordered A_ib: clip N by rhs_tab
  void inv_cached(int kind, int r0, int h) {
    std::vector<std::pair<int, int>>& own = owner[kind == OP_INV_UPPER];
    if (own.empty()) own.assign(n_pad / 16 + 1, {-1, -1});
    bool valid = true;
    for (int g = r0 / 16; g < (r0 + h + 15) / 16; ++g) valid = valid && own[g] == std::make_pair(r0, h);
    if (valid) return;
    for (int g = r0 / 16; g < (r0 + h + 15) / 16; ++g) own[g] = {r0, h};
    inv(kind, r0, h);
  }
  // colb: the columns are LU columns (< n_pad), whose U rows start at gcol16 (kmode 8)
  void trsm_lower(int r0, int h, int lo, int hi, bool colb = false) {
    if (hi <= lo) return;
    if (h <= TRI_BLOCK) {
      inv_cached(OP_INV_LOWER, r0, h);
      gemm(OP_GEMM_SET, r0, 0, r0, lo, r0, lo, h, hi - lo, h, dyn_rhs ? r0 + h : 0);
      return;
    }
    const int h1 = split16_host(h);
    trsm_lower(r0, h1, lo, hi, colb);
    // (no prefix clipping: these are pivot rows, whose first nonzero does not
    // follow their position once interchanged; the per-row g table does)
    if (tilek) { Op o{}; o.kind = OP_GMIN16; o.a = r0 + h1; o.b = r0 + h; ops.push_back(o); }
    gemm(OP_GEMM_SUB, r0 + h1, r0, r0, lo, r0 + h1, lo, h - h1, hi - lo, h1, dyn_rhs ? r0 + h1 : 0,
         (dyn_rhs ? 1 : 0) | (tilek ? 4 : 0) | (tilek && colk && colb ? 8 : 0));
    trsm_lower(r0 + h1, h - h1, lo, hi, colb);
  }
  void trsm_upper(int r0, int h, int lo, int hi) {
    if (hi <= lo) return;
    if (h <= TRI_BLOCK) {
      inv_cached(OP_INV_UPPER, r0, h);
      gemm(OP_GEMM_SET, n_pad + r0, 0, r0, lo, r0, lo, h, hi - lo, h);
      return;
    }
    const int h1 = split16_host(h);
    trsm_upper(r0 + h1, h - h1, lo, hi);
    gemm(OP_GEMM_SUB, r0, r0 + h1, r0 + h1, lo, r0, lo, h1, hi - lo, h - h1);
    trsm_upper(r0, h1, lo, hi);
  }
  void lu(int c0, int w, int NR) {
    if (w <= small_panel) { small(c0, w); return; }
    const int h = split16_host(w);
    lu(c0, h, NR);
    swaps(c0, h, c0 + h, c0 + w);
    trsm_lower(c0, h, c0 + h, c0 + w, true);
    // trailing update: only rows with a nonzero left of column c0 + h (sorted equations),
    // each row tile from the first nonzero column of its rows
    const int r_end = std::min(NR, rlim(c0 + h));
    if (tilek && r_end > c0 + h) {
      Op o{}; o.kind = OP_GMIN16; o.a = c0 + h; o.b = r_end; ops.push_back(o);
    }
    gemm(OP_GEMM_SUB, c0 + h, c0, c0, c0 + h, c0 + h, c0 + h, r_end - c0 - h, w - h, h, 0,
         tilek ? (colk ? 12 : 4) : 0);
    lu(c0 + h, w - h, NR);
    swaps(c0 + h, w - h, c0, c0 + h);
  }
};

// Matrix-free collocation rows: w = A_rows(coeffs) [u_int ; u_b] per leaf
// (the explicit half of a Crank-Nicolson step, reference problems.py:473-505:
// explicit_rows @ full with the leaf's interior + boundary values scattered into
// the p^d grid, corner/edge nodes zero).  Warp per interior row.
__global__ void __launch_bounds__(256) hps_apply_kernel(LeafParams P) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int npat = pattern_size(P);
  for (long long item = gw; item < (long long)P.n_leaves * P.n; item += nw) {
    const int leaf = (int)(item / P.n), r = (int)(item - (long long)leaf * P.n);
    const double* cf = P.coeffs + (size_t)leaf * P.ncoef * P.n;
    const double* ui = P.in0 + (size_t)leaf * P.n;
    const double* ub = P.in1 + (size_t)leaf * P.m;
    int I[3];
    interior_multi(P, r, I);
    const RowCoef rc = row_coef(P, cf, r);
    const double* D1s = P.D1;
    const double* D2s = P.D2;
    double acc = 0.0;
    for (int e = lane; e < npat; e += 32) {
      int J[3];
      if (!pattern_item(P, I, e, J)) continue;
      double x;
      if (is_interior(P, J)) {
        int flat = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (k < P.d) flat = flat * P.q + (J[k] - 1);
        x = ui[flat];
      } else {
        int a = 0, nd = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (k < P.d && J[k] != I[k]) { a = k; ++nd; }
        if (nd != 1) continue;  // corner / edge nodes carry no value in drop mode
        x = ub[boundary_index(P, a, pick3(J, a) == P.p - 1 ? 1 : 0, I)];
      }
      acc += op_entry(P, rc, D1s, D2s, I, J) * x;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) P.out0[(size_t)leaf * P.n + r] = acc;
  }
}

// ---------------------------------------------------------------------------
// Host side: plan + C ABI
// ---------------------------------------------------------------------------

thread_local std::string g_last_error;

int fail(const std::string& msg) {
  g_last_error = msg;
  return -1;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t _e = (call);                                                          \
    if (_e != cudaSuccess) return fail(std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

}  // namespace

struct hps_plan_s {
  int device = 0;
  int d = 0, p = 0, q = 0, n = 0, m = 0, n_pad = 0, m_pad = 0, wb = 8;
  int has_first = 0, has_zeroth = 0, ncoef = 0;
  int legendre = 0, has_cross = 0, nb = 0, nb_pad = 0;
  double *Q = nullptr, *a_bi_pad = nullptr;  // legendre: [nb_pad][m_pad], [m_pad][n_pad]
  int* bpos = nullptr;                        // legendre: [p^d]
  int sms = 0, slots = 0;
  size_t budget = 0;
  double *D1 = nullptr, *D2 = nullptr, *a_bi = nullptr, *a_bb = nullptr;
  // workspace (sized for the largest mode requested so far)
  double* work = nullptr;
  size_t work_doubles = 0;
  int* piv = nullptr;
  int colperm[N_MODES] = {};
  int rowperm[N_MODES] = {};
  double* scratch = nullptr;
  int ws_slots = 0;
  // unrolled LU programs per mode (device copies)
  Op* prog[N_MODES] = {};
  int prog_len[N_MODES] = {};
  double* h_stage = nullptr;
  unsigned long long* prof = nullptr;  // diagnostics counters (device), optional
  int* leaf_counter = nullptr;  // [0] next leaf, [32] CTAs without a leaf (endgame sharing)
  // DtN drop-mode orderings (device copies; host copies for the program builder)
  int *rowpos = nullptr, *colpos = nullptr, *colnat = nullptr, *fsort = nullptr, *eqpos = nullptr;
  std::vector<int> h_rowlim;  // [n_pad + 1]: equations with a nonzero left of column k
  std::vector<int> h_gsorted;  // [n_pad]: first nonzero column of the equation in row p
  int* gsorted = nullptr;
  std::vector<int> h_fsort;  // first nonzero slot row of each slot column's line, non-decreasing
  int wt = 0, RW = 0;        // W-trick DtN (drop mode) and its boundary-row block
  ShareSlot* share = nullptr;
  int share_cap = 0;
  // streamed host-buffer DtN: device copies of all inputs / outputs (grow-only)
  double* s_coef = nullptr;
  double* s_out = nullptr;
  double* s_stats = nullptr;
  int* s_done = nullptr;
  size_t s_leaves = 0;
  TmaMaps maps[N_MODES];
  int maps_ok[N_MODES] = {};
  // completion of the plan's last launch: every launch waits on it first, so
  // launches on different streams (device calls on torch's stream, the host-buffer
  // path's own streams) never overlap on the shared slot workspace and counters
  cudaEvent_t last = nullptr;
  bool last_recorded = false;
};

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

#ifndef HPS_L2_PROMO
#define HPS_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
static int make_map(CUtensorMap* map, double* base, uint64_t cols, uint64_t rows, uint64_t slots,
                    uint64_t ld, uint64_t slot_stride, uint32_t box_cols, uint32_t box_rows,
                    bool swizzle128 = false) {
  auto fn = encode_fn();
  if (!fn) return fail("cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[3] = {cols, rows, slots};
  cuuint64_t strides[2] = {ld * 8, slot_stride * 8};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  HPS_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return 0;
}

static int round16(int x) { return (x + 15) / 16 * 16; }

static void mode_dims(const hps_plan_s* P, int mode, int* NR, int* NC) {
  if (mode == MODE_DTN || mode == MODE_SOLOP || mode == MODE_FACTORS) {
    *NR = P->n_pad;
    *NC = P->n_pad + P->m_pad + (P->legendre ? P->nb_pad : 0);
  } else {
    *NR = P->n_pad;
    *NC = P->n_pad + RHS_COLS;
  }
}

// Rows allocated per slot: the LU rows, or more when the legendre T region
// (m_pad rows) does not fit below them.
static int rows_alloc(const hps_plan_s* P, int mode) {
  int NR, NC;
  mode_dims(P, mode, &NR, &NC);
  if (P->legendre && (mode == MODE_DTN || mode == MODE_FACTORS) && P->m_pad > NR) return P->m_pad;
  if (!P->legendre && mode == MODE_DTN && P->wt) return NR + P->RW;  // W-block rows
  return NR;
}

static size_t slot_doubles(const hps_plan_s* P, int mode) {
  int NR, NC;
  mode_dims(P, mode, &NR, &NC);
  return (size_t)rows_alloc(P, mode) * NC;
}

static int piv_stride(const hps_plan_s* P) {
  return P->n_pad + P->n_pad / 16 + 16 + P->m_pad + P->RW + P->n_pad + 2 * (P->n_pad / 16 + 16) + 1;
}

static int ensure_workspace(hps_plan_s* P, int mode, int want_slots) {
  const size_t per = slot_doubles(P, mode);
  size_t slot_bytes = per * 8 + (size_t)piv_stride(P) * 4 + (size_t)2 * P->n_pad * TRI_BLOCK * 8;
  int slots = want_slots;
  if (P->budget > 0) {
    const size_t fit = P->budget / slot_bytes;
    if (fit < 1) return fail("memory budget cannot hold one leaf workspace");
    if ((size_t)slots > fit) slots = (int)fit;
  }
  {
    // never claim more than ~85% of the currently free device memory (large p:
    // a p = 22 slot is ~0.7 GB); memory already held by this plan counts as free
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      free_b += P->work_doubles * 8;
      const size_t fit = free_b / 100 * 85 / slot_bytes;
      if (fit < 1) return fail("device memory cannot hold one leaf workspace");
      if ((size_t)slots > fit) slots = (int)fit;
    }
  }
  if (P->work && P->work_doubles >= per * (size_t)slots && P->ws_slots >= slots) {
    if (!P->maps_ok[mode]) {
      int NR, NC;
      mode_dims(P, mode, &NR, &NC);
      NR = rows_alloc(P, mode);
      TmaMaps& m = P->maps[mode];
      if (make_map(&m.a_work, P->work, NC, NR, P->ws_slots, NC, per, A_STRIDE, TM, !A_PAD) ||
          make_map(&m.b_work, P->work, NC, NR, P->ws_slots, NC, per, B_STRIDE, KC) ||
          make_map(&m.a_scratch, P->scratch, TRI_BLOCK, 2 * P->n_pad, P->ws_slots, TRI_BLOCK,
                   (size_t)2 * P->n_pad * TRI_BLOCK, A_STRIDE, TM, !A_PAD) ||
          make_map(&m.c_red, P->work, NC, NR, P->ws_slots, NC, per, 16, 8) ||
          make_map(&m.b_scratch, P->scratch, TRI_BLOCK, 2 * P->n_pad, P->ws_slots, TRI_BLOCK,
                   (size_t)2 * P->n_pad * TRI_BLOCK, B_STRIDE, KC) ||
          make_map(&m.a_work_t, P->work, NC, NR, P->ws_slots, NC, per, GemmTall::AS, GemmTall::TM_) ||
          make_map(&m.b_scratch_t, P->scratch, TRI_BLOCK, 2 * P->n_pad, P->ws_slots, TRI_BLOCK,
                   (size_t)2 * P->n_pad * TRI_BLOCK, GemmTall::BS, GemmTall::KC_) ||
          make_map(&m.a_work_n, P->work, NC, NR, P->ws_slots, NC, per, GemmNarrow::AS,
                   GemmNarrow::TM_) ||
          make_map(&m.b_work_n, P->work, NC, NR, P->ws_slots, NC, per, GemmNarrow::BS,
                   GemmNarrow::KC_) ||
          make_map(&m.a_work_h, P->work, NC, NR, P->ws_slots, NC, per, GemmHalf::AS, GemmHalf::TM_) ||
          make_map(&m.b_work_h, P->work, NC, NR, P->ws_slots, NC, per, GemmHalf::BS, GemmHalf::KC_) ||
          make_map(&m.a_scratch_h, P->scratch, TRI_BLOCK, 2 * P->n_pad, P->ws_slots, TRI_BLOCK,
                   (size_t)2 * P->n_pad * TRI_BLOCK, GemmHalf::AS, GemmHalf::TM_) ||
          make_map(&m.b_scratch_h, P->scratch, TRI_BLOCK, 2 * P->n_pad, P->ws_slots, TRI_BLOCK,
                   (size_t)2 * P->n_pad * TRI_BLOCK, GemmHalf::BS, GemmHalf::KC_) ||
          make_map(&m.a_work_s, P->work, NC, NR, P->ws_slots, NC, per, A_STRIDE, 8, !A_PAD) ||
          make_map(&m.a_scratch_s, P->scratch, TRI_BLOCK, 2 * P->n_pad, P->ws_slots, TRI_BLOCK,
                   (size_t)2 * P->n_pad * TRI_BLOCK, A_STRIDE, 8, !A_PAD) ||
          make_map(&m.b_work_s, P->work, NC, NR, P->ws_slots, NC, per, B_STRIDE, 4) ||
          make_map(&m.b_scratch_s, P->scratch, TRI_BLOCK, 2 * P->n_pad, P->ws_slots, TRI_BLOCK,
                   (size_t)2 * P->n_pad * TRI_BLOCK, B_STRIDE, 4))
        return -1;
      if (P->legendre &&
          (make_map(&m.a_abi, P->a_bi_pad, P->n_pad, P->m_pad, 1, P->n_pad,
                    (size_t)P->m_pad * P->n_pad, A_STRIDE, TM, !A_PAD) ||
           make_map(&m.b_q, P->Q, P->m_pad, P->nb_pad, 1, P->m_pad, (size_t)P->nb_pad * P->m_pad,
                    B_STRIDE, KC)))
        return -1;
      P->maps_ok[mode] = 1;
    }
    return slots;
  }
  if (P->work) cudaFree(P->work);
  if (P->piv) cudaFree(P->piv);
  if (P->scratch) cudaFree(P->scratch);
  P->work = nullptr; P->piv = nullptr; P->scratch = nullptr;
  CK(cudaMalloc(&P->work, per * (size_t)slots * 8));
  CK(cudaMalloc(&P->piv, (size_t)piv_stride(P) * slots * 4));
  CK(cudaMalloc(&P->scratch, (size_t)2 * P->n_pad * TRI_BLOCK * slots * 8));
  P->work_doubles = per * (size_t)slots;
  P->ws_slots = slots;
  for (int k = 0; k < N_MODES; ++k) P->maps_ok[k] = 0;
  return ensure_workspace(P, mode, want_slots);
}

static int ensure_program(hps_plan_s* P, int mode) {
  if (P->prog[mode]) return 0;
  int NR, NC;
  mode_dims(P, mode, &NR, &NC);
  ProgramBuilder b;
  b.n_pad = P->n_pad;
  // working columns: [A_ii | A_ib or rhs]; legendre adds an R_b / T region after them
  const bool leg_op = P->legendre && (mode == MODE_DTN || mode == MODE_SOLOP || mode == MODE_FACTORS);
  const int NW = leg_op ? P->n_pad + P->m_pad : NC;
  const int col_rb = P->n_pad + P->m_pad;
  if (leg_op)  // A_ib = R_b Q
    b.gemm(OP_GEMM_SET_Q, 0, col_rb, 0, 0, 0, P->n_pad, P->n_pad, P->m_pad, P->nb_pad);
  const char* dbg = getenv("HPS_DEBUG");
  P->colperm[mode] = (mode == MODE_DTN && !P->legendre && !(dbg && (atoi(dbg) & 4))) ? 1 : 0;
  // interior order with the LU's zero skipping: every drop-mode program (the
  // solve modes keep natural rhs / output order through the tables)
  P->rowperm[mode] = (!P->legendre && !(dbg && (atoi(dbg) & 4))) ? 1 : 0;
  if (P->rowperm[mode] && !(dbg && (atoi(dbg) & 256))) b.tilek = true;
  if (dbg && (atoi(dbg) & 512)) b.colk = false;
  if (const char* sp = getenv("HPS_SMALL_PANEL")) b.small_panel = std::max(16, std::min(32, atoi(sp)));
  if (const char* sa = getenv("HPS_SPLIT_ALIGN")) g_split_align = std::max(16, atoi(sa) / 16 * 16);
  if (const char* sp = getenv("HPS_SPLIT_PCT")) g_split_pct = std::max(20, std::min(80, atoi(sp)));
  b.lu(0, P->n_pad, NR);
  if (P->colperm[mode]) {
    Op o{};
    o.kind = OP_RHS_PROFILE;
    b.ops.push_back(o);
    b.dyn_rhs = true;
  }
  b.swaps(0, P->n_pad, P->n_pad, NW);
  b.trsm_lower(0, P->n_pad, P->n_pad, NW);
  b.dyn_rhs = false;
  const bool use_wt = mode == MODE_DTN && !P->legendre && P->wt && P->colperm[mode];
  if (use_wt) {
    // T = A_bb - W Y by blocks of RW sorted boundary DOFs (no backward solve)
    for (int s0 = 0; s0 < P->m; s0 += P->RW) {
      const int R = (P->m - s0 < P->RW) ? P->m - s0 : P->RW;
      const int cst = P->h_fsort[s0] / 16 * 16;
      Op o{};
      o.kind = OP_WBLOCK_INIT; o.a = s0; o.b = R; o.c = cst;
      b.ops.push_back(o);
      b.trsm_right(0, P->n_pad, cst, R);
      b.gemm(OP_GEMM_SUB, P->n_pad, cst, cst, P->n_pad, P->n_pad, P->n_pad, R, P->m, P->n_pad - cst, 0, 3);
      Op w{};
      w.kind = OP_WBLOCK_OUT; w.a = s0; w.b = R;
      b.ops.push_back(w);
    }
  } else {
    b.trsm_upper(0, P->n_pad, P->n_pad, NW);
  }
  if (leg_op && (mode == MODE_DTN || mode == MODE_FACTORS)) {  // T = a_bb - a_bi X in the (now free) R_b region
    Op o{};
    o.kind = OP_COPY_ABB;
    o.a = col_rb;
    b.ops.push_back(o);
    b.gemm(OP_GEMM_SUB_ABI, 0, 0, 0, P->n_pad, 0, col_rb, P->m_pad, P->m_pad, P->n_pad);
  }
  if (dbg && (atoi(dbg) & 128)) {  // diagnostics: op histogram of the program
    int hist[16] = {0};
    for (const Op& o : b.ops) hist[o.kind & 15]++;
    fprintf(stderr, "hps program mode %d: %zu ops:", mode, b.ops.size());
    for (int k = 0; k < 16; ++k)
      if (hist[k]) fprintf(stderr, " k%d=%d", k, hist[k]);
    fprintf(stderr, "\n");
  }
  CK(cudaMalloc(&P->prog[mode], b.ops.size() * sizeof(Op)));
  CK(cudaMemcpy(P->prog[mode], b.ops.data(), b.ops.size() * sizeof(Op), cudaMemcpyHostToDevice));
  P->prog_len[mode] = (int)b.ops.size();
  return 0;
}

static int launch(hps_plan_s* P, int mode, int n_leaves, const double* coeffs, const double* in0,
                  const double* in1, double* out0, double* out1, double* stats, cudaStream_t stream,
                  int* done_counts = nullptr, int done_chunk = 1) {
  if (n_leaves <= 0) return 0;
  CK(cudaSetDevice(P->device));
  if (ensure_program(P, mode) != 0) return -1;
  int want = P->slots;
  {
    const char* dbg = getenv("HPS_DEBUG");
    if (dbg && (atoi(dbg) & 8) && want > P->sms) want = P->sms;  // diagnostics: one CTA per SM
  }
  if (want > n_leaves) want = n_leaves;
  // dynamic shared memory: the largest of the GEMM stages, the panel and the inverses
  const int panel_bytes = ((P->n_pad * P->wb > 1024 ? P->n_pad * P->wb : 1024) + 32 * P->wb) * 8;
  int smem = GEMM_SMEM_BYTES;
  if (panel_bytes > smem) smem = panel_bytes;
  if ((2 * TRI_BLOCK * TRI_LD + 32 * TRI_BLOCK / 2) * 8 > smem) smem = (2 * TRI_BLOCK * TRI_LD + 32 * TRI_BLOCK / 2) * 8;
  CK(cudaFuncSetAttribute(hps_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(hps_leaf_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  {
    // the grid is persistent and CTAs wait on each other (endgame sharing): every
    // CTA must be resident at once, so never launch more than the occupancy allows
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hps_leaf_kernel, NT, smem));
    if (occ < 1) return fail("hps_leaf_kernel does not fit on an SM");
    if (want > occ * P->sms) want = occ * P->sms;
  }
  // ordered after the plan's previous launch, whatever stream that was on
  if (P->last_recorded) CK(cudaStreamWaitEvent(stream, P->last, 0));
  const int slots = ensure_workspace(P, mode, want);
  if (slots < 0) return -1;
  LeafParams L;
  memset(&L, 0, sizeof(L));
  L.mode = mode;
  L.d = P->d; L.p = P->p; L.q = P->q; L.n = P->n; L.m = P->m;
  L.n_pad = P->n_pad; L.m_pad = P->m_pad;
  mode_dims(P, mode, &L.NR, &L.NC);
  L.ld = L.NC;
  L.wb = P->wb;
  L.has_first = P->has_first; L.has_zeroth = P->has_zeroth; L.ncoef = P->ncoef;
  L.legendre = P->legendre; L.has_cross = P->has_cross; L.nb = P->nb;
  L.col_rb = P->n_pad + P->m_pad; L.Q = P->Q; L.bpos = P->bpos;
  L.n_leaves = n_leaves;
  L.slot_stride = slot_doubles(P, mode);
  L.work = P->work; L.piv = P->piv; L.scratch = P->scratch;
  L.piv_stride = piv_stride(P);
  L.colperm = P->colperm[mode];
  L.rowperm = P->rowperm[mode];
  L.rowpos = P->rowpos;
  L.colpos = P->colpos;
  L.colnat = P->colnat;
  L.eqpos = P->eqpos;
  L.gsorted = P->gsorted;
  L.pivot_tau = HPS_PIVOT_TAU;
  if (const char* t = getenv("HPS_PIVOT_TAU")) L.pivot_tau = atof(t);
  L.fsort = P->fsort;
  L.wt = (mode == MODE_DTN && !P->legendre && P->wt && P->colperm[mode]) ? 1 : 0;
  L.RW = P->RW;
  L.D1 = P->D1; L.D2 = P->D2; L.a_bi = P->a_bi; L.a_bb = P->a_bb;
  L.prof = P->prof;
  L.leaf_counter = P->leaf_counter;
  L.share_finished = P->leaf_counter + 32;
  L.done_counts = done_counts;
  L.done_chunk = done_chunk;
  CK(cudaMemsetAsync(P->leaf_counter, 0, 64 * sizeof(int), stream));
  {
    // Endgame GEMM sharing is opt-in (HPS_SHARE=1): repeated runs at p = 20 with it on
    // changed ~1 leaf in 5000 (profiles/r02c_determinism_p20.jsonl), never with it off
    const char* dbg = getenv("HPS_DEBUG");
    const char* shr = getenv("HPS_SHARE");
    const bool share_off = (dbg && (atoi(dbg) & 16)) || !(shr && atoi(shr) == 1);
    if (!share_off) {
      if (P->share_cap < slots) {
        cudaFree(P->share);
        P->share = nullptr;
        P->share_cap = 0;
        CK(cudaMalloc(&P->share, sizeof(ShareSlot) * (size_t)slots));
        P->share_cap = slots;
      }
      CK(cudaMemsetAsync(P->share, 0, sizeof(ShareSlot) * (size_t)slots, stream));
      L.share = P->share;
    }
  }
  L.coeffs = coeffs; L.in0 = in0; L.in1 = in1; L.out0 = out0; L.out1 = out1; L.stats = stats;
  L.smem_doubles = smem / 8;
  if (const char* dbg = getenv("HPS_DEBUG")) L.debug = atoi(dbg);
  hps_leaf_kernel<<<slots, NT, smem, stream>>>(L, P->prog[mode], P->prog_len[mode], P->maps[mode]);
  CK(cudaGetLastError());
  CK(cudaEventRecord(P->last, stream));
  P->last_recorded = true;
  return 0;
}

// Free the slot workspace and the streaming buffers (they are re-allocated by
// the next launch); templates, orderings and op programs stay.
static void release_workspace(hps_plan_s* P) {
  if (P->last_recorded) cudaEventSynchronize(P->last);
  cudaFree(P->work); cudaFree(P->piv); cudaFree(P->scratch);
  P->work = nullptr; P->piv = nullptr; P->scratch = nullptr;
  P->work_doubles = 0; P->ws_slots = 0;
  for (int k = 0; k < N_MODES; ++k) P->maps_ok[k] = 0;
  cudaFree(P->share); P->share = nullptr; P->share_cap = 0;
  cudaFree(P->s_coef); cudaFree(P->s_out); cudaFree(P->s_stats); cudaFree(P->s_done);
  P->s_coef = nullptr; P->s_out = nullptr; P->s_stats = nullptr; P->s_done = nullptr;
  P->s_leaves = 0;
}


// ---------------------------------------------------------------------------
// Interface assembly on the device: scatter-add of the leaves' DtN blocks into
// the CSR values of T (and of the Dirichlet coupling C), reference
// condensation.py:230-246.  T is block sparse at face granularity — every face
// is a contiguous id range and a leaf's boundary concatenates its faces — so a
// job is one (row face, column face) block of one leaf: nr x nc doubles read
// row by row from the DtN map and added to out[base + a * stride + b].  Each
// entry of T has at most two contributors (the two leaves of a face), and
// 0 + x + y == 0 + y + x in IEEE arithmetic, so the atomics give the host
// COO -> CSR sum bit for bit.  HBM-bound: 8 bytes read + one 8-byte atomic
// per element; warps walk rows, lanes walk columns (coalesced both sides).
__global__ void __launch_bounds__(256) hps_interface_scatter_kernel(
    const double* __restrict__ blocks, long long ld, long long block_stride, long long leaf0,
    const long long* __restrict__ jobs, double* __restrict__ out0, double* __restrict__ out1) {
  const long long* j = jobs + 8 * (long long)blockIdx.x;
  const long long leaf = j[0] - leaf0, r0 = j[1], c0 = j[2];
  const int nr = (int)j[3], nc = (int)j[4];
  double* out = (j[5] ? out1 : out0) + j[6];
  const long long stride = j[7];
  const double* src = blocks + leaf * block_stride + r0 * ld + c0;
  // flattened over the block so that narrow faces (nc < 32 at low p) keep
  // every lane busy; consecutive threads stay on consecutive columns
  const int total = nr * nc;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int a = e / nc, b = e - a * nc;
    atomicAdd(out + a * stride + b, __ldg(src + a * ld + b));
  }
}

extern "C" {

const char* hps_last_error(void) { return g_last_error.c_str(); }

int hps_abi_version(void) { return HPS_ABI_VERSION; }

int hps_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

// Orderings for the DtN drop mode.  Interior nodes: growing cubes from a leaf
// corner (key max_k I_k, then the natural index) — the lines of every face
// family start late in this order, so the forward solve's zero prefixes are
// long (sum (n - f)^2 = 0.463 n^2 m at p = 16 vs 0.545 for the natural order).
// A_ib columns: sorted by the first slot row f of their line (stable), so the
// columns with a nonzero above any row form a prefix.  HPS_DEBUG & 32 keeps
// the natural interior order (columns still sorted).
static int build_orderings(hps_plan_s* P) {
  const int q = P->q, d = P->d, n = P->n, m = P->m;
  const char* dbg = getenv("HPS_DEBUG");
  const bool natural = dbg && (atoi(dbg) & 32);
  std::vector<int> rowpos(n), colpos(m), colnat(m);
  std::vector<int> shell(n);
  auto coords = [&](int v, int* I) {
    I[0] = I[1] = I[2] = 0;
    for (int k = d - 1; k >= 0; --k) { I[k] = v % q; v /= q; }
  };
  // g[v]: first slot position among the nodes on v's d grid lines (v's row's
  // first structural nonzero, and v's column's first nonzero row)
  auto first_nonzero = [&](const std::vector<int>& pos, std::vector<int>& g) {
    for (int v = 0; v < n; ++v) {
      int I[3];
      coords(v, I);
      int mn = pos[v];
      for (int a = 0; a < d; ++a) {
        int J[3] = {I[0], I[1], I[2]};
        for (int x = 0; x < q; ++x) {
          J[a] = x;
          int flat = 0;
          for (int k = 0; k < d; ++k) flat = flat * q + J[k];
          mn = std::min(mn, pos[flat]);
        }
      }
      g[v] = mn;
    }
  };
  auto rank_by = [&](auto less, std::vector<int>& pos) {
    std::vector<int> idx(n);
    for (int i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), less);
    for (int r = 0; r < n; ++r) pos[idx[r]] = r;
  };
  for (int v = 0; v < n; ++v) {
    int I[3];
    coords(v, I);
    shell[v] = std::max(I[0], std::max(I[1], d == 3 ? I[2] : 0));
  }
  std::vector<int> g(n);
  if (natural) {
    for (int v = 0; v < n; ++v) rowpos[v] = v;
  } else {
    // growing cubes from a leaf corner (shell = max coordinate) ...
    std::vector<int> corner(n);
    rank_by([&](int a, int b) { return shell[a] != shell[b] ? shell[a] < shell[b] : a < b; }, corner);
    // ... and within a shell by first nonzero, so each 64-row tile of the LU's
    // trailing updates starts its k loop late (per-tile k offsets from g)
    first_nonzero(corner, g);
    rank_by([&](int a, int b) {
      if (shell[a] != shell[b]) return shell[a] < shell[b];
      if (g[a] != g[b]) return g[a] < g[b];
      return a < b;
    }, rowpos);
  }
  first_nonzero(rowpos, g);
  // equations in the same order as the unknowns (diagonal pivots stay in place)
  std::vector<int> eqpos(rowpos);
  P->h_gsorted.assign(P->n_pad, 0);
  for (int v = 0; v < n; ++v) P->h_gsorted[rowpos[v]] = g[v];
  for (int r = n; r < P->n_pad; ++r) P->h_gsorted[r] = r;
  const int fd = (d == 3) ? q * q : q;
  std::vector<int> f(m);
  for (int b = 0; b < m; ++b) {
    const int face = b / fd, t = b - face * fd, a = face >> 1;
    int base, stride;
    if (d == 3) {
      if (a == 0) { base = t; stride = q * q; }
      else if (a == 1) { base = (t / q) * q * q + t % q; stride = q; }
      else { base = t * q; stride = 1; }
    } else {
      if (a == 0) { base = t; stride = q; }
      else { base = t * q; stride = 1; }
    }
    int mn = n;
    for (int k = 0; k < q; ++k) mn = std::min(mn, rowpos[base + k * stride]);
    f[b] = mn;
  }
  for (int b = 0; b < m; ++b) colnat[b] = b;
  std::stable_sort(colnat.begin(), colnat.end(), [&](int a, int b) { return f[a] < f[b]; });
  P->h_fsort.assign(P->m_pad, 0x7fffffff);
  for (int sc = 0; sc < m; ++sc) { colpos[colnat[sc]] = sc; P->h_fsort[sc] = f[colnat[sc]]; }
  if (cudaMalloc(&P->rowpos, (size_t)n * 4) != cudaSuccess ||
      cudaMalloc(&P->colpos, (size_t)m * 4) != cudaSuccess ||
      cudaMalloc(&P->colnat, (size_t)m * 4) != cudaSuccess ||
      cudaMalloc(&P->fsort, (size_t)P->m_pad * 4) != cudaSuccess)
    return fail("device allocation of orderings failed");
  cudaMemcpy(P->fsort, P->h_fsort.data(), (size_t)P->m_pad * 4, cudaMemcpyHostToDevice);
  if (cudaMalloc(&P->eqpos, (size_t)n * 4) != cudaSuccess ||
      cudaMalloc(&P->gsorted, (size_t)P->n_pad * 4) != cudaSuccess)
    return fail("device allocation of orderings failed");
  cudaMemcpy(P->eqpos, eqpos.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(P->gsorted, P->h_gsorted.data(), (size_t)P->n_pad * 4, cudaMemcpyHostToDevice);
  // W blocks pay off from p ~ 15 on (small leaves: the per-block op overheads dominate)
  // W-block Schur complement from n_pad >= HPS_WT_MIN_N (default 1536: p >= 14; p = 14
  // +2.3% with it, p = 12 -6%, p = 10 -11%: profiles/r02c_variant_sweep.jsonl); below it
  // the backward solve and the line-sparse output phase are faster
  const char* wte = getenv("HPS_WT_MIN_N");
  const int wt_min = wte ? atoi(wte) : 1536;
  P->wt = (dbg && (atoi(dbg) & 64)) ? 0 : (P->n_pad >= wt_min ? 1 : 0);
  {
    // boundary rows per W block (HPS_RW_ROWS overrides the compile-time default, for tuning)
    const char* rwe = getenv("HPS_RW_ROWS");
    const int rw = rwe ? std::max(16, atoi(rwe) / 16 * 16) : HPS_RW;
    P->RW = P->m_pad < rw ? P->m_pad : rw;
  }
  cudaMemcpy(P->rowpos, rowpos.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(P->colpos, colpos.data(), (size_t)m * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(P->colnat, colnat.data(), (size_t)m * 4, cudaMemcpyHostToDevice);
  return 0;
}

static int plan_create(hps_plan_t* out, int device, int dim, int p, int legendre, int has_cross,
                       int has_first, int has_zeroth, const double* D1, const double* D2,
                       const double* a_bi, const double* a_bb, const double* Q, int n_bnd,
                       const int* bpos, int max_slots, size_t workspace_budget_bytes) {
  if (!out) return fail("null plan pointer");
  *out = nullptr;
  if (dim != 2 && dim != 3) return fail("dimension must be 2 or 3");
  if (p < 4) return fail("p must be >= 4");
  if (has_cross && !legendre) return fail("cross terms require legendre face grids");
  hps_plan_s* P = new hps_plan_s();
  P->device = device;
  P->d = dim; P->p = p; P->q = p - 2;
  P->legendre = legendre ? 1 : 0;
  P->has_cross = has_cross ? 1 : 0;
  P->n = 1; for (int k = 0; k < dim; ++k) P->n *= P->q;
  const int fq = legendre ? p - 1 : p - 2;
  const int fd = (dim == 3) ? fq * fq : fq;
  P->m = 2 * dim * fd;
  P->n_pad = round16(P->n);
  P->m_pad = round16(P->m);
  P->nb = legendre ? n_bnd : 0;
  P->nb_pad = legendre ? round16(n_bnd) : 0;
  if (legendre && P->nb_pad < P->m_pad) P->nb_pad = P->m_pad;  // region also hosts T
  P->has_first = has_first ? 1 : 0;
  P->has_zeroth = has_zeroth ? 1 : 0;
  P->ncoef = dim + (has_cross ? dim * (dim - 1) / 2 : 0) + (has_first ? dim : 0) + (has_zeroth ? 1 : 0);
  int wb = 8;
  while (wb > 1 && ((size_t)P->n_pad * wb + 32 * wb) * 8 > PANEL_SMEM_CAP) wb >>= 1;
  // (the panel step also needs max(n_pad*wb, 1024) + 32*wb doubles; 1024 + 256 always fits)
  P->wb = wb;
  P->budget = workspace_budget_bytes;
  if (cudaSetDevice(device) != cudaSuccess) { delete P; return fail("cudaSetDevice failed"); }
  if (cudaEventCreateWithFlags(&P->last, cudaEventDisableTiming) != cudaSuccess) {
    delete P;
    return fail("cudaEventCreate failed");
  }
  cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, device);
  P->slots = (max_slots > 0 && max_slots < CTAS_PER_SM * P->sms) ? max_slots : CTAS_PER_SM * P->sms;
  const size_t tab = (size_t)dim * p * p * 8;
  if (cudaMalloc(&P->D1, tab) != cudaSuccess || cudaMalloc(&P->D2, tab) != cudaSuccess ||
      cudaMalloc(&P->a_bi, (size_t)P->m * P->n * 8) != cudaSuccess ||
      cudaMalloc(&P->a_bb, (size_t)P->m * P->m * 8) != cudaSuccess ||
      cudaMalloc(&P->leaf_counter, 64 * sizeof(int)) != cudaSuccess) {
    hps_plan_destroy(P);
    return fail("device allocation of templates failed");
  }
  cudaMemcpy(P->D1, D1, tab, cudaMemcpyHostToDevice);
  cudaMemcpy(P->D2, D2, tab, cudaMemcpyHostToDevice);
  cudaMemcpy(P->a_bi, a_bi, (size_t)P->m * P->n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(P->a_bb, a_bb, (size_t)P->m * P->m * 8, cudaMemcpyHostToDevice);
  if (legendre) {
    // zero-padded copies for the TMA-fed GEMMs: Q [nb_pad][m_pad], a_bi [m_pad][n_pad]
    std::vector<double> qp((size_t)P->nb_pad * P->m_pad, 0.0), ap((size_t)P->m_pad * P->n_pad, 0.0);
    for (int g = 0; g < n_bnd; ++g)
      for (int c = 0; c < P->m; ++c) qp[(size_t)g * P->m_pad + c] = Q[(size_t)g * P->m + c];
    for (int b = 0; b < P->m; ++b)
      for (int k = 0; k < P->n; ++k) ap[(size_t)b * P->n_pad + k] = a_bi[(size_t)b * P->n + k];
    size_t full = 1;
    for (int k = 0; k < dim; ++k) full *= p;
    if (cudaMalloc(&P->Q, qp.size() * 8) != cudaSuccess ||
        cudaMalloc(&P->a_bi_pad, ap.size() * 8) != cudaSuccess ||
        cudaMalloc(&P->bpos, full * 4) != cudaSuccess) {
      hps_plan_destroy(P);
      return fail("device allocation of legendre templates failed");
    }
    cudaMemcpy(P->Q, qp.data(), qp.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(P->a_bi_pad, ap.data(), ap.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(P->bpos, bpos, full * 4, cudaMemcpyHostToDevice);
  }
  if (!legendre && build_orderings(P) != 0) { hps_plan_destroy(P); return -1; }
  if (cudaGetLastError() != cudaSuccess) { hps_plan_destroy(P); return fail("template upload failed"); }
  *out = P;
  return 0;
}

int hps_plan_create(hps_plan_t* out, int device, int dim, int p, int has_first, int has_zeroth,
                    const double* D1, const double* D2, const double* a_bi, const double* a_bb,
                    int max_slots, size_t workspace_budget_bytes) {
  return plan_create(out, device, dim, p, 0, 0, has_first, has_zeroth, D1, D2, a_bi, a_bb, nullptr,
                     0, nullptr, max_slots, workspace_budget_bytes);
}

int hps_plan_create_legendre(hps_plan_t* out, int device, int dim, int p, int has_cross,
                             int has_first, int has_zeroth, const double* D1, const double* D2,
                             const double* a_bi, const double* a_bb, const double* Q, int n_bnd,
                             const int* bpos, int max_slots, size_t workspace_budget_bytes) {
  if (!Q || !bpos || n_bnd <= 0) return fail("legendre plan needs Q and the boundary position table");
  return plan_create(out, device, dim, p, 1, has_cross, has_first, has_zeroth, D1, D2, a_bi, a_bb, Q,
                     n_bnd, bpos, max_slots, workspace_budget_bytes);
}

int hps_plan_destroy(hps_plan_t P) {
  if (!P) return 0;
  cudaSetDevice(P->device);
  release_workspace(P);
  if (P->last) cudaEventDestroy(P->last);
  cudaFree(P->D1); cudaFree(P->D2); cudaFree(P->a_bi); cudaFree(P->a_bb);
  cudaFree(P->leaf_counter);
  cudaFree(P->share);
  cudaFree(P->rowpos);
  cudaFree(P->colpos);
  cudaFree(P->colnat);
  cudaFree(P->fsort);
  cudaFree(P->eqpos);
  cudaFree(P->gsorted);
  cudaFree(P->s_coef); cudaFree(P->s_out); cudaFree(P->s_stats); cudaFree(P->s_done);
  cudaFree(P->Q); cudaFree(P->a_bi_pad); cudaFree(P->bpos);
  cudaFree(P->work); cudaFree(P->piv); cudaFree(P->scratch);
  for (int k = 0; k < N_MODES; ++k) cudaFree(P->prog[k]);
  if (P->h_stage) cudaFreeHost(P->h_stage);
  delete P;
  return 0;
}

int hps_plan_release(hps_plan_t P) {
  if (!P) return fail("null plan");
  CK(cudaSetDevice(P->device));
  release_workspace(P);
  return 0;
}

int hps_plan_workspace(hps_plan_t P, size_t* bytes, int* slots) {
  if (!P) return fail("null plan");
  const size_t per_slot = (size_t)piv_stride(P) * 4 + (size_t)2 * P->n_pad * TRI_BLOCK * 8;
  if (bytes) *bytes = P->work_doubles * 8 + per_slot * P->ws_slots + sizeof(ShareSlot) * P->share_cap +
                      P->s_leaves * ((size_t)P->ncoef * P->n * 8 + (size_t)P->m * P->m * 8 + 16 + 4);
  if (slots) *slots = P->ws_slots;
  return 0;
}

int hps_plan_set_profile(hps_plan_t P, unsigned long long* counters) {
  if (!P) return fail("null plan");
  P->prof = counters;
  return 0;
}

int hps_plan_info(hps_plan_t P, int* n_interior, int* n_boundary, int* ncoef, int* slots,
                  size_t* dtn_slot_bytes, size_t* solve_slot_bytes) {
  if (!P) return fail("null plan");
  if (n_interior) *n_interior = P->n;
  if (n_boundary) *n_boundary = P->m;
  if (ncoef) *ncoef = P->ncoef;
  if (slots) *slots = P->slots;
  if (dtn_slot_bytes) *dtn_slot_bytes = slot_doubles(P, MODE_DTN) * 8;
  if (solve_slot_bytes) *solve_slot_bytes = slot_doubles(P, MODE_REDUCE) * 8;
  return 0;
}

int hps_leaf_dtn(hps_plan_t P, int n_leaves, const double* coeffs, double* dtn, double* stats,
                 void* stream) {
  if (!P) return fail("null plan");
  return launch(P, MODE_DTN, n_leaves, coeffs, nullptr, nullptr, dtn, nullptr, stats,
                (cudaStream_t)stream);
}

int hps_leaf_factors(hps_plan_t P, int n_leaves, const double* coeffs, double* dtn, double* s,
                     double* stats, void* stream) {
  if (!P) return fail("null plan");
  return launch(P, MODE_FACTORS, n_leaves, coeffs, nullptr, nullptr, dtn, s, stats,
                (cudaStream_t)stream);
}

int hps_leaf_reduce_load(hps_plan_t P, int n_leaves, const double* coeffs, const double* f,
                         double* v, double* flux, double* stats, void* stream) {
  if (!P) return fail("null plan");
  return launch(P, MODE_REDUCE, n_leaves, coeffs, f, nullptr, v, flux, stats, (cudaStream_t)stream);
}

int hps_leaf_solution_operator(hps_plan_t P, int n_leaves, const double* coeffs, double* s,
                               double* stats, void* stream) {
  if (!P) return fail("null plan");
  return launch(P, MODE_SOLOP, n_leaves, coeffs, nullptr, nullptr, s, nullptr, stats,
                (cudaStream_t)stream);
}

int hps_leaf_interior_solve(hps_plan_t P, int n_leaves, const double* coeffs, const double* ub,
                            const double* v, double* u, double* stats, void* stream) {
  if (!P) return fail("null plan");
  return launch(P, MODE_INTERIOR, n_leaves, coeffs, ub, v, u, nullptr, stats, (cudaStream_t)stream);
}

int hps_leaf_apply(hps_plan_t P, int n_leaves, const double* coeffs, const double* u_int,
                   const double* u_b, double* w, void* stream) {
  if (!P) return fail("null plan");
  if (P->legendre) return fail("hps_leaf_apply supports corner-dropping face grids");
  if (n_leaves <= 0) return 0;
  CK(cudaSetDevice(P->device));
  LeafParams L;
  memset(&L, 0, sizeof(L));
  L.d = P->d; L.p = P->p; L.q = P->q; L.n = P->n; L.m = P->m;
  L.has_first = P->has_first; L.has_zeroth = P->has_zeroth; L.ncoef = P->ncoef;
  L.has_cross = 0; L.legendre = 0;
  L.D1 = P->D1; L.D2 = P->D2;
  L.coeffs = coeffs; L.in0 = u_int; L.in1 = u_b; L.out0 = w; L.n_leaves = n_leaves;
  const long long warps = (long long)n_leaves * P->n;
  long long blocks = (warps + 7) / 8;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  hps_apply_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(L);
  CK(cudaGetLastError());
  return 0;
}

static PFN_cuStreamWaitValue32_v11070 wait_value_fn() {
  static PFN_cuStreamWaitValue32_v11070 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
  }
  return fn;
}

// Chunked fallback: chunks of `chunk_leaves` leaves flow H2D (input stream) ->
// kernel (compute stream) -> D2H (output stream), double-buffered.
static int dtn_host_chunked(hps_plan_t P, int n_leaves, const double* coeffs_host, double* dtn_host,
                            double* stats_host, int chunk_leaves) {
  if (chunk_leaves <= 0) chunk_leaves = P->slots * 4;
  if (chunk_leaves > n_leaves) chunk_leaves = n_leaves;
  const size_t cbytes = (size_t)P->ncoef * P->n * 8, tbytes = (size_t)P->m * P->m * 8;
  double *d_coef[2] = {nullptr, nullptr}, *d_dtn[2] = {nullptr, nullptr}, *d_stats[2] = {nullptr, nullptr};
  cudaStream_t s_in, s_comp, s_out;
  cudaEvent_t ev_in[2], ev_done[2], ev_out[2];
  CK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    CK(cudaMalloc(&d_coef[b], cbytes * chunk_leaves));
    CK(cudaMalloc(&d_dtn[b], tbytes * chunk_leaves));
    CK(cudaMalloc(&d_stats[b], 16 * (size_t)chunk_leaves));
    CK(cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_done[b], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming));
  }
  int rc = 0;
  const int nchunks = (n_leaves + chunk_leaves - 1) / chunk_leaves;
  for (int ci = 0; ci < nchunks && rc == 0; ++ci) {
    const int b = ci & 1;
    const int l0 = ci * chunk_leaves;
    const int cnt = (n_leaves - l0 < chunk_leaves) ? (n_leaves - l0) : chunk_leaves;
    if (ci >= 2) cudaStreamWaitEvent(s_in, ev_done[b], 0);
    cudaMemcpyAsync(d_coef[b], coeffs_host + (size_t)l0 * P->ncoef * P->n, cbytes * cnt,
                    cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(ev_in[b], s_in);
    cudaStreamWaitEvent(s_comp, ev_in[b], 0);
    if (ci >= 2) cudaStreamWaitEvent(s_comp, ev_out[b], 0);
    rc = launch(P, MODE_DTN, cnt, d_coef[b], nullptr, nullptr, d_dtn[b], nullptr, d_stats[b], s_comp);
    cudaEventRecord(ev_done[b], s_comp);
    cudaStreamWaitEvent(s_out, ev_done[b], 0);
    cudaMemcpyAsync(dtn_host + (size_t)l0 * P->m * P->m, d_dtn[b], tbytes * cnt,
                    cudaMemcpyDeviceToHost, s_out);
    if (stats_host)
      cudaMemcpyAsync(stats_host + 2 * (size_t)l0, d_stats[b], 16 * (size_t)cnt,
                      cudaMemcpyDeviceToHost, s_out);
    cudaEventRecord(ev_out[b], s_out);
  }
  cudaError_t e0 = cudaStreamSynchronize(s_in);
  cudaError_t e1 = cudaStreamSynchronize(s_comp);
  cudaError_t e2 = cudaStreamSynchronize(s_out);
  for (int b = 0; b < 2; ++b) {
    cudaFree(d_coef[b]); cudaFree(d_dtn[b]); cudaFree(d_stats[b]);
    cudaEventDestroy(ev_in[b]); cudaEventDestroy(ev_done[b]); cudaEventDestroy(ev_out[b]);
  }
  cudaStreamDestroy(s_in);
  cudaStreamDestroy(s_comp);
  cudaStreamDestroy(s_out);
  if (rc != 0) return rc;
  const cudaError_t e = e0 != cudaSuccess ? e0 : (e1 != cudaSuccess ? e1 : e2);
  if (e != cudaSuccess) return fail(std::string("streamed dtn failed: ") + cudaGetErrorString(e));
  return 0;
}

// Host-buffer DtN with the two-level schedule on the device.  Preferred path:
// ONE persistent launch over all leaves (no chunk-boundary tails); the kernel
// counts finished leaves per output chunk in device memory and the D2H stream
// waits on those counters (cuStreamWaitValue32), so each chunk of DtN maps is
// copied to the host while later leaves are still being reduced.  Falls back
// to chunked launches when the outputs do not fit in device memory or stream
// memory operations are unavailable.
int hps_leaf_dtn_host(hps_plan_t P, int n_leaves, const double* coeffs_host, double* dtn_host,
                      double* stats_host, int chunk_leaves) {
  if (!P) return fail("null plan");
  if (n_leaves <= 0) return 0;
  CK(cudaSetDevice(P->device));
  const size_t cbytes = (size_t)P->ncoef * P->n * 8, tbytes = (size_t)P->m * P->m * 8;
  auto wait_fn = wait_value_fn();
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t need = (size_t)n_leaves * (cbytes + tbytes + 16);
  const size_t have = P->s_leaves >= (size_t)n_leaves ? need : 0;
  if (!wait_fn || (have == 0 && need > free_b / 10 * 6))
    return dtn_host_chunked(P, n_leaves, coeffs_host, dtn_host, stats_host, chunk_leaves);
  if (P->s_leaves < (size_t)n_leaves) {
    cudaFree(P->s_coef); cudaFree(P->s_out); cudaFree(P->s_stats); cudaFree(P->s_done);
    P->s_coef = nullptr; P->s_out = nullptr; P->s_stats = nullptr; P->s_done = nullptr;
    P->s_leaves = 0;
    CK(cudaMalloc(&P->s_coef, cbytes * n_leaves));
    CK(cudaMalloc(&P->s_out, tbytes * n_leaves));
    CK(cudaMalloc(&P->s_stats, 16 * (size_t)n_leaves));
    CK(cudaMalloc(&P->s_done, sizeof(int) * ((size_t)n_leaves + 1)));
    P->s_leaves = n_leaves;
  }
  int chunk = chunk_leaves > 0 ? chunk_leaves : P->slots / 2;
  if (chunk < 1) chunk = 1;
  const int nchunks = (n_leaves + chunk - 1) / chunk;
  cudaStream_t s_comp, s_out;
  CK(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
  cudaEvent_t ev_start;
  CK(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
  CK(cudaMemsetAsync(P->s_done, 0, sizeof(int) * nchunks, s_comp));
  CK(cudaMemcpyAsync(P->s_coef, coeffs_host, cbytes * n_leaves, cudaMemcpyHostToDevice, s_comp));
  cudaEventRecord(ev_start, s_comp);  // counters zeroed before any wait is evaluated
  cudaStreamWaitEvent(s_out, ev_start, 0);
  int rc = launch(P, MODE_DTN, n_leaves, P->s_coef, nullptr, nullptr, P->s_out, nullptr, P->s_stats,
                  s_comp, P->s_done, chunk);
  bool waits_ok = true;
  for (int k = 0; k < nchunks && rc == 0; ++k) {
    const int l0 = k * chunk, cnt = (n_leaves - l0 < chunk) ? n_leaves - l0 : chunk;
    if (waits_ok &&
        wait_fn((CUstream)s_out, (CUdeviceptr)(P->s_done + k), (cuuint32_t)cnt, CU_STREAM_WAIT_VALUE_GEQ) !=
            CUDA_SUCCESS) {
      waits_ok = false;  // cannot wait on counters: copy after the kernel instead
      cudaEvent_t ev_k;
      cudaEventCreateWithFlags(&ev_k, cudaEventDisableTiming);
      cudaEventRecord(ev_k, s_comp);
      cudaStreamWaitEvent(s_out, ev_k, 0);
      cudaEventDestroy(ev_k);
    }
    cudaMemcpyAsync(dtn_host + (size_t)l0 * P->m * P->m, P->s_out + (size_t)l0 * P->m * P->m,
                    tbytes * cnt, cudaMemcpyDeviceToHost, s_out);
    if (stats_host)
      cudaMemcpyAsync(stats_host + 2 * (size_t)l0, P->s_stats + 2 * (size_t)l0, 16 * (size_t)cnt,
                      cudaMemcpyDeviceToHost, s_out);
  }
  cudaError_t e1 = cudaStreamSynchronize(s_comp);
  cudaError_t e2 = cudaStreamSynchronize(s_out);
  cudaEventDestroy(ev_start);
  cudaStreamDestroy(s_comp);
  cudaStreamDestroy(s_out);
  if (rc != 0) return rc;
  const cudaError_t e = e1 != cudaSuccess ? e1 : e2;
  if (e != cudaSuccess) return fail(std::string("streamed dtn failed: ") + cudaGetErrorString(e));
  return 0;
}

int hps_interface_scatter(int device, const double* blocks, long long ld, long long block_stride,
                          long long leaf0, int n_jobs, const long long* jobs, double* out_t,
                          double* out_c, void* stream) {
  if (n_jobs < 0 || ld <= 0 || block_stride < 0) return fail("hps_interface_scatter: bad sizes");
  if (n_jobs == 0) return 0;
  if (!blocks || !jobs || !out_t) return fail("hps_interface_scatter: null pointer");
  CK(cudaSetDevice(device));
  hps_interface_scatter_kernel<<<n_jobs, 256, 0, (cudaStream_t)stream>>>(blocks, ld, block_stride, leaf0, jobs,
                                                                        out_t, out_c ? out_c : out_t);
  CK(cudaGetLastError());
  return 0;
}

}  // extern "C"
