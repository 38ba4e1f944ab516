// gsot_internal.cuh — shared declarations of the sm_100a solver library.
//
// Device layout: the cost lives in HBM column-tiled: for
// group l and 32-column chunk c, a tile of g_l x 32 entries starting at
// element 32 * (nw * off_l + c * g_l) (columns >= n are zero padding). Inside
// the tile the four 8-column quarters are stored one after the other, each
// g_l x 8 row-major (64-byte rows): a quarter is ONE contiguous run of
// g_l * 64 bytes, so an evaluation can fetch only the quarters that hold a
// possibly-nonzero block (cost_index below).
// Snapshot norms and per-block partials are [l][j] (j fastest) so that the
// per-block kernels, which put consecutive target columns on consecutive
// lanes, read and write them coalesced. Bitmasks are [l][c] words over
// 32-column chunks c = j / 32: bit (j % 32) of word (l, c).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "gsot.h"

namespace gsot {

// Exception carrying a gsot_status; converted to a status code at the C ABI.
struct Error : std::runtime_error {
  int status;
  gsot_error_detail detail{};
  Error(int st, const std::string& what) : std::runtime_error(what), status(st) {
    detail.status = st;
    detail.index = -1;
  }
};

#define GSOT_CUDA_CHECK(expr)                                                              \
  do {                                                                                    \
    cudaError_t gsot_e_ = (expr);                                                         \
    if (gsot_e_ != cudaSuccess) {                                                         \
      if (gsot_e_ == cudaErrorMemoryAllocation)                                           \
        throw ::gsot::Error(GSOT_ERR_OUT_OF_MEMORY,                                       \
                            std::string("CUDA out of memory at " #expr ": ") +            \
                                cudaGetErrorString(gsot_e_));                             \
      throw ::gsot::Error(GSOT_ERR_CUDA, std::string(#expr " failed: ") +                 \
                                             cudaGetErrorString(gsot_e_));                \
    }                                                                                     \
  } while (0)

// Tile geometry: columns per quarter plane; consecutive rows of one column are
// kRowStride elements apart.
constexpr int kPlaneCols = 8;
constexpr int kRowStride = kPlaneCols;
// Element index of cost entry (row o0 + r of the group at rows [o0, o0 + g),
// column j) in the tiled layout.
__host__ __device__ inline int64_t cost_index(int64_t nw, int64_t o0, int64_t g, int64_t j,
                                              int64_t r) {
  return 32 * (nw * o0 + (j >> 5) * g) + ((j & 31) >> 3) * (kPlaneCols * g) + kRowStride * r +
         (j & (kPlaneCols - 1));
}

// Read-only view of the resident instance passed to every kernel by value.
struct DevProblem {
  const double* C;        // column-tiled cost, 32 * nw * m doubles
  int64_t m, n;           // instance shape
  int32_t L;              // groups
  int32_t nw;             // 32-column chunks: ceil(n / 32)
  const int32_t* off;     // L+1 row offsets
  const int32_t* row_group;  // m: group of each row
  const double* sqrt_g;   // L: sqrt(g_l) (screening.hpp:79)
  const double* a;        // m
  const double* b;        // n
  double gamma, mu, tau;  // tau = mu * gamma (core.hpp:70)
  double half_inv_gamma;  // 0.5 / gamma (fast-mode psi)
  unsigned long long* tl; // diagnostic timeline (GSOT_PHASE_CLOCKS builds only), else null
  // provably-zero blocks: cmin[l * n + j] <= min_{i in l} c_ij
  // (float, rounded down), amax[l] = max_{i in l} alpha_i (NaN if any is NaN)
  const float* cmin;
  const double* amax;
  const float* cmn;  // per (group, chunk): min of cmin over the chunk's valid columns
};

// Device scalars written by the reduction kernels and read back with one
// D2H copy per evaluation.
struct EvalScalars {
  double objective;  // a.alpha + b.beta - psi
  double slope;      // grad . d (line search), when requested
  double dot_aa, dot_bb, psi_sum;
  double extra[3];   // pair kernel: s.y, s.s, y.y
  unsigned long long counters[4];  // in_active, skipped, unskipped, upper_bounds
  unsigned long long surv_rows;  // sum of g_l over surviving blocks (bytes accounting)
  unsigned long long task_rows;  // sum of g_l over work-list tasks
  unsigned long long zero_rows;  // cost rows of surviving blocks not read (provably zero)
  unsigned long long read_qrows; // 64-byte quarter rows of cost the evaluation fetched
  int ntasks;        // screened work-list length
  int next_task;     // dynamic scheduler cursor
  unsigned int ticket;  // last-block-done counter
  int audit_violation;  // audit: first violating block + 1 (l * n + j + 1)
  long long audit_where;
  // deferred folds, done by k_publish: per-block partials left by k_finalize
  // (fin_blocks blocks x 4), by k_lbfgs_step (step_blocks CTAs x 2), and the
  // screen's counter slots (cnt_pending). Not cleared by the per-evaluation
  // reset (it covers the fields above only).
  int fin_blocks;
  int step_blocks;
  int cnt_pending;
  int pad_;
};
constexpr size_t kEvalScalarsResetBytes = offsetof(EvalScalars, fin_blocks);

// One evaluation task: block row group l x 32-column chunk c, with what the
// eval kernel's producer needs to start the tile copy in one 32-byte load.
struct alignas(16) TaskDesc {
  int l, c, o0, g;  // group, chunk, first row, rows
  uint32_t word;    // survivor bits of the chunk's columns
  int pad[3];
};

// Launch with programmatic stream serialisation (PDL) unless GSOT_PDL=0.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- kernels (gsot_kernels.cu) ---------------------------------------------

// Per-kernel-class counters for gsot_profile_*.
enum KernelKind {
  K_EVAL = 0,
  K_SNAPSHOT = 1,
  K_BOUNDS = 2,
  K_ACTIVE = 3,
  K_FINALIZE = 4,
  K_LBFGS = 5,
  K_DELTA = 6,
  K_MISC = 7,
  K_NKINDS = 8,
  // statistics only (not a launch kind): the K_EVAL launches that read at
  // least half the dense bytes (near-dense evaluations, bandwidth-bound)
  K_EVAL_NEAR_DENSE = 8,
  // statistics only: the K_EVAL launches again, with bytes = the cost bytes
  // they actually fetched (whole 8-column quarters of the tasks they read)
  K_EVAL_FETCHED = 9,
  K_NSTATS = 10
};

void launch_relayout(const DevProblem& P, const double* src_colmajor, int64_t j0, int64_t ncols,
                     double* C, unsigned long long* first_bad, cudaStream_t s);
// lazy: provably-zero blocks not read; rows_read: 64 slots counting the cost
// rows a lazy snapshot read (bytes accounting)
void launch_snapshot(const DevProblem& P, const double* x, double* zs, double* ks, double* os,
                     bool lazy, unsigned long long* rows_read, cudaStream_t s);
void launch_block_z(const DevProblem& P, const double* x, double* zout, cudaStream_t s);
// Screened evaluations start from zeroed per-evaluation cursors of sc
// (ntasks, next_task, ticket, audit fields): k_publish resets them after it
// copies them out, the context starts zeroed, other paths use a memset.
void launch_delta(const DevProblem& P, const double* x, const double* xs, double* dpos,
                  double* dfull, double* dneg, double* dbeta, EvalScalars* sc, uint32_t* gmask,
                  cudaStream_t s);
void launch_active(const DevProblem& P, const double* ks, const double* os, const double* dfull,
                   const double* dneg, const double* dbeta, uint32_t* active_words,
                   EvalScalars* sc, cudaStream_t s);
// Upper-bound screen (screening.hpp:252-275): survivor words + counters.
// Counters accumulate into 64 slots x 8 (cnt_slots); the objective kernel
// folds them into EvalScalars and zeroes the slots.
// Per-group chunk masks gmask[l][c / 32] bit c % 32: chunk (l, c) non-empty.
void launch_screen(const DevProblem& P, const double* zs, const uint32_t* aw, const double* dpos,
                   const double* dbeta, double ub_offset, uint32_t* words, TaskDesc* tasks,
                   EvalScalars* sc, unsigned long long* cnt_slots, uint32_t* gmask,
                   uint32_t* cmask, const double* x, const double* xs, int dbeta_ready,
                   const double* xe, const double* dpre, const double2* zmm, const double* dbx3,
                   int num_sms, cudaStream_t s);
bool screen_uses_summaries(const DevProblem& P, int num_sms);
// zmm[l * nw + c] = (min, max) of z~ over the chunk's columns: after every snapshot
void launch_chunk_minmax(const DevProblem& P, const double* zs, double2* zmm,
                         const unsigned char* zero_chunk, cudaStream_t s);
// dpre: optional, the fast-mode group delta norms precomputed by launch_group_amax
// xe: the evaluation state (the provably-zero test; P.amax must hold its
// group maxima). Fused evaluation over the non-empty chunks of `words` (gsot_kernels.cu).
int eval_buf_rows(int gmax);
// qrows: 0, or the quarter pipeline's rows per quarter segment (variant 3)
size_t eval_smem_bytes(int buf_rows, int qrows);
// quarter pipeline geometry for a tallest group of gmax rows: rows per quarter
// segment, and the tallest group still evaluated as a whole tile
int eval_qrows_for(int gmax);
int eval_q_short_rows(int qrows);
// k_eval variant for a context: 0 in place / 4 consumer warps, 1 recomputing
// (tiles taller than a segment; superseded by 3, kept for comparison), 2 in
// place / 2 consumer warps (short tiles), 3 the quarter pipeline k_eval_q
int eval_variant(int gmax, int seg, bool recompute);
int eval_blocks_per_sm(size_t smem, int variant);
// ntasks >= 0: `tasks` holds that many entries (dense list); -1: the
// screened list, length *ntasks_dev (written by the screen kernel).
void launch_eval(const DevProblem& P, const double* x, const TaskDesc* tasks, int ntasks,
                 const int* ntasks_dev, const uint32_t* words, double* rowpart, double* colpart,
                 double* psi, int seg, int qrows, int variant, int grid, int* next_task,
                 bool pz_done, cudaStream_t s);
// pz_done: the work list comes from the chunk-summary screen, which already
// dropped the provably-zero columns from the survivor words
// grad, psi columns, objective and slope (dvec may be null) in one kernel.
void launch_finalize(const DevProblem& P, const double* x, const uint32_t* words,
                     const uint32_t* gmask, uint32_t* cmask, int clear_cmask,
                     const double* rowpart, const double* colpart, const double* psi,
                     double* grad, const double* dvec, double* partials, EvalScalars* sc,
                     int cnt_pending, cudaStream_t s);
// plan_diagnostics at x: per-chunk row sums into rowpart, per-block column
// sums into colpart, all-zero block count added to *zero_blocks; the fold
// writes plan row sums to sums[0, m) and column sums to sums[m, m + n).
void launch_plan_diag(const DevProblem& P, const double* x, double* rowpart, double* colpart,
                      unsigned long long* zero_blocks, cudaStream_t s);
// primal_objective at x: each block's share of <T, C> + regularizer into colpart.
void launch_plan_primal(const DevProblem& P, const double* x, double* colpart, cudaStream_t s);
void launch_plan_diag_fold(const DevProblem& P, const double* rowpart, const double* colpart,
                           double* sums, cudaStream_t s);
void launch_plan_columns(const DevProblem& P, const double* x, int64_t j0, int64_t ncols,
                         double* out, cudaStream_t s);
void launch_audit_skips(const DevProblem& P, const double* x, const uint32_t* words,
                        const uint32_t* active_words, EvalScalars* sc, cudaStream_t s);
void launch_audit_active(const DevProblem& P, const double* x, const uint32_t* active_words,
                         EvalScalars* sc, cudaStream_t s);
void launch_fill_words(uint32_t* words, int32_t L, int32_t nw, int64_t n, cudaStream_t s);
// Provably-zero blocks: the per-block minimum cost (once per upload) and the
// per-group maximum of alpha (per evaluation, programmatic launch).
void launch_block_min(const DevProblem& P, float* cmin, cudaStream_t s);
// zero_me: optional L counters the kernel also clears (the lazy snapshot's list lengths)
// xs, dfast: optional; dfast[l] = |[x_l - xs_l]+| (the fast-mode screen's group delta norm)
void launch_group_amax(const DevProblem& P, const double* x, double* amax, cudaStream_t s,
                       unsigned int* zero_me = nullptr, const double* xs = nullptr,
                       double* dfast = nullptr, const double* dbeta = nullptr,
                       double* dbx3 = nullptr);
// dbeta, dbx3: optional; dbx3[3 c ..] = (min dbeta, max dbeta, max beta) of chunk c,
// for the chunk-summary screen
// shorter groups are walked by the marking kernel itself (measured: 64 -> 8
// takes config 3 from 22.8 to 21.1 ms and config 4 from 52.0 to 50.3 ms)
constexpr int kSnapListMinRows = 8;
// lazy snapshot through per-group lists of the blocks that are not provably
// zero (list: L * n column indices; count: L lengths, cleared by the preceding
// launch_group_amax)
void launch_snapshot_lazy2(const DevProblem& P, const double* x, double* zs, double* ks, double* os,
                           uint32_t* list, unsigned int* count, unsigned long long* rows_read,
                           unsigned char* zero_chunk, double2* zmm, double* bmaxc,
                           cudaStream_t s);
// zero_chunk[l * nw + c] = 1: the chunk's z~ k~ o~ hold zeros (maintained by the
// listed lazy snapshot; cleared by the caller whenever another form writes them)
void launch_fill_gmask(uint32_t* gmask, int32_t L, int32_t nw, cudaStream_t s);
// Per-chunk group masks cmask[c][l / 32] bit l % 32: (l, c) non-empty.
void launch_fill_cmask(uint32_t* cmask, int32_t L, int32_t nw, cudaStream_t s);
void launch_dense_tasks(const DevProblem& P, TaskDesc* tasks, const int32_t* group_order,
                        cudaStream_t s);

// L-BFGS vector kernels (gsot_lbfgs.cu).
constexpr int kMaxMemory = 64;

// Device-resident curvature-pair history (lbfgs.hpp:73-74, :243-255): a ring
// of mem+1 vector slots, `order` lists the k live pairs oldest first and
// `scratch` is the slot the next pair is written to before the acceptance
// test. The pair kernel decides acceptance and evicts on the device, so the
// per-iteration graph needs no host round trip.
struct HistState {
  int k;
  int mem;
  int scratch;
  int accepted;  // last pair: 1 pushed, 0 rejected by the s.y test
  int order[kMaxMemory + 1];
  double rho[kMaxMemory + 1];  // 1 / s.y, by logical position
  double sy[kMaxMemory + 1];   // s.y, by logical position
  double yy[kMaxMemory + 1];   // y.y, by logical position
  double last_sy, last_ss, last_yy;
};

// Everything the host reads after one device sequence, in one D2H copy.
struct DevSync {
  EvalScalars sc;
  HistState h;
  double tl[2];  // two-loop: g.d, d.d
  double t;      // line-search step: host-owned, copied in by the solver
};

// Copy the scalar block into mapped host memory and then bump the host-visible
// completion counter (system-scope release): the host spins on the counter
// instead of a D2H copy + stream synchronisation.
// First the pending folds (EvalScalars::fin_blocks / step_blocks /
// cnt_pending) in a fixed order.
void launch_publish(DevSync* src, DevSync* host_dst, unsigned long long* dev_count,
                    unsigned long long* host_flag, const double* fin_partials,
                    const double* step_partials, unsigned long long* cnt_slots,
                    unsigned long long* tl, cudaStream_t s);

// Column-sharded contexts (gsot_lbfgs.cu): fold the pending
// partials into `tail` (kShardTail doubles, presence flags per group) before
// the sum all-reduce, and write the reduced groups back after it.
constexpr int kShardTail = 16;
void launch_shard_pack(DevSync* src, const double* fin_partials, const double* step_partials,
                       unsigned long long* cnt_slots, double* tail, cudaStream_t s);
void launch_shard_unpack(DevSync* src, const double* tail, cudaStream_t s);

// trial.x = x + t * d with t read from device memory; with dbeta != null also
// dbeta_j = out[m + j] - snap[m + j] for the screen.
void launch_axpy_point(const double* x, const double* t, const double* d, double* out,
                       int64_t dim, int64_t m, const double* snap, double* dbeta, cudaStream_t s);
void launch_hist_reset(HistState* h, int mem, cudaStream_t s);
void launch_dot(const double* a, const double* b, int64_t dim, double* partials, int nblocks,
                EvalScalars* sc, int slot, cudaStream_t s);
void launch_absmax(const double* a, int64_t dim, double* partials, int nblocks, EvalScalars* sc,
                   int slot, cudaStream_t s);

// Cost-matrix construction (gsot_data.cu).
// tiled == nullptr: column-major m x n output; otherwise the column-tiled
// layout of that problem.
void launch_cost_matrix(const double* src, int64_t m, const double* tgt, int64_t n, int64_t d,
                        const DevProblem* tiled, double* out, cudaStream_t s);
void launch_max_reduce(const double* C, int64_t count, double* partials, int nblocks,
                       double* out, unsigned int* ticket, cudaStream_t s);
void launch_scale_div(double* C, int64_t count, const double* divisor, cudaStream_t s);
// validate_instance's cost scan over the tiled layout: first offender (j*m+i).
void launch_scan_bad(const DevProblem& P, unsigned long long* first_bad, cudaStream_t s);

}  // namespace gsot

namespace gsot {

// Compact (Byrd-Nocedal-Schnabel) representation of the same L-BFGS
// operator the two-loop recursion applies (fast mode): R = upper triangle of
// S^T Y, D = diag(R), YY = Y^T Y, kept by logical pair position on the
// device, plus the current u = S^T g, v = Y^T g and the direction
// coefficients d = gam * g + S p - Y w (w already scaled by gam).
struct CompactState {
  double R[kMaxMemory * kMaxMemory];   // R[i * kMaxMemory + j] = s_i . y_j, i <= j
  double YY[kMaxMemory * kMaxMemory];  // y_i . y_j
  double u[kMaxMemory + 1], v[kMaxMemory + 1];
  double p[kMaxMemory], w[kMaxMemory];
  double gam;
  int k;
};

constexpr int kStepMaxGrid = 1024;  // CTAs of the cooperative step kernel, at most
// Doubles of partials the step kernel needs for a history of `mem` pairs.
size_t lbfgs_step_partials(int mem);
// The fast-mode direction update in one cooperative launch (gsot_lbfgs.cu):
// pair != 0 first forms the pending curvature pair s = x - xprev,
// y = gprev - g into the scratch slot, tests it and updates the ring and
// R / YY (lbfgs.hpp:243-255); then the compact coefficients for g, the
// direction d, out[0] = g.d, out[1] = d.d, and xt = x + t d when xt != null.
void launch_lbfgs_step(int pair, const double* x, const double* xprev, const double* g,
                       const double* gprev, double* S, double* Y, int64_t stride, HistState* h,
                       CompactState* cs, double* d, const double* t, double* xt, int64_t dim,
                       double* out, EvalScalars* sc, double* part, int mem,
                       unsigned long long* tl, int64_t m, const double* snap, double* dbeta,
                       cudaStream_t s, int split = 0, int64_t dot_lo = 0,
                       double* red_io = nullptr);

}  // namespace gsot
