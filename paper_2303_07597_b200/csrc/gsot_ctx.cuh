// gsot_ctx.cuh — the resident-instance context shared by the context/eval
// code (gsot_ctx.cu) and the solver (gsot_solver.cu).
#pragma once

#include <atomic>

#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gsot_internal.cuh"
#include "gsot_exact2.cuh"

namespace gsot {

// One captured device sequence (CUDA graph) plus the timing marks it records
// through external event nodes when profiling.
struct Mark {
  cudaEvent_t a, b;
  int kind;
  double bytes;  // < 0: screened eval, bytes from the synced counters
};

struct Sequence {
  cudaGraphExec_t exec = nullptr;
  std::vector<Mark> marks;
  int kernels = 0;
  int publishes = 0;
  ~Sequence() {
    if (exec) cudaGraphExecDestroy(exec);
    for (auto& m : marks) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
  }
};

// Persistent solver workspace (lives as long as the context so captured
// graphs stay valid across solves).
struct SolverWorkspace {
  int64_t dim = 0;
  int mem = 0;
  double* X[2] = {nullptr, nullptr};  // iterate / trial, alternating roles
  double* G[2] = {nullptr, nullptr};
  double* lo_x = nullptr;  // line-search points kept by value (lbfgs.hpp:157, :166)
  double* lo_g = nullptr;
  double* prev_x = nullptr;
  double* prev_g = nullptr;
  double* d = nullptr;     // direction
  double* S = nullptr;     // (mem + 1) pair slots of dim doubles
  double* Y = nullptr;
  double* audit_g = nullptr;
  CompactState* cs = nullptr;   // compact L-BFGS state (fast mode)
  double* cpart = nullptr;      // step-kernel partials (lbfgs_step_partials)
  std::map<std::string, std::unique_ptr<Sequence>> graphs;
  ~SolverWorkspace();
};

// A sharded context's communicator (gsot_comm.cu).
struct ShardComm {
  enum { kNccl = 1, kHost = 2 };
  int kind = 0;
  int rank = 0, world = 1;
  void* nccl_comm = nullptr;  // ncclComm_t
  gsot_allreduce_fn fn = nullptr;
  void* user = nullptr;
  double* host_buf = nullptr;  // pinned staging of the host transport
  size_t host_cap = 0;
  double* d_tail = nullptr;  // kShardTail doubles (k_shard_pack / k_shard_unpack)
  double* d_red = nullptr;   // the step kernel's folded dots, (kMaxMemory + 1) * 5
  double* d_n = nullptr;
  int64_t n_global = 0;      // columns over all ranks
  // In-place all-reduce of `count` device doubles on stream s (GSOT_REDUCE_*).
  void allreduce(double* d, int64_t count, int op, cudaStream_t s);
  void group_begin();  // NCCL group (no-op for the host transport)
  void group_end();
  ~ShardComm();
};

}  // namespace gsot

struct gsot_ctx {
  int device = 0;
  double ub_offset = 0.0;  // FastGradDispatcher upper_bound_offset for gsot_eval (screening.hpp:211)
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  int64_t m = 0, n = 0;
  int32_t L = 0, nw = 0;
  double gamma = 1.0, mu = 1.0;
  std::vector<int32_t> sizes, off;
  size_t bytes = 0;

  // resident instance
  double* C = nullptr;
  int32_t *d_off = nullptr, *d_row_group = nullptr, *d_group_order = nullptr;
  double *d_sqrt_g = nullptr, *d_a = nullptr, *d_b = nullptr;
  // evaluation buffers
  double *x_eval = nullptr, *g_eval = nullptr;
  double *rowpart = nullptr, *colpart = nullptr, *psi = nullptr, *psicol = nullptr;
  double* partials = nullptr;
  unsigned long long* cnt_partials = nullptr;  // spare counter partials
  unsigned long long* cnt_slots = nullptr;     // screen counters, 64 x 8
  uint32_t *words = nullptr, *dense_words = nullptr;
  uint32_t *gmask = nullptr, *dense_gmask = nullptr;  // per-group non-empty chunk masks
  uint32_t *cmask = nullptr, *dense_cmask = nullptr;  // per-chunk non-empty group masks
  double* d_one = nullptr;  // device constant 1.0 (t_init of direction sequences)
  double* staging = nullptr;            // host-cost upload staging (column chunks)
  unsigned long long* d_bad = nullptr;  // first invalid cost entry (validation)
  unsigned long long* tl = nullptr;  // diagnostic kernel timeline (GSOT_TIMELINE=1, diag builds)
  gsot::TaskDesc* dense_tasks = nullptr;  // every chunk, largest groups first
  gsot::TaskDesc* tasks = nullptr;        // screened work list (non-empty chunks)
  // screening state
  double *snap_x = nullptr, *zs = nullptr, *ks = nullptr, *os = nullptr;
  double *dpos = nullptr, *dfull = nullptr, *dneg = nullptr, *dbeta = nullptr;
  // provably-zero blocks: per block min cost (float, rounded down; computed
  // once per upload) and per group max alpha (per evaluation)
  float* cmin = nullptr;
  double* amax = nullptr;
  bool snap_lazy = false;  // the current snapshot skipped provably-zero blocks
  unsigned long long* snap_rows = nullptr;  // 64 slots: cost rows read by lazy snapshots
  uint32_t* snap_list = nullptr;            // lazy snapshots: per group, the columns of its blocks that are not provably zero
  unsigned int* snap_cnt = nullptr;         // L list lengths
  double* dpos_fast = nullptr;              // L: fast-mode screen's group delta norms (k_group_amax)
  float* cmn = nullptr;                     // L * nw: per-chunk minimum of cmin
  double2* zmm = nullptr;                   // L * nw: per-chunk (min, max) of the snapshot's z~
  unsigned char* snap_zero = nullptr;       // L * nw: the chunk's z~ k~ o~ currently hold zeros
  double* bmaxc = nullptr;                  // nw: per-chunk maximum of beta (lazy snapshot's chunk test)
  double* dbx3 = nullptr;                   // 3 nw: per-chunk (min dbeta, max dbeta, max beta) for the screen
  uint32_t* active_words = nullptr;
  int64_t active_count = 0;
  bool have_snapshot = false;
  // scalars: one device block, one pinned mirror
  gsot::DevSync* dsync = nullptr;
  gsot::DevSync* h_sync = nullptr;      // mapped pinned mirror, written by k_publish
  gsot::DevSync* h_sync_dev = nullptr;  // its device address
  unsigned long long* h_flag = nullptr;      // mapped completion counter
  unsigned long long* h_flag_dev = nullptr;
  unsigned long long* d_pub_count = nullptr;  // device copy of the counter
  unsigned long long pub_expected = 0;        // publishes enqueued so far
  gsot::EvalScalars* sc = nullptr;    // &dsync->sc
  gsot::EvalScalars* h_sc = nullptr;  // &h_sync->sc
  int eval_grid = 148 * 4;
  int eval_buf = 96;  // rows per shared-memory segment in k_eval
  bool eval_recompute = false;  // k_eval<true>: some block is taller than a segment
  int eval_variant = 0;         // gsot::eval_variant (0 / 1 recompute / 2 short tiles / 3 quarters)
  int eval_qrows = 0;           // variant 3: rows per quarter segment
  int red_blocks = 148 * 2;
  // exact-order mode buffers (gsot_exact2.cu), allocated on first use
  gsot::ExactWs ex;
  bool ex_ready = false;
  // solver
  std::unique_ptr<gsot::SolverWorkspace> ws;
  uint64_t graph_epoch = 0;  // bumped when baked-in parameters change
  bool cacheable = false;    // created from data (gsot_create / _device): may be parked
  // measurement
  bool profile = false;
  unsigned profile_mask = 0;  // kinds bracketed with events (bit per KernelKind)
  std::vector<gsot::Mark> marks;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[gsot::K_NSTATS] = {};
  double prof_bytes[gsot::K_NSTATS] = {};
  int64_t prof_launches[gsot::K_NSTATS] = {};
  int64_t launches = 0;
  cudaEvent_t timer_a = nullptr, timer_b = nullptr;
  // stream capture in progress: marks/kernels go to the sequence
  gsot::Sequence* capturing = nullptr;
  // column-sharded solve (gsot_comm.cu): the communicator, and the gradient
  // whose head the next publication all-reduces (set by enqueue_eval)
  std::unique_ptr<gsot::ShardComm> comm;
  double* pending_grad = nullptr;
  // dots over [alpha; beta_p] start here: the replicated alpha part counts on rank 0 only
  int64_t dot_lo() const { return comm && comm->rank != 0 ? m : 0; }
  int64_t n_global() const { return comm ? comm->n_global : n; }

  gsot::DevProblem problem() const {
    gsot::DevProblem P;
    P.C = C;
    P.m = m;
    P.n = n;
    P.L = L;
    P.nw = nw;
    P.off = d_off;
    P.row_group = d_row_group;
    P.sqrt_g = d_sqrt_g;
    P.a = d_a;
    P.b = d_b;
    P.gamma = gamma;
    P.mu = mu;
    P.tau = mu * gamma;
    P.half_inv_gamma = 0.5 / gamma;
    P.tl = tl;
    P.cmin = cmin;
    P.amax = amax;
    P.cmn = cmn;
    return P;
  }

  // Exact-order buffers (never during stream capture: the solver and the
  // eval entry points call this before they enqueue).
  void ensure_exact() {
    if (ex_ready) return;
    if (capturing) throw gsot::Error(GSOT_ERR_STATE, "exact-order buffers allocated during capture");
    GSOT_CUDA_CHECK(cudaStreamSynchronize(stream));
    gsot::exact_ws_alloc(ex, problem(), sizes, &bytes);
    ex_ready = true;
  }

  cudaEvent_t take_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    GSOT_CUDA_CHECK(cudaEventCreate(&e));
    return e;
  }

  // Enqueue one kernel launch; bracket it with events when profiling (event
  // record nodes when capturing); count launches.
  template <typename F>
  void launch(int kind, double bytes_alg, F&& f) {
    const bool timed = profile && ((profile_mask >> kind) & 1u);
    if (capturing) {
      ++capturing->kernels;
      if (timed) {
        gsot::Mark mk{nullptr, nullptr, kind, bytes_alg};
        GSOT_CUDA_CHECK(cudaEventCreate(&mk.a));
        GSOT_CUDA_CHECK(cudaEventCreate(&mk.b));
        GSOT_CUDA_CHECK(cudaEventRecordWithFlags(mk.a, stream, cudaEventRecordExternal));
        f();
        GSOT_CUDA_CHECK(cudaGetLastError());
        GSOT_CUDA_CHECK(cudaEventRecordWithFlags(mk.b, stream, cudaEventRecordExternal));
        capturing->marks.push_back(mk);
      } else {
        f();
        GSOT_CUDA_CHECK(cudaGetLastError());
      }
      return;
    }
    ++launches;
    if (!timed) {
      f();
      GSOT_CUDA_CHECK(cudaGetLastError());
      return;
    }
    gsot::Mark mk{take_event(), take_event(), kind, bytes_alg};
    GSOT_CUDA_CHECK(cudaEventRecord(mk.a, stream));
    f();
    GSOT_CUDA_CHECK(cudaGetLastError());
    GSOT_CUDA_CHECK(cudaEventRecord(mk.b, stream));
    marks.push_back(mk);
  }

  double screened_eval_bytes() const {
    // screen: z~ of every bound-checked block + the survivor words; then the
    // surviving blocks' cost rows, the non-empty chunks' row partials and
    // the per-block column / psi partials
    const double surv_blocks = static_cast<double>(h_sc->counters[0] + h_sc->counters[2]);
    return 8.0 * static_cast<double>(h_sc->counters[3]) + 4.0 * static_cast<double>(L) * nw +
           8.0 * static_cast<double>(h_sc->surv_rows) +
           8.0 * static_cast<double>(h_sc->task_rows) + 16.0 * surv_blocks;
  }

  void account(const gsot::Mark& mk) {
    float ms = 0.f;
    GSOT_CUDA_CHECK(cudaEventElapsedTime(&ms, mk.a, mk.b));
    double bytes = mk.bytes < 0 ? screened_eval_bytes() : mk.bytes;
    if (mk.kind == gsot::K_SNAPSHOT && mk.bytes == -2.0) {  // lazy: the rows it read
      unsigned long long rows[64];
      GSOT_CUDA_CHECK(cudaMemcpy(rows, snap_rows, sizeof(rows), cudaMemcpyDeviceToHost));
      GSOT_CUDA_CHECK(cudaMemset(snap_rows, 0, sizeof(rows)));
      double r = 0.0;
      for (unsigned long long v : rows) r += static_cast<double>(v);
      const double Ln = static_cast<double>(L) * n;
      bytes = 8.0 * r + 28.0 * Ln + 8.0 * (m + n);  // rows, cmin + z~ k~ o~, x
    }
    if (mk.kind == gsot::K_EVAL)  // rows of provably-zero blocks are not read
      bytes -= 8.0 * static_cast<double>(h_sc->zero_rows);
    prof_ms[mk.kind] += ms;
    prof_bytes[mk.kind] += bytes;
    prof_launches[mk.kind] += 1;
    if (mk.kind == gsot::K_EVAL) {
      prof_ms[gsot::K_EVAL_FETCHED] += ms;
      prof_bytes[gsot::K_EVAL_FETCHED] += 64.0 * static_cast<double>(h_sc->read_qrows);
      prof_launches[gsot::K_EVAL_FETCHED] += 1;
    }
    if (mk.kind == gsot::K_EVAL && bytes >= 4.0 * static_cast<double>(m) * static_cast<double>(n)) {
      prof_ms[gsot::K_EVAL_NEAR_DENSE] += ms;
      prof_bytes[gsot::K_EVAL_NEAR_DENSE] += bytes;
      prof_launches[gsot::K_EVAL_NEAR_DENSE] += 1;
    }
  }

  // After a synchronisation: fold eager marks into the counters.
  void collect_marks() {
    if (marks.empty()) return;
    GSOT_CUDA_CHECK(cudaStreamSynchronize(stream));
    for (auto& mk : marks) {
      account(mk);
      event_pool.push_back(mk.a);
      event_pool.push_back(mk.b);
    }
    marks.clear();
  }

  void sync() { GSOT_CUDA_CHECK(cudaStreamSynchronize(stream)); }
  void fetch_scalars() {
    enqueue_fetch();
    wait_published();
    collect_marks();
  }
  // Enqueue the publication of the scalar block to the host mirror.
  void enqueue_fetch() {
    if (comm) {  // sharded: fold, sum over the ranks, write back, then publish
      launch(gsot::K_MISC, 0.0, [&] {
        gsot::launch_shard_pack(dsync, partials, ws ? ws->cpart : nullptr, cnt_slots,
                                comm->d_tail, stream);
      });
      comm->group_begin();
      if (pending_grad) comm->allreduce(pending_grad, m, GSOT_REDUCE_SUM, stream);
      comm->allreduce(comm->d_tail, gsot::kShardTail, GSOT_REDUCE_SUM, stream);
      comm->group_end();
      pending_grad = nullptr;
      launch(gsot::K_MISC, 0.0, [&] { gsot::launch_shard_unpack(dsync, comm->d_tail, stream); });
    }
    launch(gsot::K_MISC, 0.0, [&] {
      gsot::launch_publish(dsync, h_sync_dev, d_pub_count, h_flag_dev, partials,
                           ws ? ws->cpart : nullptr, cnt_slots, tl, stream);
    });
    if (capturing)
      ++capturing->publishes;
    else
      ++pub_expected;
  }
  // Wait until every enqueued publication has landed in the host mirror:
  // spin on the mapped counter (the stream is polled for errors meanwhile).
  void wait_published() {
    const volatile unsigned long long* f = h_flag;
    for (uint64_t spin = 0;; ++spin) {
      if (*f >= pub_expected) break;
      if ((spin & 1023u) == 1023u) {
        const cudaError_t st = cudaStreamQuery(stream);
        if (st == cudaSuccess) {
          if (*f >= pub_expected) break;
          throw gsot::Error(GSOT_ERR_CUDA, "publication counter out of step with the stream");
        }
        if (st != cudaErrorNotReady) GSOT_CUDA_CHECK(st);
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  }
  void reset_scalars() {
    GSOT_CUDA_CHECK(cudaMemsetAsync(sc, 0, gsot::kEvalScalarsResetBytes, stream));
  }

  ~gsot_ctx();
};

// guard() of gsot_ctx.cu for the entry points of other translation units.
int gsot_guard_call(const std::function<void()>& f);

namespace gsot {

struct EvalOut {
  double objective = 0.0;
  double slope = 0.0;
  gsot_call_stats stats{};
};

// Enqueue the fused evaluation at device state d_x (length m+n) into d_grad,
// with the line-search slope against d_dir when non-null. No sync; the
// scalars land in c->dsync->sc.
// dbeta_ready: the kernel that produced d_x also wrote c->dbeta (fast solves).
void enqueue_eval(gsot_ctx* c, const double* d_x, int mode, double* d_grad, const double* d_dir,
                  double ub_offset, bool use_active, bool dbeta_ready = false);
// Read back the result of the last enqueue_eval after c->fetch_scalars().
EvalOut eval_result(gsot_ctx* c, int mode);
EvalOut eval_device(gsot_ctx* c, const double* d_x, int mode, double* d_grad,
                    const double* d_dir, double ub_offset, bool use_active);
// lazy: provably-zero blocks not read (the solver's own snapshots)
void enqueue_snapshot(gsot_ctx* c, const double* d_x, bool lazy);
void init_snapshot_device(gsot_ctx* c, const double* d_x, bool lazy);
void enqueue_refresh(gsot_ctx* c, const double* d_x, bool use_active, bool lazy);
void refresh_device(gsot_ctx* c, const double* d_x, bool use_active);

template <typename T>
T* dalloc(size_t count, size_t* tally) {
  T* p = nullptr;
  if (count == 0) count = 1;
  GSOT_CUDA_CHECK(cudaMalloc(&p, sizeof(T) * count));
  if (tally) *tally += sizeof(T) * count;
  return p;
}

void run_solve(gsot_ctx* c, const gsot_solver_options& o, double* x_out, gsot_solve_result* res,
               int64_t* history, int64_t history_cap);

}  // namespace gsot
