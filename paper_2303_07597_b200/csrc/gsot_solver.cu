// gsot_solver.cu — solve() on the device (solver.hpp:92-293).
//
// The host runs the scalar control flow of the reference's L-BFGS ascent
// (lbfgs.hpp:61-274) verbatim: two-loop direction, strong-Wolfe bracketing
// and zoom, retry from steepest ascent, the curvature-pair test, chunk hooks
// and the infinity-norm stop test. Every vector operation and every
// evaluation runs on the device. Each host decision point needs exactly one
// device round trip: the work between two decisions is one CUDA graph
//   DT   two-loop -> trial point -> fused evaluation -> scalars to host
//   PDT  curvature pair + ring update -> DT            (after an acceptance)
//   T    trial point -> fused evaluation -> scalars    (further line-search steps)
//   RF   active set + snapshot (chunk hook) -> |g|_inf -> scalars
// captured once per context and replayed (the line-search step t and the
// pair history live in device memory, so the graphs never change). Audit
// mode runs the same sequences eagerly and re-verifies every evaluation.
#include <cstdio>
#include <cstdlib>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#include "gsot_ctx.cuh"

namespace gsot {

namespace {

struct Pt {  // lbfgs.hpp:40-46
  double t = 0.0, value = 0.0, slope = 0.0;
  bool vec = false;  // vectors valid in this point's buffer
};

class Solver {
 public:
  Solver(gsot_ctx* c, const gsot_solver_options& o, gsot_solve_result* res, int64_t* hist,
         int64_t hist_cap)
      : c_(c), o_(o), res_(res), hist_(hist), hist_cap_(hist_cap) {
    screened_ = o.mode != GSOT_MODE_BASELINE;
    use_active_ = o.mode == GSOT_MODE_FAST ||
                  (o.mode == GSOT_MODE_AUDIT && !(o.flags & GSOT_SOLVE_NO_ACTIVE_SET));
    audit_ = o.mode == GSOT_MODE_AUDIT;
    exact_ = (o.flags & GSOT_SOLVE_EXACT) != 0;
    // a sharded context (gsot_comm.cu): every publication sums over the ranks;
    // the host transport synchronises, so its sequences run eagerly
    sharded_ = c->comm != nullptr;
    if (sharded_ && (exact_ || audit_))
      throw Error(GSOT_ERR_INVALID_ARGUMENT,
                  "sharded solves support the baseline and fast modes (no exact-order / audit)");
    graphs_ = !audit_ && !(sharded_ && c->comm->kind == ShardComm::kHost);
    mode_eval_ = (screened_ ? GSOT_EVAL_SCREENED : GSOT_EVAL_DENSE) | (exact_ ? GSOT_EVAL_EXACT : 0);
    mem_ = std::max(1, o.lbfgs_memory);
    if (exact_) c_->ensure_exact();
    ensure_workspace();
    w_ = c_->ws.get();
    key_ = std::to_string(o.mode) + "/" + std::to_string(o.lbfgs_memory) + "/" +
           std::to_string(o.upper_bound_offset) + "/" + std::to_string(c_->profile ? c_->profile_mask : 0u) +
           (exact_ ? "/exact" : "") + (use_active_ ? "" : "/nolb") + (sharded_ ? "/shard" : "");
  }

  ~Solver() {
    if (diag_) {
      cudaEventDestroy(diag_ev_[0]);
      cudaEventDestroy(diag_ev_[1]);
    }
  }

  void run(double* x_out) {
    if (std::getenv("GSOT_DIAG_SEQ") && graphs_) {
      diag_ = true;
      GSOT_CUDA_CHECK(cudaEventCreate(&diag_ev_[0]));
      GSOT_CUDA_CHECK(cudaEventCreate(&diag_ev_[1]));
    }
    const int64_t dim = w_->dim;
    r_ = 0;
    GSOT_CUDA_CHECK(cudaMemsetAsync(w_->X[0], 0, sizeof(double) * dim, c_->stream));
    c_->launch(K_LBFGS, 0.0, [&] { launch_hist_reset(&c_->dsync->h, mem_, c_->stream); });
    if (screened_) init_snapshot_device(c_, w_->X[0], true);  // solver.hpp:141-144
    // initial gradient + objective (lbfgs.hpp:70-71): one fused evaluation
    enqueue_eval(c_, w_->X[0], mode_eval_, w_->G[0], nullptr, o_.upper_bound_offset, use_active_);
    c_->fetch_scalars();
    EvalOut e0 = eval_result(c_, mode_eval_);
    record(e0);
    if (audit_) audit_call(w_->X[0], w_->G[0], e0);
    res_value_ = e0.objective;

    const auto t0 = std::chrono::steady_clock::now();
    maximize();
    const auto t1 = std::chrono::steady_clock::now();
    if (diag_)
      std::fprintf(stderr, "[gsot diag] sequences %ld  device %.1f us/seq  host round trip %.1f us/seq\n",
                   (long)diag_n_, 1e6 * diag_dev_ / std::max<int64_t>(1, diag_n_),
                   1e6 * diag_host_ / std::max<int64_t>(1, diag_n_));
    res_->wall_seconds = std::chrono::duration<double>(t1 - t0).count();
    if (x_out)
      GSOT_CUDA_CHECK(cudaMemcpyAsync(x_out, w_->X[r_], sizeof(double) * dim,
                                      cudaMemcpyDeviceToHost, c_->stream));
    c_->sync();
    // finish_solution's dual_objective(x*) (solver.hpp:78) equals the
    // accepted point's value: screened and dense evaluations agree bitwise.
    res_->objective = res_value_;
    res_->outer_loops = res_->chunks;
  }

 private:
  bool diag_ = false;
  cudaEvent_t diag_ev_[2] = {nullptr, nullptr};
  double diag_dev_ = 0.0, diag_host_ = 0.0;
  int64_t diag_n_ = 0;

  void ensure_workspace() {
    const int64_t dim = c_->m + c_->n;
    const int mem = std::max(1, o_.lbfgs_memory);
    auto& ws = c_->ws;
    if (ws && ws->dim == dim && ws->mem >= mem) return;
    ws.reset(new SolverWorkspace());
    ws->dim = dim;
    ws->mem = mem;
    size_t* t = &c_->bytes;
    for (int q = 0; q < 2; ++q) {
      ws->X[q] = dalloc<double>(dim + 8, t);
      ws->G[q] = dalloc<double>(dim + 8, t);
    }
    ws->lo_x = dalloc<double>(dim, t);
    ws->lo_g = dalloc<double>(dim, t);
    ws->prev_x = dalloc<double>(dim, t);
    ws->prev_g = dalloc<double>(dim, t);
    ws->d = dalloc<double>(dim + 8, t);
    ws->S = dalloc<double>(static_cast<size_t>(mem + 1) * dim, t);
    ws->Y = dalloc<double>(static_cast<size_t>(mem + 1) * dim, t);
    ws->cs = dalloc<CompactState>(1, t);
    ws->cpart = dalloc<double>(lbfgs_step_partials(mem), t);
  }

  // ---- device sequences ----------------------------------------------------

  // Run `body` (which enqueues work ending with enqueue_fetch) as a captured
  // graph keyed by name and iterate parity, or eagerly in audit mode; then
  // synchronise and account the timing marks.
  void run_seq(const char* name, const std::function<void()>& body) {
    if (!graphs_) {
      body();
      c_->wait_published();
      c_->sync();
      c_->collect_marks();
      return;
    }
    // per-solve lookup cache by (name literal, buffer parity): the string key
    // and map search run once per sequence kind, not once per launch
    Sequence* cached = nullptr;
    for (const auto& ce : seq_cache_)
      if (ce.name == name && ce.r == r_) {
        cached = ce.seq;
        break;
      }
    if (cached) {
      launch_seq(*cached);
      return;
    }
    const std::string key =
        std::string(name) + "/" + std::to_string(r_) + "/" + key_ + "/" + std::to_string(c_->graph_epoch);
    auto it = w_->graphs.find(key);
    if (it == w_->graphs.end()) {
      std::unique_ptr<Sequence> sq(new Sequence());
      GSOT_CUDA_CHECK(cudaStreamBeginCapture(c_->stream, cudaStreamCaptureModeThreadLocal));
      c_->capturing = sq.get();
      try {
        body();
      } catch (...) {
        c_->capturing = nullptr;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(c_->stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      c_->capturing = nullptr;
      cudaGraph_t g = nullptr;
      GSOT_CUDA_CHECK(cudaStreamEndCapture(c_->stream, &g));
      GSOT_CUDA_CHECK(cudaGraphInstantiate(&sq->exec, g, 0));
      GSOT_CUDA_CHECK(cudaGraphDestroy(g));
      it = w_->graphs.emplace(key, std::move(sq)).first;
    }
    seq_cache_.push_back({name, r_, it->second.get()});
    launch_seq(*it->second);
  }

  struct SeqCacheEntry {
    const char* name;
    int r;
    Sequence* seq;
  };
  std::vector<SeqCacheEntry> seq_cache_;

  void launch_seq(Sequence& sq) {
    if (diag_) GSOT_CUDA_CHECK(cudaEventRecord(diag_ev_[0], c_->stream));
    const auto h0 = std::chrono::steady_clock::now();
    GSOT_CUDA_CHECK(cudaGraphLaunch(sq.exec, c_->stream));
    if (diag_) GSOT_CUDA_CHECK(cudaEventRecord(diag_ev_[1], c_->stream));
    c_->launches += sq.kernels;
    c_->pub_expected += static_cast<unsigned long long>(sq.publishes);
    if (sq.publishes > 0) c_->wait_published();
    if (sq.publishes == 0 || !sq.marks.empty()) c_->sync();
    if (diag_) {  // GSOT_DIAG_SEQ: device time vs host round trip per sequence
      c_->sync();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, diag_ev_[0], diag_ev_[1]);
      diag_dev_ += ms * 1e-3;
      diag_host_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
      diag_n_ += 1;
    }
    for (const auto& mk : sq.marks) c_->account(mk);
  }

  // The line-search step: the host writes it into the pinned mirror, a copy
  // node moves it to the device (GPU reads of mapped host memory measured
  // ~100 us per sequence on the B200 boxes; the copy node costs far less).
  void enqueue_t() {
    GSOT_CUDA_CHECK(cudaMemcpyAsync(&c_->dsync->t, &c_->h_sync->t, sizeof(double),
                                    cudaMemcpyHostToDevice, c_->stream));
  }
  const double* t_dev() const { return &c_->dsync->t; }
  // the first trial of a direction sequence uses t_init = 1 (lbfgs.hpp:150):
  // a device constant, so those graphs carry no copy node
  const double* t_one() const { return c_->d_one; }
  // fast screened solves: the step / trial kernels also write dbeta for the screen
  bool fast_screen() const { return screened_ && !exact_; }
  void enqueue_trial() {  // trial = X[r] + t d into X[1-r], evaluated into G[1-r]
    const int q = 1 - r_;
    enqueue_t();
    c_->launch(K_LBFGS, 24.0 * w_->dim, [&] {
      launch_axpy_point(w_->X[r_], t_dev(), w_->d, w_->X[q], w_->dim, c_->m, c_->snap_x,
                        fast_screen() ? c_->dbeta : nullptr, c_->stream);
    });
    enqueue_eval(c_, w_->X[q], mode_eval_, w_->G[q], w_->d, o_.upper_bound_offset, use_active_,
                 fast_screen());
  }

  // The search direction (lbfgs.hpp:109-126), optionally preceded by the
  // pending curvature pair of the last acceptance (lbfgs.hpp:243-255) and
  // followed by the first trial point x + t d into the trial buffer.
  // Exact mode: the reference's two-loop with sequential dots. Fast mode:
  // the compact representation in one cooperative launch (gsot_lbfgs.cu).
  void enqueue_direction(bool pair, bool trial) {
    const int q = 1 - r_;
    if (exact_) {
      ExactDirArgs a;
      a.pair = pair ? 1 : 0;
      a.x = w_->X[r_];
      a.xprev = w_->X[q];
      a.g = w_->G[r_];
      a.gprev = w_->G[q];
      a.S = w_->S;
      a.Y = w_->Y;
      a.stride = w_->dim;
      a.h = &c_->dsync->h;
      a.d = w_->d;
      a.dim = w_->dim;
      a.out = c_->dsync->tl;
      a.sc = c_->sc;
      c_->launch(K_LBFGS, 8.0 * w_->dim * (4.0 * w_->mem + 10.0),
                 [&] { launch_exact_direction(a, c_->ex, c_->stream); });
      if (trial)
        c_->launch(K_LBFGS, 24.0 * w_->dim, [&] {
          launch_axpy_point(w_->X[r_], t_one(), w_->d, w_->X[q], w_->dim, c_->m, c_->snap_x,
                            nullptr, c_->stream);
        });
      return;
    }
    // sharded: phase (1) -> the dots summed over the ranks -> phases (2)-(3)
    const int splits = sharded_ ? 2 : 0;
    for (int sp = splits ? 1 : 0; sp <= splits; ++sp) {
      if (sp == 2)
        c_->comm->allreduce(c_->comm->d_red, (mem_ + 1) * 5, GSOT_REDUCE_SUM, c_->stream);
      c_->launch(K_LBFGS, 8.0 * w_->dim * (4.0 * w_->mem + 10.0), [&] {
        launch_lbfgs_step(pair ? 1 : 0, w_->X[r_], w_->X[q], w_->G[r_], w_->G[q], w_->S, w_->Y,
                          w_->dim, &c_->dsync->h, w_->cs, w_->d, t_one(),
                          trial ? w_->X[q] : nullptr, w_->dim, c_->dsync->tl, c_->sc, w_->cpart,
                          mem_, c_->tl, c_->m, c_->snap_x, fast_screen() ? c_->dbeta : nullptr,
                          c_->stream, sp, c_->dot_lo(), sharded_ ? c_->comm->d_red : nullptr);
      });
    }
  }
  // |g|_inf over the ranks (alpha is replicated: max is idempotent)
  void reduce_extra0(int op) {
    if (sharded_) c_->comm->allreduce(&c_->sc->extra[0], 1, op, c_->stream);
  }

  // ---- bookkeeping ---------------------------------------------------------

  void record(const EvalOut& e) {  // GradStats (screening.hpp:280-287, solver.hpp:117-119)
    const int64_t row = res_->grad_calls;
    if (hist_ && row < hist_cap_) {
      hist_[row * 4 + 0] = e.stats.in_active;
      hist_[row * 4 + 1] = e.stats.skipped;
      hist_[row * 4 + 2] = e.stats.unskipped;
      hist_[row * 4 + 3] = e.stats.upper_bounds;
    }
    res_->blocks_in_active_set += e.stats.in_active;
    res_->blocks_skipped += e.stats.skipped;
    res_->blocks_unskipped += e.stats.unskipped;
    res_->upper_bounds_evaluated += e.stats.upper_bounds;
    ++res_->grad_calls;
    if ((mode_eval_ & 1) == GSOT_EVAL_SCREENED) {
      res_->eval_blocks += e.stats.in_active + e.stats.unskipped;
      res_->eval_tasks += c_->h_sc->ntasks;
    } else {
      res_->eval_blocks += static_cast<int64_t>(c_->L) * c_->n;  // this rank's blocks
      res_->eval_tasks += static_cast<int64_t>(c_->L) * c_->nw;
    }
  }

  double* px(int which) { return which == 0 ? w_->X[1 - r_] : which == 1 ? w_->lo_x : w_->prev_x; }
  double* pg(int which) { return which == 0 ? w_->G[1 - r_] : which == 1 ? w_->lo_g : w_->prev_g; }
  // dst = src for line-search points 0 trial, 1 lo, 2 prev (value copy).
  void assign(Pt* pts, int dst, int src) {
    if (dst == src) return;
    pts[dst] = pts[src];
    if (pts[src].vec) {
      const size_t b = sizeof(double) * w_->dim;
      GSOT_CUDA_CHECK(
          cudaMemcpyAsync(px(dst), px(src), b, cudaMemcpyDeviceToDevice, c_->stream));
      GSOT_CUDA_CHECK(
          cudaMemcpyAsync(pg(dst), pg(src), b, cudaMemcpyDeviceToDevice, c_->stream));
    }
  }

  // eval_at (lbfgs.hpp:84-90) for a further step of the current search.
  void eval_trial(double t, Pt& trial) {
    c_->h_sync->t = t;
    run_seq("T", [&] {
      enqueue_trial();
      c_->enqueue_fetch();
    });
    take_trial(t, trial);
  }
  void take_trial(double t, Pt& trial) {
    EvalOut e = eval_result(c_, mode_eval_);
    trial.t = t;
    trial.value = e.objective;
    trial.slope = e.slope;
    trial.vec = true;
    record(e);
    if (audit_) audit_call(w_->X[1 - r_], w_->G[1 - r_], e);
  }

  double norm_inf_now() {  // lpNorm<Infinity> of the iterate's gradient
    run_seq("N", [&] {
      c_->reset_scalars();
      c_->launch(K_LBFGS, 8.0 * w_->dim, [&] {
        launch_absmax(w_->G[r_], w_->dim, c_->partials, c_->red_blocks, c_->sc, 0, c_->stream);
      });
      reduce_extra0(GSOT_REDUCE_MAX);
      c_->enqueue_fetch();
    });
    return c_->h_sc->extra[0];
  }

  // chunk hook (solver.hpp:212-241) + the stop test (lbfgs.hpp:263-267)
  double hook_and_norm() {
    if (!screened_) return norm_inf_now();
    run_seq("RF", [&] {
      enqueue_refresh(c_, w_->X[r_], use_active_, true);
      c_->launch(K_LBFGS, 8.0 * w_->dim, [&] {
        launch_absmax(w_->G[r_], w_->dim, c_->partials, c_->red_blocks, c_->sc, 0, c_->stream);
      });
      reduce_extra0(GSOT_REDUCE_MAX);
      c_->enqueue_fetch();
    });
    const double nrm = c_->h_sc->extra[0];
    if (use_active_) c_->active_count = static_cast<int64_t>(c_->h_sc->counters[0]);
    if (audit_ && use_active_) audit_active(w_->X[r_]);
    return nrm;
  }

  void clear_history() {
    c_->launch(K_LBFGS, 0.0, [&] { launch_hist_reset(&c_->dsync->h, mem_, c_->stream); });
    hk_ = 0;
  }

  // ---- audit (solver.hpp:172-201, :215-240) ---------------------------------

  void audit_call(const double* d_x, const double* d_g, const EvalOut& e) {
    const DevProblem P = c_->problem();
    const gsot::DevSync saved = *c_->h_sync;
    c_->reset_scalars();
    c_->launch(K_MISC, 0.0, [&] {
      launch_audit_skips(P, d_x, c_->words, c_->active_words, c_->sc, c_->stream);
    });
    c_->fetch_scalars();
    res_->audit_skip_checks += static_cast<int64_t>(c_->h_sc->counters[0]);
    if (c_->h_sc->audit_violation) {
      const long long wv = c_->h_sc->audit_where;
      throw Error(GSOT_ERR_AUDIT_VIOLATION,
                  "audit violation: skipped block (l=" + std::to_string(wv / c_->n) +
                      ", j=" + std::to_string(wv % c_->n) +
                      ") has nonzero exact gradient at call " + std::to_string(res_->grad_calls));
    }
    if (!w_->audit_g) w_->audit_g = dalloc<double>(w_->dim + 8, &c_->bytes);
    EvalOut d = eval_device(c_, d_x, GSOT_EVAL_DENSE | (exact_ ? GSOT_EVAL_EXACT : 0), w_->audit_g,
                            nullptr, 0.0, false);
    std::vector<double> a(static_cast<size_t>(w_->dim)), b(static_cast<size_t>(w_->dim));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(a.data(), d_g, sizeof(double) * w_->dim,
                                    cudaMemcpyDeviceToHost, c_->stream));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(b.data(), w_->audit_g, sizeof(double) * w_->dim,
                                    cudaMemcpyDeviceToHost, c_->stream));
    c_->sync();
    res_->audit_column_compares += c_->n;
    if (memcmp(a.data(), b.data(), sizeof(double) * w_->dim) != 0 || d.objective != e.objective)
      throw Error(GSOT_ERR_AUDIT_VIOLATION,
                  "audit violation: screened gradient differs from plain gradient at call " +
                      std::to_string(res_->grad_calls));
    ++res_->audit_gradient_calls;
    *c_->h_sync = saved;
  }

  void audit_active(const double* d_x) {
    const DevProblem P = c_->problem();
    c_->reset_scalars();
    c_->launch(K_MISC, 0.0, [&] {
      launch_audit_active(P, d_x, c_->active_words, c_->sc, c_->stream);
    });
    c_->fetch_scalars();
    res_->audit_active_checks += static_cast<int64_t>(c_->h_sc->counters[1]);
    if (c_->h_sc->audit_violation) {
      const long long wv = c_->h_sc->audit_where;
      throw Error(GSOT_ERR_AUDIT_VIOLATION,
                  "audit violation: active-set block (l=" + std::to_string(wv / c_->n) + ", j=" +
                      std::to_string(wv % c_->n) + ") has zero exact gradient at build time");
    }
  }

  // ---- lbfgs.hpp:61-274 ------------------------------------------------------

  void maximize() {
    const double c1 = 1e-4, c2 = 0.9;  // MaximizeOptions (lbfgs.hpp:16-19)
    const int max_bracket = 40, max_zoom = 12;
    bool stalled = false, zero_gradient = false;
    bool pending_pair = false;
    Pt pts[3];  // 0 trial, 1 lo, 2 prev
    Pt& trial = pts[0];
    Pt& lo = pts[1];
    Pt& prev = pts[2];
    for (int chunk = 0; chunk < o_.max_outer_loops && !stalled && !zero_gradient; ++chunk) {
      ++res_->chunks;
      for (int it = 0; it < o_.snapshot_interval; ++it) {
        bool accepted = false;
        for (int attempt = 0; attempt < 2 && !accepted; ++attempt) {
          if (attempt == 1) {  // lbfgs.hpp:100-105
            if (hk_ == 0) break;
            clear_history();
          }
          // direction (two-loop) and, once the first step is known, the first
          // trial of the search in the same device sequence
          double dir_slope, dd;
          bool have_first = false;
          if (res_->iterations == 0) {
            run_seq(pending_pair ? "PD" : "D", [&] {
              enqueue_direction(pending_pair, false);
              c_->enqueue_fetch();
            });
          } else {
            run_seq(pending_pair ? "PDT" : "DT", [&] {  // first trial at t_init = 1
              enqueue_direction(pending_pair, true);
              enqueue_eval(c_, w_->X[1 - r_], mode_eval_, w_->G[1 - r_], w_->d,
                           o_.upper_bound_offset, use_active_, fast_screen());
              c_->enqueue_fetch();
            });
            have_first = true;
          }
          pending_pair = false;
          hk_ = c_->h_sync->h.k;
          dir_slope = c_->h_sync->tl[0];
          dd = c_->h_sync->tl[1];
          if (!(dir_slope > 0.0)) {  // lbfgs.hpp:127-137
            have_first = false;      // that trial used the rejected direction
            clear_history();
            GSOT_CUDA_CHECK(cudaMemcpyAsync(w_->d, w_->G[r_], sizeof(double) * w_->dim,
                                            cudaMemcpyDeviceToDevice, c_->stream));
            c_->reset_scalars();
            c_->launch(K_LBFGS, 16.0 * w_->dim, [&] {
              if (exact_)
                launch_exact_dot2(w_->G[r_], w_->G[r_], w_->dim, c_->ex, c_->sc, 0, c_->stream);
              else
                launch_dot(w_->G[r_] + c_->dot_lo(), w_->G[r_] + c_->dot_lo(),
                           w_->dim - c_->dot_lo(), c_->partials, c_->red_blocks, c_->sc, 0,
                           c_->stream);
            });
            reduce_extra0(GSOT_REDUCE_SUM);
            c_->fetch_scalars();
            dir_slope = c_->h_sc->extra[0];
            dd = dir_slope;
            if (dir_slope == 0.0) {
              zero_gradient = true;
              break;
            }
          }
          if (have_first) take_trial(1.0, trial);

          const double f0 = res_value_;  // lbfgs.hpp:141-148
          const double armijo = c1 * dir_slope;
          auto sufficient = [&](const Pt& p) { return p.value >= f0 + armijo * p.t; };
          auto curvature_ok = [&](const Pt& p) { return std::abs(p.slope) <= c2 * dir_slope; };

          double t_init = 1.0;  // lbfgs.hpp:150-154
          if (res_->iterations == 0) {
            const double dnorm = std::sqrt(dd);
            if (dnorm > 0.0) t_init = 1.0 / dnorm;
          }
          bool have_bracket = false;
          lo = Pt{0.0, f0, dir_slope, false};
          double hi_t = 0.0;
          double t = t_init;
          assign(pts, 2, 1);
          for (int i = 0; i < max_bracket; ++i) {  // lbfgs.hpp:165-187
            if (i == 0 && have_first && t == 1.0) {
              // the first trial already ran inside the direction sequence
            } else {
              eval_trial(t, trial);
            }
            if (!sufficient(trial) || (i > 0 && trial.value <= prev.value)) {
              assign(pts, 1, 2);
              hi_t = trial.t;
              have_bracket = true;
              break;
            }
            if (curvature_ok(trial)) {
              accepted = true;
              break;
            }
            if (trial.slope <= 0.0) {
              assign(pts, 1, 0);
              hi_t = prev.t;
              have_bracket = true;
              break;
            }
            assign(pts, 2, 0);
            t *= 2.0;
          }
          if (!accepted && have_bracket) {  // lbfgs.hpp:189-231
            double hi_value = std::numeric_limits<double>::quiet_NaN();
            for (int i = 0; i < max_zoom; ++i) {
              double cand = 0.5 * (lo.t + hi_t);
              if (std::isfinite(hi_value)) {
                const double dt = hi_t - lo.t;
                const double denom = 2.0 * (lo.value + lo.slope * dt - hi_value);
                if (denom != 0.0) {
                  const double interp = lo.t + lo.slope * dt * dt / denom;
                  const double lo_guard = lo.t + 0.1 * dt;
                  const double hi_guard = hi_t - 0.1 * dt;
                  const double lim_min = std::min(lo_guard, hi_guard);
                  const double lim_max = std::max(lo_guard, hi_guard);
                  if (interp >= lim_min && interp <= lim_max) cand = interp;
                }
              }
              if (cand == lo.t || cand == hi_t) break;
              eval_trial(cand, trial);
              if (!sufficient(trial) || trial.value <= lo.value) {
                hi_t = cand;
                hi_value = trial.value;
                continue;
              }
              if (curvature_ok(trial)) {
                accepted = true;
                break;
              }
              if (trial.slope * (hi_t - lo.t) <= 0.0) {
                hi_t = lo.t;
                hi_value = lo.value;
              }
              assign(pts, 1, 0);
            }
            if (!accepted && lo.t > 0.0) {
              assign(pts, 0, 1);
              accepted = true;
            }
          }
          if (!accepted && !have_bracket && prev.t > 0.0) {
            assign(pts, 0, 2);
            accepted = true;
          }
        }
        if (zero_gradient) break;
        if (!accepted) {
          stalled = true;
          break;
        }
        // accept: the trial buffer becomes the iterate; the curvature pair
        // (lbfgs.hpp:243-255) is formed at the start of the next sequence,
        // before the old iterate's buffer is reused.
        r_ = 1 - r_;
        res_value_ = trial.value;
        ++res_->iterations;
        pending_pair = true;
        trial.vec = lo.vec = prev.vec = false;
      }
      if (stalled) break;
      if (hook_and_norm() <= o_.grad_tol) {
        res_->converged = 1;
        break;
      }
    }
    if (!res_->converged) res_->converged = norm_inf_now() <= o_.grad_tol;
    res_->line_search_failed = stalled && !res_->converged;
  }

  gsot_ctx* c_;
  gsot_solver_options o_;
  gsot_solve_result* res_;
  int64_t* hist_;
  int64_t hist_cap_;
  SolverWorkspace* w_ = nullptr;
  std::string key_;
  int mem_ = 10;  // history capacity (lbfgs_memory)
  int r_ = 0;    // iterate buffer index
  int hk_ = 0;  // history length mirrored from the device
  double res_value_ = 0.0;
  bool screened_ = false, use_active_ = false, audit_ = false, graphs_ = true, exact_ = false;
  bool sharded_ = false;
  int mode_eval_ = GSOT_EVAL_DENSE;
};

}  // namespace

void run_solve(gsot_ctx* c, const gsot_solver_options& o, double* x_out, gsot_solve_result* res,
               int64_t* history, int64_t history_cap) {
  Solver s(c, o, res, history, history_cap);
  s.run(x_out);
}

}  // namespace gsot
