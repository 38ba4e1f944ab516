// gsot_ctx.cu — resident instance, evaluation pipeline, screening state and
// the C ABI of include/gsot.h (the solver lives in gsot_solver.cu).
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <vector>
#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "gsot_ctx.cuh"

namespace gsot {
int config_features(int cfg, uint64_t seed, double* src, double* tgt, int32_t* sizes, double* a,
                    double* b);
int config_shape(int cfg, int64_t* m, int64_t* n, int32_t* L, int64_t* d);
}  // namespace gsot

using gsot::Error;

using gsot::dalloc;

namespace {

thread_local std::string g_err;
thread_local gsot_error_detail g_detail{};

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    g_detail = gsot_error_detail{};
    return GSOT_OK;
  } catch (const Error& e) {
    g_err = e.what();
    g_detail = e.detail;
    g_detail.status = e.status;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    g_detail = gsot_error_detail{};
    g_detail.status = GSOT_ERR_OUT_OF_MEMORY;
    return GSOT_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_detail = gsot_error_detail{};
    g_detail.status = GSOT_ERR_CUDA;
    return GSOT_ERR_CUDA;
  }
}


void check_params(double gamma, double mu) {  // core.hpp:61-66
  if (!(gamma > 0.0) || !std::isfinite(gamma))
    throw Error(GSOT_ERR_INVALID_ARGUMENT, "gamma must be positive, got " + std::to_string(gamma));
  if (!(mu > 0.0) || !std::isfinite(mu))
    throw Error(GSOT_ERR_INVALID_ARGUMENT, "mu must be positive, got " + std::to_string(mu));
}

double compensated_sum(const double* v, int64_t n) {  // core.hpp:85-98
  double sum = 0.0, comp = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = v[i];
    const double t = sum + x;
    if (std::abs(sum) >= std::abs(x))
      comp += (sum - t) + x;
    else
      comp += (x - t) + sum;
    sum = t;
  }
  return sum + comp;
}

// shard: a column shard's partial marginals (gsot_create_shard) are checked
// entrywise only; the sum is the driver's (the full instance's) business.
void check_marginal(const double* v, int64_t n, char which, bool shard = false) {  // core.hpp:100-112
  for (int64_t i = 0; i < n; ++i) {
    if (!(v[i] >= 0.0) || !std::isfinite(v[i])) {
      Error e(GSOT_ERR_MARGINAL_NOT_NORMALIZED,
              std::string("marginal ") + which + ": entry " + std::to_string(i) + " = " +
                  std::to_string(v[i]) + " is negative or non-finite");
      e.detail.which = which;
      e.detail.index = i;
      throw e;
    }
  }
  if (shard) return;
  const double sum = compensated_sum(v, n);
  if (std::abs(sum - 1.0) > 1e-12) {
    Error e(GSOT_ERR_MARGINAL_NOT_NORMALIZED,
            std::string("marginal ") + which + ": sum = " + std::to_string(sum) +
                " differs from 1");
    e.detail.which = which;
    e.detail.index = -1;
    throw e;
  }
}

}  // namespace


int gsot_guard_call(const std::function<void()>& f) { return guard(f); }

gsot_ctx::~gsot_ctx() {
  if (stream) cudaStreamSynchronize(stream);
  ws.reset();
  for (auto& mk : marks) {
    cudaEventDestroy(mk.a);
    cudaEventDestroy(mk.b);
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  if (timer_a) cudaEventDestroy(timer_a);
  if (timer_b) cudaEventDestroy(timer_b);
  void* ptrs[] = {C,        d_off,   d_group_order, d_row_group, d_sqrt_g, d_a,     d_b,
                  x_eval,   g_eval,  rowpart,       colpart,     psi,      psicol,  partials,
                  words,    dense_words, dense_tasks, tasks, snap_x,   zs,      ks,
                  os,       dpos,    dfull,         dneg,        dbeta,    active_words, dsync,
                  cnt_partials, cnt_slots, d_pub_count, gmask, dense_gmask, cmask, dense_cmask, tl,
                  d_one, staging, d_bad, cmin, amax, snap_rows, snap_list, snap_cnt, dpos_fast, cmn, zmm, snap_zero, bmaxc, dbx3};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ex_ready) gsot::exact_ws_free(ex);
  if (h_sync) cudaFreeHost(h_sync);
  if (stream) cudaStreamDestroy(stream);
}

gsot::SolverWorkspace::~SolverWorkspace() {
  graphs.clear();
  void* ptrs[] = {X[0], X[1], G[0], G[1], lo_x, lo_g, prev_x, prev_g, d, S, Y, audit_g, cs, cpart};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

namespace {

// Partition + RegParams checks in the reference's constructor order
// (GroupPartition core.hpp:19-30, then RegParams :61-66), then layout.
void setup_shape(gsot_ctx* c, int64_t m, int64_t n, const int32_t* sizes, int32_t L, double gamma,
                 double mu) {
  if (L < 1 || sizes == nullptr) throw Error(GSOT_ERR_PARTITION_MISMATCH, "group partition: at least one group required");
  for (int32_t l = 0; l < L; ++l)
    if (sizes[l] < 1)
      throw Error(GSOT_ERR_PARTITION_MISMATCH,
                  "group partition: group " + std::to_string(l) + " has non-positive size " +
                      std::to_string(sizes[l]));
  check_params(gamma, mu);
  if (m < 1 || n < 1)
    throw Error(GSOT_ERR_DIMENSION_MISMATCH, "dimension mismatch: empty cost matrix");
  c->m = m;
  c->n = n;
  c->L = L;
  c->gamma = gamma;
  c->mu = mu;
  c->nw = static_cast<int32_t>((n + 31) / 32);
  c->sizes.assign(sizes, sizes + L);
  c->off.assign(static_cast<size_t>(L) + 1, 0);
  for (int32_t l = 0; l < L; ++l) c->off[l + 1] = c->off[l] + sizes[l];
}

void init_device(gsot_ctx* c) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    throw Error(GSOT_ERR_CUDA, "no CUDA device available (libgsot has no CPU fallback)");
  GSOT_CUDA_CHECK(cudaGetDevice(&c->device));
  GSOT_CUDA_CHECK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  GSOT_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->red_blocks = c->num_sms * 2;
}

void alloc_buffers(gsot_ctx* c) {
  size_t* t = &c->bytes;
  const int64_t m = c->m, n = c->n, L = c->L, nw = c->nw, dim = m + n;
  const size_t celems = static_cast<size_t>(32) * nw * m;  // column-tiled, n padded to 32
  c->C = dalloc<double>(celems, t);
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->C, 0, sizeof(double) * celems, c->stream));
  c->d_off = dalloc<int32_t>(L + 1, t);
  c->d_group_order = dalloc<int32_t>(L, t);
  c->d_row_group = dalloc<int32_t>(m, t);
  c->d_sqrt_g = dalloc<double>(L, t);
  c->d_a = dalloc<double>(m, t);
  c->d_b = dalloc<double>(n, t);
  c->x_eval = dalloc<double>(dim + 8, t);
  c->g_eval = dalloc<double>(dim + 8, t);
  c->rowpart = dalloc<double>(static_cast<size_t>(nw) * m, t);
  c->colpart = dalloc<double>(static_cast<size_t>(L) * n, t);
  c->psi = dalloc<double>(static_cast<size_t>(L) * n, t);
  c->psicol = dalloc<double>(n, t);
  c->partials = dalloc<double>(
      static_cast<size_t>(std::max<int64_t>(c->red_blocks, (m + 31) / 32 + (n + 31) / 32)) * 4 +
          64,
      t);
  c->cnt_slots = dalloc<unsigned long long>(64 * 8, t);
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->cnt_slots, 0, sizeof(unsigned long long) * 64 * 8, c->stream));
  c->cnt_partials = dalloc<unsigned long long>(
      static_cast<size_t>(std::max<int64_t>(c->num_sms * 64, L * ((nw + 7) / 8))) * 8, t);
  c->words = dalloc<uint32_t>(static_cast<size_t>(L) * nw, t);
  c->dense_words = dalloc<uint32_t>(static_cast<size_t>(L) * nw, t);
  c->gmask = dalloc<uint32_t>(static_cast<size_t>(L) * ((nw + 31) / 32), t);
  c->dense_gmask = dalloc<uint32_t>(static_cast<size_t>(L) * ((nw + 31) / 32), t);
  c->cmask = dalloc<uint32_t>(static_cast<size_t>(nw) * ((L + 31) / 32), t);
  c->dense_cmask = dalloc<uint32_t>(static_cast<size_t>(nw) * ((L + 31) / 32), t);
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->cmask, 0, sizeof(uint32_t) * nw * ((L + 31) / 32), c->stream));
  c->dense_tasks = dalloc<gsot::TaskDesc>(static_cast<size_t>(L) * nw, t);
  c->tasks = dalloc<gsot::TaskDesc>(static_cast<size_t>(L) * nw, t);
  c->snap_x = dalloc<double>(dim + 8, t);
  c->zs = dalloc<double>(static_cast<size_t>(L) * n, t);
  c->ks = dalloc<double>(static_cast<size_t>(L) * n, t);
  c->os = dalloc<double>(static_cast<size_t>(L) * n, t);
  c->dpos = dalloc<double>(L, t);
  c->dfull = dalloc<double>(L, t);
  c->dneg = dalloc<double>(L, t);
  c->dbeta = dalloc<double>(n, t);
  c->cmin = dalloc<float>(static_cast<size_t>(L) * n, t);
  c->snap_rows = dalloc<unsigned long long>(64, t);
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->snap_rows, 0, sizeof(unsigned long long) * 64, c->stream));
  if (!std::getenv("GSOT_SNAP_SCATTERED")) {  // (GSOT_SNAP_SCATTERED=1: the one-kernel lazy form)
    c->snap_list = dalloc<uint32_t>(static_cast<size_t>(L) * n, t);
    c->snap_cnt = dalloc<unsigned int>(L, t);
  }
  c->amax = dalloc<double>(L, t);
  c->dpos_fast = dalloc<double>(L, t);
  c->cmn = dalloc<float>(static_cast<size_t>(L) * nw, t);
  c->zmm = dalloc<double2>(static_cast<size_t>(L) * nw, t);
  c->bmaxc = dalloc<double>(nw, t);
  c->dbx3 = dalloc<double>(3 * static_cast<size_t>(nw), t);
  c->snap_zero = dalloc<unsigned char>(static_cast<size_t>(L) * nw, t);
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->snap_zero, 0, static_cast<size_t>(L) * nw, c->stream));
  c->active_words = dalloc<uint32_t>(static_cast<size_t>(L) * nw, t);
  c->dsync = dalloc<gsot::DevSync>(1, t);
  GSOT_CUDA_CHECK(cudaHostAlloc(&c->h_sync, sizeof(gsot::DevSync) + 128, cudaHostAllocMapped));
  c->h_flag = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(c->h_sync) +
                                                    sizeof(gsot::DevSync) + 64 -
                                                    sizeof(gsot::DevSync) % 64);
  GSOT_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_sync_dev), c->h_sync, 0));
  GSOT_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_flag_dev), c->h_flag, 0));
  c->d_pub_count = dalloc<unsigned long long>(1, t);
  c->d_one = dalloc<double>(1, t);
  {
    const double one = 1.0;
    GSOT_CUDA_CHECK(cudaMemcpy(c->d_one, &one, sizeof(double), cudaMemcpyHostToDevice));
  }
#ifdef GSOT_PHASE_CLOCKS
  if (std::getenv("GSOT_TIMELINE")) {  // diagnostic kernel timeline
    c->tl = dalloc<unsigned long long>(64, t);
    unsigned long long init[64] = {};
    for (int k = 0; k < 8; ++k) init[2 * k] = ~0ull;
    GSOT_CUDA_CHECK(cudaMemcpy(c->tl, init, sizeof(init), cudaMemcpyHostToDevice));
  }
#endif
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->d_pub_count, 0, sizeof(unsigned long long), c->stream));
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->dsync, 0, sizeof(gsot::DevSync), c->stream));
  memset(c->h_sync, 0, sizeof(gsot::DevSync) + 128);
  c->pub_expected = 0;
  c->sc = &c->dsync->sc;
  c->h_sc = &c->h_sync->sc;
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->x_eval, 0, sizeof(double) * (dim + 8), c->stream));
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->snap_x, 0, sizeof(double) * (dim + 8), c->stream));

  std::vector<int32_t> row_group(static_cast<size_t>(m)), order(static_cast<size_t>(L));
  std::vector<double> sqrt_g(static_cast<size_t>(L));
  for (int32_t l = 0; l < L; ++l) {
    sqrt_g[l] = std::sqrt(static_cast<double>(c->sizes[l]));  // screening.hpp:79
    for (int32_t r = 0; r < c->sizes[l]; ++r) row_group[c->off[l] + r] = l;
    order[l] = l;
  }
  // dense work list: largest groups (longest per-lane chains) first
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t p, int32_t q) { return c->sizes[p] > c->sizes[q]; });
  GSOT_CUDA_CHECK(cudaMemcpyAsync(c->d_off, c->off.data(), sizeof(int32_t) * (L + 1),
                                  cudaMemcpyHostToDevice, c->stream));
  GSOT_CUDA_CHECK(cudaMemcpyAsync(c->d_group_order, order.data(), sizeof(int32_t) * L,
                                  cudaMemcpyHostToDevice, c->stream));
  GSOT_CUDA_CHECK(cudaMemcpyAsync(c->d_row_group, row_group.data(), sizeof(int32_t) * m,
                                  cudaMemcpyHostToDevice, c->stream));
  GSOT_CUDA_CHECK(cudaMemcpyAsync(c->d_sqrt_g, sqrt_g.data(), sizeof(double) * L,
                                  cudaMemcpyHostToDevice, c->stream));
  c->launch(gsot::K_MISC, 0, [&] { gsot::launch_fill_words(c->dense_words, c->L, c->nw, c->n, c->stream); });
  c->launch(gsot::K_MISC, 0, [&] { gsot::launch_fill_gmask(c->dense_gmask, c->L, c->nw, c->stream); });
  c->launch(gsot::K_MISC, 0, [&] { gsot::launch_fill_cmask(c->dense_cmask, c->L, c->nw, c->stream); });
  c->launch(gsot::K_MISC, 0, [&] { gsot::launch_dense_tasks(c->problem(), c->dense_tasks, c->d_group_order, c->stream); });
  // Persistent eval grid: two shared-memory segments of up to 128 rows per
  // CTA (the tallest group when it fits), as many CTAs per SM as shared
  // memory allows (GSOT_EVAL_SEG overrides the segment rows for tuning).
  {
    const int gmax = *std::max_element(c->sizes.begin(), c->sizes.end());
    int seg = gsot::eval_buf_rows(gmax);
    if (const char* ev = std::getenv("GSOT_EVAL_SEG")) seg = std::max(8, std::min(128, std::atoi(ev)));
    // tiles taller than a segment: the recomputing variant (k_eval<true>)
    bool rec = gmax > seg;
    if (const char* ev = std::getenv("GSOT_EVAL_RECOMPUTE")) rec = std::atoi(ev) != 0;
    int var = gsot::eval_variant(gmax, seg, rec);
    int qrows = 0;
    // groups taller than a whole-tile segment: the quarter pipeline
    // (GSOT_EVAL_TALL_OLD=1 keeps the two-pass recomputing variant, for comparison)
    if (var == 1 && !std::getenv("GSOT_EVAL_TALL_OLD")) {
      var = 3;
      qrows = gsot::eval_qrows_for(gmax);
      seg = gsot::eval_q_short_rows(qrows);
    }
    const int bps = gsot::eval_blocks_per_sm(gsot::eval_smem_bytes(seg, qrows), var);
    c->eval_recompute = rec;
    c->eval_variant = var;
    c->eval_buf = seg;
    c->eval_qrows = qrows;
    c->eval_grid = c->num_sms * bps;
    if (std::getenv("GSOT_DIAG_SEQ"))
      std::fprintf(stderr, "[gsot diag] eval: %d rows per segment, %d CTAs per SM, %zu B shared, variant %d\n",
                   seg, bps, gsot::eval_smem_bytes(seg, qrows), var);
  }
  c->sync();
}

void set_marginals(gsot_ctx* c, const double* a, const double* b) {
  GSOT_CUDA_CHECK(cudaMemcpyAsync(c->d_a, a, sizeof(double) * c->m, cudaMemcpyHostToDevice, c->stream));
  GSOT_CUDA_CHECK(cudaMemcpyAsync(c->d_b, b, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
}

// validate_instance (core.hpp:117-139) order: cost scan (first offender in
// j-major order, computed on device during the upload), a, b, partition.
void finish_validation(gsot_ctx* c, unsigned long long* d_first_bad, const double* a,
                       const double* b, const double* d_src_for_value, bool shard = false) {
  unsigned long long first_bad = 0;
  GSOT_CUDA_CHECK(cudaMemcpyAsync(&first_bad, d_first_bad, sizeof(first_bad),
                                  cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (first_bad != ~0ull) {
    const int64_t row = static_cast<int64_t>(first_bad % static_cast<unsigned long long>(c->m));
    const int64_t col = static_cast<int64_t>(first_bad / static_cast<unsigned long long>(c->m));
    double value = 0.0;
    int32_t l = 0;
    while (c->off[l + 1] <= row) ++l;
    const int64_t o0 = c->off[l], g = c->sizes[l];
    const int64_t el = gsot::cost_index(c->nw, o0, g, col, row - o0);
    GSOT_CUDA_CHECK(cudaMemcpy(&value, c->C + el, sizeof(double), cudaMemcpyDeviceToHost));
    (void)d_src_for_value;
    Error e(GSOT_ERR_NEGATIVE_COST, "cost(" + std::to_string(row) + "," + std::to_string(col) +
                                        ") = " + std::to_string(value) +
                                        " is negative or non-finite");
    e.detail.row = row;
    e.detail.col = col;
    e.detail.value = value;
    throw e;
  }
  check_marginal(a, c->m, 'a', shard);
  check_marginal(b, c->n, 'b', shard);
  if (c->off[c->L] != c->m)
    throw Error(GSOT_ERR_PARTITION_MISMATCH,
                "group partition: partition covers " + std::to_string(c->off[c->L]) +
                    " indices, cost has " + std::to_string(c->m) + " rows");
  // the per-block minimum cost of the valid instance (provably-zero blocks)
  c->launch(gsot::K_MISC, 8.0 * c->m * c->n, [&] { gsot::launch_block_min(c->problem(), c->cmin, c->stream); });
}

// Context cache: gsot_destroy parks a context's device state (buffers,
// stream, captured graphs) and gsot_create of the same shape and partition
// on the same device takes it back, re-uploading only the data. Repeated
// solves of same-shape instances then skip allocation, frees and graph
// capture (like a caching allocator). GSOT_CTX_CACHE=0 disables it.
namespace {
std::mutex g_cache_mu;
std::vector<gsot_ctx*> g_cache;
constexpr size_t kCacheMax = 2;

bool cache_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GSOT_CTX_CACHE");
    return !(e && e[0] == '0');
  }();
  return on;
}

gsot_ctx* cache_take(int64_t m, int64_t n, const int32_t* sizes, int32_t L) {
  if (!cache_enabled()) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(g_cache_mu);
  for (size_t k = 0; k < g_cache.size(); ++k) {
    gsot_ctx* c = g_cache[k];
    if (c->device == dev && c->m == m && c->n == n && c->L == L &&
        std::equal(c->sizes.begin(), c->sizes.end(), sizes)) {
      g_cache.erase(g_cache.begin() + k);
      return c;
    }
  }
  return nullptr;
}

// Free every parked context (all devices). Returns how many were freed.
size_t cache_drain() {
  std::vector<gsot_ctx*> victims;
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    victims.swap(g_cache);
  }
  for (gsot_ctx* v : victims) delete v;
  return victims.size();
}
}  // namespace

void park_or_delete(gsot_ctx* c) {
  if (!c) return;
  if (c->comm) {  // a communicator never outlives its owner's handle
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->comm.reset();
    c->pending_grad = nullptr;
    ++c->graph_epoch;
  }
  if (!cache_enabled() || !c->cacheable || cudaStreamSynchronize(c->stream) != cudaSuccess) {
    delete c;
    return;
  }
  gsot_ctx* evict = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    g_cache.push_back(c);
    if (g_cache.size() > kCacheMax) {
      evict = g_cache.front();
      g_cache.erase(g_cache.begin());
    }
  }
  delete evict;
}

gsot_ctx* create_common(const double* cost, bool cost_on_device, int64_t m, int64_t n,
                        const int32_t* sizes, int32_t L, const double* a, const double* b,
                        double gamma, double mu, bool shard = false) {
  gsot_ctx* c = (sizes && L > 0 && m > 0 && n > 0) ? cache_take(m, n, sizes, L) : nullptr;
  const bool reused = c != nullptr;
  if (!c) c = new gsot_ctx();
  c->cacheable = false;  // until the new data is in
  try {
    if (reused) {  // same shape and partition: device state as parked
      check_params(gamma, mu);
      if (gamma != c->gamma || mu != c->mu) {
        c->gamma = gamma;
        c->mu = mu;
        if (c->ws) c->ws->graphs.clear();  // graphs bake (gamma, mu) into kernel parameters
      }
      c->have_snapshot = false;
      c->active_count = 0;
      GSOT_CUDA_CHECK(cudaMemsetAsync(c->sc, 0, sizeof(gsot::EvalScalars), c->stream));
      GSOT_CUDA_CHECK(cudaMemsetAsync(c->cnt_slots, 0, sizeof(unsigned long long) * 64 * 8, c->stream));
      GSOT_CUDA_CHECK(cudaMemsetAsync(
          c->cmask, 0, sizeof(uint32_t) * c->nw * ((c->L + 31) / 32), c->stream));
    } else {
      setup_shape(c, m, n, sizes, L, gamma, mu);
    }
    if (c->off[L] != m) {
      // The reference checks the cover last (core.hpp:134-138) but the
      // layout needs it; the scan order of the remaining checks is kept.
      if (!cost_on_device && cost) {
        for (int64_t j = 0; j < n; ++j)
          for (int64_t i = 0; i < m; ++i) {
            const double v = cost[i + j * m];
            if (!(v >= 0.0) || !std::isfinite(v)) {
              Error e(GSOT_ERR_NEGATIVE_COST, "cost(" + std::to_string(i) + "," +
                                                  std::to_string(j) + ") = " +
                                                  std::to_string(v) + " is negative or non-finite");
              e.detail.row = i;
              e.detail.col = j;
              e.detail.value = v;
              throw e;
            }
          }
      }
      check_marginal(a, m, 'a', shard);
      check_marginal(b, n, 'b', shard);
      throw Error(GSOT_ERR_PARTITION_MISMATCH,
                  "group partition: partition covers " + std::to_string(c->off[L]) +
                      " indices, cost has " + std::to_string(m) + " rows");
    }
    if (!reused) {
      try {
        init_device(c);
        alloc_buffers(c);
      } catch (const Error& e) {
        // Parked contexts hold HBM (a config-5 cost alone is 40 GB): on an
        // allocation failure free them all and retry once on a fresh context.
        if (e.status != GSOT_ERR_OUT_OF_MEMORY || cache_drain() == 0) throw;
        cudaGetLastError();
        delete c;
        c = new gsot_ctx();
        setup_shape(c, m, n, sizes, L, gamma, mu);
        init_device(c);
        alloc_buffers(c);
      }
    }
    set_marginals(c, a, b);
    // Upload in column chunks through a staging buffer (bounded extra HBM;
    // kept by the context for the next upload of a cached context).
    if (!c->d_bad) GSOT_CUDA_CHECK(cudaMalloc(&c->d_bad, sizeof(unsigned long long)));
    unsigned long long* d_bad = c->d_bad;
    GSOT_CUDA_CHECK(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), c->stream));
    const int64_t chunk_cols =
        std::max<int64_t>(1, std::min<int64_t>(n, (int64_t(256) << 20) / (8 * m)));
    if (!cost_on_device && !c->staging)
      GSOT_CUDA_CHECK(cudaMalloc(&c->staging, sizeof(double) * m * chunk_cols));
    double* staging = c->staging;
    for (int64_t j0 = 0; j0 < n; j0 += chunk_cols) {
      const int64_t nc = std::min(chunk_cols, n - j0);
      const double* src = nullptr;
      if (cost_on_device) {
        src = cost + j0 * m;
      } else {
        GSOT_CUDA_CHECK(cudaMemcpyAsync(staging, cost + j0 * m, sizeof(double) * m * nc,
                                        cudaMemcpyHostToDevice, c->stream));
        src = staging;
      }
      c->launch(gsot::K_MISC, 16.0 * m * nc, [&] {
        gsot::launch_relayout(c->problem(), src, j0, nc, c->C, d_bad, c->stream);
      });
    }
    finish_validation(c, d_bad, a, b, nullptr, shard);
    c->cacheable = true;
    return c;
  } catch (...) {
    delete c;
    throw;
  }
}

// ------------------------------------------------------------------ eval

}  // namespace

namespace gsot {

void enqueue_eval(gsot_ctx* c, const double* d_x, int mode_flags, double* d_grad,
                  const double* d_dir, double ub_offset, bool use_active, bool dbeta_ready) {
  const bool exact = (mode_flags & GSOT_EVAL_EXACT) != 0;
  const int mode = mode_flags & 1;
  if (exact && c->comm)
    throw Error(GSOT_ERR_INVALID_ARGUMENT, "exact-order evaluation of a sharded context");
  if (c->comm) c->pending_grad = d_grad;  // its head is summed over the ranks at publication
  if (exact) c->ensure_exact();
  if (mode == GSOT_EVAL_SCREENED && !c->have_snapshot)
    throw Error(GSOT_ERR_STATE, "screened evaluation requires a snapshot (gsot_init_snapshot)");
  const DevProblem P = c->problem();
  if (mode != GSOT_EVAL_SCREENED || exact) c->reset_scalars();  // screened: zeroed by k_publish
  // per-group max alpha for the provably-zero block test (k_block_min): read
  // by the screen and the evaluation
  const bool fused = mode == GSOT_EVAL_SCREENED && dbeta_ready && !exact;
  const bool summ = mode == GSOT_EVAL_SCREENED && screen_uses_summaries(P, c->num_sms);
  const bool pre = fused && summ;  // delta norms once per group
  // Fast solves fuse the group delta norms into the screen (the step / trial
  // kernel wrote dbeta); every other screened evaluation -- exact mode and
  // the API's gsot_eval -- takes the reference-order norms of k_delta, so
  // its decisions and counters are the reference's bit for bit.
  if (mode == GSOT_EVAL_SCREENED && !fused)
    c->launch(K_DELTA, 16.0 * (c->m + c->n) + 32.0 * c->L + 8.0 * c->n, [&] {
      launch_delta(P, d_x, c->snap_x, c->dpos, c->dfull, c->dneg, c->dbeta, nullptr, nullptr,
                   c->stream);
    });
  // (after dbeta is final: the chunk role reads it)
  c->launch(K_MISC, 8.0 * c->m, [&] {
    launch_group_amax(P, d_x, c->amax, c->stream, nullptr, pre ? c->snap_x : nullptr,
                      pre ? c->dpos_fast : nullptr, summ ? c->dbeta : nullptr,
                      summ ? c->dbx3 : nullptr);
  });
  const uint32_t* words = c->dense_words;
  const double Ln = static_cast<double>(c->L) * c->n;
  if (mode == GSOT_EVAL_SCREENED) {
    c->launch(K_BOUNDS, 8.0 * Ln + 8.0 * c->L * c->nw, [&] {
      launch_screen(P, c->zs, use_active ? c->active_words : nullptr, c->dpos, c->dbeta,
                    ub_offset, c->words, c->tasks, c->sc, c->cnt_slots, c->gmask,
                    c->cmask, fused ? d_x : nullptr, fused ? c->snap_x : nullptr,
                    fused ? 1 : 0, d_x, pre ? c->dpos_fast : nullptr, c->zmm, c->dbx3, c->num_sms,
                    c->stream);
    });
    words = c->words;
  }
  if (exact) {  // the reference's order of operations (gsot_exact2.cu)
    const bool scr = mode == GSOT_EVAL_SCREENED;
    c->launch(K_EVAL, 0.0, [&] {
      launch_exact_eval2(P, c->ex, d_x, scr ? c->words : c->dense_words,
                         scr ? c->gmask : c->dense_gmask, scr ? c->cmask : c->dense_cmask,
                         scr ? 1 : 0, d_grad, d_dir, c->sc, scr ? c->cnt_slots : nullptr,
                         c->stream);
    });
    return;
  }
  const double dense_bytes = 8.0 * c->m * c->n + 8.0 * c->m * c->nw + 16.0 * Ln;
  c->launch(K_EVAL, mode == GSOT_EVAL_DENSE ? dense_bytes : -1.0, [&] {
    if (mode == GSOT_EVAL_SCREENED)
      launch_eval(P, d_x, c->tasks, -1, &c->sc->ntasks, words, c->rowpart, c->colpart, c->psi,
                  c->eval_buf, c->eval_qrows, c->eval_variant, c->eval_grid, &c->sc->next_task,
                  screen_uses_summaries(P, c->num_sms), c->stream);
    else
      launch_eval(P, d_x, c->dense_tasks, c->L * c->nw, nullptr, words, c->rowpart, c->colpart,
                  c->psi, c->eval_buf, c->eval_qrows, c->eval_variant, c->eval_grid, &c->sc->next_task,
                  false, c->stream);
  });
  c->launch(K_FINALIZE, 16.0 * (c->m + c->n), [&] {
    const bool scr = mode == GSOT_EVAL_SCREENED;
    launch_finalize(P, d_x, words, scr ? c->gmask : c->dense_gmask,
                    scr ? c->cmask : c->dense_cmask, scr ? 1 : 0, c->rowpart, c->colpart,
                    c->psi, d_grad, d_dir, c->partials, c->sc, scr ? 1 : 0, c->stream);
  });
}

EvalOut eval_result(gsot_ctx* c, int mode_flags) {
  const int mode = mode_flags & 1;
  EvalOut o;
  o.objective = c->h_sc->objective;
  o.slope = c->h_sc->slope;
  if (mode == GSOT_EVAL_SCREENED) {
    o.stats.in_active = static_cast<int64_t>(c->h_sc->counters[0]);
    o.stats.skipped = static_cast<int64_t>(c->h_sc->counters[1]);
    o.stats.unskipped = static_cast<int64_t>(c->h_sc->counters[2]);
    o.stats.upper_bounds = static_cast<int64_t>(c->h_sc->counters[3]);
  } else {
    o.stats.unskipped = static_cast<int64_t>(c->L) * c->n_global();  // solver.hpp:117-119
  }
  return o;
}

EvalOut eval_device(gsot_ctx* c, const double* d_x, int mode, double* d_grad,
                    const double* d_dir, double ub_offset, bool use_active) {
  enqueue_eval(c, d_x, mode, d_grad, d_dir, ub_offset, use_active);
  c->fetch_scalars();
  return eval_result(c, mode);
}

void enqueue_snapshot(gsot_ctx* c, const double* d_x, bool lazy) {  // take_snapshot (screening.hpp:24-50)
  const DevProblem P = c->problem();
  const double Ln = static_cast<double>(c->L) * c->n;
  unsigned int* list_len = c->snap_cnt;
  // (short groups are walked by the marking kernel itself; they still gain its
  // chunk-level zero test and flags)
  const bool listed = lazy && c->snap_list != nullptr;
  if (lazy)
    c->launch(K_MISC, 8.0 * c->m, [&] {
      launch_group_amax(P, d_x, c->amax, c->stream, listed ? list_len : nullptr);
    });
  c->launch(K_SNAPSHOT, lazy ? -2.0 : 8.0 * c->m * c->n + 24.0 * Ln + 8.0 * (c->m + c->n), [&] {
    if (listed) ++c->launches;  // two kernels
    if (listed)
      launch_snapshot_lazy2(P, d_x, c->zs, c->ks, c->os, c->snap_list, list_len, c->snap_rows,
                            c->snap_zero, c->zmm, c->bmaxc, c->stream);
    if (listed) ++c->launches;  // k_chunk_bmax
    else
      launch_snapshot(P, d_x, c->zs, c->ks, c->os, lazy, c->snap_rows, c->stream);
  });
  // per-chunk extremes of z~ for the screen's whole-chunk decisions
  if (!listed)  // the arrays were written in full: no chunk is known to hold zeros
    GSOT_CUDA_CHECK(cudaMemsetAsync(c->snap_zero, 0, static_cast<size_t>(c->L) * c->nw, c->stream));
  if (screen_uses_summaries(P, c->num_sms))
    c->launch(K_MISC, 8.0 * Ln, [&] {
      launch_chunk_minmax(P, c->zs, c->zmm, listed ? c->snap_zero : nullptr, c->stream);
    });
  c->snap_lazy = lazy;
  if (d_x != c->snap_x)
    GSOT_CUDA_CHECK(cudaMemcpyAsync(c->snap_x, d_x, sizeof(double) * (c->m + c->n),
                                    cudaMemcpyDeviceToDevice, c->stream));
  c->have_snapshot = true;
}

void init_snapshot_device(gsot_ctx* c, const double* d_x, bool lazy) {  // screening.hpp:220-227
  enqueue_snapshot(c, d_x, lazy);
  GSOT_CUDA_CHECK(cudaMemsetAsync(c->active_words, 0,
                                  sizeof(uint32_t) * static_cast<size_t>(c->L) * c->nw, c->stream));
  c->active_count = 0;
}

// FastGradDispatcher::refresh (screening.hpp:231-235): active set from the
// lower bounds against the current snapshot, then the new snapshot. The
// active-set size lands in sc->counters[0] (reset first).
void enqueue_refresh(gsot_ctx* c, const double* d_x, bool use_active, bool lazy) {
  if (!c->have_snapshot) throw Error(GSOT_ERR_STATE, "refresh requires a snapshot");
  const DevProblem P = c->problem();
  c->reset_scalars();
  if (use_active) {
    c->launch(K_DELTA, 16.0 * (c->m + c->n), [&] {
      launch_delta(P, d_x, c->snap_x, c->dpos, c->dfull, c->dneg, c->dbeta, nullptr, nullptr,
                   c->stream);
    });
    c->launch(K_ACTIVE, 16.0 * c->L * c->n + 4.0 * c->L * c->nw, [&] {
      launch_active(P, c->ks, c->os, c->dfull, c->dneg, c->dbeta, c->active_words, c->sc,
                    c->stream);
    });
  }
  enqueue_snapshot(c, d_x, lazy);
}

void refresh_device(gsot_ctx* c, const double* d_x, bool use_active) {
  enqueue_refresh(c, d_x, use_active, false);
  c->fetch_scalars();
  if (use_active) c->active_count = static_cast<int64_t>(c->h_sc->counters[0]);
}

}  // namespace gsot

using gsot::EvalOut;
using gsot::eval_device;
using gsot::init_snapshot_device;
using gsot::refresh_device;

namespace {

gsot_ctx* checked(gsot_ctx* c) {
  if (!c) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null context");
  return c;
}

void upload_x(gsot_ctx* c, const double* x) {
  if (!x) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null state");
  GSOT_CUDA_CHECK(cudaMemcpyAsync(c->x_eval, x, sizeof(double) * (c->m + c->n),
                                  cudaMemcpyHostToDevice, c->stream));
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

GSOT_API const char* gsot_last_error(void) { return g_err.c_str(); }

GSOT_API int gsot_last_error_detail(gsot_error_detail* out) {
  if (out) *out = g_detail;
  return GSOT_OK;
}

GSOT_API const char* gsot_version(void) { return "gsot-b200 0.1 (sm_100a)"; }

GSOT_API int gsot_params_from_rho(double gamma, double rho, double* gamma_eff, double* mu_eff) {
  return guard([&] {
    if (!(rho > 0.0) || !(rho < 1.0)) {  // core.hpp:148-151, errors.hpp:49-56
      Error e(GSOT_ERR_RHO_OUT_OF_RANGE,
              "rho = " + std::to_string(rho) + " is outside the open interval (0,1)");
      e.detail.value = rho;  // RhoOutOfRange::rho
      throw e;
    }
    const double g = gamma * (1.0 - rho), mu = rho / (1.0 - rho);
    check_params(g, mu);
    if (gamma_eff) *gamma_eff = g;
    if (mu_eff) *mu_eff = mu;
  });
}

GSOT_API int gsot_create(const double* cost, int64_t m, int64_t n, const int32_t* group_sizes,
                         int32_t L, const double* a, const double* b, double gamma, double mu,
                         gsot_ctx** out) {
  return guard([&] {
    if (!out || !cost || !a || !b) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    *out = create_common(cost, false, m, n, group_sizes, L, a, b, gamma, mu);
  });
}

GSOT_API int gsot_create_device(const double* d_cost, int64_t m, int64_t n,
                                const int32_t* group_sizes, int32_t L, const double* a,
                                const double* b, double gamma, double mu, gsot_ctx** out) {
  return guard([&] {
    if (!out || !d_cost || !a || !b) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    *out = create_common(d_cost, true, m, n, group_sizes, L, a, b, gamma, mu);
  });
}

GSOT_API int gsot_create_shard(const double* cost, int64_t m, int64_t n_shard,
                               const int32_t* group_sizes, int32_t L, const double* a,
                               const double* b_shard, double gamma, double mu, gsot_ctx** out) {
  return guard([&] {
    if (!out || !cost || !a || !b_shard) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    *out = create_common(cost, false, m, n_shard, group_sizes, L, a, b_shard, gamma, mu, true);
  });
}

GSOT_API int gsot_create_shard_device(const double* d_cost, int64_t m, int64_t n_shard,
                                      const int32_t* group_sizes, int32_t L, const double* a,
                                      const double* b_shard, double gamma, double mu,
                                      gsot_ctx** out) {
  return guard([&] {
    if (!out || !d_cost || !a || !b_shard) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    *out = create_common(d_cost, true, m, n_shard, group_sizes, L, a, b_shard, gamma, mu, true);
  });
}

GSOT_API void gsot_destroy(gsot_ctx* ctx) { park_or_delete(ctx); }

GSOT_API int64_t gsot_cache_clear(void) { return static_cast<int64_t>(cache_drain()); }

extern "C" __attribute__((visibility("default"))) int gsot_debug_seq_prof(unsigned long long* out8) {
  return guard([&] { gsot::read_seq_prof(out8); });
}

GSOT_API int gsot_sequential_sum(gsot_ctx* ctx, const double* terms, int64_t n, double s0,
                                 double* out) {
  return guard([&] {
    checked(ctx);
    if (n < 0 || (n > 0 && !terms) || !out) throw Error(GSOT_ERR_INVALID_ARGUMENT, "bad arguments");
    ctx->ensure_exact();
    double* d = dalloc<double>(static_cast<size_t>(n) + 1, nullptr);
    double* r = dalloc<double>(1, nullptr);
    try {
      if (n > 0)
        GSOT_CUDA_CHECK(cudaMemcpyAsync(d, terms, sizeof(double) * n, cudaMemcpyHostToDevice,
                                        ctx->stream));
      ctx->launch(gsot::K_MISC, 8.0 * n, [&] { gsot::launch_seqsum(d, n, s0, ctx->ex, r, ctx->stream); });
      GSOT_CUDA_CHECK(cudaMemcpyAsync(out, r, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
    } catch (...) {
      cudaFree(d);
      cudaFree(r);
      throw;
    }
    cudaFree(d);
    cudaFree(r);
  });
}

GSOT_API int gsot_set_upper_bound_offset(gsot_ctx* ctx, double offset) {
  return guard([&] {
    checked(ctx);
    if (!std::isfinite(offset)) throw Error(GSOT_ERR_INVALID_ARGUMENT, "non-finite offset");
    ctx->ub_offset = offset;
  });
}

GSOT_API int gsot_set_params(gsot_ctx* ctx, double gamma, double mu) {
  return guard([&] {
    checked(ctx);
    check_params(gamma, mu);
    if (gamma != ctx->gamma || mu != ctx->mu) {
      ctx->gamma = gamma;
      ctx->mu = mu;
      if (ctx->ws) ctx->ws->graphs.clear();  // graphs bake (gamma, mu) into kernel parameters
    }
  });
}

GSOT_API int gsot_shape(const gsot_ctx* ctx, int64_t* m, int64_t* n, int32_t* L,
                        int64_t* device_bytes) {
  return guard([&] {
    if (!ctx) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null context");
    if (m) *m = ctx->m;
    if (n) *n = ctx->n;
    if (L) *L = ctx->L;
    if (device_bytes) *device_bytes = static_cast<int64_t>(ctx->bytes);
  });
}

GSOT_API int gsot_eval(gsot_ctx* ctx, const double* x, int mode, double* objective, double* grad,
                       gsot_call_stats* stats) {
  return guard([&] {
    checked(ctx);
    if (mode < 0 || mode > 3) throw Error(GSOT_ERR_INVALID_ARGUMENT, "unknown eval mode");
    upload_x(ctx, x);
    EvalOut e = eval_device(ctx, ctx->x_eval, mode, ctx->g_eval, nullptr, ctx->ub_offset, true);
    if (grad) {
      GSOT_CUDA_CHECK(cudaMemcpyAsync(grad, ctx->g_eval, sizeof(double) * (ctx->m + ctx->n),
                                      cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
    }
    if (objective) *objective = e.objective;
    if (stats) *stats = e.stats;
  });
}

GSOT_API int gsot_eval_device(gsot_ctx* ctx, const double* d_x, int mode, double* objective,
                              double* d_grad, gsot_call_stats* stats) {
  return guard([&] {
    checked(ctx);
    if (!d_x || !d_grad) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null device pointer");
    if (mode < 0 || mode > 3) throw Error(GSOT_ERR_INVALID_ARGUMENT, "unknown eval mode");
    GSOT_CUDA_CHECK(cudaMemcpyAsync(ctx->x_eval, d_x, sizeof(double) * (ctx->m + ctx->n),
                                    cudaMemcpyDeviceToDevice, ctx->stream));
    EvalOut e = eval_device(ctx, ctx->x_eval, mode, d_grad, nullptr, ctx->ub_offset, true);
    if (objective) *objective = e.objective;
    if (stats) *stats = e.stats;
  });
}

GSOT_API int gsot_init_snapshot(gsot_ctx* ctx, const double* x) {
  return guard([&] {
    checked(ctx);
    upload_x(ctx, x);
    init_snapshot_device(ctx, ctx->x_eval, false);
    ctx->sync();
  });
}

GSOT_API int gsot_refresh(gsot_ctx* ctx, const double* x, int use_active_set) {
  return guard([&] {
    checked(ctx);
    upload_x(ctx, x);
    refresh_device(ctx, ctx->x_eval, use_active_set != 0);
    ctx->sync();
  });
}

GSOT_API int gsot_snapshot_norms(gsot_ctx* ctx, double* z, double* k, double* o) {
  return guard([&] {
    checked(ctx);
    if (!ctx->have_snapshot) throw Error(GSOT_ERR_STATE, "no snapshot taken");
    if (ctx->snap_lazy) {  // the solver's last snapshot skipped zero blocks: retake it in full
      gsot::enqueue_snapshot(ctx, ctx->snap_x, false);
      ctx->sync();
    }
    const int64_t Ln = static_cast<int64_t>(ctx->L) * ctx->n;
    std::vector<double> tmp(static_cast<size_t>(Ln));
    double* srcs[3] = {ctx->zs, ctx->ks, ctx->os};
    double* dsts[3] = {z, k, o};
    for (int q = 0; q < 3; ++q) {
      if (!dsts[q]) continue;
      GSOT_CUDA_CHECK(cudaMemcpyAsync(tmp.data(), srcs[q], sizeof(double) * Ln,
                                      cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      for (int32_t l = 0; l < ctx->L; ++l)
        for (int64_t j = 0; j < ctx->n; ++j) dsts[q][l + j * ctx->L] = tmp[l * ctx->n + j];
    }
  });
}

GSOT_API int gsot_active_set(gsot_ctx* ctx, uint8_t* member, int64_t* count) {
  return guard([&] {
    checked(ctx);
    if (count) *count = ctx->active_count;
    if (!member) return;
    const int64_t nwords = static_cast<int64_t>(ctx->L) * ctx->nw;
    std::vector<uint32_t> w(static_cast<size_t>(nwords));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(w.data(), ctx->active_words, sizeof(uint32_t) * nwords,
                                    cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    for (int32_t l = 0; l < ctx->L; ++l)
      for (int64_t j = 0; j < ctx->n; ++j)
        member[l + j * ctx->L] = (w[l * ctx->nw + (j >> 5)] >> (j & 31)) & 1u;
  });
}

GSOT_API int gsot_block_mask(gsot_ctx* ctx, const double* x, uint8_t* nonzero) {
  return guard([&] {
    checked(ctx);
    if (!nonzero) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null output");
    upload_x(ctx, x);
    const gsot::DevProblem P = ctx->problem();
    // reuse colpart as scratch for the per-block z
    ctx->launch(gsot::K_MISC, 8.0 * ctx->m * ctx->n,
                [&] { gsot::launch_block_z(P, ctx->x_eval, ctx->colpart, ctx->stream); });
    const int64_t Ln = static_cast<int64_t>(ctx->L) * ctx->n;
    std::vector<double> z(static_cast<size_t>(Ln));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(z.data(), ctx->colpart, sizeof(double) * Ln,
                                    cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    const double tau = ctx->mu * ctx->gamma;
    for (int32_t l = 0; l < ctx->L; ++l)
      for (int64_t j = 0; j < ctx->n; ++j) nonzero[l + j * ctx->L] = z[l * ctx->n + j] > tau;
  });
}

GSOT_API int gsot_plan_columns(gsot_ctx* ctx, const double* x, int64_t j0, int64_t j1,
                               double* out) {
  return guard([&] {
    checked(ctx);
    if (j0 < 0 || j1 > ctx->n || j0 > j1)
      throw Error(GSOT_ERR_DIMENSION_MISMATCH, "dimension mismatch: column range");
    if (!out) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null output");
    upload_x(ctx, x);
    const gsot::DevProblem P = ctx->problem();
    // Stream through rowpart (nw * m doubles) as scratch: nw columns a step.
    const int64_t step = std::max<int64_t>(1, ctx->nw);
    for (int64_t a = j0; a < j1; a += step) {
      const int64_t nc = std::min(step, j1 - a);
      ctx->launch(gsot::K_MISC, 16.0 * ctx->m * nc, [&] {
        gsot::launch_plan_columns(P, ctx->x_eval, a, nc, ctx->rowpart, ctx->stream);
      });
      GSOT_CUDA_CHECK(cudaMemcpyAsync(out + (a - j0) * ctx->m, ctx->rowpart,
                                      sizeof(double) * ctx->m * nc, cudaMemcpyDeviceToHost,
                                      ctx->stream));
    }
    ctx->sync();
  });
}

GSOT_API int gsot_plan_diagnostics(gsot_ctx* ctx, const double* x, gsot_plan_diag* out) {
  return guard([&] {
    checked(ctx);
    if (!out) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null output");
    upload_x(ctx, x);
    const gsot::DevProblem P = ctx->problem();
    const int64_t m = ctx->m, n = ctx->n;
    GSOT_CUDA_CHECK(cudaMemsetAsync(ctx->cnt_partials, 0, sizeof(unsigned long long), ctx->stream));
    ctx->launch(gsot::K_MISC, 16.0 * m * n, [&] {
      gsot::launch_plan_diag(P, ctx->x_eval, ctx->rowpart, ctx->colpart, ctx->cnt_partials,
                             ctx->stream);
    });
    ctx->launch(gsot::K_MISC, 8.0 * (static_cast<double>(ctx->nw) * m + static_cast<double>(ctx->L) * n),
                [&] {
                  gsot::launch_plan_diag_fold(P, ctx->rowpart, ctx->colpart, ctx->g_eval,
                                              ctx->stream);
                });
    std::vector<double> sums(static_cast<size_t>(m + n)), a(static_cast<size_t>(m)),
        b(static_cast<size_t>(n));
    unsigned long long zero = 0;
    GSOT_CUDA_CHECK(cudaMemcpyAsync(sums.data(), ctx->g_eval, sizeof(double) * (m + n),
                                    cudaMemcpyDeviceToHost, ctx->stream));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(a.data(), ctx->d_a, sizeof(double) * m, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(b.data(), ctx->d_b, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(&zero, ctx->cnt_partials, sizeof(zero), cudaMemcpyDeviceToHost,
                                    ctx->stream));
    ctx->sync();
    // (T 1 - a).cwiseAbs().maxCoeff(), (T' 1 - b)..., T.sum() (dual.hpp:143-147)
    double ra = std::abs(sums[0] - a[0]), rb = std::abs(sums[m] - b[0]), mass = 0.0;
    for (int64_t i = 0; i < m; ++i) ra = std::max(ra, std::abs(sums[i] - a[i]));
    for (int64_t j = 0; j < n; ++j) {
      rb = std::max(rb, std::abs(sums[m + j] - b[j]));
      mass += sums[m + j];
    }
    out->marginal_res_a = ra;
    out->marginal_res_b = rb;
    out->group_sparsity = static_cast<double>(zero) /
                          (static_cast<double>(ctx->L) * static_cast<double>(n));
    out->mass = mass;
  });
}

GSOT_API int gsot_primal_objective(gsot_ctx* ctx, const double* x, double* out) {
  return guard([&] {
    checked(ctx);
    if (!out) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null output");
    upload_x(ctx, x);
    const gsot::DevProblem P = ctx->problem();
    const int64_t m = ctx->m, n = ctx->n;
    ctx->launch(gsot::K_MISC, 8.0 * m * n, [&] {
      gsot::launch_plan_primal(P, ctx->x_eval, ctx->colpart, ctx->stream);
    });
    ctx->launch(gsot::K_MISC, 8.0 * static_cast<double>(ctx->L) * n, [&] {
      gsot::launch_plan_diag_fold(P, ctx->rowpart, ctx->colpart, ctx->g_eval, ctx->stream);
    });
    std::vector<double> cols(static_cast<size_t>(n));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(cols.data(), ctx->g_eval + m, sizeof(double) * n,
                                    cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    double v = 0.0;
    for (int64_t j = 0; j < n; ++j) v += cols[j];
    *out = v;
  });
}

GSOT_API void gsot_default_solver_options(gsot_solver_options* o) {
  if (!o) return;
  o->snapshot_interval = 10;  // solver.hpp:26-30
  o->grad_tol = 1e-6;
  o->max_outer_loops = 200;
  o->lbfgs_memory = 10;
  o->mode = GSOT_MODE_FAST;
  o->upper_bound_offset = 0.0;
  o->flags = 0;
}

GSOT_API int gsot_solve(gsot_ctx* ctx, const gsot_solver_options* opts, double* x_out,
                        gsot_solve_result* result, int64_t* history, int64_t history_cap) {
  return guard([&] {
    checked(ctx);
    gsot_solver_options o;
    gsot_default_solver_options(&o);
    if (opts) o = *opts;
    if (o.mode < 0 || o.mode > 3) throw Error(GSOT_ERR_INVALID_ARGUMENT, "unknown solver mode");
    if (o.lbfgs_memory > gsot::kMaxMemory)
      throw Error(GSOT_ERR_INVALID_ARGUMENT, "lbfgs_memory above the supported maximum");
    gsot_solve_result r{};
    gsot::run_solve(ctx, o, x_out, &r, history, history_cap);
    if (result) *result = r;
  });
}

GSOT_API int gsot_config_shape(int32_t cfg, int64_t* m, int64_t* n, int32_t* L, int64_t* d) {
  return guard([&] { gsot::config_shape(cfg, m, n, L, d); });
}

GSOT_API int gsot_config_features(int32_t cfg, uint64_t seed, double* src, double* tgt,
                                  int32_t* sizes, double* a, double* b) {
  return guard([&] {
    if (!src || !tgt || !sizes || !a || !b) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    gsot::config_features(cfg, seed, src, tgt, sizes, a, b);
  });
}

GSOT_API int gsot_cost_matrix_device(const double* src, int64_t m, const double* tgt, int64_t n,
                                     int64_t d, int normalize, double* d_cost) {
  return guard([&] {
    if (!src || !tgt || !d_cost) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t s;
    GSOT_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double *ds = nullptr, *dt = nullptr, *part = nullptr;
    unsigned int* ticket = nullptr;
    GSOT_CUDA_CHECK(cudaMalloc(&ds, sizeof(double) * m * d));
    GSOT_CUDA_CHECK(cudaMalloc(&dt, sizeof(double) * n * d));
    GSOT_CUDA_CHECK(cudaMalloc(&part, sizeof(double) * (148 * 8 + 1)));
    GSOT_CUDA_CHECK(cudaMalloc(&ticket, sizeof(unsigned int)));
    GSOT_CUDA_CHECK(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), s));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(ds, src, sizeof(double) * m * d, cudaMemcpyHostToDevice, s));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(dt, tgt, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
    gsot::launch_cost_matrix(ds, m, dt, n, d, nullptr, d_cost, s);
    if (normalize) {
      gsot::launch_max_reduce(d_cost, m * n, part, 148 * 8, part + 148 * 8, ticket, s);
      gsot::launch_scale_div(d_cost, m * n, part + 148 * 8, s);
    }
    GSOT_CUDA_CHECK(cudaGetLastError());
    GSOT_CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFree(ds);
    cudaFree(dt);
    cudaFree(part);
    cudaFree(ticket);
    cudaStreamDestroy(s);
  });
}

namespace {
// make_instance on the device (data_io.hpp:157-181): cost_matrix from the
// features straight into the tiled layout (k-sequential, no FMA, bitwise the
// reference's), C /= max(C) when normalize and max > 0, then
// validate_instance (core.hpp:117-139) in the reference's order: the cost
// scan (first offender, j-major), the marginals, the partition.
gsot_ctx* create_from_features(const double* src, int64_t m, const double* tgt, int64_t n,
                               int64_t d, const int32_t* sizes, int32_t L, const double* a,
                               const double* b, bool normalize, double gamma, double mu) {
  if (!src || !tgt || !sizes || !a || !b) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
  if (m <= 0 || n <= 0 || d <= 0) throw Error(GSOT_ERR_DIMENSION_MISMATCH, "empty instance");
  auto* c = new gsot_ctx();
  double *ds = nullptr, *dt = nullptr, *part = nullptr;
  unsigned int* ticket = nullptr;
  try {
    setup_shape(c, m, n, sizes, L, gamma, mu);
    if (c->off[L] != m)
      throw Error(GSOT_ERR_PARTITION_MISMATCH,
                  "group partition: partition covers " + std::to_string(c->off[L]) +
                      " indices, cost has " + std::to_string(m) + " rows");
    init_device(c);
    alloc_buffers(c);
    set_marginals(c, a, b);
    GSOT_CUDA_CHECK(cudaMalloc(&ds, sizeof(double) * m * d));
    GSOT_CUDA_CHECK(cudaMalloc(&dt, sizeof(double) * n * d));
    GSOT_CUDA_CHECK(cudaMalloc(&part, sizeof(double) * (148 * 8 + 1)));
    GSOT_CUDA_CHECK(cudaMalloc(&ticket, sizeof(unsigned int)));
    GSOT_CUDA_CHECK(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), c->stream));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(ds, src, sizeof(double) * m * d, cudaMemcpyHostToDevice,
                                    c->stream));
    GSOT_CUDA_CHECK(cudaMemcpyAsync(dt, tgt, sizeof(double) * n * d, cudaMemcpyHostToDevice,
                                    c->stream));
    const gsot::DevProblem TP = c->problem();
    c->launch(gsot::K_MISC, 0, [&] { gsot::launch_cost_matrix(ds, m, dt, n, d, &TP, c->C, c->stream); });
    if (normalize) {
      // padding columns are zero (memset at allocation) and the max over the
      // padded buffer is max(C) whenever max(C) >= 0
      const int64_t count = static_cast<int64_t>(32) * c->nw * m;
      c->launch(gsot::K_MISC, 0, [&] {
        gsot::launch_max_reduce(c->C, count, part, 148 * 8, part + 148 * 8, ticket, c->stream);
      });
      c->launch(gsot::K_MISC, 0, [&] { gsot::launch_scale_div(c->C, count, part + 148 * 8, c->stream); });
    }
    if (!c->d_bad) GSOT_CUDA_CHECK(cudaMalloc(&c->d_bad, sizeof(unsigned long long)));
    GSOT_CUDA_CHECK(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), c->stream));
    c->launch(gsot::K_MISC, 0, [&] { gsot::launch_scan_bad(TP, c->d_bad, c->stream); });
    c->sync();
    cudaFree(ds);
    cudaFree(dt);
    cudaFree(part);
    cudaFree(ticket);
    ds = dt = part = nullptr;
    ticket = nullptr;
    finish_validation(c, c->d_bad, a, b, nullptr);
    c->cacheable = false;
    return c;
  } catch (...) {
    if (ds) cudaFree(ds);
    if (dt) cudaFree(dt);
    if (part) cudaFree(part);
    if (ticket) cudaFree(ticket);
    delete c;
    throw;
  }
}
}  // namespace

GSOT_API int gsot_create_features(const double* src, int64_t m, const double* tgt, int64_t n,
                                  int64_t d, const int32_t* group_sizes, int32_t L,
                                  const double* a, const double* b, int normalize, double gamma,
                                  double mu, gsot_ctx** out) {
  return guard([&] {
    if (!out) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    *out = create_from_features(src, m, tgt, n, d, group_sizes, L, a, b, normalize != 0, gamma,
                                mu);
  });
}

GSOT_API int gsot_create_config(int32_t cfg, uint64_t seed, double gamma, double mu,
                                gsot_ctx** out) {
  return guard([&] {
    if (!out) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    int64_t m, n, d;
    int32_t L;
    gsot::config_shape(cfg, &m, &n, &L, &d);
    std::vector<double> src(static_cast<size_t>(m * d)), tgt(static_cast<size_t>(n * d));
    std::vector<double> a(static_cast<size_t>(m)), b(static_cast<size_t>(n));
    std::vector<int32_t> sizes(static_cast<size_t>(L));
    gsot::config_features(cfg, seed, src.data(), tgt.data(), sizes.data(), a.data(), b.data());
    *out = create_from_features(src.data(), m, tgt.data(), n, d, sizes.data(), L, a.data(),
                                b.data(), true, gamma, mu);
  });
}

GSOT_API int gsot_profile_enable(gsot_ctx* ctx, int enable) {
  return guard([&] {
    checked(ctx);
    ctx->collect_marks();
    ctx->profile = enable != 0;
    // negative = every kernel class, positive = bit mask (1 << kind)
    ctx->profile_mask = enable < 0 ? 0xffffffffu : static_cast<unsigned>(enable);
    if (ctx->ws) ctx->ws->graphs.clear();  // graphs carry their event nodes
  });
}

GSOT_API int gsot_profile_read(gsot_ctx* ctx, int kind, double* ms, double* bytes,
                               int64_t* launches) {
  return guard([&] {
    checked(ctx);
    if (kind < 0 || kind >= gsot::K_NSTATS) throw Error(GSOT_ERR_INVALID_ARGUMENT, "bad kind");
    ctx->collect_marks();
    if (ms) *ms = ctx->prof_ms[kind];
    if (bytes) *bytes = ctx->prof_bytes[kind];
    if (launches) *launches = ctx->prof_launches[kind];
  });
}

GSOT_API int gsot_profile_reset(gsot_ctx* ctx) {
  return guard([&] {
    checked(ctx);
    ctx->collect_marks();
    for (int k = 0; k < gsot::K_NSTATS; ++k) {
      ctx->prof_ms[k] = 0;
      ctx->prof_bytes[k] = 0;
      ctx->prof_launches[k] = 0;
    }
  });
}

GSOT_API int64_t gsot_kernel_launches(const gsot_ctx* ctx) { return ctx ? ctx->launches : 0; }

GSOT_API int gsot_set_device(int32_t device) {
  return guard([&] { GSOT_CUDA_CHECK(cudaSetDevice(device)); });
}

GSOT_API int gsot_timer(gsot_ctx* ctx, int op, double* ms) {
  return guard([&] {
    checked(ctx);
    if (!ctx->timer_a) {
      GSOT_CUDA_CHECK(cudaEventCreate(&ctx->timer_a));
      GSOT_CUDA_CHECK(cudaEventCreate(&ctx->timer_b));
    }
    if (op == 0) {
      GSOT_CUDA_CHECK(cudaEventRecord(ctx->timer_a, ctx->stream));
      return;
    }
    GSOT_CUDA_CHECK(cudaEventRecord(ctx->timer_b, ctx->stream));
    GSOT_CUDA_CHECK(cudaEventSynchronize(ctx->timer_b));
    float e = 0.f;
    GSOT_CUDA_CHECK(cudaEventElapsedTime(&e, ctx->timer_a, ctx->timer_b));
    if (ms) *ms = e;
  });
}

}  // extern "C"

#ifdef GSOT_PHASE_CLOCKS
// Diagnostic builds: the folded kernel timeline (64 words, see gsot_device.cuh).
extern "C" __attribute__((visibility("default"))) int gsot_debug_timeline(gsot_ctx* c,
                                                                          unsigned long long* out) {
  if (!c || !c->tl) return GSOT_ERR_STATE;
  cudaStreamSynchronize(c->stream);
  cudaMemcpy(out, c->tl, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 0;
}
#endif
