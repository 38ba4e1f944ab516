// gsot_kernels.cu — sm_100a kernels of the group-sparse OT dual evaluation.
//
// Parity contract: every per-block quantity the reference
// computes sequentially — the residual f = (alpha_i + beta_j) - c_ij
// (regularizer.hpp:55-58), the norms z, k, o (:23-45), the threshold test
// z <= tau (:67), the scale (1 - tau/z)/gamma (:71) and each plan entry
// scale * f (:72) — is computed by ONE thread, in ascending row order, with
// one IEEE rounding per operation (the library is built with --fmad=false
// and the hot expressions use explicit _rn intrinsics). Those values are
// therefore bitwise the reference's. Only the sums ACROSS blocks
// (grad_alpha, grad_beta, the objective) are re-associated; their
// association is fixed by block position and is independent of which
// blocks the screen skipped, so screened and dense evaluations agree
// bitwise on every output.
#include <cooperative_groups.h>

#include "gsot_internal.cuh"

namespace gsot {

namespace {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// f = (alpha_i + beta_j) - c_ij, regularizer.hpp:57.
__device__ __forceinline__ double residual(double alpha_i, double beta_j, double c) {
  return dsub(dadd(alpha_i, beta_j), c);
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// Streaming load: the cost is read once per pass; do not let it evict the
// small reused vectors from L1.
__device__ __forceinline__ double2 ldcs2(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}

// Warp-wide 32x32 transpose-reduce: on entry lane t holds v[k] = value of
// row k for column t; on exit v[0] on lane t = sum over the 32 columns of
// row t. The butterfly tree is fixed by lane position, so it is independent
// of which lanes hold exact zeros.
__device__ __forceinline__ void transpose_reduce32(double (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const double send = up ? v[k] : v[k + o];
      const double keep = up ? v[k + o] : v[k];
      v[k] = dadd(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  // Fixed-tree block reduction (warp butterfly, then warps in order).
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < NT / 32; ++w) r = dadd(r, sh[w]);
  }
  return r;  // valid on thread 0
}

}  // namespace

// ---------------------------------------------------------------- relayout
// Column-major m x n (device) -> group-padded layout, plus the first
// offending entry of validate_instance's j-major scan (core.hpp:118-123):
// the minimum linear index j*m + i with !(c >= 0) || !isfinite(c).
__global__ void k_relayout(const double* __restrict__ src, int64_t m, int64_t j0, int64_t ncols,
                           const int32_t* __restrict__ row_to_prow, int64_t ldc,
                           double* __restrict__ C, unsigned long long* first_bad) {
  const int64_t total = m * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jj = e / m;
    const int64_t i = e - jj * m;
    const double c = src[e];
    C[(j0 + jj) * ldc + row_to_prow[i]] = c;
    if (!(c >= 0.0) || !isfinite(c)) atomicMin(first_bad, (unsigned long long)((j0 + jj) * m + i));
  }
}

void launch_relayout(const double* src, int64_t m, int64_t j0, int64_t ncols,
                     const int32_t* row_to_prow, int64_t ldc, double* C,
                     unsigned long long* first_bad, cudaStream_t s) {
  const int64_t total = m * ncols;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (grid < 1) grid = 1;
  k_relayout<<<grid, 256, 0, s>>>(src, m, j0, ncols, row_to_prow, ldc, C, first_bad);
}

// ---------------------------------------------------------------- snapshot
// take_snapshot (screening.hpp:24-50): z~ = |[f]+|, k~ = |f|, o~ = |[f]-|
// per block, each a sequential sum over the block's rows. One thread per
// (l, j); consecutive lanes are consecutive columns.
__global__ void __launch_bounds__(256) k_snapshot(DevProblem P, const double* __restrict__ x,
                                                  double* __restrict__ zs,
                                                  double* __restrict__ ks,
                                                  double* __restrict__ os) {
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  const int g = P.off[l + 1] - P.off[l];
  const double* __restrict__ al = x + P.off[l];
  const double bj = x[P.m + j];
  const double* __restrict__ cp = P.C + j * P.ldc + P.poff[l];
  double az = 0.0, ak = 0.0, ao = 0.0;
#define GSOT_SNAP_STEP(ALPHA, CVAL)            \
  {                                            \
    const double f = residual((ALPHA), bj, (CVAL)); \
    const double sq = dmul(f, f);              \
    ak = dadd(ak, sq);                         \
    az = dadd(az, f > 0.0 ? sq : 0.0);         \
    ao = dadd(ao, f < 0.0 ? sq : 0.0);         \
  }
  int r = 0;
  for (; r + 8 <= g; r += 8) {
    const double2 c0 = ldcs2(cp + r), c1 = ldcs2(cp + r + 2), c2 = ldcs2(cp + r + 4),
                  c3 = ldcs2(cp + r + 6);
    GSOT_SNAP_STEP(__ldg(al + r), c0.x);
    GSOT_SNAP_STEP(__ldg(al + r + 1), c0.y);
    GSOT_SNAP_STEP(__ldg(al + r + 2), c1.x);
    GSOT_SNAP_STEP(__ldg(al + r + 3), c1.y);
    GSOT_SNAP_STEP(__ldg(al + r + 4), c2.x);
    GSOT_SNAP_STEP(__ldg(al + r + 5), c2.y);
    GSOT_SNAP_STEP(__ldg(al + r + 6), c3.x);
    GSOT_SNAP_STEP(__ldg(al + r + 7), c3.y);
  }
  for (; r < g; ++r) GSOT_SNAP_STEP(__ldg(al + r), __ldcs(cp + r));
#undef GSOT_SNAP_STEP
  const int64_t idx = (int64_t)l * P.n + j;
  zs[idx] = sqrt(az);
  ks[idx] = sqrt(ak);
  os[idx] = sqrt(ao);
}

void launch_snapshot(const DevProblem& P, const double* x, double* zs, double* ks, double* os,
                     cudaStream_t s) {
  dim3 grid((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  k_snapshot<<<grid, 256, 0, s>>>(P, x, zs, ks, os);
}

// z per block only (block mask, audits): pos_part_norm of each block.
__global__ void __launch_bounds__(256) k_block_z(DevProblem P, const double* __restrict__ x,
                                                 double* __restrict__ zout) {
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  const int g = P.off[l + 1] - P.off[l];
  const double* __restrict__ al = x + P.off[l];
  const double bj = x[P.m + j];
  const double* __restrict__ cp = P.C + j * P.ldc + P.poff[l];
  double az = 0.0;
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, __ldcs(cp + r));
    const double v = f > 0.0 ? f : 0.0;
    az = dadd(az, dmul(v, v));
  }
  zout[(int64_t)l * P.n + j] = sqrt(az);
}

void launch_block_z(const DevProblem& P, const double* x, double* zout, cudaStream_t s) {
  dim3 grid((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  k_block_z<<<grid, 256, 0, s>>>(P, x, zout);
}

// ---------------------------------------------------------------- deltas
// compute_delta_norms (screening.hpp:63-83): per group the sequential
// pos/full/neg norms of alpha - alpha~, and dbeta = beta - beta~.
__global__ void k_delta(DevProblem P, const double* __restrict__ x, const double* __restrict__ xs,
                        double* __restrict__ dpos, double* __restrict__ dfull,
                        double* __restrict__ dneg, double* __restrict__ dbeta) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < P.L) {
    const int l = (int)t;
    const int o0 = P.off[l], g = P.off[l + 1] - o0;
    double ap = 0.0, af = 0.0, an = 0.0;
    for (int r = 0; r < g; ++r) {
      const double da = dsub(x[o0 + r], xs[o0 + r]);
      const double sq = dmul(da, da);
      af = dadd(af, sq);
      ap = dadd(ap, da > 0.0 ? sq : 0.0);
      an = dadd(an, da < 0.0 ? sq : 0.0);
    }
    dpos[l] = sqrt(ap);
    dfull[l] = sqrt(af);
    dneg[l] = sqrt(an);
  }
  const int64_t j = t - P.L;
  if (j >= 0 && j < P.n) dbeta[j] = dsub(x[P.m + j], xs[P.m + j]);
}

void launch_delta(const DevProblem& P, const double* x, const double* xs, double* dpos,
                  double* dfull, double* dneg, double* dbeta, cudaStream_t s) {
  const int64_t total = P.L + P.n;
  k_delta<<<(unsigned)((total + 127) / 128), 128, 0, s>>>(P, x, xs, dpos, dfull, dneg, dbeta);
}

// ---------------------------------------------------------------- active set
// build_active_set (screening.hpp:147-166) with lower_bound (:99-105)
// evaluated left to right, unclamped; strict > tau.
__global__ void __launch_bounds__(256) k_active(DevProblem P, const double* __restrict__ ks,
                                                const double* __restrict__ os,
                                                const double* __restrict__ dfull,
                                                const double* __restrict__ dneg,
                                                const double* __restrict__ dbeta,
                                                uint32_t* __restrict__ aw, EvalScalars* sc) {
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool in = false;
  if (j < P.n) {
    const int64_t idx = (int64_t)l * P.n + j;
    const double db = dbeta[j];
    const double db_neg = db < 0.0 ? -db : 0.0;
    const double sg = P.sqrt_g[l];
    const double lb = dsub(dsub(dsub(dsub(dsub(ks[idx], dfull[l]), dmul(sg, fabs(db))), os[idx]),
                                dneg[l]),
                           dmul(sg, db_neg));
    in = lb > P.tau;
  }
  const unsigned w = __ballot_sync(0xffffffffu, in);
  const int64_t c = j >> 5;
  if (lane == 0 && c < P.nw) {
    aw[(int64_t)l * P.nw + c] = w;
    if (w) atomicAdd(&sc->counters[0], (unsigned long long)__popc(w));
  }
}

void launch_active(const DevProblem& P, const double* ks, const double* os, const double* dfull,
                   const double* dneg, const double* dbeta, uint32_t* aw, EvalScalars* sc,
                   cudaStream_t s) {
  dim3 grid((unsigned)((P.nw * 32 + 255) / 256), (unsigned)P.L);
  k_active<<<grid, 256, 0, s>>>(P, ks, os, dfull, dneg, dbeta, aw, sc);
}

// ---------------------------------------------------------------- bounds
// FastGradDispatcher::column's per-block decision (screening.hpp:252-275):
// active-set members are computed without a bound; every other block gets
// z_bar = (z~ + |[dalpha_l]+|) + sqrt(g_l) * [dbeta_j]+ (+ offset) and is
// skipped iff z_bar <= tau. Writes the survivor word of each (l, c) chunk
// and appends non-empty chunks to the work list (order irrelevant: every
// task writes fixed slots).
__global__ void __launch_bounds__(256) k_bounds(DevProblem P, const double* __restrict__ zs,
                                                const uint32_t* __restrict__ aw,
                                                const double* __restrict__ dpos,
                                                const double* __restrict__ dbeta,
                                                double ub_offset, uint32_t* __restrict__ words,
                                                int2* __restrict__ tasks, EvalScalars* sc) {
  __shared__ unsigned long long cnt[4];
  __shared__ int wtask[8];
  __shared__ int base;
  if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = j >> 5;
  const bool valid = j < P.n;
  bool in_active = false;
  if (valid && aw != nullptr) in_active = (aw[(int64_t)l * P.nw + c] >> lane) & 1u;
  const bool evaluated = valid && !in_active;
  bool surv = in_active;
  if (evaluated) {
    const double db = dbeta[j];
    const double db_pos = db > 0.0 ? db : 0.0;
    const double zbar =
        dadd(dadd(dadd(zs[(int64_t)l * P.n + j], dpos[l]), dmul(P.sqrt_g[l], db_pos)), ub_offset);
    surv = !(zbar <= P.tau);
  }
  const unsigned wa = __ballot_sync(0xffffffffu, in_active);
  const unsigned we = __ballot_sync(0xffffffffu, evaluated);
  const unsigned ws = __ballot_sync(0xffffffffu, surv);
  if (lane == 0) {
    if (c < P.nw) words[(int64_t)l * P.nw + c] = ws;
    atomicAdd(&cnt[0], (unsigned long long)__popc(wa));
    atomicAdd(&cnt[1], (unsigned long long)__popc(we & ~ws));
    atomicAdd(&cnt[2], (unsigned long long)__popc(we & ws));
    atomicAdd(&cnt[3], (unsigned long long)__popc(we));
    wtask[warp] = (ws != 0u && c < P.nw) ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nt = 0;
    for (int w = 0; w < 8; ++w) nt += wtask[w];
    base = nt ? atomicAdd(&sc->ntasks, nt) : 0;
    for (int q = 0; q < 4; ++q)
      if (cnt[q]) atomicAdd(&sc->counters[q], cnt[q]);
  }
  __syncthreads();
  if (lane == 0 && wtask[warp]) {
    int pos = base;
    for (int w = 0; w < warp; ++w) pos += wtask[w];
    tasks[pos] = make_int2(l, (int)c);
  }
}

void launch_bounds(const DevProblem& P, const double* zs, const uint32_t* aw, const double* dpos,
                   const double* dbeta, double ub_offset, uint32_t* words, int2* tasks,
                   EvalScalars* sc, cudaStream_t s) {
  dim3 grid((unsigned)((P.nw * 32 + 255) / 256), (unsigned)P.L);
  k_bounds<<<grid, 256, 0, s>>>(P, zs, aw, dpos, dbeta, ub_offset, words, tasks, sc);
}

// Dense mode: every word full (bits only for j < n), every chunk a task.
__global__ void k_fill_words(uint32_t* words, int32_t L, int32_t nw, int64_t n) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)L * nw) return;
  const int64_t c = t % nw;
  const int64_t rem = n - c * 32;
  words[t] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}
void launch_fill_words(uint32_t* words, int32_t L, int32_t nw, int64_t n, cudaStream_t s) {
  const int64_t total = (int64_t)L * nw;
  k_fill_words<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(words, L, nw, n);
}
__global__ void k_dense_tasks(int2* tasks, int32_t L, int32_t nw) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)L * nw) return;
  tasks[t] = make_int2((int)(t / nw), (int)(t % nw));
}
void launch_dense_tasks(int2* tasks, int32_t L, int32_t nw, cudaStream_t s) {
  const int64_t total = (int64_t)L * nw;
  k_dense_tasks<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(tasks, L, nw);
}

// ---------------------------------------------------------------- fused eval
// One warp per (group l, 32-column chunk c) task; lane = column j = 32c+lane,
// active iff its survivor bit is set. Pass 1 (sequential over the block's
// rows): z^2 = sum [f]+^2 and sum [f]+. Then scale = (1 - tau/z)/gamma when
// z > tau (grad_block, regularizer.hpp:64-74), psi = (z - tau)^2 / (2 gamma)
// (the closed form of psi_block, regularizer.hpp:78-91),
// column partial scale * sum [f]+. Pass 2 (32 rows at a time): plan entries
// T = scale * [f]+, transpose-reduced across the warp into per-row partials
// of the chunk, stored at rowpart[c * m + row]. The plan is never stored.
__global__ void __launch_bounds__(256) k_eval(DevProblem P, const double* __restrict__ x,
                                              const int2* __restrict__ tasks, int dense_ntasks,
                                              const uint32_t* __restrict__ words,
                                              double* __restrict__ rowpart,
                                              double* __restrict__ colpart,
                                              double* __restrict__ psi, EvalScalars* sc) {
  const int lane = threadIdx.x & 31;
  const int ntasks = dense_ntasks >= 0 ? dense_ntasks : sc->ntasks;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(&sc->next_task, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= ntasks) break;
    const int2 tk = tasks[t];
    const int l = tk.x, c = tk.y;
    const uint32_t word = words[(int64_t)l * P.nw + c];
    const int64_t j = (int64_t)c * 32 + lane;
    const bool act = (word >> lane) & 1u;
    const int o0 = P.off[l];
    const int g = P.off[l + 1] - o0;
    const double* __restrict__ al = x + o0;
    const double bj = act ? x[P.m + j] : 0.0;
    const double* __restrict__ cp = P.C + (act ? j : 0) * P.ldc + P.poff[l];

    // pass 1
    double z2 = 0.0, sv = 0.0;
    if (act) {
#define GSOT_P1(ALPHA, CVAL)                          \
  {                                                   \
    const double f = residual((ALPHA), bj, (CVAL));   \
    const double v = f > 0.0 ? f : 0.0;               \
    z2 = dadd(z2, dmul(v, v));                        \
    sv = dadd(sv, v);                                 \
  }
      int r = 0;
      for (; r + 8 <= g; r += 8) {
        const double2 c0 = ldg2(cp + r), c1 = ldg2(cp + r + 2), c2 = ldg2(cp + r + 4),
                      c3 = ldg2(cp + r + 6);
        GSOT_P1(__ldg(al + r), c0.x);
        GSOT_P1(__ldg(al + r + 1), c0.y);
        GSOT_P1(__ldg(al + r + 2), c1.x);
        GSOT_P1(__ldg(al + r + 3), c1.y);
        GSOT_P1(__ldg(al + r + 4), c2.x);
        GSOT_P1(__ldg(al + r + 5), c2.y);
        GSOT_P1(__ldg(al + r + 6), c3.x);
        GSOT_P1(__ldg(al + r + 7), c3.y);
      }
      for (; r < g; ++r) GSOT_P1(__ldg(al + r), __ldg(cp + r));
#undef GSOT_P1
    }
    const double z = sqrt(z2);
    const bool nz = act && z > P.tau;
    const double scale = nz ? ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma) : 0.0;
    if (act) {
      const int64_t idx = (int64_t)l * P.n + j;
      colpart[idx] = dmul(scale, sv);
      double ps = 0.0;
      if (nz) {
        const double e = dsub(z, P.tau);
        ps = ddiv(dmul(e, e), dmul(2.0, P.gamma));
      }
      psi[idx] = ps;
    }
    double* __restrict__ rp = rowpart + (int64_t)c * P.m + o0;
    const unsigned nzm = __ballot_sync(0xffffffffu, nz);
    if (nzm == 0u) {
      for (int r = lane; r < g; r += 32) rp[r] = 0.0;
      continue;
    }
    // pass 2
    for (int r0 = 0; r0 < g; r0 += 32) {
      double v[32];
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        const int r = r0 + k;
        double2 cc = make_double2(0.0, 0.0);
        if (nz && r < g) cc = ldg2(cp + r);  // r even, rows r, r+1 within the padded block
        const double a0 = r < g ? __ldg(al + r) : 0.0;
        const double a1 = r + 1 < g ? __ldg(al + r + 1) : 0.0;
        const double f0 = residual(a0, bj, cc.x);
        const double f1 = residual(a1, bj, cc.y);
        v[k] = (nz && r < g && f0 > 0.0) ? dmul(scale, f0) : 0.0;
        v[k + 1] = (nz && r + 1 < g && f1 > 0.0) ? dmul(scale, f1) : 0.0;
      }
      transpose_reduce32(v, lane);
      if (r0 + lane < g) rp[r0 + lane] = v[0];
    }
  }
}

int eval_blocks_per_sm() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_eval, 256, 0) != cudaSuccess) return 2;
  return n;
}

void launch_eval(const DevProblem& P, const double* x, const int2* tasks, int dense_ntasks,
                 const uint32_t* words, double* rowpart, double* colpart, double* psi,
                 EvalScalars* sc, int grid, cudaStream_t s) {
  k_eval<<<grid, 256, 0, s>>>(P, x, tasks, dense_ntasks, words, rowpart, colpart, psi, sc);
}

// ---------------------------------------------------------------- finalize
// grad_alpha_i = a_i - sum over non-empty chunks c (ascending) of
// rowpart[c*m+i]; grad_beta_j = b_j - sum over surviving l (ascending) of
// colpart[l][j]; psicol_j = sum over surviving l of psi[l][j]. Empty
// chunks and skipped blocks contribute exact zeros, so omitting them is
// exact: the result does not depend on the screen.
__global__ void __launch_bounds__(256) k_finalize(DevProblem P, const uint32_t* __restrict__ words,
                                                  const double* __restrict__ rowpart,
                                                  const double* __restrict__ colpart,
                                                  const double* __restrict__ psi,
                                                  double* __restrict__ grad,
                                                  double* __restrict__ psicol) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < P.m) {
    const int64_t i = t;
    const int l = P.row_group[i];
    const uint32_t* __restrict__ wl = words + (int64_t)l * P.nw;
    double acc = 0.0;
    for (int c = 0; c < P.nw; ++c)
      if (wl[c]) acc = dadd(acc, rowpart[(int64_t)c * P.m + i]);
    grad[i] = dsub(P.a[i], acc);
    return;
  }
  const int64_t j = t - P.m;
  if (j >= P.n) return;
  const int64_t c = j >> 5;
  const int lane = (int)(j & 31);
  double acc = 0.0, ps = 0.0;
  for (int l = 0; l < P.L; ++l) {
    if ((words[(int64_t)l * P.nw + c] >> lane) & 1u) {
      acc = dadd(acc, colpart[(int64_t)l * P.n + j]);
      ps = dadd(ps, psi[(int64_t)l * P.n + j]);
    }
  }
  grad[P.m + j] = dsub(P.b[j], acc);
  psicol[j] = ps;
}

void launch_finalize(const DevProblem& P, const double* x, const uint32_t* words,
                     const double* rowpart, const double* colpart, const double* psi,
                     double* grad, double* psicol, cudaStream_t s) {
  (void)x;
  const int64_t total = P.m + P.n;
  k_finalize<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(P, words, rowpart, colpart, psi,
                                                            grad, psicol);
}

// Objective a.alpha + b.beta - sum psi (dual.hpp:51) and optionally the
// line-search slope grad.d, as fixed-structure reductions: grid-stride
// partials per block, then the last block to finish sums the partials in
// block order.
__global__ void __launch_bounds__(256) k_objective(DevProblem P, const double* __restrict__ x,
                                                   const double* __restrict__ psicol,
                                                   const double* __restrict__ grad,
                                                   const double* __restrict__ dvec,
                                                   double* __restrict__ partials,
                                                   EvalScalars* sc) {
  __shared__ double sh[8];
  __shared__ bool last;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t dim = P.m + P.n;
  double pa = 0.0, pb = 0.0, pp = 0.0, pd = 0.0;
  for (int64_t i = t0; i < P.m; i += stride) pa = dadd(pa, dmul(x[i], P.a[i]));
  for (int64_t j = t0; j < P.n; j += stride) {
    pb = dadd(pb, dmul(x[P.m + j], P.b[j]));
    pp = dadd(pp, psicol[j]);
  }
  if (dvec)
    for (int64_t i = t0; i < dim; i += stride) pd = dadd(pd, dmul(grad[i], dvec[i]));
  const double ra = block_sum<256>(pa, sh);
  const double rb = block_sum<256>(pb, sh);
  const double rp = block_sum<256>(pp, sh);
  const double rd = block_sum<256>(pd, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x * 4 + 0] = ra;
    partials[blockIdx.x * 4 + 1] = rb;
    partials[blockIdx.x * 4 + 2] = rp;
    partials[blockIdx.x * 4 + 3] = rd;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double sa = 0.0, sb = 0.0, sp = 0.0, sd = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      sa = dadd(sa, partials[b * 4 + 0]);
      sb = dadd(sb, partials[b * 4 + 1]);
      sp = dadd(sp, partials[b * 4 + 2]);
      sd = dadd(sd, partials[b * 4 + 3]);
    }
    sc->dot_aa = sa;
    sc->dot_bb = sb;
    sc->psi_sum = sp;
    sc->objective = dsub(dadd(sa, sb), sp);
    sc->slope = sd;
    sc->ticket = 0u;
  }
}

void launch_objective(const DevProblem& P, const double* x, const double* psicol,
                      const double* grad, const double* dvec, double* partials, int nblocks,
                      EvalScalars* sc, cudaStream_t s) {
  k_objective<<<nblocks, 256, 0, s>>>(P, x, psicol, grad, dvec, partials, sc);
}

// ---------------------------------------------------------------- plan
// recover_plan columns [j0, j0+ncols): out (m x ncols column-major) =
// grad_block of every block (regularizer.hpp:64-74), bitwise.
__global__ void __launch_bounds__(256) k_plan(DevProblem P, const double* __restrict__ x,
                                              int64_t j0, int64_t ncols,
                                              double* __restrict__ out) {
  const int l = blockIdx.y;
  const int64_t jj = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (jj >= ncols) return;
  const int64_t j = j0 + jj;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const double* __restrict__ al = x + o0;
  const double bj = x[P.m + j];
  const double* __restrict__ cp = P.C + j * P.ldc + P.poff[l];
  double z2 = 0.0;
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[r]);
    const double v = f > 0.0 ? f : 0.0;
    z2 = dadd(z2, dmul(v, v));
  }
  const double z = sqrt(z2);
  double* __restrict__ o = out + jj * P.m + o0;
  if (z <= P.tau) {
    for (int r = 0; r < g; ++r) o[r] = 0.0;
    return;
  }
  const double scale = ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma);
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[r]);
    o[r] = f > 0.0 ? dmul(scale, f) : 0.0;
  }
}

void launch_plan_columns(const DevProblem& P, const double* x, int64_t j0, int64_t ncols,
                         double* out, cudaStream_t s) {
  dim3 grid((unsigned)((ncols + 255) / 256), (unsigned)P.L);
  k_plan<<<grid, 256, 0, s>>>(P, x, j0, ncols, out);
}

// ---------------------------------------------------------------- audit
// audit_solve (solver.hpp:172-201): every block the screen skipped must
// have z <= tau at the evaluated state; counts checks into counters[0].
__global__ void __launch_bounds__(256) k_audit_skips(DevProblem P, const double* __restrict__ x,
                                                     const uint32_t* __restrict__ words,
                                                     const uint32_t* __restrict__ aw,
                                                     EvalScalars* sc) {
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  const int64_t c = j >> 5;
  const int lane = (int)(j & 31);
  const bool surv = (words[(int64_t)l * P.nw + c] >> lane) & 1u;
  if (surv) return;
  const int g = P.off[l + 1] - P.off[l];
  const double* __restrict__ al = x + P.off[l];
  const double bj = x[P.m + j];
  const double* __restrict__ cp = P.C + j * P.ldc + P.poff[l];
  double z2 = 0.0;
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[r]);
    const double v = f > 0.0 ? f : 0.0;
    z2 = dadd(z2, dmul(v, v));
  }
  atomicAdd(&sc->counters[0], 1ull);
  if (!(sqrt(z2) <= P.tau)) {
    if (atomicCAS(&sc->audit_violation, 0, 1) == 0) sc->audit_where = (long long)l * P.n + j;
  }
  (void)aw;
}

void launch_audit_skips(const DevProblem& P, const double* x, const uint32_t* words,
                        const uint32_t* aw, EvalScalars* sc, cudaStream_t s) {
  dim3 grid((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  k_audit_skips<<<grid, 256, 0, s>>>(P, x, words, aw, sc);
}

// solver.hpp:215-240: every active-set member has z > tau at build time.
__global__ void __launch_bounds__(256) k_audit_active(DevProblem P, const double* __restrict__ x,
                                                      const uint32_t* __restrict__ aw,
                                                      EvalScalars* sc) {
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  const bool in = (aw[(int64_t)l * P.nw + (j >> 5)] >> (j & 31)) & 1u;
  if (!in) return;
  const int g = P.off[l + 1] - P.off[l];
  const double* __restrict__ al = x + P.off[l];
  const double bj = x[P.m + j];
  const double* __restrict__ cp = P.C + j * P.ldc + P.poff[l];
  double z2 = 0.0;
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[r]);
    const double v = f > 0.0 ? f : 0.0;
    z2 = dadd(z2, dmul(v, v));
  }
  atomicAdd(&sc->counters[1], 1ull);
  if (!(sqrt(z2) > P.tau)) {
    if (atomicCAS(&sc->audit_violation, 0, 2) == 0) sc->audit_where = (long long)l * P.n + j;
  }
}

void launch_audit_active(const DevProblem& P, const double* x, const uint32_t* aw,
                         EvalScalars* sc, cudaStream_t s) {
  dim3 grid((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  k_audit_active<<<grid, 256, 0, s>>>(P, x, aw, sc);
}

}  // namespace gsot
