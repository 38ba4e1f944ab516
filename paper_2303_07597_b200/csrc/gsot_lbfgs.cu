// gsot_lbfgs.cu — device side of the L-BFGS ascent (lbfgs.hpp:61-274) in
// fast mode. The host keeps the scalar control flow of `maximize`; every
// O(m+n) vector operation of one direction update runs in ONE cooperative
// launch (k_lbfgs_step), so only scalars cross PCIe.
//
// The direction uses the compact representation of the L-BFGS inverse
// Hessian (Byrd, Nocedal & Schnabel 1994) instead of the two-loop recursion:
// the same matrix H_k = gam I + [S Y] M [S Y]^T, but the 4k dots it needs
// are independent (one pass over the history) and the direction is one
// combine pass: d = gam g + S p - Y (gam w), with w = R^-1 (S^T g),
// p = R^-T ((D + gam Y^T Y) w - gam Y^T g), R = triu(S^T Y). R and Y^T Y are
// kept by logical position and updated by one column per accepted pair.
// Exact mode (gsot_exact2.cu) keeps the reference's two-loop instead.
//
// Determinism: each dot is reduced by fixed warp trees, per-CTA results are
// folded in CTA order, the grid is a fixed function of the device.
#include <cooperative_groups.h>

#include "gsot_device.cuh"

namespace cg = cooperative_groups;

namespace gsot {

// trial.x = x + t * d (lbfgs.hpp:86).
__global__ void k_axpy_point(const double* __restrict__ x, const double* __restrict__ tp,
                             const double* __restrict__ d, double* __restrict__ out, int64_t dim,
                             int64_t m, const double* __restrict__ snap,
                             double* __restrict__ dbeta) {
  pdl_trigger();
  const double t = *tp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = dadd(x[e], dmul(t, d[e]));
    out[e] = v;
    if (dbeta && e >= m) dbeta[e - m] = dsub(v, snap[e]);  // compute_delta_norms' dbeta
  }
}

void launch_axpy_point(const double* x, const double* t, const double* d, double* out,
                       int64_t dim, int64_t m, const double* snap, double* dbeta, cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((dim + 255) / 256, 148 * 4);
  k_axpy_point<<<grid, 256, 0, s>>>(x, t, d, out, dim, m, snap, dbeta);
}

#ifdef GSOT_PHASE_CLOCKS
// Diagnostic build only: per-phase SM clocks of CTA 0 / thread 0, summed.
__device__ unsigned long long g_phase_clk[16];
#define PHASE_MARK(i)                                                   \
  do {                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                          \
      const long long now = clock64();                                  \
      atomicAdd(&g_phase_clk[i], (unsigned long long)(now - clk_prev)); \
      clk_prev = now;                                                   \
    }                                                                   \
  } while (0)
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif

// Warp-wide: sum of part[i * stride] for i in [0, n) -- lane runs of
// consecutive entries (loads in flight together), then a fixed xor tree.
__device__ __forceinline__ double warp_fold(const double* part, int n, int stride) {
  const int lane = threadIdx.x & 31;
  const int run = (n + 31) / 32;
  const int i0 = lane * run, i1 = min(n, i0 + run);
  double s = 0.0;
  for (int ib = i0; ib < i1; ib += 16) {
    double q[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) q[u] = ib + u < i1 ? __ldcg(part + (int64_t)(ib + u) * stride) : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (ib + u < i1) s = dadd(s, q[u]);
  }
#pragma unroll
  for (int o = 1; o <= 16; o <<= 1) s = dadd(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}

// The pending folds (EvalScalars::fin_blocks / step_blocks / cnt_pending),
// in a fixed order, by all 256 threads of one CTA: k_publish, and k_shard_pack
// before a sharded context's all-reduce. Returns with the CTA synchronised.
__device__ __forceinline__ void publish_fold(DevSync* __restrict__ src,
                                             const double* __restrict__ fin_partials,
                                             const double* __restrict__ step_partials,
                                             unsigned long long* cnt_slots) {
  EvalScalars* sc = &src->sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fin = sc->fin_blocks, step = sc->step_blocks, cnt = sc->cnt_pending;
  __shared__ double f[6];
  __shared__ double fw[8][4];
  if (fin > 0) {  // a.alpha, b.beta, psi, g.d (dual.hpp:51): every thread folds a
    // contiguous run of unit partials (all loads in flight), then a fixed xor
    // tree per warp and the warps in order
    const int run = (fin + 255) / 256;
    const int i0 = min(fin, (int)threadIdx.x * run), i1 = min(fin, i0 + run);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int ib = i0; ib < i1; ib += 8) {
      double2 q[8][2];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2 z{0.0, 0.0};
        const double2* pp = reinterpret_cast<const double2*>(fin_partials + 4ll * (ib + u));
        q[u][0] = ib + u < i1 ? __ldcg(pp) : z;
        q[u][1] = ib + u < i1 ? __ldcg(pp + 1) : z;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (ib + u < i1) {
          a0 = dadd(a0, q[u][0].x);
          a1 = dadd(a1, q[u][0].y);
          a2 = dadd(a2, q[u][1].x);
          a3 = dadd(a3, q[u][1].y);
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      a0 = dadd(a0, __shfl_xor_sync(0xffffffffu, a0, o));
      a1 = dadd(a1, __shfl_xor_sync(0xffffffffu, a1, o));
      a2 = dadd(a2, __shfl_xor_sync(0xffffffffu, a2, o));
      a3 = dadd(a3, __shfl_xor_sync(0xffffffffu, a3, o));
    }
    if (lane == 0) {
      fw[warp][0] = a0;
      fw[warp][1] = a1;
      fw[warp][2] = a2;
      fw[warp][3] = a3;
    }
  }
  if (step > 0 && (warp == 4 || warp == 5)) {  // g.d, d.d of the new direction
    const double v = warp_fold(step_partials + (warp - 4), step, 2);
    if (lane == 0) f[warp] = v;
  }
  if (cnt && warp == 6) fold_counter_slots(cnt_slots, sc);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (fin > 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double v = fw[0][q];
        for (int w = 1; w < 8; ++w) v = dadd(v, fw[w][q]);
        f[q] = v;
      }
      sc->dot_aa = f[0];
      sc->dot_bb = f[1];
      sc->psi_sum = f[2];
      sc->objective = dsub(dadd(f[0], f[1]), f[2]);
      sc->slope = f[3];
    }
    if (step > 0) {
      src->tl[0] = f[4];
      src->tl[1] = f[5];
    }
    sc->fin_blocks = 0;
    sc->step_blocks = 0;
    sc->cnt_pending = 0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_publish(DevSync* __restrict__ src, DevSync* host_dst,
                                                 unsigned long long* dev_count,
                                                 unsigned long long* host_flag,
                                                 const double* __restrict__ fin_partials,
                                                 const double* __restrict__ step_partials,
                                                 unsigned long long* cnt_slots,
                                                 unsigned long long* tl) {
  static_assert(offsetof(DevSync, t) % 8 == 0, "DevSync is copied as 8-byte words");
#ifdef GSOT_PHASE_CLOCKS
  long long clk_prev = clock64();
#endif
  // the completion counter is written only by earlier publishes, which
  // completed before this sequence was launched: read it before the wait
  unsigned long long count0 = 0;
  if (threadIdx.x == 0) count0 = *dev_count;
  pdl_wait();
  TL_ENTER(tl, TL_PUBLISH);
  EvalScalars* sc = &src->sc;
  publish_fold(src, fin_partials, step_partials, cnt_slots);
  PHASE_MARK(11);
  // what the host reads: the scalar block, the ring's counters, the slopes
  // (t is host-owned; it is copied to the device by the solver)
  constexpr int kSc = (int)(sizeof(EvalScalars) / 8);
  constexpr int kH = (int)(offsetof(HistState, order) / 8);
  static_assert(sizeof(EvalScalars) % 8 == 0 && offsetof(HistState, order) % 8 == 0, "8-byte words");
  const unsigned long long* a = reinterpret_cast<const unsigned long long*>(src);
  volatile unsigned long long* b = reinterpret_cast<volatile unsigned long long*>(host_dst);
  constexpr int kHOff = (int)(offsetof(DevSync, h) / 8), kTlOff = (int)(offsetof(DevSync, tl) / 8);
  const int i = threadIdx.x;
  if (i < kSc) b[i] = a[i];
  else if (i < kSc + kH) b[kHOff + i - kSc] = a[kHOff + i - kSc];
  else if (i < kSc + kH + 2) b[kTlOff + i - kSc - kH] = a[kTlOff + i - kSc - kH];
  __syncthreads();
  PHASE_MARK(12);
  if (threadIdx.x == 0) {  // one system-scope fence (cumulative over the CTA's writes)
    sc->ntasks = 0;        // the next screened evaluation starts from zeroed cursors
    sc->next_task = 0;
    sc->zero_rows = 0ull;
    sc->read_qrows = 0ull;
    sc->ticket = 0u;
    sc->audit_violation = 0;
    sc->audit_where = 0;
    const unsigned long long c = count0 + 1;
    *dev_count = c;
    __threadfence_system();
    PHASE_MARK(13);
    *reinterpret_cast<volatile unsigned long long*>(host_flag) = c;
#ifdef GSOT_PHASE_CLOCKS
    if (tl) {  // fold this sequence's kernel windows into offsets from its first entry
      TL_EXIT(tl, TL_PUBLISH);
      unsigned long long s0 = ~0ull;
      for (int k = 0; k < 8; ++k) s0 = tl[2 * k] < s0 ? tl[2 * k] : s0;
      if (tl[2 * TL_EVAL] != ~0ull && tl[2 * TL_EVAL + 1] - tl[2 * TL_EVAL] < 40000ull) {
        tl[56] += tl[2 * TL_EVAL + 1] - tl[2 * TL_EVAL];  // steady-state (sparse) evaluations
        tl[57] += 1;
        tl[58] += tl[2 * TL_PUBLISH + 1] - s0;  // and their sequence span
        for (int k = 0; k < 4; ++k) {  // screen, eval, finalize, publish windows
          tl[48 + 2 * k] += tl[2 * k] - s0;
          tl[49 + 2 * k] += tl[2 * k + 1] - s0;
        }
        if (tl[2 * TL_STEP] != ~0ull) {
          tl[59] += tl[2 * TL_STEP] - s0;
          tl[60] += tl[2 * TL_STEP + 1] - s0;
          tl[61] += 1;
        }
      }
      for (int k = 0; k < 8; ++k)
        if (tl[2 * k] != ~0ull) {
          tl[16 + 4 * k] += tl[2 * k] - s0;
          tl[16 + 4 * k + 1] += tl[2 * k + 1] - s0;
          tl[16 + 4 * k + 2] += 1;
          tl[2 * k] = ~0ull;
          tl[2 * k + 1] = 0;
        }
      tl[63] += 1;
    }
#endif
  }
}

void launch_publish(DevSync* src, DevSync* host_dst, unsigned long long* dev_count,
                    unsigned long long* host_flag, const double* fin_partials,
                    const double* step_partials, unsigned long long* cnt_slots,
                    unsigned long long* tl, cudaStream_t s) {
  launch_pdl(k_publish, dim3(1), dim3(256), 0, s, src, host_dst, dev_count, host_flag,
             fin_partials, step_partials, cnt_slots, tl);
}

// ---- column-sharded contexts: the scalars of one device
// sequence, summed over the ranks. k_shard_pack folds this rank's pending
// partials exactly as k_publish would and lays the folded values out in
// `tail` (kShardTail doubles) with one presence flag per group; after the sum
// all-reduce k_shard_unpack writes back the groups present (identical on every
// rank, so every rank's host takes the same decisions). The objective's terms
// add up over ranks because only rank 0's shard carries a (a.alpha) and every
// shard's b_p.beta_p - psi_p covers its own columns; g.d adds up because the
// gradient head is linear in the per-rank row sums (dual.hpp:91, :96).
__global__ void __launch_bounds__(256) k_shard_pack(DevSync* __restrict__ src,
                                                    const double* __restrict__ fin_partials,
                                                    const double* __restrict__ step_partials,
                                                    unsigned long long* cnt_slots,
                                                    double* __restrict__ tail) {
  EvalScalars* sc = &src->sc;
  const int fin = sc->fin_blocks, step = sc->step_blocks, cnt = sc->cnt_pending;
  publish_fold(src, fin_partials, step_partials, cnt_slots);
  if (threadIdx.x == 0) {
    double t[kShardTail];
    for (int i = 0; i < kShardTail; ++i) t[i] = 0.0;
    if (fin > 0) {
      t[0] = sc->dot_aa;
      t[1] = sc->dot_bb;
      t[2] = sc->psi_sum;
      t[3] = sc->slope;
      t[4] = 1.0;
    }
    if (step > 0) {
      t[5] = src->tl[0];
      t[6] = src->tl[1];
      t[7] = 1.0;
    }
    if (cnt) {
      for (int q = 0; q < 4; ++q) t[8 + q] = static_cast<double>(sc->counters[q]);
      t[12] = 1.0;
    }
    for (int i = 0; i < kShardTail; ++i) tail[i] = t[i];
  }
}

__global__ void k_shard_unpack(DevSync* __restrict__ src, const double* __restrict__ tail) {
  EvalScalars* sc = &src->sc;
  if (tail[4] > 0.0) {
    sc->dot_aa = tail[0];
    sc->dot_bb = tail[1];
    sc->psi_sum = tail[2];
    sc->objective = dsub(dadd(tail[0], tail[1]), tail[2]);
    sc->slope = tail[3];
  }
  if (tail[7] > 0.0) {
    src->tl[0] = tail[5];
    src->tl[1] = tail[6];
  }
  if (tail[12] > 0.0)
    for (int q = 0; q < 4; ++q) sc->counters[q] = static_cast<unsigned long long>(tail[8 + q]);
}

void launch_shard_pack(DevSync* src, const double* fin_partials, const double* step_partials,
                       unsigned long long* cnt_slots, double* tail, cudaStream_t s) {
  k_shard_pack<<<1, 256, 0, s>>>(src, fin_partials, step_partials, cnt_slots, tail);
}

void launch_shard_unpack(DevSync* src, const double* tail, cudaStream_t s) {
  k_shard_unpack<<<1, 1, 0, s>>>(src, tail);
}

__global__ void k_hist_reset(HistState* h, int mem) {
  h->k = 0;
  h->mem = mem;
  h->scratch = 0;
  h->accepted = 0;
}

void launch_hist_reset(HistState* h, int mem, cudaStream_t s) { k_hist_reset<<<1, 1, 0, s>>>(h, mem); }

// Plain deterministic dot into sc->extra[slot].
__global__ void __launch_bounds__(256) k_dot(const double* __restrict__ a,
                                             const double* __restrict__ b, int64_t dim,
                                             double* __restrict__ partials, EvalScalars* sc,
                                             int slot) {
  double p[1] = {0.0};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x)
    p[0] = dadd(p[0], dmul(a[e], b[e]));
  double out[1];
  if (last_block_reduce<256, 1>(p, partials, &sc->ticket, out)) sc->extra[slot] = out[0];
}

void launch_dot(const double* a, const double* b, int64_t dim, double* partials, int nblocks,
                EvalScalars* sc, int slot, cudaStream_t s) {
  k_dot<<<nblocks, 256, 0, s>>>(a, b, dim, partials, sc, slot);
}

// max |a_e| into sc->extra[slot] (lpNorm<Infinity>; exact in any order).
__global__ void __launch_bounds__(256) k_absmax(const double* __restrict__ a, int64_t dim,
                                                double* __restrict__ partials, EvalScalars* sc,
                                                int slot) {
  double p[1] = {0.0};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x)
    p[0] = fmax(p[0], fabs(a[e]));
  double out[1];
  if (last_block_reduce<256, 1>(p, partials, &sc->ticket, out, true)) sc->extra[slot] = out[0];
}

void launch_absmax(const double* a, int64_t dim, double* partials, int nblocks, EvalScalars* sc,
                   int slot, cudaStream_t s) {
  k_absmax<<<nblocks, 256, 0, s>>>(a, dim, partials, sc, slot);
}


// ============================================================ fused L-BFGS step
// One cooperative launch (one CTA per SM) does the whole direction update:
//   (1) each CTA owns a slice of the vectors; one warp per history row
//       computes s_i.y_new, y_i.y_new, s_i.g, y_i.g, and one warp the new
//       pair s = x - x_prev, y = g_prev - g (written into the scratch slot)
//       with s.y, s.s, y.y, s.g, y.g;            -- grid barrier --
//   (2) CTA 0 folds the per-CTA partials in CTA order, applies the
//       acceptance test and ring update (lbfgs.hpp:243-255), maintains R and
//       YY and solves for p, gam w (warp 0, lanes own rows); -- grid barrier --
//   (3) every CTA forms its slice of d and of the first trial point x + t d
//       (lbfgs.hpp:86) and the slopes g.d, d.d;  -- grid barrier --
//   (4) CTA 0 folds the slope partials.
namespace {
constexpr int kStepThreads = 512;
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kStepBatch = 8;  // elements per lane per load batch (phase 1)
int g_step_grid = 0;
size_t g_step_smem = 0;
}  // namespace

struct StepArgs {
  int pair;
  const double *x, *xprev, *g, *gprev;  // accepted point and the previous one
  double *S, *Y;
  int64_t stride;
  HistState* h;
  CompactState* cs;
  double* d;
  const double* t;  // line-search step (device)
  double* xt;       // first trial point, or null
  int64_t dim;
  double* out;      // [0] g.d, [1] d.d
  EvalScalars* sc;
  double* part;     // [kStepMaxGrid][2] slope partials, then [grid][KS * 5] dot partials
  int ks;           // memory + 1: leading dimension of R / YY in shared memory
  unsigned long long* tl;  // diagnostic timeline or null
  int64_t m;               // with dbeta: dbeta_j = xt[m + j] - snap[m + j]
  const double* snap;
  double* dbeta;
  // column-sharded contexts: split 1 runs phase (1) and leaves
  // the folded dots in red_io ((memory + 1) * 5 doubles) for the sum
  // all-reduce, split 2 runs phases (2)-(3) from the reduced red_io; 0 = the
  // whole update. Dots and slopes skip elements below dot_lo (m on every rank
  // but rank 0: the replicated alpha part counts once over the ranks).
  int split;
  int64_t dot_lo;
  double* red_io;
};


// CTA-wide: out[v] = sum over c in [0, nc) of part[c * ld + v], v < nv.
// Thread (sub, v) = (tid / 64, tid % 64) sums a contiguous run of CTAs for
// value v (64 consecutive threads read 64 consecutive values: coalesced, all
// loads of the run in flight), then the 8 runs are added in a fixed tree.
__device__ __forceinline__ void grid_fold(const double* part, int nc, int ld, int nv,
                                          double* out) {
  __shared__ double fs[8][64];
  const int sub = threadIdx.x >> 6, vl = threadIdx.x & 63;
  const int run = (nc + 7) / 8;
  for (int v0 = 0; v0 < nv; v0 += 64) {
    const int v = v0 + vl;
    double s = 0.0;
    if (v < nv) {
      const int c0 = sub * run, c1 = min(nc, c0 + run);
      for (int cb = c0; cb < c1; cb += 24) {
        double q[24];
#pragma unroll
        for (int u = 0; u < 24; ++u) q[u] = cb + u < c1 ? __ldcg(part + (int64_t)(cb + u) * ld + v) : 0.0;
#pragma unroll
        for (int u = 0; u < 24; ++u)
          if (cb + u < c1) s = dadd(s, q[u]);
      }
    }
    fs[sub][vl] = s;
    __syncthreads();
    if (threadIdx.x < 64 && v0 + threadIdx.x < nv)
      out[v0 + threadIdx.x] = dadd(dadd(dadd(fs[0][threadIdx.x], fs[1][threadIdx.x]),
                                        dadd(fs[2][threadIdx.x], fs[3][threadIdx.x])),
                                   dadd(dadd(fs[4][threadIdx.x], fs[5][threadIdx.x]),
                                        dadd(fs[6][threadIdx.x], fs[7][threadIdx.x])));
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kStepThreads) k_lbfgs_step(const StepArgs A) {
  cg::grid_group grid = cg::this_grid();
  pdl_trigger();  // the screen may launch early; it waits for this grid
  TL_ENTER(A.tl, TL_STEP);
#ifdef GSOT_PHASE_CLOCKS
  long long clk_prev = clock64();
#endif
  const int nc = (int)gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KS = A.ks;
  const int ld = KS * 5;
  __shared__ double warp_sh[2 * kStepWarps];
  __shared__ const double* sp[kMaxMemory + 1];
  __shared__ const double* yp[kMaxMemory + 1];
  // slices: multiples of 32 elements so that lanes stay aligned
  const int64_t per = ((A.dim + nc - 1) / nc + 31) / 32 * 32;
  const int64_t lo = min(A.dim, blockIdx.x * per), hi = min(A.dim, lo + per);
  const int k = A.h->k;  // read by every CTA before CTA 0 rewrites the ring
  const int scratch = A.h->scratch;
  // the step: one read per CTA, issued now, stored after phase 1
  __shared__ double t_sh, gam_sh;
  double t_reg = 0.0;
  if (threadIdx.x == 32 && A.xt) t_reg = *A.t;
  // every CTA stages the ring state and R / YY (logical positions) now: the
  // solve runs redundantly in every CTA after the grid barrier (identical
  // inputs, identical bits), so no second barrier is needed; CTA 0 alone
  // writes the state back (after the barrier, so no CTA reads it late)
  extern __shared__ double step_dyn[];  // R, YY: KS x KS each
  double* R = step_dyn;
  double* YY = R + KS * KS;
  __shared__ double red[(kMaxMemory + 1) * 5];
  __shared__ double uu[kMaxMemory + 1], vv[kMaxMemory + 1];
  __shared__ double lc[2 * kMaxMemory + 2];  // p, gam w, gam
  __shared__ HistState hs;
  __shared__ int fl[3];  // accepted, evicted-first, count after
  // (loads issued now into registers, stored after phase 1: the latency overlaps it)
  constexpr int kHsWords = (int)(sizeof(HistState) / sizeof(int));
  static_assert(kHsWords <= 2 * kStepThreads, "HistState staging");
  int hs_reg[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = threadIdx.x + q * kStepThreads;
    hs_reg[q] = t < kHsWords ? reinterpret_cast<const int*>(A.h)[t] : 0;
  }
  double r_reg = 0.0, y_reg = 0.0;  // R / YY entry tid (k^2 <= 512; longer memories below)
  if (threadIdx.x < k * k) {
    const int i = threadIdx.x / k, jj = threadIdx.x % k;
    r_reg = A.cs->R[i * kMaxMemory + jj];
    y_reg = A.cs->YY[i * kMaxMemory + jj];
  }
  if (threadIdx.x < k) {
    sp[threadIdx.x] = A.S + A.h->order[threadIdx.x] * A.stride;
    yp[threadIdx.x] = A.Y + A.h->order[threadIdx.x] * A.stride;
  }
  __syncthreads();
  // (1) one warp per row, lanes striding the slice kStepBatch elements at a time
  const int nrows = k + (A.pair ? 1 : 0);
  const int64_t dlo = A.dot_lo;
  for (int r = warp; r < nrows && A.split != 2; r += kStepWarps) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (r == k) {  // the new pair, written into the scratch slot
      double* __restrict__ sv = A.S + scratch * A.stride;
      double* __restrict__ yv = A.Y + scratch * A.stride;
      for (int64_t e0 = lo + lane; e0 < hi; e0 += 32 * kStepBatch) {
        double xs[kStepBatch], xp[kStepBatch], gs[kStepBatch], gp[kStepBatch];
#pragma unroll
        for (int u = 0; u < kStepBatch; ++u) {
          const int64_t e = e0 + 32 * u;
          const bool in = e < hi;
          xs[u] = in ? A.x[e] : 0.0;
          xp[u] = in ? A.xprev[e] : 0.0;
          gs[u] = in ? A.g[e] : 0.0;
          gp[u] = in ? A.gprev[e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kStepBatch; ++u) {
          const int64_t e = e0 + 32 * u;
          if (e >= hi) break;
          const double s = dsub(xs[u], xp[u]), y = dsub(gp[u], gs[u]);
          sv[e] = s;
          yv[e] = y;
          if (e < dlo) continue;
          acc[0] = dadd(acc[0], dmul(s, y));
          acc[1] = dadd(acc[1], dmul(s, s));
          acc[2] = dadd(acc[2], dmul(y, y));
          acc[3] = dadd(acc[3], dmul(s, gs[u]));
          acc[4] = dadd(acc[4], dmul(y, gs[u]));
        }
      }
    } else {  // history row r: s_r.y_new, y_r.y_new, s_r.g, y_r.g
      const double* __restrict__ si = sp[r];
      const double* __restrict__ yi = yp[r];
      for (int64_t e0 = lo + lane; e0 < hi; e0 += 32 * kStepBatch) {
        double ss[kStepBatch], ys[kStepBatch], gs[kStepBatch], gp[kStepBatch];
#pragma unroll
        for (int u = 0; u < kStepBatch; ++u) {
          const int64_t e = e0 + 32 * u;
          const bool in = e < hi;
          ss[u] = in ? si[e] : 0.0;
          ys[u] = in ? yi[e] : 0.0;
          gs[u] = in ? A.g[e] : 0.0;
          gp[u] = (in && A.pair) ? A.gprev[e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kStepBatch; ++u) {
          const int64_t e = e0 + 32 * u;
          if (e >= hi) break;
          if (e < dlo) continue;
          if (A.pair) {
            const double yn = dsub(gp[u], gs[u]);
            acc[0] = dadd(acc[0], dmul(ss[u], yn));
            acc[1] = dadd(acc[1], dmul(ys[u], yn));
          }
          acc[2] = dadd(acc[2], dmul(ss[u], gs[u]));
          acc[3] = dadd(acc[3], dmul(ys[u], gs[u]));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      double v = acc[q];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) A.part[2 * kStepMaxGrid + (int64_t)blockIdx.x * ld + r * 5 + q] = v;
    }
  }
  if (threadIdx.x == 32) t_sh = t_reg;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = threadIdx.x + q * kStepThreads;
    if (t < kHsWords) reinterpret_cast<int*>(&hs)[t] = hs_reg[q];
  }
  if (threadIdx.x < k * k) {
    const int i = threadIdx.x / k, jj = threadIdx.x % k;
    R[i * KS + jj] = r_reg;
    YY[i * KS + jj] = y_reg;
  }
  for (int t = threadIdx.x + kStepThreads; t < k * k; t += kStepThreads) {
    const int i = t / k, jj = t % k;
    R[i * KS + jj] = A.cs->R[i * kMaxMemory + jj];
    YY[i * KS + jj] = A.cs->YY[i * kMaxMemory + jj];
  }
  PHASE_MARK(0);
  grid.sync();
  PHASE_MARK(1);
  if (A.split == 1) {  // sharded: this rank's folded dots, then the all-reduce
    if (blockIdx.x == 0) {
      grid_fold(A.part + 2 * kStepMaxGrid, nc, ld, nrows * 5, red);
      __syncthreads();
      for (int i = threadIdx.x; i < KS * 5; i += blockDim.x) A.red_io[i] = i < nrows * 5 ? red[i] : 0.0;
    }
    return;
  }
  // (2) every CTA: fold, ring update, R / YY maintenance, compact solve
  {
    if (A.split == 2) {
      for (int i = threadIdx.x; i < nrows * 5; i += blockDim.x) red[i] = __ldcg(A.red_io + i);
    } else {
      grid_fold(A.part + 2 * kStepMaxGrid, nc, ld, nrows * 5, red);
    }
    __syncthreads();
    PHASE_MARK(2);
    if (threadIdx.x == 32) {  // gam (lbfgs.hpp:116-119) of the newest pair, beside the ring update
      bool fresh = false;
      double sy = 0.0, yy = 0.0;
      if (A.pair) {
        sy = red[k * 5 + 0];
        yy = red[k * 5 + 2];
        fresh = sy > 1e-10 * sqrt(red[k * 5 + 1]) * sqrt(yy);  // the acceptance test below
      }
      if (!fresh) {  // no new pair: thread 0 leaves the ring's sy / yy untouched
        sy = k > 0 ? hs.sy[k - 1] : 0.0;
        yy = k > 0 ? hs.yy[k - 1] : 0.0;
      }
      gam_sh = (fresh || k > 0) && yy > 0.0 ? sy / yy : 1.0;
    }
    if (threadIdx.x == 0) {
      int accept = 0, first = 0, kk = k;
      if (A.pair) {
        const double sy = red[k * 5 + 0], ss = red[k * 5 + 1], yy = red[k * 5 + 2];
        if (blockIdx.x == 0) {
          A.sc->extra[0] = sy;
          A.sc->extra[1] = ss;
          A.sc->extra[2] = yy;
        }
        hs.last_sy = sy;
        hs.last_ss = ss;
        hs.last_yy = yy;
        accept = sy > 1e-10 * sqrt(ss) * sqrt(yy);  // lbfgs.hpp:246
        hs.accepted = accept;
        if (accept) {
          if (k == hs.mem) {  // evict the oldest (lbfgs.hpp:247-251)
            first = 1;
            const int ev = hs.order[0];
            for (int i = 1; i < k; ++i) {
              hs.order[i - 1] = hs.order[i];
              hs.rho[i - 1] = hs.rho[i];
              hs.sy[i - 1] = hs.sy[i];
              hs.yy[i - 1] = hs.yy[i];
            }
            hs.order[k - 1] = scratch;
            hs.scratch = ev;
          } else {
            hs.order[k] = scratch;
            int next = 0;
            for (;; ++next) {
              bool used = false;
              for (int i = 0; i <= k; ++i) used |= hs.order[i] == next;
              if (!used) break;
            }
            hs.scratch = next;
          }
          kk = k - first;
          hs.rho[kk] = 1.0 / sy;
          hs.sy[kk] = sy;
          hs.yy[kk] = yy;
          hs.k = kk + 1;
        }
      }
      fl[0] = accept;
      fl[1] = first;
      fl[2] = accept ? kk + 1 : k;
    }
    __syncthreads();
    PHASE_MARK(3);
    const int accept = fl[0], first = fl[1], kn = fl[2];
    if (accept && first) {  // shift R and YY up-left by one
      const int n1 = k - 1;
      double tr[8], ty[8];
      int c = 0;
      for (int t = threadIdx.x; t < n1 * n1; t += blockDim.x, ++c) {
        const int i = t / n1 + 1, jj = t % n1 + 1;
        tr[c] = R[i * KS + jj];
        ty[c] = YY[i * KS + jj];
      }
      __syncthreads();
      c = 0;
      for (int t = threadIdx.x; t < n1 * n1; t += blockDim.x, ++c) {
        const int i = t / n1, jj = t % n1;
        R[i * KS + jj] = tr[c];
        YY[i * KS + jj] = ty[c];
      }
    }
    __syncthreads();
    const int c0 = kn - 1;  // logical position of the new pair
    for (int i = threadIdx.x; i < kn; i += blockDim.x) {
      const int src = accept ? (i < c0 ? i + first : k) : i;
      const bool nw = accept && i == c0;
      uu[i] = red[src * 5 + (nw ? 3 : 2)];  // s_i . g
      vv[i] = red[src * 5 + (nw ? 4 : 3)];  // y_i . g
      if (accept && i < c0) {
        R[i * KS + c0] = red[src * 5 + 0];   // s_i . y_new
        YY[i * KS + c0] = red[src * 5 + 1];  // y_i . y_new
        YY[c0 * KS + i] = red[src * 5 + 1];
      }
      if (nw) {
        R[c0 * KS + c0] = hs.sy[c0];
        YY[c0 * KS + c0] = hs.yy[c0];
      }
    }
    __syncthreads();
    PHASE_MARK(4);
    if (warp == 0) {
      // gam (lbfgs.hpp:116-119); w = R^-1 u, z = (D + gam YY) w - gam v,
      // p = R^-T z. Lane i owns row i; substitutions are column oriented
      // (one broadcast per step), diagonal reciprocals computed up front.
      const double gam = gam_sh;
      if (kn <= 32) {
        const bool act = lane < kn;
        const double rii = act ? R[lane * KS + lane] : 1.0;
        const double rinv = act ? hs.rho[lane] : 1.0;  // 1 / s_i.y_i, kept with the ring
        double tv = act ? uu[lane] : 0.0;
        double wl = 0.0;
        for (int i = kn - 1; i >= 0; --i) {
          const double wi = __shfl_sync(0xffffffffu, dmul(tv, rinv), i);
          if (lane == i) wl = wi;
          if (lane < i) tv = dsub(tv, dmul(R[lane * KS + i], wi));
        }
        PHASE_MARK(6);
        double z = act ? dsub(dmul(rii, wl), dmul(gam, vv[lane])) : 0.0;
        for (int j = 0; j < kn; ++j) {
          const double wj = __shfl_sync(0xffffffffu, wl, j);
          if (act) z = dadd(z, dmul(dmul(gam, YY[lane * KS + j]), wj));
        }
        PHASE_MARK(8);
        double pl = 0.0;
        for (int j = 0; j < kn; ++j) {
          const double pj = __shfl_sync(0xffffffffu, dmul(z, rinv), j);
          if (lane == j) pl = pj;
          if (act && lane > j) z = dsub(z, dmul(R[j * KS + lane], pj));
        }
        PHASE_MARK(9);
        if (act) {
          lc[lane] = pl;
          lc[kMaxMemory + lane] = dmul(gam, wl);
        }
      } else {  // long memories: the same substitutions through shared memory
        __shared__ double tv[kMaxMemory + 1], wv[kMaxMemory + 1], pv[kMaxMemory + 1];
        for (int i = lane; i < kn; i += 32) tv[i] = uu[i];
        __syncwarp();
        for (int i = kn - 1; i >= 0; --i) {
          const double wi = dmul(tv[i], 1.0 / R[i * KS + i]);
          __syncwarp();
          if (lane == 0) wv[i] = wi;
          for (int j = lane; j < i; j += 32) tv[j] = dsub(tv[j], dmul(R[j * KS + i], wi));
          __syncwarp();
        }
        for (int i = lane; i < kn; i += 32) {
          double z = dsub(dmul(R[i * KS + i], wv[i]), dmul(gam, vv[i]));
          for (int j = 0; j < kn; ++j) z = dadd(z, dmul(dmul(gam, YY[i * KS + j]), wv[j]));
          tv[i] = z;
        }
        __syncwarp();
        for (int j = 0; j < kn; ++j) {
          const double pj = dmul(tv[j], 1.0 / R[j * KS + j]);
          __syncwarp();
          if (lane == 0) pv[j] = pj;
          for (int i = j + 1 + lane; i < kn; i += 32) tv[i] = dsub(tv[i], dmul(R[j * KS + i], pj));
          __syncwarp();
        }
        for (int i = lane; i < kn; i += 32) {
          lc[i] = pv[i];
          lc[kMaxMemory + i] = dmul(gam, wv[i]);
        }
      }
      if (lane == 0) lc[2 * kMaxMemory] = gam;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
      for (int t = threadIdx.x; t < (int)(sizeof(HistState) / sizeof(int)); t += blockDim.x)
        reinterpret_cast<int*>(A.h)[t] = reinterpret_cast<const int*>(&hs)[t];
      for (int t = threadIdx.x; t < kn * kn; t += blockDim.x) {  // R, YY back
        const int i = t / kn, jj = t % kn;
        A.cs->R[i * kMaxMemory + jj] = R[i * KS + jj];
        A.cs->YY[i * kMaxMemory + jj] = YY[i * KS + jj];
      }
    }
    if (threadIdx.x < kn) {  // this CTA's pointers to the (new) ring order
      sp[threadIdx.x] = A.S + hs.order[threadIdx.x] * A.stride;
      yp[threadIdx.x] = A.Y + hs.order[threadIdx.x] * A.stride;
    }
    PHASE_MARK(5);
  }
  __syncthreads();
  PHASE_MARK(7);
  const int kk = fl[2];
  const double gam = lc[2 * kMaxMemory];
  const double t = t_sh;
  double pg = 0.0, pd = 0.0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += kStepThreads) {
    const double ge = A.g[e];
    const double xe = A.xt ? A.x[e] : 0.0;
    double de = dmul(gam, ge);
    for (int i0 = 0; i0 < kk; i0 += 16) {
      double vs[16], vy[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        vs[u] = i0 + u < kk ? __ldcg(sp[i0 + u] + e) : 0.0;
        vy[u] = i0 + u < kk ? __ldcg(yp[i0 + u] + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (i0 + u < kk) de = dadd(de, dmul(lc[i0 + u], vs[u]));
      if (i0 + 16 >= kk) {  // the y terms after every s term (fixed order)
        for (int j0 = 0; j0 < i0; j0 += 16)
          for (int u = 0; u < 16; ++u)
            if (j0 + u < kk) de = dsub(de, dmul(lc[kMaxMemory + j0 + u], __ldcg(yp[j0 + u] + e)));
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (i0 + u < kk) de = dsub(de, dmul(lc[kMaxMemory + i0 + u], vy[u]));
      }
    }
    A.d[e] = de;
    if (A.xt) {
      const double v = dadd(xe, dmul(t, de));  // lbfgs.hpp:86
      A.xt[e] = v;
      if (A.dbeta && e >= A.m) A.dbeta[e - A.m] = dsub(v, A.snap[e]);
    }
    if (e >= dlo) {
      pg = dadd(pg, dmul(ge, de));
      pd = dadd(pd, dmul(de, de));
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    pg = dadd(pg, __shfl_xor_sync(0xffffffffu, pg, o));
    pd = dadd(pd, __shfl_xor_sync(0xffffffffu, pd, o));
  }
  if (lane == 0) {
    warp_sh[warp] = pg;
    warp_sh[kStepWarps + warp] = pd;
  }
  __syncthreads();
  if (threadIdx.x < 2) {  // CTA partial; k_publish folds them (fixed order)
    double v = warp_sh[threadIdx.x * kStepWarps];
    for (int w = 1; w < kStepWarps; ++w) v = dadd(v, warp_sh[threadIdx.x * kStepWarps + w]);
    A.part[blockIdx.x * 2 + threadIdx.x] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) A.sc->step_blocks = nc;
  PHASE_MARK(10);
  TL_EXIT(A.tl, TL_STEP);
}

#ifdef GSOT_PHASE_CLOCKS
extern "C" __attribute__((visibility("default"))) int gsot_debug_phase_clocks(unsigned long long* out,
                                                                               int n) {
  if (out) cudaMemcpyFromSymbol(out, g_phase_clk, sizeof(unsigned long long) * (n < 16 ? n : 16));
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_phase_clk, z, sizeof(z));
  return 0;
}
#endif

// One CTA per SM (the kernel needs all 64K registers of an SM per CTA).
int lbfgs_step_grid() {
  if (g_step_grid == 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_step_grid = std::max(1, std::min(sms, kStepMaxGrid));
  }
  return g_step_grid;
}

size_t lbfgs_step_partials(int mem) {
  return (size_t)kStepMaxGrid * ((size_t)(mem + 1) * 5 + 2);
}

void launch_lbfgs_step(int pair, const double* x, const double* xprev, const double* g,
                       const double* gprev, double* S, double* Y, int64_t stride, HistState* h,
                       CompactState* cs, double* d, const double* t, double* xt, int64_t dim,
                       double* out, EvalScalars* sc, double* part, int mem,
                       unsigned long long* tl, int64_t m, const double* snap, double* dbeta,
                       cudaStream_t s, int split, int64_t dot_lo, double* red_io) {
  const int grid = lbfgs_step_grid();
  StepArgs A{pair, x, xprev, g, gprev, S, Y, stride, h, cs, d, t, xt, dim, out, sc, part, mem + 1,
             tl, m, snap, dbeta, split, dot_lo, red_io};
  const size_t smem = sizeof(double) * 2 * (size_t)(mem + 1) * (mem + 1);
  if (smem > 48 * 1024 && smem > g_step_smem) {
    cudaFuncSetAttribute(k_lbfgs_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    g_step_smem = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kStepThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_lbfgs_step, A);
}

}  // namespace gsot
