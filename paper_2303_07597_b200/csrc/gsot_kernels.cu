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
//
// Cost layout: column-tiled. For group l (rows off_l ..
// off_l + g_l) and 32-column chunk c, the tile is g_l rows x 32 columns
// stored row-major; tile (l, c) starts at element 32 * (nw * off_l + c * g_l).
// A warp (lane = column) walking the block rows reads one contiguous 256-byte
// row of the tile per load.
#include <cooperative_groups.h>
#include <cstdlib>

#include "gsot_device.cuh"

namespace cg = cooperative_groups;

namespace gsot {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GSOT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ---------------------------------------------------------------- relayout
// Column-major m x n (device) chunk [j0, j0+ncols) -> column-tiled layout,
// through a 32 x 32 shared-memory transpose (coalesced on both sides), plus
// validate_instance's first offending entry in j-major order
// (core.hpp:118-123): min over j*m + i of !(c >= 0) || !isfinite(c).
__global__ void __launch_bounds__(256) k_relayout(DevProblem P, const double* __restrict__ src,
                                                  int64_t j0, int64_t ncols,
                                                  double* __restrict__ C,
                                                  unsigned long long* first_bad) {
  __shared__ double tile[32][33];
  const int64_t i0 = blockIdx.x * 32ll, jj0 = blockIdx.y * 32ll;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  unsigned long long bad = ~0ull;
  for (int k = ty; k < 32; k += 8) {  // read: lanes along rows
    const int64_t i = i0 + tx, jj = jj0 + k;
    double v = 0.0;
    if (i < P.m && jj < ncols) {
      v = src[jj * P.m + i];
      if (!(v >= 0.0) || !isfinite(v)) {
        const unsigned long long e = (unsigned long long)((j0 + jj) * P.m + i);
        bad = e < bad ? e : bad;
      }
    }
    tile[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {  // write: lanes along columns
    const int64_t i = i0 + k, jj = jj0 + tx;
    if (i < P.m && jj < ncols) {
      const int l = P.row_group[i];
      const int o0 = P.off[l], g = P.off[l + 1] - o0;
      const int64_t j = j0 + jj;
      C[cost_index(P.nw, o0, g, j, i - o0)] = tile[tx][k];
    }
  }
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, bad, o);
    bad = w < bad ? w : bad;
  }
  if (tx == 0 && bad != ~0ull) atomicMin(first_bad, bad);
}

void launch_relayout(const DevProblem& P, const double* src, int64_t j0, int64_t ncols,
                     double* C, unsigned long long* first_bad, cudaStream_t s) {
  dim3 grid((unsigned)((P.m + 31) / 32), (unsigned)((ncols + 31) / 32));
  k_relayout<<<grid, 256, 0, s>>>(P, src, j0, ncols, C, first_bad);
}

// ---------------------------------------------------------------- snapshot
// take_snapshot (screening.hpp:24-50): z~ = |[f]+|, k~ = |f|, o~ = |[f]-|
// per block, each a sequential sum over the block's rows. One thread per
// (l, j); a warp covers one 32-column tile and reads one 256-byte tile row per
// load.
// lazy (the solver's own snapshots): a provably-zero block (every
// residual <= 0, so z~ = 0 and k~ == o~ bit for bit) is not read and gets
// z~ = k~ = o~ = 0. Only the bounds read these, and with k~ == o~ the lower
// bound ((((k~ - A) - B) - o~) - C) - D is <= 0 < tau whatever their common
// value, as the reference's is: every decision and counter is unchanged.
// API snapshots are taken in full (gsot_snapshot_norms returns the reference's
// values; a lazy snapshot is retaken in full on request).
// One block of take_snapshot: three sequential sums over the block's rows, U
// cost loads in flight per thread. kPipe: the next batch is loaded while the
// current one is summed (the walk of a tall column is a chain of memory round
// trips: deeper batches, fewer trips).
template <int U = 8, bool kPipe = false>
__device__ __forceinline__ void snapshot_block(const DevProblem& P, const double* __restrict__ x,
                                               int o0, int g, int l, int64_t j,
                                               double* __restrict__ zs, double* __restrict__ ks,
                                               double* __restrict__ os) {
  const double bj = x[P.m + j];
  const double* __restrict__ al = x + o0;
  const double* __restrict__ cp = block_ptr(P, o0, g, j);
  double az = 0.0, ak = 0.0, ao = 0.0;
#define GSOT_SNAP_STEP(ALPHA, CVAL)                 \
  {                                                 \
    const double f = residual((ALPHA), bj, (CVAL)); \
    const double sq = dmul(f, f);                   \
    ak = dadd(ak, sq);                              \
    az = dadd(az, f > 0.0 ? sq : 0.0);              \
    ao = dadd(ao, f < 0.0 ? sq : 0.0);              \
  }
  int r = 0;
  if constexpr (kPipe) {
    double c[U], cn[U];
    if (g >= U) {
#pragma unroll
      for (int k = 0; k < U; ++k) c[k] = __ldcs(cp + kRowStride * k);
    }
    for (; r + U <= g; r += U) {
      const bool more = r + 2 * U <= g;
      if (more) {
#pragma unroll
        for (int k = 0; k < U; ++k) cn[k] = __ldcs(cp + kRowStride * (r + U + k));
      }
#pragma unroll
      for (int k = 0; k < U; ++k) GSOT_SNAP_STEP(__ldg(al + r + k), c[k]);
      if (more) {
#pragma unroll
        for (int k = 0; k < U; ++k) c[k] = cn[k];
      }
    }
  } else {
    for (; r + U <= g; r += U) {
      double c[U];
#pragma unroll
      for (int k = 0; k < U; ++k) c[k] = __ldcs(cp + kRowStride * (r + k));
#pragma unroll
      for (int k = 0; k < U; ++k) GSOT_SNAP_STEP(__ldg(al + r + k), c[k]);
    }
  }
  for (; r < g; ++r) GSOT_SNAP_STEP(__ldg(al + r), __ldcs(cp + kRowStride * r));
#undef GSOT_SNAP_STEP
  const int64_t idx = (int64_t)l * P.n + j;
  zs[idx] = sqrt(az);
  ks[idx] = sqrt(ak);
  os[idx] = sqrt(ao);
}

__global__ void __launch_bounds__(256) k_snapshot(DevProblem P, const double* __restrict__ x,
                                                  double* __restrict__ zs,
                                                  double* __restrict__ ks,
                                                  double* __restrict__ os, int lazy,
                                                  unsigned long long* __restrict__ rows_read) {
  if (lazy) pdl_wait();  // after the group maxima of x (k_group_amax)
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const bool in = j < P.n;
  if (lazy) {
    const bool zero = !in || dadd(P.amax[l], x[P.m + j]) <= (double)P.cmin[(int64_t)l * P.n + j];
    const unsigned read = __ballot_sync(0xffffffffu, !zero);  // bytes accounting (slots)
    if ((threadIdx.x & 31) == 0 && read)
      atomicAdd(rows_read + (blockIdx.x & 63), (unsigned long long)__popc(read) * g);
    if (zero) {
      if (in) {
        const int64_t idx = (int64_t)l * P.n + j;
        zs[idx] = 0.0;
        ks[idx] = 0.0;
        os[idx] = 0.0;
      }
      return;
    }
  }
  if (!in) return;
  snapshot_block(P, x, o0, g, l, j, zs, ks, os);
}

// The lazy snapshot in two kernels (contexts with a block list).
// k_snapshot_mark tests every block: a provably-zero one gets z~ = k~ = o~ = 0,
// the others (about 1 % of them during a solve) are appended to their group's
// list (one atomic per warp; groups of fewer than kSnapListMinRows rows are
// walked on the spot). k_snapshot_walk then takes one block per thread
// from the lists, group by group, so every warp of the sequential walks is
// full and walks columns of one height (in k_snapshot's lazy form a live lane
// walks its column while the other lanes of its warp have exited). Each
// block is still one thread's sequential sum: the same bits.
__global__ void __launch_bounds__(256) k_snapshot_mark(DevProblem P, const double* __restrict__ x,
                                                       double* __restrict__ zs,
                                                       double* __restrict__ ks,
                                                       double* __restrict__ os,
                                                       uint32_t* __restrict__ list,
                                                       unsigned int* __restrict__ count,
                                                       unsigned long long* __restrict__ rows_read,
                                                       unsigned char* __restrict__ zero_chunk,
                                                       double2* __restrict__ zmm,
                                                       const double* __restrict__ bmaxc) {
  pdl_wait();  // after k_group_amax: the group maxima of x, the chunk maxima of beta, count[] = 0
  pdl_trigger();
  // one warp = 32 consecutive chunks of group l, lane = chunk: a chunk whose
  // largest beta passes against its smallest cmin is provably zero whole; if
  // its z~ k~ o~ already hold zeros (zero_chunk: kept here, cleared whenever
  // another snapshot form writes the arrays) there is nothing to do. The other
  // chunks are walked one by one (lane = column).
  const int l = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t c = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32 + lane;
  const bool cvalid = c < P.nw;
  const int64_t t = (int64_t)l * P.nw + c;
  const double amx = P.amax[l];
  const bool pass = cvalid && dadd(amx, bmaxc[cvalid ? c : 0]) <= (double)P.cmn[cvalid ? t : 0];
  const bool flagged = cvalid && zero_chunk[cvalid ? t : 0] != 0;
  uint32_t fill = __ballot_sync(0xffffffffu, pass && !flagged);   // zeros to write
  uint32_t mixed = __ballot_sync(0xffffffffu, cvalid && !pass);   // column by column
  const int64_t c0 = c - lane;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  while (fill) {
    const int ci = __ffs(fill) - 1;
    fill &= fill - 1u;
    const int64_t j = (c0 + ci) * 32 + lane;
    if (j < P.n) {
      const int64_t idx = (int64_t)l * P.n + j;
      zs[idx] = 0.0;
      ks[idx] = 0.0;
      os[idx] = 0.0;
    }
    if (lane == 0) {
      zero_chunk[t + ci] = 1;
      zmm[t + ci] = make_double2(0.0, 0.0);
    }
  }
  while (mixed) {
    const int ci = __ffs(mixed) - 1;
    mixed &= mixed - 1u;
    const int64_t j = (c0 + ci) * 32 + lane;
    const bool in = j < P.n;
    const int64_t idx = (int64_t)l * P.n + j;
    const bool zero = !in || dadd(amx, x[P.m + j]) <= (double)P.cmin[idx];
    const unsigned livem = __ballot_sync(0xffffffffu, !zero);
    if (zero && in) {
      zs[idx] = 0.0;
      ks[idx] = 0.0;
      os[idx] = 0.0;
    }
    if (lane == 0) {
      zero_chunk[t + ci] = livem == 0u ? 1 : 0;
      if (livem == 0u) zmm[t + ci] = make_double2(0.0, 0.0);
    }
    if (livem == 0u) continue;
    if (lane == 0)
      atomicAdd(rows_read + (blockIdx.x & 63), (unsigned long long)__popc(livem) * (unsigned)g);
    if (g < kSnapListMinRows) {  // a short column: walked here (listing it costs more than it saves)
      if (!zero) snapshot_block(P, x, o0, g, l, j, zs, ks, os);
      continue;
    }
    unsigned int base = 0;
    if (lane == 0) base = atomicAdd(count + l, (unsigned int)__popc(livem));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (!zero) list[(int64_t)l * P.n + base + __popc(livem & ((1u << lane) - 1u))] = (uint32_t)j;
  }
}

// Per chunk: the largest beta of its valid columns (+inf if one is NaN), for
// the snapshot's whole-chunk zero test. One warp per chunk.
__global__ void __launch_bounds__(256) k_chunk_bmax(DevProblem P, const double* __restrict__ x,
                                                    double* __restrict__ bmaxc) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= P.nw) return;
  const int64_t j = c * 32 + lane;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double b = -inf;
  if (j < P.n) {
    const double v = x[P.m + j];
    b = v != v ? inf : v;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  if (lane == 0) bmaxc[c] = b;
}

constexpr int kSnapWalkX = 8;  // CTAs per group
__global__ void __launch_bounds__(128) k_snapshot_walk(DevProblem P, const double* __restrict__ x,
                                                       double* __restrict__ zs,
                                                       double* __restrict__ ks,
                                                       double* __restrict__ os,
                                                       const uint32_t* __restrict__ list,
                                                       const unsigned int* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int l = blockIdx.y;
  const unsigned int n_live = count[l];
  if (blockIdx.x * blockDim.x >= n_live) return;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  for (unsigned int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_live;
       t += gridDim.x * blockDim.x) {
    const int64_t j = (int64_t)list[(int64_t)l * P.n + t];
    if (g >= 128)
      snapshot_block<32, true>(P, x, o0, g, l, j, zs, ks, os);
    else
      snapshot_block<8, false>(P, x, o0, g, l, j, zs, ks, os);
  }
}

void launch_snapshot_lazy2(const DevProblem& P, const double* x, double* zs, double* ks, double* os,
                           uint32_t* list, unsigned int* count, unsigned long long* rows_read,
                           unsigned char* zero_chunk, double2* zmm, double* bmaxc,
                           cudaStream_t s) {
  launch_pdl(k_chunk_bmax, dim3((unsigned)((P.nw + 7) / 8)), dim3(256), 0, s, P, x, bmaxc);
  dim3 grid((unsigned)((P.nw + 255) / 256), (unsigned)P.L);  // 256 chunks per CTA
  launch_pdl(k_snapshot_mark, grid, dim3(256), 0, s, P, x, zs, ks, os, list, count, rows_read,
             zero_chunk, zmm, (const double*)bmaxc);
  launch_pdl(k_snapshot_walk, dim3(kSnapWalkX, (unsigned)P.L), dim3(128), 0, s, P, x, zs, ks, os,
             (const uint32_t*)list, (const unsigned int*)count);
}

void launch_snapshot(const DevProblem& P, const double* x, double* zs, double* ks, double* os,
                     bool lazy, unsigned long long* rows_read, cudaStream_t s) {
  dim3 grid((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  if (lazy)
    launch_pdl(k_snapshot, grid, dim3(256), 0, s, P, x, zs, ks, os, 1, rows_read);
  else
    k_snapshot<<<grid, 256, 0, s>>>(P, x, zs, ks, os, 0, rows_read);
}

// Sequential z of one block (pos_part_norm over the block rows).
__device__ __forceinline__ double block_z(const DevProblem& P, const double* __restrict__ x, int l,
                                          int64_t j) {
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const double* __restrict__ al = x + o0;
  const double bj = x[P.m + j];
  const double* __restrict__ cp = block_ptr(P, o0, g, j);
  double az = 0.0;
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[kRowStride * r]);
    const double v = f > 0.0 ? f : 0.0;
    az = dadd(az, dmul(v, v));
  }
  return sqrt(az);
}

// z per block (block mask).
__global__ void __launch_bounds__(256) k_block_z(DevProblem P, const double* __restrict__ x,
                                                 double* __restrict__ zout) {
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  zout[(int64_t)l * P.n + j] = block_z(P, x, l, j);
}

void launch_block_z(const DevProblem& P, const double* x, double* zout, cudaStream_t s) {
  dim3 grid((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  k_block_z<<<grid, 256, 0, s>>>(P, x, zout);
}

// ---------------------------------------------------------------- deltas
// compute_delta_norms (screening.hpp:63-83): per group the sequential
// pos/full/neg norms of alpha - alpha~ (one warp per group: the lanes load
// and square 32 rows at a time, lane 0 runs the three ascending chains), and
// dbeta = beta - beta~ elementwise.
__global__ void __launch_bounds__(256) k_delta(DevProblem P, const double* __restrict__ x,
                                               const double* __restrict__ xs,
                                               double* __restrict__ dpos,
                                               double* __restrict__ dfull,
                                               double* __restrict__ dneg,
                                               double* __restrict__ dbeta, int group_blocks,
                                               EvalScalars* sc, uint32_t* __restrict__ gmask) {
  pdl_trigger();
  (void)sc;
  (void)gmask;
  if ((int)blockIdx.x >= group_blocks) {
    const int64_t j = ((int64_t)blockIdx.x - group_blocks) * blockDim.x + threadIdx.x;
    if (j < P.n) dbeta[j] = dsub(x[P.m + j], xs[P.m + j]);
    return;
  }
  constexpr int kBatch = 4;  // 32-row chunks loaded per round trip
  __shared__ double sq_sh[8][kBatch * 32];
  __shared__ signed char sg_sh[8][kBatch * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = blockIdx.x * 8 + warp;
  if (l >= P.L) return;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  double ap = 0.0, af = 0.0, an = 0.0;
  for (int r0 = 0; r0 < g; r0 += kBatch * 32) {
    double xv[kBatch], sv[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int r = r0 + b * 32 + lane;
      xv[b] = r < g ? x[o0 + r] : 0.0;
      sv[b] = r < g ? xs[o0 + r] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const double da = dsub(xv[b], sv[b]);
      sq_sh[warp][b * 32 + lane] = dmul(da, da);
      sg_sh[warp][b * 32 + lane] = da > 0.0 ? 1 : (da < 0.0 ? -1 : 0);
    }
    __syncwarp();
    if (lane == 0) {
      const int cnt = min(kBatch * 32, g - r0);
      for (int k = 0; k < cnt; ++k) {
        const double s = sq_sh[warp][k];
        const signed char sg = sg_sh[warp][k];
        af = dadd(af, s);
        ap = dadd(ap, sg > 0 ? s : 0.0);
        an = dadd(an, sg < 0 ? s : 0.0);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    dpos[l] = sqrt(ap);
    dfull[l] = sqrt(af);
    dneg[l] = sqrt(an);
  }
}

void launch_delta(const DevProblem& P, const double* x, const double* xs, double* dpos,
                  double* dfull, double* dneg, double* dbeta, EvalScalars* sc, uint32_t* gmask,
                  cudaStream_t s) {
  const int gb = (P.L + 7) / 8;
  const int bb = (int)((P.n + 255) / 256);
  k_delta<<<gb + bb, 256, 0, s>>>(P, x, xs, dpos, dfull, dneg, dbeta, gb, sc, gmask);
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

// ---------------------------------------------------------------- screen (small)
// FastGradDispatcher::column's per-block decision (screening.hpp:252-275),
// layout for small problems (few CTAs of the transposed kernel below):
// active-set members are computed without a bound; every other block gets
// z_bar = (z~ + |[dalpha_l]+|) + sqrt(g_l) * [dbeta_j]+ (+ offset) and is
// skipped iff z_bar <= tau. CTA (k, l) screens the 64 chunks of group l
// covered by chunk-mask words 2k, 2k+1 (2048 columns); each warp takes eight
// chunks with all loads in flight and writes their survivor words. The CTA
// writes its chunk-mask words, (fast mode) marks its non-empty chunks in the
// per-chunk group masks, reserves their work-list slots with ONE atomic, and
// adds its GradStats::PerCall counters into one of 64 slots (integers:
// order-free). One CTA per unit keeps every unit's short dependency chain
// overlapped with the others on the SM.
__global__ void __launch_bounds__(256) k_screen_rows(DevProblem P, const double* __restrict__ zs,
                                                const uint32_t* __restrict__ aw,
                                                const double* __restrict__ dpos,
                                                const double* __restrict__ dbeta,
                                                double ub_offset, uint32_t* __restrict__ words,
                                                TaskDesc* __restrict__ tasks, EvalScalars* sc,
                                                unsigned long long* __restrict__ cnt_slots,
                                                uint32_t* __restrict__ gmask,
                                                uint32_t* __restrict__ cmask,
                                                const double* __restrict__ x,
                                                const double* __restrict__ xs, int dbeta_ready) {
  __shared__ unsigned long long cnt[8][6];
  __shared__ uint32_t cw[64];  // survivor word of each of the CTA's chunks
  __shared__ double dsh[8];
  __shared__ int base;
  pdl_wait();
  pdl_trigger();
  TL_ENTER(P.tl, TL_SCREEN);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int l = blockIdx.y;
  const int cb = blockIdx.x * 64;  // first chunk (two chunk-mask words per CTA)
  const int o0 = P.off[l];
  const unsigned long long g = (unsigned long long)(P.off[l + 1] - o0);
  // dbeta from memory (exact mode: k_delta; fast solves: the step / trial
  // kernels), else inline from x and the snapshot
  const bool db_inline = x != nullptr && !dbeta_ready;
  double zv[8], db[8];
  uint32_t am[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {  // chunk cb + warp + 8u, all loads first
    const int c = cb + warp + 8 * u;
    const int64_t j = (int64_t)c * 32 + lane;
    const bool valid = c < P.nw && j < P.n;
    am[u] = (c < P.nw && aw != nullptr) ? aw[(int64_t)l * P.nw + c] : 0u;
    zv[u] = valid ? zs[(int64_t)l * P.n + j] : 0.0;
    db[u] = valid ? (db_inline ? dsub(x[P.m + j], xs[P.m + j]) : dbeta[j]) : 0.0;
  }
  double dp;
  if (x) {
    // fused delta (fast mode): |[alpha_l - alpha~_l]+| over the group's rows,
    // per-thread strided chains, then a fixed tree (every CTA of the group
    // computes the same bits)
    double acc = 0.0;
    for (int r = threadIdx.x; r < (int)g; r += blockDim.x) {
      const double d = dsub(x[o0 + r], xs[o0 + r]);
      if (d > 0.0) acc = dadd(acc, dmul(d, d));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc = dadd(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) dsh[warp] = acc;
    __syncthreads();
    double t = dsh[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) t = dadd(t, dsh[w]);
    dp = sqrt(t);
  } else {
    dp = dpos[l];  // k_delta's reference-order norm (exact mode)
  }
  const double sg = P.sqrt_g[l];
  uint32_t my[6] = {0u, 0u, 0u, 0u, 0u, 0u};  // per CTA: at most 2048 blocks x g rows
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int c = cb + warp + 8 * u;
    const int64_t j0 = (int64_t)c * 32;
    // valid columns of the chunk; active-set members come straight from the word
    const uint32_t vmask = c >= P.nw ? 0u : (P.n - j0 >= 32 ? 0xffffffffu : ((1u << (P.n - j0)) - 1u));
    const uint32_t wa = am[u] & vmask;
    const uint32_t we = vmask & ~wa;
    bool surv = false;
    if ((we >> lane) & 1u) {
      const double zbar = dadd(dadd(dadd(zv[u], dp), dmul(sg, relu(db[u]))), ub_offset);
      surv = !(zbar <= P.tau);
    }
    const uint32_t ws = __ballot_sync(0xffffffffu, surv) | wa;
    if (lane == 0) {
      if (c < P.nw) words[(int64_t)l * P.nw + c] = ws;
      cw[warp + 8 * u] = ws;
      const uint32_t ns = __popc(ws), ne = __popc(we), nsv = __popc(we & ws);
      my[0] += __popc(wa);
      my[1] += ne - nsv;
      my[2] += nsv;
      my[3] += ne;
      my[4] += ns * (uint32_t)g;      // survivors' rows
      my[5] += ws ? (uint32_t)g : 0u;  // task rows
    }
  }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) cnt[warp][k] = my[k];  // widened
  __syncthreads();
  if (warp == 0) {  // chunk-mask words, work-list slots (chunk order within the CTA)
    const uint32_t w0 = cw[lane], w1 = cw[32 + lane];
    const unsigned ne0 = __ballot_sync(0xffffffffu, w0 != 0u);
    const unsigned ne1 = __ballot_sync(0xffffffffu, w1 != 0u);
    const int nmw = (P.nw + 31) / 32;
    if (lane == 0) {
      gmask[(int64_t)l * nmw + 2 * blockIdx.x] = ne0;
      if (2 * (int)blockIdx.x + 1 < nmw) gmask[(int64_t)l * nmw + 2 * blockIdx.x + 1] = ne1;
      const int tot = __popc(ne0) + __popc(ne1);
      base = tot ? atomicAdd(&sc->ntasks, tot) : 0;
    }
    const int nlw = (P.L + 31) / 32;
    if (cmask) {
      if (w0 != 0u) atomicOr(cmask + (int64_t)(cb + lane) * nlw + (l >> 5), 1u << (l & 31));
      if (w1 != 0u) atomicOr(cmask + (int64_t)(cb + 32 + lane) * nlw + (l >> 5), 1u << (l & 31));
    }
    __syncwarp();
    TaskDesc d;
    d.l = l;
    d.o0 = o0;
    d.g = (int)g;
    d.pad[0] = d.pad[1] = d.pad[2] = 0;
    if (w0 != 0u) {
      d.c = cb + lane;
      d.word = w0;
      tasks[base + __popc(ne0 & ((1u << lane) - 1u))] = d;
    }
    if (w1 != 0u) {
      d.c = cb + 32 + lane;
      d.word = w1;
      tasks[base + __popc(ne0) + __popc(ne1 & ((1u << lane) - 1u))] = d;
    }
  } else if (warp == 1 && lane < 6) {
    unsigned long long s = 0ull;
    for (int w = 0; w < 8; ++w) s += cnt[w][lane];
    if (s) atomicAdd(cnt_slots + ((blockIdx.y * gridDim.x + blockIdx.x) & 63u) * 8 + lane, s);
  }
  TL_EXIT(P.tl, TL_SCREEN);
}

// ---------------------------------------------------------------- screen
// FastGradDispatcher::column's per-block decision (screening.hpp:252-275):
// active-set members are computed without a bound; every other block gets
// z_bar = (z~ + |[dalpha_l]+|) + sqrt(g_l) * [dbeta_j]+ (+ offset) and is
// skipped iff z_bar <= tau.
// CTA (kx, ky) covers groups 8 ky .. 8 ky + 7 (one warp each) and the 32
// chunks of chunk-mask word kx (one lane each). Whole chunks are decided from
// per-chunk summaries (the extremes of z~, dbeta, beta and cmin; rounding is
// monotone, so the decisions are the reference's); only mixed chunks are walked
// column by column (lane = column, one ballot per chunk). Per warp: the
// survivor words, the group's chunk-mask word (one ballot); per CTA: one atomic
// reserving the non-empty chunks' work-list slots, the per-chunk group masks
// (one atomic per chunk), and the GradStats::PerCall counters into one of 64
// slots (integers: order-free). The group's delta norm comes from
// k_group_amax (fast mode: fixed tree) or k_delta (reference order).
constexpr int kScrWarps = 8;   // groups per CTA

__global__ void __launch_bounds__(256) k_screen(DevProblem P, const double* __restrict__ zs,
                                                const uint32_t* __restrict__ aw,
                                                const double* __restrict__ dpos,
                                                const double* __restrict__ dbeta,
                                                double ub_offset, uint32_t* __restrict__ words,
                                                TaskDesc* __restrict__ tasks, EvalScalars* sc,
                                                unsigned long long* __restrict__ cnt_slots,
                                                uint32_t* __restrict__ gmask,
                                                uint32_t* __restrict__ cmask,
                                                const double* __restrict__ x,
                                                const double* __restrict__ xs, int dbeta_ready,
                                                const double* __restrict__ xe,
                                                const double* __restrict__ dpre,
                                                const double2* __restrict__ zmm,
                                                const double* __restrict__ dbx3) {
  __shared__ unsigned long long cnt[kScrWarps][6];
  __shared__ int wn[kScrWarps];                        // non-empty chunks per warp
  __shared__ uint32_t gbits[kScrWarps][32];            // for the per-chunk group masks
  __shared__ int base;
  pdl_wait();
  pdl_trigger();
  TL_ENTER(P.tl, TL_SCREEN);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 32;
  const int l = blockIdx.y * kScrWarps + warp;
  const bool lvalid = l < P.L;
  const int c = c0 + lane;  // this lane's chunk
  const bool cvalid = c < P.nw;
  const bool db_inline = x != nullptr && !dbeta_ready;
  const int o0 = lvalid ? P.off[l] : 0;
  const int g = lvalid ? P.off[l + 1] - o0 : 0;
  const uint32_t am = (lvalid && cvalid && aw != nullptr) ? aw[(int64_t)l * P.nw + c] : 0u;
  double dp = 0.0;
  if (x && dpre) {
    dp = lvalid ? dpre[l] : 0.0;  // fast mode: the same norm, computed once per group (k_group_amax)
  } else if (x) {
    // fused delta (fast mode): |[alpha_l - alpha~_l]+| over the group's rows,
    // lane-strided chains, then a fixed xor tree
    double acc = 0.0;
    for (int r = lane; r < g; r += 32) {
      const double d = dsub(x[o0 + r], xs[o0 + r]);
      if (d > 0.0) acc = dadd(acc, dmul(d, d));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc = dadd(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    dp = sqrt(acc);
  } else if (lvalid) {
    dp = dpos[l];  // k_delta's reference-order norm (exact mode)
  }
  const double sg = lvalid ? P.sqrt_g[l] : 0.0;
  // Per-chunk summaries first (lane = chunk): with the chunk's extreme z~
  // (k_chunk_minmax, once per snapshot) and extreme dbeta, monotone rounding
  // gives the bound of every column between zbar(zmin, dbmin) and zbar(zmax,
  // dbmax): a chunk whose largest bound is <= tau is skipped whole, one whose
  // smallest is > tau kept whole -- the reference's decisions, without reading
  // the 32 z~. Only mixed chunks are walked (lane = column, one ballot each).
  // (the chunks' dbeta / beta extremes come from k_group_amax's chunk role)
  double dbmn = 0.0, dbmx = 0.0, bemx = 0.0;
  if (cvalid) {
    dbmn = dbx3[3 * (int64_t)c];
    dbmx = dbx3[3 * (int64_t)c + 1];
    bemx = dbx3[3 * (int64_t)c + 2];
  }
  auto zbar_of = [&](double z, double db) {
    return dadd(dadd(dadd(z, dp), dmul(sg, relu(db))), ub_offset);
  };
  uint32_t surv = 0u;  // evaluated columns with z_bar > tau
  {
    double2 zm = make_double2(0.0, 0.0);
    if (lvalid && cvalid) zm = zmm[(int64_t)l * P.nw + c];
    const bool all_skip = zbar_of(zm.y, dbmx) <= P.tau;
    const bool all_keep = !(zbar_of(zm.x, dbmn) <= P.tau);
    surv = all_skip ? 0u : 0xffffffffu;
    uint32_t need = __ballot_sync(0xffffffffu, lvalid && cvalid && !all_skip && !all_keep);
    const double* __restrict__ zrow = zs + (int64_t)(lvalid ? l : 0) * P.n;
    while (need) {  // mixed chunks, four at a time (independent loads)
      int cis[4];
      double z[4], db[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cis[u] = need ? __ffs(need) - 1 : -1;
        need &= need - 1u;
        z[u] = 0.0;
        db[u] = 0.0;
        if (cis[u] >= 0) {
          const int64_t j = (int64_t)(c0 + cis[u]) * 32 + lane;
          if (j < P.n) {
            z[u] = zrow[j];
            db[u] = db_inline ? dsub(x[P.m + j], xs[P.m + j]) : dbeta[j];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (cis[u] < 0) break;  // warp-uniform
        const uint32_t bs = __ballot_sync(0xffffffffu, !(zbar_of(z[u], db[u]) <= P.tau));
        if (lane == cis[u]) surv = bs;
      }
    }
  }
  // masks of this lane's chunk (the reference's decisions)
  const int64_t j0 = (int64_t)c * 32;
  const uint32_t vmask = (!lvalid || !cvalid) ? 0u
                         : (P.n - j0 >= 32 ? 0xffffffffu : ((1u << (P.n - j0)) - 1u));
  const uint32_t wa = am & vmask;
  const uint32_t we = vmask & ~wa;
  const uint32_t wd = (surv & we) | wa;  // the reference's decisions (counters)
  // provably-zero blocks among the chunk's computed columns:
  // max alpha + beta_j <= cmin. A chunk with nothing to compute needs no test;
  // one whose largest beta passes against its smallest cmin (k_block_min's
  // per-chunk minimum) is zero whole; the others are walked.
  uint32_t pz = 0u;  // columns possibly nonzero
  {
    const double amx = lvalid ? P.amax[l] : 0.0;
    bool detail = false;
    if (wd != 0u) detail = !(dadd(amx, bemx) <= (double)P.cmn[(int64_t)l * P.nw + c]);
    uint32_t need = __ballot_sync(0xffffffffu, detail);
    const float* __restrict__ crow = P.cmin + (int64_t)(lvalid ? l : 0) * P.n;
    while (need) {
      int cis[4];
      double be[4];
      float cm[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cis[u] = need ? __ffs(need) - 1 : -1;
        need &= need - 1u;
        be[u] = 0.0;
        cm[u] = 0.0f;
        if (cis[u] >= 0) {
          const int64_t j = (int64_t)(c0 + cis[u]) * 32 + lane;
          if (j < P.n) {
            be[u] = xe[P.m + j];
            cm[u] = crow[j];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (cis[u] < 0) break;
        const uint32_t bp = __ballot_sync(0xffffffffu, !(dadd(amx, be[u]) <= (double)cm[u]));
        if (lane == cis[u]) pz = bp;
      }
    }
  }
  const uint32_t ws = wd & pz;           // what the evaluation reads
  if (lvalid && cvalid) words[(int64_t)l * P.nw + c] = ws;
  const unsigned ne = __ballot_sync(0xffffffffu, ws != 0u);
  if (lvalid && lane == 0) gmask[(int64_t)l * ((P.nw + 31) / 32) + blockIdx.x] = ne;
  // GradStats counters of this lane's chunk, warp-reduced
  unsigned long long v[6];
  const uint32_t nsv = __popc(we & wd), nev = __popc(we);
  v[0] = __popc(wa);
  v[1] = nev - nsv;
  v[2] = nsv;
  v[3] = nev;
  v[4] = (unsigned long long)__popc(ws) * (unsigned)g;  // survivors' rows
  v[5] = ws ? (unsigned long long)g : 0ull;             // task rows
#pragma unroll
  for (int q = 0; q < 6; ++q) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) cnt[warp][q] = v[q];
    wn[warp] = __popc(ne);
  }
  gbits[warp][lane] = ws ? (1u << (l & 31)) : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kScrWarps; ++w) tot += wn[w];
    base = tot ? atomicAdd(&sc->ntasks, tot) : 0;
  }
  if (threadIdx.x >= 32 && threadIdx.x < 38) {
    const int q = threadIdx.x - 32;
    unsigned long long s = 0ull;
    for (int w = 0; w < kScrWarps; ++w) s += cnt[w][q];
    if (s) atomicAdd(cnt_slots + ((blockIdx.y * gridDim.x + blockIdx.x) & 63u) * 8 + q, s);
  }
  if (cmask && warp == 1) {  // per-chunk group masks: one atomic per chunk
    // groups 8 ky .. 8 ky + 7 share one mask word (8 divides 32)
    uint32_t bits = 0u;
#pragma unroll
    for (int w = 0; w < kScrWarps; ++w) bits |= gbits[w][lane];
    if (bits && cvalid)
      atomicOr(cmask + (int64_t)c * ((P.L + 31) / 32) + ((blockIdx.y * kScrWarps) >> 5), bits);
  }
  __syncthreads();
  if (ws != 0u) {
    int pos = base + __popc(ne & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += wn[w];
    TaskDesc d;
    d.l = l;
    d.c = c;
    d.o0 = o0;
    d.g = g;
    d.word = ws;
    d.pad[0] = d.pad[1] = d.pad[2] = 0;
    tasks[pos] = d;
  }
  TL_EXIT(P.tl, TL_SCREEN);
}

// The chunk-summary screen (k_screen) runs when its grid has at least 64 CTAs;
// smaller instances take k_screen_rows, which needs neither the per-chunk
// extremes nor the precomputed group delta norms.
bool screen_uses_summaries(const DevProblem& P, int num_sms) {
  // (GSOT_SCREEN_SUMMARIES=1 / 0 forces the choice: tests run k_screen on small instances)
  if (const char* ev = std::getenv("GSOT_SCREEN_SUMMARIES")) return std::atoi(ev) != 0;
  const int64_t gx = (P.nw + 31) / 32, gy = (P.L + kScrWarps - 1) / kScrWarps;
  // measured: config 2 (130 CTAs) 16.7 -> 14.8 ms with the summaries, config 1
  // (2 CTAs) 5.8 -> 7.5 ms: from about half a wave of CTAs upwards
  (void)num_sms;
  return gx * gy >= 64;
}

void launch_screen(const DevProblem& P, const double* zs, const uint32_t* aw, const double* dpos,
                   const double* dbeta, double ub_offset, uint32_t* words, TaskDesc* tasks,
                   EvalScalars* sc, unsigned long long* cnt_slots, uint32_t* gmask,
                   uint32_t* cmask, const double* x, const double* xs, int dbeta_ready,
                   const double* xe, const double* dpre, const double2* zmm, const double* dbx3,
                   int num_sms, cudaStream_t s) {
  const dim3 grid((unsigned)((P.nw + 31) / 32), (unsigned)((P.L + kScrWarps - 1) / kScrWarps));
  if (!screen_uses_summaries(P, num_sms)) {  // small: one CTA per (group, 2048 columns)
    const dim3 g2((unsigned)((P.nw + 63) / 64), (unsigned)P.L);
    launch_pdl(k_screen_rows, g2, dim3(256), 0, s, P, zs, aw, dpos, dbeta, ub_offset, words, tasks,
               sc, cnt_slots, gmask, cmask, x, xs, dbeta_ready);
    return;
  }
  launch_pdl(k_screen, grid, dim3(32 * kScrWarps), 0, s, P, zs, aw, dpos, dbeta, ub_offset, words,
             tasks, sc, cnt_slots, gmask, cmask, x, xs, dbeta_ready, xe, dpre, zmm, dbx3);
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

// Dense chunk masks: every chunk of every group.
__global__ void k_fill_gmask(uint32_t* gmask, int32_t L, int32_t nw) {
  const int nmw = (nw + 31) / 32;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)L * nmw) return;
  const int k = (int)(t % nmw);
  const int rem = nw - 32 * k;
  gmask[t] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}
void launch_fill_gmask(uint32_t* gmask, int32_t L, int32_t nw, cudaStream_t s) {
  const int64_t total = (int64_t)L * ((nw + 31) / 32);
  k_fill_gmask<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(gmask, L, nw);
}

// Dense per-chunk group masks: every group of every chunk.
__global__ void k_fill_cmask(uint32_t* cmask, int32_t L, int32_t nw) {
  const int nlw = (L + 31) / 32;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nw * nlw) return;
  const int k = (int)(t % nlw);
  const int rem = L - 32 * k;
  cmask[t] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}
void launch_fill_cmask(uint32_t* cmask, int32_t L, int32_t nw, cudaStream_t s) {
  const int64_t total = (int64_t)nw * ((L + 31) / 32);
  k_fill_cmask<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(cmask, L, nw);
}

// Dense task order: largest groups first (long chains start early).
__global__ void k_dense_tasks(DevProblem P, TaskDesc* tasks, const int32_t* __restrict__ order) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)P.L * P.nw) return;
  TaskDesc d;
  d.l = order[t / P.nw];
  d.c = (int)(t % P.nw);
  d.o0 = P.off[d.l];
  d.g = P.off[d.l + 1] - d.o0;
  const int64_t rem = P.n - (int64_t)d.c * 32;
  d.word = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
  d.pad[0] = d.pad[1] = d.pad[2] = 0;
  tasks[t] = d;
}
void launch_dense_tasks(const DevProblem& P, TaskDesc* tasks, const int32_t* order,
                        cudaStream_t s) {
  const int64_t total = (int64_t)P.L * P.nw;
  k_dense_tasks<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(P, tasks, order);
}

// ---------------------------------------------------------------- provably-zero blocks
// A block (l, j) whose every residual is non-positive has z = 0 exactly, so
// its plan entries, psi and column / row contributions are exact zeros: the
// evaluation need not read its cost. f_ij = RN(RN(alpha_i + beta_j) - c_ij) <= 0
// iff RN(alpha_i + beta_j) <= c_ij (a difference of doubles rounds to 0 only
// when they are equal), and rounding is monotone, so
//   RN(max_{i in l} alpha_i + beta_j) <= cmin[l][j] <= min_{i in l} c_ij
// proves it for the whole block (cmin rounded down to float: conservative; a
// NaN anywhere fails the test). On the BASELINE configs this holds for ~99 %
// of the blocks at every state of a solve (tools/zero_block_fraction.py).
__global__ void __launch_bounds__(256) k_block_min(DevProblem P, float* __restrict__ cmin) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);  // tile l * nw + c
  if (t >= (int64_t)P.L * P.nw) return;
  const int l = (int)(t / P.nw), c = (int)(t % P.nw);
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const double* __restrict__ tile = P.C + cost_index(P.nw, o0, g, 32ll * c + lane, 0);
  double v = __longlong_as_double(0x7ff0000000000000ll);  // +inf
#pragma unroll 8
  for (int r = 0; r < g; ++r) v = fmin(v, tile[kRowStride * r]);
  const int64_t j = (int64_t)c * 32 + lane;
  const float f = __double2float_rd(v);
  if (j < P.n) cmin[(int64_t)l * P.n + j] = f;
  // the chunk's smallest (valid columns): the screen's whole-chunk test
  float fm = j < P.n ? f : __int_as_float(0x7f800000);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) fm = fminf(fm, __shfl_xor_sync(0xffffffffu, fm, o));
  if (lane == 0) const_cast<float*>(P.cmn)[t] = fm;
}

// Per (group, chunk): the smallest and largest z~ of the chunk's valid columns
// (a NaN makes them -inf / +inf: the screen then walks the chunk). Once per
// snapshot, for the screen's whole-chunk decisions.
__global__ void __launch_bounds__(256) k_chunk_minmax(DevProblem P, const double* __restrict__ zs,
                                                      double2* __restrict__ zmm,
                                                      const unsigned char* __restrict__ zero_chunk) {
  pdl_wait();
  pdl_trigger();
  // one warp = 32 consecutive (group, chunk) pairs, lane = pair: the pairs that
  // are not known to hold zeros (k_snapshot_mark wrote (0, 0) for those) are
  // reduced one by one, lane = column
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)P.L * P.nw;
  const int64_t t0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
  const int64_t tl = t0 + lane;
  uint32_t todo = __ballot_sync(0xffffffffu, tl < total && !(zero_chunk && zero_chunk[tl]));
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  while (todo) {
    const int ti = __ffs(todo) - 1;
    todo &= todo - 1u;
    const int64_t t = t0 + ti;
    const int l = (int)(t / P.nw), c = (int)(t % P.nw);
    const int64_t j = (int64_t)c * 32 + lane;
    double mn = inf, mx = -inf;
    if (j < P.n) {
      const double z = zs[(int64_t)l * P.n + j];
      mn = z != z ? -inf : z;
      mx = z != z ? inf : z;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) zmm[t] = make_double2(mn, mx);
  }
}

void launch_chunk_minmax(const DevProblem& P, const double* zs, double2* zmm,
                         const unsigned char* zero_chunk, cudaStream_t s) {
  const int64_t tiles = (int64_t)P.L * P.nw;
  launch_pdl(k_chunk_minmax, dim3((unsigned)((tiles + 255) / 256)), dim3(256), 0, s, P, zs, zmm,
             zero_chunk);
}

void launch_block_min(const DevProblem& P, float* cmin, cudaStream_t s) {
  const int64_t tiles = (int64_t)P.L * P.nw;
  k_block_min<<<(unsigned)((tiles + 7) / 8), 256, 0, s>>>(P, cmin);
}

// amax[l] = max over the group's alpha (a NaN propagates: no block of the
// group is then provably zero). One warp per group.
// One stride-S scan of rows [o0, o1) by a thread starting at o0 + first: the
// maximum of alpha (NaN propagates) and, with xs, the chain of [alpha - alpha~]+^2
// in row order; eight loads in flight.
template <int S>
__device__ __forceinline__ void amax_scan(const double* __restrict__ x, const double* __restrict__ xs,
                                          int i, int o1, double& v, double& acc) {
  for (; i + 7 * S < o1; i += 8 * S) {
    double a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a[k] = x[i + S * k];
      b[k] = xs ? xs[i + S * k] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v = (a[k] > v || a[k] != a[k]) ? a[k] : v;
      const double d = dsub(a[k], b[k]);
      if (xs && d > 0.0) acc = dadd(acc, dmul(d, d));
    }
  }
  for (; i < o1; i += S) {
    const double a = x[i];
    v = (a > v || a != a) ? a : v;
    if (xs) {
      const double d = dsub(a, xs[i]);
      if (d > 0.0) acc = dadd(acc, dmul(d, d));
    }
  }
}

constexpr int kAmaxTall = 1024;  // taller groups are scanned by the whole CTA
__global__ void __launch_bounds__(256) k_group_amax(DevProblem P, const double* __restrict__ x,
                                                    double* __restrict__ amax,
                                                    unsigned int* __restrict__ zero_me,
                                                    const double* __restrict__ xs,
                                                    double* __restrict__ dfast,
                                                    const double* __restrict__ dbeta,
                                                    double* __restrict__ dbx3) {
  __shared__ double sh_v[8], sh_a[8];
  pdl_wait();
  pdl_trigger();
  const int ga = (P.L + 7) / 8;  // CTAs of the group role; the rest: chunk role
  if ((int)blockIdx.x >= ga) {
    // per chunk, for the screen's whole-chunk decisions: the extremes of dbeta
    // and the largest beta over the chunk's valid columns (a NaN makes them
    // -inf / +inf: the chunk is then walked). One warp per chunk.
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x - ga) * 8 + (threadIdx.x >> 5);
    if (c >= P.nw) return;
    const int64_t j = c * 32 + lane;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    double dmn = inf, dmx = -inf, bmx = -inf;
    if (j < P.n) {
      const double db = dbeta[j], be = x[P.m + j];
      dmn = db != db ? -inf : db;
      dmx = db != db ? inf : db;
      bmx = be != be ? inf : be;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
      dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
      bmx = fmax(bmx, __shfl_xor_sync(0xffffffffu, bmx, o));
    }
    if (lane == 0) {
      dbx3[3 * c] = dmn;
      dbx3[3 * c + 1] = dmx;
      dbx3[3 * c + 2] = bmx;
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double ninf = -__longlong_as_double(0x7ff0000000000000ll);
  // fast solves: the group's |[alpha_l - alpha~_l]+| for the screen (xs: the
  // snapshot state), strided chains in row order, then fixed trees -- once per
  // group here instead of once per screen CTA. CTA b takes groups b, b + ga,
  // b + 2 ga, ... (neighbouring groups, often of similar height, go to
  // different CTAs): a warp per group, but a group taller than kAmaxTall rows
  // by the CTA's eight warps together (config 4's 4000-row group is otherwise
  // a 16-round-trip chain for one warp).
  __shared__ int so0[8], so1[8];
  if (threadIdx.x < 8) {
    const int lt = (int)threadIdx.x * ga + (int)blockIdx.x;
    so0[threadIdx.x] = lt < P.L ? P.off[lt] : 0;
    so1[threadIdx.x] = lt < P.L ? P.off[lt + 1] : 0;
  }
  __syncthreads();
  {
    const int l = warp * ga + (int)blockIdx.x;
    const int o0 = so0[warp], o1 = so1[warp];
    if (l < P.L && o1 - o0 <= kAmaxTall) {
      double v = ninf, acc = 0.0;
      amax_scan<32>(x, xs, o0 + lane, o1, v, acc);
      if (xs) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) acc = dadd(acc, __shfl_xor_sync(0xffffffffu, acc, o));
        if (lane == 0) dfast[l] = sqrt(acc);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = (w > v || w != w) ? w : v;
      }
      if (lane == 0) {
        amax[l] = v;
        if (zero_me) zero_me[l] = 0u;  // the lazy snapshot's list length of the group
      }
    }
  }
  for (int gi = 0; gi < 8; ++gi) {  // the CTA's tall groups, one after the other
    const int l = gi * ga + (int)blockIdx.x;
    const int o0 = so0[gi], o1 = so1[gi];
    if (l >= P.L || o1 - o0 <= kAmaxTall) continue;  // (uniform over the CTA)
    double v = ninf, acc = 0.0;
    amax_scan<256>(x, xs, o0 + (int)threadIdx.x, o1, v, acc);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      acc = dadd(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      const double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = (w > v || w != w) ? w : v;
    }
    if (lane == 0) {
      sh_v[warp] = v;
      sh_a[warp] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double vv = sh_v[0], aa = sh_a[0];
      for (int w = 1; w < 8; ++w) {
        vv = (sh_v[w] > vv || sh_v[w] != sh_v[w]) ? sh_v[w] : vv;
        aa = dadd(aa, sh_a[w]);
      }
      amax[l] = vv;
      if (xs) dfast[l] = sqrt(aa);
      if (zero_me) zero_me[l] = 0u;
    }
    __syncthreads();
  }
}

void launch_group_amax(const DevProblem& P, const double* x, double* amax, cudaStream_t s,
                       unsigned int* zero_me, const double* xs, double* dfast,
                       const double* dbeta, double* dbx3) {
  const int ga = (P.L + 7) / 8, gc = dbx3 ? (P.nw + 7) / 8 : 0;
  launch_pdl(k_group_amax, dim3(ga + gc), dim3(256), 0, s, P, x, amax, zero_me, xs, dfast, dbeta,
             dbx3);
}

// ---------------------------------------------------------------- fused eval
// Persistent, warp-specialised CTAs drain the task list (the compact
// screened list, or every chunk in dense mode) through a global cursor; ONE
// CTA per task = (group l, 32-column chunk c). The task's g_l x 32 tile is
// contiguous in HBM, so a producer warp stages it -- with the g_l entries of
// alpha -- into shared memory with TMA bulk copies (cp.async.bulk + mbarrier
// complete_tx) in segments of at most `seg` rows through two slots (full /
// empty mbarriers), running ahead into the next task; four consumer warps
// compute. Within a segment, consumer warp w owns a contiguous run of rows;
// lane = column j = 32c + lane, active iff its survivor bit is set.
//   pass 1: [f]+ = max(alpha_i + beta_j - C_ij, 0) replaces the cost in
//   shared memory; z^2 = sum [f]+^2 and sum [f]+ per column (per-warp chains
//   over the warp's rows, segment after segment; the warp partials then added
//   in warp order); scale = (1 - tau/z)/gamma when z > tau (grad_block,
//   regularizer.hpp:64-74); psi = (z - tau)^2 / (2 gamma) (closed form of
//   psi_block, regularizer.hpp:78-91); column partial
//   scale * sum [f]+;
//   pass 2: row partials sum_j scale_j [f]+_ij of the chunk (T summed over
//   the chunk's columns), stored at rowpart[c*m + row]. A tile that fits one
//   segment is still resident; a taller one is streamed again.
// Every association depends only on g_l and the segment size, never on
// which blocks survived: dense and screened evaluations agree bitwise.
// The plan is never stored.
struct EvalArgs {
  DevProblem P;
  const double* x;
  const TaskDesc* order;  // task list
  const uint32_t* words;  // survivor words (dense: all valid columns)
  double* rowpart;
  double* colpart;
  double* psi;
  int seg;          // rows per shared-memory segment (<= kEvalMaxSeg)
  int qrows;        // quarter pipeline (k_eval_q): rows per quarter segment
  int qrec;         // quarter pipeline: resident quarters recompute [f]+ in pass 2 (no in-place store)
  int pz_done;      // the screen already applied the provably-zero test: the words hold only possibly-nonzero columns
  int* next_task;   // global claim cursor (zeroed per evaluation)
  int ntasks;       // >= 0: list length; -1: read *ntasks_dev (screened)
  const int* ntasks_dev;
  unsigned long long* zero_rows;  // bytes accounting: cost rows not read (provably zero)
  unsigned long long* read_qrows; // bytes accounting: 64-byte quarter rows actually fetched
};

// consumer warps per CTA: 4, or 2 for short tiles (at most kEvalShortRows rows:
// fewer warps per tile, more tiles in flight per SM); + one producer warp
__host__ __device__ constexpr int eval_threads(int nw) { return 32 * (nw + 1); }
constexpr int kEvalShortRows = 64;
constexpr int kEvalMaxSeg = 128;
// alpha slot length in doubles: seg + 2 (aligned superset), even (16-byte slots)
__host__ __device__ constexpr int aslot_len(int seg) { return (seg + 3) & ~1; }
// A slot holds a segment as four quarter planes of [rows][8] (the tile's own
// order). Plane length in doubles: an odd number of 64-byte rows,
// so the planes of a half warp's 16 lanes fall on disjoint banks.
__host__ __device__ constexpr int plane_len(int seg) { return 8 * ((seg + 1) | 1); }

struct EvalTask {
  int l, c, g, o0, nseg, valid;
  uint32_t word;
  uint32_t qm;  // quarters (8 columns) holding a surviving, possibly-nonzero block: only these are read
  int zero;  // every surviving block of the task provably zero: nothing is read
};

template <int NW>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// kRecompute (used when some block is taller than a segment): pass 1 leaves
// the cost in shared memory and pass 2 recomputes [f]+ from it, so a tile
// streamed twice needs no in-place rewrite either -- about half the shared
// memory traffic per element of such tiles, for more registers (3 CTAs per
// SM). Otherwise pass 1 writes [f]+ in place and pass 2 reads it (4 CTAs).
template <bool kRecompute, int kEvalWarps>
__global__ void __launch_bounds__(eval_threads(kEvalWarps), kRecompute ? 3 : (kEvalWarps == 4 ? 4 : 7))
    k_eval(const EvalArgs A) {
  extern __shared__ __align__(128) unsigned char eval_smem[];
  const DevProblem& P = A.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int PS = plane_len(A.seg);
  double* slots = reinterpret_cast<double*>(eval_smem);  // [2][4][PS] cost segments (quarter planes)
  double* aslots = slots + 2 * (size_t)4 * PS;           // [2][seg + 2] alpha segments
  double* bslots = aslots + 2 * (size_t)aslot_len(A.seg);     // [2][34] the task's beta chunk
  __shared__ uint64_t full[2], empty[2];
  __shared__ EvalTask tinfo[2];  // by the slot of the task's first segment
  __shared__ double zsh[kEvalWarps][32], ssh[kEvalWarps][32];
  __shared__ double scale_sh[32];
  if (threadIdx.x == 0) {  // barrier set-up overlaps the predecessor's tail
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], kEvalWarps);
    mbar_init(&empty[1], kEvalWarps);
    mbar_fence_init();
  }
  // the cost slots start zeroed (a quarter that is never fetched must not
  // hold NaN / Inf bit patterns); generic-proxy writes before the TMA's
  for (int i = threadIdx.x; i < 2 * 4 * PS; i += blockDim.x) slots[i] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  TL_ENTER(P.tl, TL_EVAL);
  if (warp == kEvalWarps) {  // ---- producer (the whole warp; lane 0 issues)
    const int ntasks = A.ntasks >= 0 ? A.ntasks : *(volatile const int*)A.ntasks_dev;
    auto fetch = [&](int t) {  // claimed task -> descriptor (one 32-byte load)
      EvalTask T{};
      T.valid = t < ntasks;
      if (T.valid) {
        const int4 a = __ldg(reinterpret_cast<const int4*>(A.order + t));
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(A.order + t) + 4);
        T.l = a.x;
        T.c = a.y;
        T.o0 = a.z;
        T.g = a.w;
        T.word = w;
        T.nseg = (T.g + A.seg - 1) / A.seg;
        // provably zero (k_block_min): every surviving column's
        // max alpha + beta_j <= its block's min cost -- lane = column
        const int64_t j = 32ll * T.c + lane;
        const bool act = (w >> lane) & 1u;
        const bool maybe =
            act && (A.pz_done ||
                    !(dadd(P.amax[T.l], A.x[P.m + j]) <= (double)P.cmin[(int64_t)T.l * P.n + j]));
        const uint32_t mb = __ballot_sync(0xffffffffu, maybe);
        T.qm = ((mb & 0xffu) ? 1u : 0u) | ((mb & 0xff00u) ? 2u : 0u) | ((mb & 0xff0000u) ? 4u : 0u) |
               ((mb & 0xff000000u) ? 8u : 0u);
        T.zero = T.qm == 0u;
      }
      return T;
    };
    // CTA b starts with tasks b and b + grid; further tasks are claimed from
    // 2 * grid onwards, the claim (one atomic, lane 0) in flight while the
    // next task's descriptor is fetched
    const int G = (int)gridDim.x;
    const uint64_t pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
    uint32_t e = 0;
    EvalTask T = fetch(blockIdx.x);
    int tn = T.valid ? G + (int)blockIdx.x : ntasks;  // one task ahead
    for (;;) {
      const double* tile = P.C + 32 * ((int64_t)P.nw * T.o0 + (int64_t)T.c * T.g);
      const int ne = (!T.valid || T.zero) ? 1 : T.nseg == 1 ? 1 : 2 * T.nseg;
      EvalTask Tn{};
      for (int k = 0; k < ne; ++k, ++e) {
        const int slot = e & 1u;
        if (e >= 2) mbar_wait_sleep(&empty[slot], ((e >> 1) - 1) & 1u);
        if (k == 0 && lane == 0) tinfo[slot] = T;
        if (!T.valid) {
          if (lane == 0) mbar_arrive(&full[slot]);  // end marker
          goto producer_done;
        }
        if (T.zero) {
          if (lane == 0) {
            mbar_arrive(&full[slot]);  // no bytes: the consumers write zeros
            atomicAdd(A.zero_rows, (unsigned long long)__popc(T.word) * (unsigned long long)T.g);
          }
        } else if (lane == 0) {
          if (k == 0) {  // bytes accounting: surviving columns in quarters that are not read
            uint32_t dead = 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (!((T.qm >> q) & 1u)) dead |= 0xffu << (8 * q);
            if (dead & T.word)
              atomicAdd(A.zero_rows,
                        (unsigned long long)__popc(T.word & dead) * (unsigned long long)T.g);
            atomicAdd(A.read_qrows, (unsigned long long)__popc(T.qm) * (unsigned long long)T.g *
                                        (unsigned long long)(T.nseg == 1 ? 1 : 2));
          }
          // alpha rides along with each cost segment (x is 16-byte aligned)
          const int r0 = (k < T.nseg ? k : 2 * T.nseg - 1 - k) * A.seg, rows = min(A.seg, T.g - r0);
          const int64_t a0 = (T.o0 + r0) & ~1ll;  // 16-byte aligned superset of the rows
          const uint32_t abytes = (uint32_t)(((T.o0 + r0 + rows - a0) + 1) & ~1ll) * 8u;
          // the task's beta chunk rides along with its first segment
          const int64_t b0 = (P.m + 32ll * T.c) & ~1ll;
          const int64_t bn = P.m + P.n - b0 < 34 ? P.m + P.n - b0 : 34;
          const uint32_t bbytes = k == 0 ? (uint32_t)((bn + 1) & ~1ll) * 8u : 0u;
          mbar_expect_tx(&full[slot], (uint32_t)rows * 64u * (uint32_t)__popc(T.qm) + abytes + bbytes);
          // a tile streamed twice stays in L2 between its passes (evict_last
          // on the first pass); everything else is read once (evict_first)
          const uint64_t pol = (T.nseg > 1 && k < T.nseg) ? pol_keep : pol_stream;
#pragma unroll
          for (int q = 0; q < 4; ++q)  // one contiguous run per live quarter
            if ((T.qm >> q) & 1u)
              tma_load_1d_hint(slots + ((size_t)slot * 4 + q) * PS,
                               tile + (int64_t)q * kPlaneCols * T.g + (int64_t)r0 * kRowStride,
                               (uint32_t)rows * 64u, &full[slot], pol);
          tma_load_1d(aslots + (size_t)slot * aslot_len(A.seg), A.x + a0, abytes, &full[slot]);
          if (k == 0) tma_load_1d(bslots + (size_t)slot * 34, A.x + b0, bbytes, &full[slot]);
        }
        if (k == 0) {
          // decode the next task and claim the one after while this one loads
          int tc = 0;
          if (lane == 0) tc = atomicAdd(A.next_task, 1);
          Tn = fetch(tn);
          tn = 2 * G + __shfl_sync(0xffffffffu, tc, 0);
        }
      }
      T = Tn;
    }
  producer_done:
    return;
  }
  // ---- consumers
  const int rr = lane & 15, hh = lane >> 4;  // row-reduction roles (pass 2)
  // first column of this lane's p-th column pair, rotated by rr: the eight
  // lanes of a quarter warp read eight distinct 16-byte words of their rows
  // (no bank conflicts for 16-byte shared loads)
  int pcol[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) pcol[p] = hh * 16 + 2 * ((p + rr) & 7);
  // pair p in the quarter planes: pairs with (p + rr) & 7 < 4 lie in the first
  // plane of the lane's half, the others in the second
  const int ql = lane >> 3;  // this lane's quarter (pass 1: lane = column)
  uint32_t e = 0;
  for (;;) {
    mbar_wait_sleep(&full[e & 1u], (e >> 1) & 1u);
    const EvalTask T = tinfo[e & 1u];
    if (!T.valid) break;
    if (T.zero) {  // provably zero: the exact zeros a computed block would give
      for (int r = warp * 32 + lane; r < T.g; r += 32 * kEvalWarps)
        A.rowpart[(int64_t)T.c * P.m + T.o0 + r] = 0.0;
      if (warp == 0 && ((T.word >> lane) & 1u)) {
        const int64_t idx = (int64_t)T.l * P.n + (int64_t)T.c * 32 + lane;
        A.colpart[idx] = 0.0;
        A.psi[idx] = 0.0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[e & 1u]);
      ++e;
      continue;
    }
    const uint32_t s0 = e & 1u;  // the slot of the task's first segment (its beta chunk)
    const int64_t j = (int64_t)T.c * 32 + lane;
    const bool act = (T.word >> lane) & 1u;
    // a surviving column in a quarter that was not fetched is provably zero:
    // z2 = sv = 0 below give the exact zeros its computation would
    const bool qlive = (T.qm >> ql) & 1u;
    const bool live = act && qlive;
    const double bj =
        act ? bslots[(size_t)(e & 1u) * 34 + ((P.m + 32ll * T.c) & 1) + lane] : 0.0;
    double z2 = 0.0, sv = 0.0;
    double scr[16], bq[16];  // scales and betas of this lane's 8 rotated column pairs
    const int ne = T.nseg == 1 ? 1 : 2 * T.nseg;
    for (int k = 0; k < ne; ++k, ++e) {
      const int slot = e & 1u;
      if (k > 0) mbar_wait_sleep(&full[slot], (e >> 1) & 1u);
      double* __restrict__ buf = slots + (size_t)slot * 4 * PS;
      const int sgm = k < T.nseg ? k : 2 * T.nseg - 1 - k;  // pass 2 backwards (L2-warm first)
      const int r0 = sgm * A.seg, rows = min(A.seg, T.g - r0);
      const int R = (rows + kEvalWarps - 1) / kEvalWarps;
      const int w0 = min(rows, warp * R), w1 = min(rows, w0 + R);
      const double* __restrict__ as = aslots + (size_t)slot * aslot_len(A.seg) + ((T.o0 + r0) & 1);
      double* __restrict__ col = buf + ql * PS + (lane & 7);
      if constexpr (kRecompute) {
        if (live && k < T.nseg) {  // pass 1: accumulate
#pragma unroll 4
          for (int r = w0; r < w1; ++r) {
            const double v = relu(residual(as[r], bj, col[r * kRowStride]));
            z2 = dfma(v, v, z2);
            sv = dadd(sv, v);
          }
        }
      } else if (live) {
        if (k < T.nseg) {  // pass 1: accumulate ([f]+ in place of the cost)
#pragma unroll 4
          for (int r = w0; r < w1; ++r) {
            const double v = relu(residual(as[r], bj, col[r * kRowStride]));
            z2 = dfma(v, v, z2);
            sv = dadd(sv, v);
            col[r * kRowStride] = v;
          }
        } else {  // re-streamed segment: [f]+ only
#pragma unroll 4
          for (int r = w0; r < w1; ++r)
            col[r * kRowStride] = relu(residual(as[r], bj, col[r * kRowStride]));
        }
      } else if (!qlive) {
        // the columns of a quarter that was not fetched get zeros, so pass 2
        // never meets stale shared memory
#pragma unroll 4
        for (int r = w0; r < w1; ++r) col[r * kRowStride] = 0.0;
      }
      if (k == T.nseg - 1) {  // pass 1 complete: the warps in order (warp 0)
        zsh[warp][lane] = z2;
        ssh[warp][lane] = sv;
        consumer_sync<kEvalWarps>();
        if (warp == 0) {
          double zz = zsh[0][lane], ss = ssh[0][lane];
#pragma unroll
          for (int w = 1; w < kEvalWarps; ++w) {
            zz = dadd(zz, zsh[w][lane]);
            ss = dadd(ss, ssh[w][lane]);
          }
          // scale = (1 - tau/z)/gamma as (z - tau)/(gamma z) and psi =
          // (z - tau)^2/(2 gamma) with 1/(2 gamma) hoisted: one division per
          // column on the tile's serial section
          // (the recomputing variant, whose tiles are tall, keeps the
          // two-division form: measured faster there)
          const double z = sqrt(zz);
          const bool nz = act && z > P.tau;
          const double d = dsub(z, P.tau);
          const double scale = !nz ? 0.0
                               : kRecompute ? ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma)
                                            : ddiv(d, dmul(P.gamma, z));
          scale_sh[lane] = scale;
          if (act) {
            const int64_t idx = (int64_t)T.l * P.n + j;
            A.colpart[idx] = dmul(scale, ss);
            A.psi[idx] = !nz ? 0.0
                         : kRecompute ? ddiv(dmul(d, d), dmul(2.0, P.gamma))
                                      : dmul(dmul(d, d), P.half_inv_gamma);
          }
        }
        consumer_sync<kEvalWarps>();
        // scales and betas of this lane's 16 rotated columns (the task's beta
        // slot is not reused before its last segment; columns >= n: 0)
        const double* bsl = bslots + (size_t)s0 * 34 + ((P.m + 32ll * T.c) & 1);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int cq = pcol[q >> 1] + (q & 1);
          scr[q] = scale_sh[cq];
          if constexpr (kRecompute) bq[q] = 32ll * T.c + cq < P.n ? bsl[cq] : 0.0;
        }
      }
      if (T.nseg == 1 || k >= T.nseg) {
        // pass 2: row partial sum_j scale_j [f]+_ij of the chunk ([f]+ read,
        // or recomputed from the resident cost: the same bits as pass 1). Lane
        // (rr, hh) sums half hh of a row, two columns per 16-byte load (pairs in
        // rotated order: no bank conflicts), then the two halves; 16 rows at a
        // time. Inactive columns have scale 0 and a finite [f]+: an exact zero,
        // as in a dense evaluation; a quarter that was not fetched has every
        // scale 0 and holds zeros (in place) or stale finite costs
        // (recomputing variant: the slots start zeroed).
        __syncwarp();
        for (int rb = w0; rb < w1; rb += 16) {
          double acc = 0.0;
          if (rr < w1 - rb) {
            const double* __restrict__ row = buf + (rb + rr) * kRowStride;
            const double ar = kRecompute ? as[rb + rr] : 0.0;
#pragma unroll
            for (int p = 0; p < 8; ++p) {
              const double2 v = *reinterpret_cast<const double2*>(
                  row + (pcol[p] >> 3) * PS + (pcol[p] & 7));
              if constexpr (kRecompute) {
                acc = dfma(scr[2 * p], relu(residual(ar, bq[2 * p], v.x)), acc);
                acc = dfma(scr[2 * p + 1], relu(residual(ar, bq[2 * p + 1], v.y)), acc);
              } else {
                acc = dfma(scr[2 * p], v.x, acc);
                acc = dfma(scr[2 * p + 1], v.y, acc);
              }
            }
          }
          acc = dadd(acc, __shfl_xor_sync(0xffffffffu, acc, 16));
          if (hh == 0 && rr < w1 - rb) A.rowpart[(int64_t)T.c * P.m + T.o0 + r0 + rb + rr] = acc;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
    }
  }
  TL_EXIT(P.tl, TL_EVAL);
}


// ---------------------------------------------------------------- quarter pipeline
// The evaluation for instances with groups taller than a whole-tile segment
// (variant 3). The cost tile of a task is stored as four 8-column quarter
// planes, each one contiguous run of g_l * 64 bytes, so a
// group of up to `qrows` rows fits a 32 KB slot one QUARTER at a time:
//   short tasks (g <= seg): the whole tile in one slot, computed as in k_eval
//     (lane = column; [f]+ in place; row sums from shared memory);
//   tall tasks: one step per live quarter. Thread (warp w, lane) = (row slice
//     rs = lane / 8, column cj = lane % 8) walks rows 16 i + 4 w + rs in pass 1
//     ([f]+ in place, z^2 and sum [f]+ chains; a warp reads 256 contiguous
//     bytes per step); the 16 partials per column are folded by a fixed
//     butterfly (lanes) and in warp order; pass 2 is one thread per row over
//     the quarter's 8 columns (16-byte loads, pairs rotated by (lane / 2) % 4:
//     no bank conflicts), the row's sum carried in a register across the
//     task's quarters. The tile is read ONCE; quarters without a surviving,
//     possibly-nonzero block are never fetched.
//   groups taller than qrows: per quarter, 2 x ceil(g / qrows) steps (pass 2
//     streams the quarter again, from L2, and recomputes [f]+); the row sums
//     of the task's quarters are added in global memory by the thread that
//     owns the row.
// As in k_eval every association depends only on the shape (g_l, seg, qrows),
// never on the screen: quarters that are not fetched and inactive columns
// contribute exact zeros.
__global__ void __launch_bounds__(eval_threads(4), 3) k_eval_q(const EvalArgs A) {
  constexpr int NW = 4;
  extern __shared__ __align__(128) unsigned char eval_smem[];
  const DevProblem& P = A.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int PS = plane_len(A.seg), QR = A.qrows;
  const int slot_len = max(4 * PS, QR * kPlaneCols);
  const int al_len = aslot_len(max(A.seg, QR));
  double* slots = reinterpret_cast<double*>(eval_smem);  // [2][slot_len]
  double* aslots = slots + 2 * (size_t)slot_len;         // [2][al_len]
  double* bslots = aslots + 2 * (size_t)al_len;          // [2][34]
  __shared__ uint64_t full[2], empty[2];
  __shared__ EvalTask tinfo[2];
  __shared__ double zsh[NW][32], ssh[NW][32];
  __shared__ __align__(16) double scale_sh[32];
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], NW);
    mbar_init(&empty[1], NW);
    mbar_fence_init();
  }
  for (int i = threadIdx.x; i < 2 * slot_len; i += blockDim.x) slots[i] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  TL_ENTER(P.tl, TL_EVAL);
  if (warp == NW) {  // ---- producer
    const int ntasks = A.ntasks >= 0 ? A.ntasks : *(volatile const int*)A.ntasks_dev;
    auto fetch = [&](int t) {
      EvalTask T{};
      T.valid = t < ntasks;
      if (T.valid) {
        const int4 a = __ldg(reinterpret_cast<const int4*>(A.order + t));
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(A.order + t) + 4);
        T.l = a.x;
        T.c = a.y;
        T.o0 = a.z;
        T.g = a.w;
        T.word = w;
        T.nseg = T.g <= A.seg ? 1 : (T.g + QR - 1) / QR;
        const int64_t j = 32ll * T.c + lane;
        const bool act = (w >> lane) & 1u;
        const bool maybe =
            act && (A.pz_done ||
                    !(dadd(P.amax[T.l], A.x[P.m + j]) <= (double)P.cmin[(int64_t)T.l * P.n + j]));
        T.qm = quarter_mask(__ballot_sync(0xffffffffu, maybe));
        T.zero = T.qm == 0u;
      }
      return T;
    };
    // CTA b starts with tasks b and b + grid; further tasks are claimed from
    // 2 * grid onwards, the claim in flight while the next descriptor is fetched
    const int G = (int)gridDim.x;
    const uint64_t pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
    uint32_t e = 0;
    EvalTask T = fetch(blockIdx.x);
    int tn = T.valid ? G + (int)blockIdx.x : ntasks;
    // one step: wait for the slot, publish the task with its first step
    auto acquire = [&](bool first) {
      const int slot = e & 1u;
      if (e >= 2) mbar_wait_sleep(&empty[slot], ((e >> 1) - 1) & 1u);
      if (first && lane == 0) tinfo[slot] = T;
      return slot;
    };
    auto alpha_beta = [&](int slot, int r0, int rows, uint32_t& bytes) {  // lane 0
      const int64_t a0 = (T.o0 + r0) & ~1ll;
      const uint32_t abytes = (uint32_t)(((T.o0 + r0 + rows - a0) + 1) & ~1ll) * 8u;
      const int64_t b0 = (P.m + 32ll * T.c) & ~1ll;
      const int64_t bn = P.m + P.n - b0 < 34 ? P.m + P.n - b0 : 34;
      const uint32_t bbytes = (uint32_t)((bn + 1) & ~1ll) * 8u;
      bytes += abytes + bbytes;
      mbar_expect_tx(&full[slot], bytes);
      tma_load_1d(aslots + (size_t)slot * al_len, A.x + a0, abytes, &full[slot]);
      tma_load_1d(bslots + (size_t)slot * 34, A.x + b0, bbytes, &full[slot]);
    };
    for (;;) {
      EvalTask Tn{};
      bool first = true;
      auto prefetch_next = [&]() {  // decode the next task while this one loads
        int tc = 0;
        if (lane == 0) tc = atomicAdd(A.next_task, 1);
        Tn = fetch(tn);
        tn = 2 * G + __shfl_sync(0xffffffffu, tc, 0);
      };
      if (!T.valid) {
        const int slot = acquire(true);
        if (lane == 0) mbar_arrive(&full[slot]);  // end marker
        break;
      }
      const double* tile = P.C + 32 * ((int64_t)P.nw * T.o0 + (int64_t)T.c * T.g);
      if (T.zero) {
        const int slot = acquire(true);
        if (lane == 0) {
          mbar_arrive(&full[slot]);
          atomicAdd(A.zero_rows, (unsigned long long)__popc(T.word) * (unsigned long long)T.g);
        }
        ++e;
        prefetch_next();
        T = Tn;
        continue;
      }
      if (lane == 0) {  // bytes accounting
        const uint32_t dead = ~quarter_lanes(T.qm);
        if (dead & T.word)
          atomicAdd(A.zero_rows, (unsigned long long)__popc(T.word & dead) * (unsigned long long)T.g);
        atomicAdd(A.read_qrows, (unsigned long long)__popc(T.qm) * (unsigned long long)T.g *
                                    (unsigned long long)(T.nseg == 1 ? 1 : 2));
      }
      if (T.g <= A.seg) {  // short: the whole tile (its live quarters) in one step
        const int slot = acquire(true);
        if (lane == 0) {
          uint32_t bytes = (uint32_t)T.g * 64u * (uint32_t)__popc(T.qm);
          alpha_beta(slot, 0, T.g, bytes);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if ((T.qm >> q) & 1u)
              tma_load_1d_hint(slots + (size_t)slot * slot_len + (size_t)q * PS,
                               tile + (int64_t)q * kPlaneCols * T.g, (uint32_t)T.g * 64u,
                               &full[slot], pol_stream);
        }
        ++e;
        prefetch_next();
      } else {
        const int ne = T.nseg == 1 ? 1 : 2 * T.nseg;
        for (int q = 0; q < 4; ++q) {
          if (!((T.qm >> q) & 1u)) continue;
          for (int k = 0; k < ne; ++k, ++e) {
            const int slot = acquire(first);
            if (lane == 0) {
              const int r0 = (k < T.nseg ? k : 2 * T.nseg - 1 - k) * QR, rows = min(QR, T.g - r0);
              uint32_t bytes = (uint32_t)rows * 64u;
              alpha_beta(slot, r0, rows, bytes);
              tma_load_1d_hint(slots + (size_t)slot * slot_len,
                               tile + (int64_t)q * kPlaneCols * T.g + (int64_t)r0 * kRowStride,
                               (uint32_t)rows * 64u, &full[slot],
                               (T.nseg > 1 && k < T.nseg) ? pol_keep : pol_stream);
            }
            if (first) {
              first = false;
              prefetch_next();
            }
          }
        }
      }
      T = Tn;
    }
    return;
  }
  // ---- consumers
  const int rr = lane & 15, hh = lane >> 4;  // short tasks, pass 2 (as k_eval)
  int pcol[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) pcol[p] = hh * 16 + 2 * ((p + rr) & 7);
  const int ql = lane >> 3;
  const int rs = lane >> 3, cj = lane & 7;  // tall tasks, pass 1
  const int rho = (lane >> 1) & 3;          // tall tasks, pass 2: pair rotation
  const int trow = warp * 32 + lane;        // tall tasks, pass 2: first row of the thread
  uint32_t e = 0;
  for (;;) {
    mbar_wait_sleep(&full[e & 1u], (e >> 1) & 1u);
    const EvalTask T = tinfo[e & 1u];
    if (!T.valid) break;
    if (T.zero) {
      for (int r = warp * 32 + lane; r < T.g; r += 32 * NW)
        A.rowpart[(int64_t)T.c * P.m + T.o0 + r] = 0.0;
      if (warp == 0 && ((T.word >> lane) & 1u)) {
        const int64_t idx = (int64_t)T.l * P.n + (int64_t)T.c * 32 + lane;
        A.colpart[idx] = 0.0;
        A.psi[idx] = 0.0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[e & 1u]);
      ++e;
      continue;
    }
    const int boff = (int)((P.m + 32ll * T.c) & 1);
    if (T.g <= A.seg) {
      // ---- short task: one resident step, lane = column (k_eval's in-place form)
      const int slot = e & 1u;
      double* __restrict__ buf = slots + (size_t)slot * slot_len;
      const int64_t j = (int64_t)T.c * 32 + lane;
      const bool act = (T.word >> lane) & 1u;
      const bool qlive = (T.qm >> ql) & 1u;
      const bool live = act && qlive;
      const double bj = act ? bslots[(size_t)slot * 34 + boff + lane] : 0.0;
      const int rows = T.g;
      const int R = (rows + NW - 1) / NW;
      const int w0 = min(rows, warp * R), w1 = min(rows, w0 + R);
      const double* __restrict__ as = aslots + (size_t)slot * al_len + (T.o0 & 1);
      double* __restrict__ col = buf + ql * PS + cj;
      double z2 = 0.0, sv = 0.0;
      if (live) {
#pragma unroll 4
        for (int r = w0; r < w1; ++r) {
          const double v = relu(residual(as[r], bj, col[r * kRowStride]));
          z2 = dfma(v, v, z2);
          sv = dadd(sv, v);
          col[r * kRowStride] = v;
        }
      } else if (!qlive) {  // a quarter that was not fetched gets zeros
#pragma unroll 4
        for (int r = w0; r < w1; ++r) col[r * kRowStride] = 0.0;
      }
      zsh[warp][lane] = z2;
      ssh[warp][lane] = sv;
      consumer_sync<NW>();
      if (warp == 0) {
        double zz = zsh[0][lane], ss = ssh[0][lane];
#pragma unroll
        for (int w = 1; w < NW; ++w) {
          zz = dadd(zz, zsh[w][lane]);
          ss = dadd(ss, ssh[w][lane]);
        }
        const double z = sqrt(zz);
        const bool nz = act && z > P.tau;
        const double d = dsub(z, P.tau);
        const double scale = !nz ? 0.0 : ddiv(d, dmul(P.gamma, z));
        scale_sh[lane] = scale;
        if (act) {
          const int64_t idx = (int64_t)T.l * P.n + j;
          A.colpart[idx] = dmul(scale, ss);
          A.psi[idx] = !nz ? 0.0 : dmul(dmul(d, d), P.half_inv_gamma);
        }
      }
      consumer_sync<NW>();
      double scr[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) scr[q] = scale_sh[pcol[q >> 1] + (q & 1)];
      for (int rb = w0; rb < w1; rb += 16) {
        double acc = 0.0;
        if (rr < w1 - rb) {
          const double* __restrict__ row = buf + (rb + rr) * kRowStride;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const double2 v =
                *reinterpret_cast<const double2*>(row + (pcol[p] >> 3) * PS + (pcol[p] & 7));
            acc = dfma(scr[2 * p], v.x, acc);
            acc = dfma(scr[2 * p + 1], v.y, acc);
          }
        }
        acc = dadd(acc, __shfl_xor_sync(0xffffffffu, acc, 16));
        if (hh == 0 && rr < w1 - rb) A.rowpart[(int64_t)T.c * P.m + T.o0 + rb + rr] = acc;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      ++e;
      continue;
    }
    // ---- tall task: its live quarters one after the other
    if (warp == 0) {  // survivors in quarters that are not fetched: exact zeros
      if (((T.word & ~quarter_lanes(T.qm)) >> lane) & 1u) {
        const int64_t idx = (int64_t)T.l * P.n + (int64_t)T.c * 32 + lane;
        A.colpart[idx] = 0.0;
        A.psi[idx] = 0.0;
      }
    }
    const int nseg = T.nseg;
    double racc[4] = {0.0, 0.0, 0.0, 0.0};  // resident quarters: the rows' sums so far
    bool first_step = true, first_q = true;
    for (int q = 0; q < 4; ++q) {
      if (!((T.qm >> q) & 1u)) continue;
      const bool act = (T.word >> (8 * q + cj)) & 1u;
      double z2 = 0.0, sv = 0.0;
      double2 sr[4], br[4];  // this thread's rotated scale / beta pairs (pass 2)
      const int ne = nseg == 1 ? 1 : 2 * nseg;
      for (int k = 0; k < ne; ++k, ++e) {
        const int slot = e & 1u;
        if (!first_step) mbar_wait_sleep(&full[slot], (e >> 1) & 1u);
        first_step = false;
        double* __restrict__ buf = slots + (size_t)slot * slot_len;
        const int sgm = k < nseg ? k : 2 * nseg - 1 - k;
        const int r0 = sgm * QR, rows = min(QR, T.g - r0);
        const double* __restrict__ as = aslots + (size_t)slot * al_len + ((T.o0 + r0) & 1);
        const double* __restrict__ bs = bslots + (size_t)slot * 34 + boff + 8 * q;
        if (k < nseg && act) {  // pass 1
          const double bj = bs[cj];
          double* __restrict__ colp = buf + cj;
          if (nseg == 1 && !A.qrec) {
#pragma unroll 4
            for (int r = 4 * warp + rs; r < rows; r += 16) {
              const double v = relu(residual(as[r], bj, colp[r * kRowStride]));
              z2 = dfma(v, v, z2);
              sv = dadd(sv, v);
              colp[r * kRowStride] = v;
            }
          } else {
#pragma unroll 4
            for (int r = 4 * warp + rs; r < rows; r += 16) {
              const double v = relu(residual(as[r], bj, colp[r * kRowStride]));
              z2 = dfma(v, v, z2);
              sv = dadd(sv, v);
            }
          }
        }
        if (k == nseg - 1) {  // pass 1 complete: fold the 16 partials per column
          z2 = dadd(z2, __shfl_xor_sync(0xffffffffu, z2, 8));
          sv = dadd(sv, __shfl_xor_sync(0xffffffffu, sv, 8));
          z2 = dadd(z2, __shfl_xor_sync(0xffffffffu, z2, 16));
          sv = dadd(sv, __shfl_xor_sync(0xffffffffu, sv, 16));
          if (lane < 8) {
            zsh[warp][lane] = z2;
            ssh[warp][lane] = sv;
          }
          consumer_sync<NW>();
          if (warp == 0 && lane < 8) {
            double zz = zsh[0][lane], ss = ssh[0][lane];
#pragma unroll
            for (int w = 1; w < NW; ++w) {
              zz = dadd(zz, zsh[w][lane]);
              ss = dadd(ss, ssh[w][lane]);
            }
            const double z = sqrt(zz);
            const bool nz = act && z > P.tau;
            const double d = dsub(z, P.tau);
            const double scale = !nz ? 0.0 : ddiv(d, dmul(P.gamma, z));
            scale_sh[lane] = scale;
            if (act) {
              const int64_t idx = (int64_t)T.l * P.n + (int64_t)T.c * 32 + 8 * q + lane;
              A.colpart[idx] = dmul(scale, ss);
              A.psi[idx] = !nz ? 0.0 : dmul(dmul(d, d), P.half_inv_gamma);
            }
          }
          consumer_sync<NW>();
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int cp = 2 * ((p + rho) & 3);
            sr[p] = *reinterpret_cast<const double2*>(scale_sh + cp);
            // beta pair (columns >= n: 0; their scale is 0)
            const int64_t jc = 32ll * T.c + 8 * q + cp;
            br[p].x = jc < P.n ? bs[cp] : 0.0;
            br[p].y = jc + 1 < P.n ? bs[cp + 1] : 0.0;
          }
        }
        if (nseg == 1 || k >= nseg) {  // pass 2: one thread per row
#pragma unroll
          for (int ri = 0; ri < 4; ++ri) {
            const int r = trow + 128 * ri;
            if (r < rows) {
              const double* __restrict__ row = buf + r * kRowStride;
              double acc = nseg == 1 ? racc[ri] : 0.0;
              const bool inplace = nseg == 1 && !A.qrec;
              const double ar = inplace ? 0.0 : as[r];
#pragma unroll
              for (int p = 0; p < 4; ++p) {
                const double2 v = *reinterpret_cast<const double2*>(row + 2 * ((p + rho) & 3));
                if (inplace) {
                  acc = dfma(sr[p].x, v.x, acc);
                  acc = dfma(sr[p].y, v.y, acc);
                } else {
                  acc = dfma(sr[p].x, relu(residual(ar, br[p].x, v.x)), acc);
                  acc = dfma(sr[p].y, relu(residual(ar, br[p].y, v.y)), acc);
                }
              }
              if (nseg == 1) {
                racc[ri] = acc;
              } else {  // the row's owner adds the quarters in order
                double* dst = A.rowpart + (int64_t)T.c * P.m + T.o0 + r0 + r;
                *dst = first_q ? acc : dadd(*dst, acc);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
      first_q = false;
    }
    if (nseg == 1) {
#pragma unroll
      for (int ri = 0; ri < 4; ++ri) {
        const int r = trow + 128 * ri;
        if (r < T.g) A.rowpart[(int64_t)T.c * P.m + T.o0 + r] = racc[ri];
      }
    }
  }
  TL_EXIT(P.tl, TL_EVAL);
}

// rows per quarter segment of the quarter pipeline: the tallest group when a
// slot of that size still leaves three CTAs per SM, else 448
int eval_qrows_for(int gmax) { return gmax <= 500 ? std::max(gmax, 16) : 448; }
// the tallest group evaluated as a whole tile: its four padded planes fit the
// slot of a quarter segment (at least 32,000 bytes)
int eval_q_short_rows(int qrows) {
  const int h = std::max(qrows, 500) / 4;  // plane rows incl. padding: (rows + 1) | 1 <= h
  return std::min(kEvalMaxSeg, (h & 1) ? h - 1 : h - 2);
}

namespace {
int g_eval_smem_attr[4] = {0, 0, 0, 0};
}

// Rows per segment: the tallest group when it fits, else kEvalMaxSeg.
int eval_buf_rows(int gmax) { return std::max(8, std::min(gmax, kEvalMaxSeg)); }

size_t eval_smem_bytes(int seg, int qrows) {
  if (qrows > 0)  // quarter pipeline: a slot holds a whole short tile or one quarter segment
    return sizeof(double) * 2 *
           ((size_t)std::max(4 * plane_len(seg), qrows * kPlaneCols) +
            aslot_len(std::max(seg, qrows)) + 34);
  return sizeof(double) * 2 * ((size_t)4 * plane_len(seg) + aslot_len(seg) + 34);
}

// variant: 0 in place (4 consumer warps), 1 recomputing (4), 2 in place (2)
static void (*eval_kernel(int variant))(const EvalArgs) {
  return variant == 3   ? k_eval_q
         : variant == 1 ? k_eval<true, 4>
         : variant == 2 ? k_eval<false, 2>
                        : k_eval<false, 4>;
}
static int eval_nthreads(int variant) { return eval_threads(variant == 2 ? 2 : 4); }

int eval_variant(int gmax, int seg, bool recompute) {
  if (recompute) return 1;
  if (const char* ev = std::getenv("GSOT_EVAL_NW")) return std::atoi(ev) == 2 && gmax <= kEvalShortRows ? 2 : 0;
  return gmax <= kEvalShortRows && seg >= gmax ? 2 : 0;
}

int eval_blocks_per_sm(size_t smem, int variant) {
  auto kern = eval_kernel(variant);
  if ((int)smem > g_eval_smem_attr[variant]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // all of the unified L1 / shared array as shared memory: one more CTA
    // (one more tile in flight) per SM
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    g_eval_smem_attr[variant] = (int)smem;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, eval_nthreads(variant), smem) !=
          cudaSuccess ||
      n < 1)
    n = 1;
  return n;
}

void launch_eval(const DevProblem& P, const double* x, const TaskDesc* tasks, int ntasks,
                 const int* ntasks_dev, const uint32_t* words, double* rowpart, double* colpart,
                 double* psi, int seg, int qrows, int variant, int grid, int* next_task,
                 bool pz_done, cudaStream_t s) {
  if ((reinterpret_cast<uintptr_t>(x) & 15u) != 0)
    throw Error(GSOT_ERR_INVALID_ARGUMENT, "eval: x must be 16-byte aligned (TMA source)");
  // next_task is EvalScalars::next_task: zero_rows lives in the same block
  EvalScalars* sc = reinterpret_cast<EvalScalars*>(reinterpret_cast<char*>(next_task) -
                                                   offsetof(EvalScalars, next_task));
  static const int qrec = [] {
    // measured: recomputing [f]+ in pass 2 (no in-place store in pass 1) is
    // 2 % faster on config 5; GSOT_EVAL_Q_RECOMPUTE=0 keeps the in-place form
    const char* ev = std::getenv("GSOT_EVAL_Q_RECOMPUTE");
    return ev ? std::atoi(ev) : 1;
  }();
  EvalArgs A{P, x, tasks, words, rowpart, colpart, psi, seg, qrows, qrec, pz_done ? 1 : 0, next_task, ntasks, ntasks_dev,
             &sc->zero_rows, &sc->read_qrows};
  const size_t smem = eval_smem_bytes(seg, qrows);
  if ((int)smem > g_eval_smem_attr[variant]) eval_blocks_per_sm(smem, variant);
  launch_pdl(eval_kernel(variant), dim3(grid), dim3(eval_nthreads(variant)), smem, s, A);
}

// ---------------------------------------------------------------- finalize
// grad_alpha_i = a_i - sum over non-empty chunks c of rowpart[c*m+i];
// grad_beta_j = b_j - sum over surviving l of colpart[l][j]; psicol_j = sum
// over surviving l of psi[l][j]. Each sum has a FIXED association: 8
// slices (c = s mod 8 resp. l = s mod 8), each sequential in ascending
// order, then the 8 slice partials in slice order. Empty chunks and skipped
// blocks contribute exact zeros, so omitting them leaves every partial
// unchanged: the result does not depend on the screen. Rows find their
// group's non-empty chunks in the per-group chunk masks (staged in shared
// memory), columns in the survivor words.
// In the same kernel: per-block partials of a.alpha, b.beta, sum psi
// (dual.hpp:51) and the line-search slope grad.d; k_publish folds them in
// block order (and the screen's counter slots) before the host reads them.
// Block (32, 8): blocks [0, m/32) handle 32 rows, the rest 32 columns.
#ifndef GSOT_FIN_SLICES
#define GSOT_FIN_SLICES 2
#endif
// threads per row / column = slices of the sums. Measured on config 5 (fast
// solve / baseline-mode solve): 8 slices 83.2 / 650 ms, 4: 80.0 / 642, 2: 77.0 /
// 682, 1: 77.4 / 739 -- fewer threads per unit mean fewer CTA waves of this
// latency-bound kernel; dense evaluations (long sums) prefer more slices.
constexpr int kFinSlices = GSOT_FIN_SLICES;
static_assert(kFinSlices == 8 || kFinSlices == 4 || kFinSlices == 2 || kFinSlices == 1, "slices");
constexpr int kFinUnitT = 32 * kFinSlices;   // threads per unit
// the bits of a 32-bit mask word whose index is 0 mod kFinSlices
constexpr uint32_t kFinSel = kFinSlices == 8 ? 0x01010101u : kFinSlices == 4 ? 0x11111111u : kFinSlices == 2 ? 0x55555555u : 0xffffffffu;
constexpr int kFinBatch = 8;
constexpr int kFinMaskCap = 1024;  // mask words staged per row unit
constexpr int kFinListCap = 2048 / kFinSlices;  // compacted chunks per slice (units within one group)

// Block = two independent units of (32 rows or columns) x kFinSlices slices. Everything
// that does not depend on the evaluation (x, d, marginals, the chunk masks and
// survivor words written by the screen, which completed before the evaluation
// started) is loaded before the programmatic wait.
__global__ void __launch_bounds__(64 * kFinSlices, kFinSlices == 8 ? 3 : kFinSlices == 4 ? 6 : kFinSlices == 2 ? 10 : 16) k_finalize(
    DevProblem P, const double* __restrict__ x, const uint32_t* __restrict__ words,
    const uint32_t* __restrict__ gmask, uint32_t* __restrict__ cmask, int clear_cmask,
    const double* __restrict__ rowpart, const double* __restrict__ colpart,
    const double* __restrict__ psi, double* __restrict__ grad, const double* __restrict__ dvec,
    double* __restrict__ partials, EvalScalars* sc, int cnt_pending, int row_blocks, int units) {
  __shared__ double sh[2][2][kFinSlices][33];
  __shared__ uint32_t msk[2][kFinMaskCap];
  // row unit inside one group: each slice's non-empty chunks (c = slice mod 8,
  // ascending), compacted once by the slice's warp before the programmatic
  // wait instead of every lane scanning the group's chunk mask
  __shared__ int clist[2][kFinSlices][kFinListCap];
  __shared__ int ccount[2][2 * kFinSlices];
  const int half = threadIdx.x / kFinUnitT, t = threadIdx.x % kFinUnitT;
  const int tx = t & 31, ty = t >> 5;
  const int unit = 2 * blockIdx.x + half;
  const bool is_row = unit < row_blocks;
  const bool live = unit < units;
  double obj[4] = {0.0, 0.0, 0.0, 0.0};  // a.alpha, b.beta, psi, g.d
  double acc = 0.0, ps = 0.0;
  // ---- before the wait
  int64_t i = -1, j = -1;
  double marg = 0.0, xv = 0.0, dv = 0.0;
  const int nmw = (P.nw + 31) / 32;
  int lf = 0;
  bool staged = false, coop = false;
  const int nlw = (P.L + 31) / 32;
  if (live && is_row) {
    const int64_t i0 = unit * 32ll;
    i = i0 + tx < P.m ? i0 + tx : -1;
    if (i >= 0) {
      marg = P.a[i];
      xv = x[i];
      dv = dvec ? dvec[i] : 0.0;
    }
    lf = P.row_group[i0];
    const int ll = P.row_group[P.m - 1 < i0 + 31 ? P.m - 1 : i0 + 31];
    // one group: one list of up to kFinListCap chunks per slice; two groups
    // (a group boundary inside the unit): one list per group, half the cap each
    const int per = (P.nw + kFinSlices - 1) / kFinSlices;
    coop = (lf == ll && per <= kFinListCap) || (ll == lf + 1 && per <= kFinListCap / 2);
    if (coop) {
      const uint32_t sel = kFinSel << ty;  // chunks c = ty mod 8 within a mask word
      for (int gi = 0; gi <= ll - lf; ++gi) {
        int* __restrict__ out = clist[half][ty] + gi * (kFinListCap / 2);
        int base = 0;
        for (int kb = 0; kb < nmw; kb += 32) {
          const uint32_t w = kb + tx < nmw ? gmask[(int64_t)(lf + gi) * nmw + kb + tx] & sel : 0u;
          const int cnt = __popc(w);
          int pre = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pre, o);
            if (tx >= o) pre += y;
          }
          int pos = base + pre - cnt;
          for (uint32_t ww = w; ww != 0u; ww &= ww - 1u) out[pos++] = 32 * (kb + tx) + __ffs(ww) - 1;
          base += __shfl_sync(0xffffffffu, pre, 31);
        }
        if (tx == 0) ccount[half][ty + gi * kFinSlices] = base;
      }
    } else {
      staged = (int64_t)(ll - lf + 1) * nmw <= kFinMaskCap;
      if (staged)
        for (int k = t; k < (ll - lf + 1) * nmw; k += kFinUnitT) msk[half][k] = gmask[(int64_t)lf * nmw + k];
    }
  } else if (live) {
    const int64_t c = unit - row_blocks;
    const int64_t jj = c * 32 + tx;
    j = jj < P.n ? jj : -1;
    if (j >= 0) {
      marg = P.b[j];
      xv = x[P.m + j];
      dv = dvec ? dvec[P.m + j] : 0.0;
    }
    staged = nlw <= kFinMaskCap;  // the chunk's group mask (non-empty (l, c))
    if (staged)
      for (int k = t; k < nlw; k += kFinUnitT) msk[half][k] = cmask[c * nlw + k];
  }
  __syncthreads();
  if (live && !is_row && staged && (P.L + kFinSlices - 1) / kFinSlices <= kFinListCap) {
    // column unit: the slice's non-empty groups (l = slice mod 8, ascending)
    // from the staged group mask, compacted by the slice's warp
    coop = true;
    const uint32_t sel = kFinSel << ty;
    int base = 0;
    for (int kb = 0; kb < nlw; kb += 32) {
      const uint32_t w = kb + tx < nlw ? msk[half][kb + tx] & sel : 0u;
      const int cnt = __popc(w);
      int pre = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pre, o);
        if (tx >= o) pre += y;
      }
      int pos = base + pre - cnt;
      for (uint32_t ww = w; ww != 0u; ww &= ww - 1u) clist[half][ty][pos++] = 32 * (kb + tx) + __ffs(ww) - 1;
      base += __shfl_sync(0xffffffffu, pre, 31);
    }
    if (tx == 0) ccount[half][ty] = base;
    __syncwarp();
  }
  if (clear_cmask && live && !is_row && staged)  // consumed: empty for the next screen
    for (int k = t; k < nlw; k += kFinUnitT) cmask[(unit - row_blocks) * (int64_t)nlw + k] = 0u;
  pdl_wait();
  pdl_trigger();
  TL_ENTER(P.tl, TL_FINALIZE);
  if (i >= 0 && coop) {  // the slice's compacted chunks, ascending: the same sum order
    const int gi = P.row_group[i] - lf;  // 0, or 1 past a group boundary
    const int* __restrict__ cl = clist[half][ty] + gi * (kFinListCap / 2);
    const int nc = ccount[half][ty + gi * kFinSlices];
    for (int b = 0; b < nc; b += kFinBatch) {
      double v[kFinBatch];
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q)
        v[q] = b + q < nc ? rowpart[(int64_t)cl[b + q] * P.m + i] : 0.0;
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q)
        if (b + q < nc) acc = dadd(acc, v[q]);
    }
  } else if (i >= 0) {
    const int l = P.row_group[i];
    const uint32_t* gm = staged ? msk[half] + (int64_t)(l - lf) * nmw : gmask + (int64_t)l * nmw;
    const uint32_t sel = kFinSel << ty;  // chunks c = ty mod 8 within a mask word
    int k = 0;
    uint32_t cur = nmw > 0 ? gm[0] & sel : 0u;
    for (;;) {  // batches of the slice's non-empty chunks, ascending c
      int idx[kFinBatch];
      int cnt = 0;
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q) {
        while (cur == 0u && k + 1 < nmw) cur = gm[++k] & sel;
        idx[q] = -1;
        if (cur != 0u) {
          const int b = __ffs(cur) - 1;
          cur &= cur - 1u;
          idx[q] = 32 * k + b;
          ++cnt;
        }
      }
      if (cnt == 0) break;
      double v[kFinBatch];
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q) v[q] = idx[q] >= 0 ? rowpart[(int64_t)idx[q] * P.m + i] : 0.0;
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q)
        if (idx[q] >= 0) acc = dadd(acc, v[q]);
      if (cnt < kFinBatch) break;
    }
  } else if (j >= 0 && coop) {  // the slice's compacted groups, ascending: the same sum order
    const int64_t c = j >> 5;
    const int* __restrict__ cl = clist[half][ty];
    const int nc = ccount[half][ty];
    for (int b = 0; b < nc; b += kFinBatch) {
      bool on[kFinBatch];
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q)
        on[q] = b + q < nc && ((words[(int64_t)cl[b + q] * P.nw + c] >> tx) & 1u);
      double cp[kFinBatch], pp[kFinBatch];
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q) {
        const int64_t idx = (int64_t)(on[q] ? cl[b + q] : 0) * P.n + j;
        cp[q] = on[q] ? colpart[idx] : 0.0;
        pp[q] = on[q] ? psi[idx] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q)
        if (on[q]) {
          acc = dadd(acc, cp[q]);
          ps = dadd(ps, pp[q]);
        }
    }
  } else if (j >= 0) {
    const int64_t c = j >> 5;
    const uint32_t* cm = staged ? msk[half] : cmask + c * nlw;
    const uint32_t sel = kFinSel << ty;  // groups l = ty mod 8 within a mask word
    int k = 0;
    uint32_t cur = nlw > 0 ? cm[0] & sel : 0u;
    for (;;) {  // batches of the slice's non-empty (l, c), ascending l
      int gl[kFinBatch];
      int cnt = 0;
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q) {
        while (cur == 0u && k + 1 < nlw) cur = cm[++k] & sel;
        gl[q] = -1;
        if (cur != 0u) {
          const int b = __ffs(cur) - 1;
          cur &= cur - 1u;
          gl[q] = 32 * k + b;
          ++cnt;
        }
      }
      if (cnt == 0) break;
      bool on[kFinBatch];
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q)
        on[q] = gl[q] >= 0 && ((words[(int64_t)gl[q] * P.nw + c] >> tx) & 1u);
      double cp[kFinBatch], pp[kFinBatch];
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q) {
        const int64_t idx = (int64_t)(on[q] ? gl[q] : 0) * P.n + j;
        cp[q] = on[q] ? colpart[idx] : 0.0;
        pp[q] = on[q] ? psi[idx] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kFinBatch; ++q)
        if (on[q]) {
          acc = dadd(acc, cp[q]);
          ps = dadd(ps, pp[q]);
        }
      if (cnt < kFinBatch) break;
    }
  }
  sh[half][0][ty][tx] = acc;
  sh[half][1][ty][tx] = ps;
  __syncthreads();
  if (ty == 0 && live) {
    if (i >= 0 || j >= 0) {
      double s = sh[half][0][0][tx], p = sh[half][1][0][tx];
      for (int q = 1; q < kFinSlices; ++q) {
        s = dadd(s, sh[half][0][q][tx]);
        p = dadd(p, sh[half][1][q][tx]);
      }
      const double gv = dsub(marg, s);
      if (i >= 0) {
        grad[i] = gv;
        obj[0] = dmul(xv, marg);
      } else {
        grad[P.m + j] = gv;
        obj[1] = dmul(xv, marg);
        obj[2] = p;
      }
      if (dvec) obj[3] = dmul(gv, dv);
    }
    // warp 0 of the unit holds its 32 rows / columns: fixed xor tree
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int o = 1; o <= 16; o <<= 1) obj[q] = dadd(obj[q], __shfl_xor_sync(0xffffffffu, obj[q], o));
    }
    if (tx < 4) partials[unit * 4 + tx] = obj[tx == 0 ? 0 : tx == 1 ? 1 : tx == 2 ? 2 : 3];
    if (unit == 0 && tx == 0) {
      sc->fin_blocks = units;
      sc->cnt_pending = cnt_pending;
    }
  }
  TL_EXIT(P.tl, TL_FINALIZE);
}

void launch_finalize(const DevProblem& P, const double* x, const uint32_t* words,
                     const uint32_t* gmask, uint32_t* cmask, int clear_cmask,
                     const double* rowpart, const double* colpart, const double* psi,
                     double* grad, const double* dvec, double* partials, EvalScalars* sc,
                     int cnt_pending, cudaStream_t s) {
  const int rb = (int)((P.m + 31) / 32);
  const int cb = (int)((P.n + 31) / 32);
  const int units = rb + cb;
  launch_pdl(k_finalize, dim3((units + 1) / 2), dim3(64 * kFinSlices), 0, s, P, x, words, gmask,
             cmask, clear_cmask, rowpart, colpart, psi, grad, dvec, partials, sc, cnt_pending, rb,
             units);
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
  const double* __restrict__ cp = block_ptr(P, o0, g, j);
  const double z = block_z(P, x, l, j);
  double* __restrict__ o = out + jj * P.m + o0;
  if (z <= P.tau) {
    for (int r = 0; r < g; ++r) o[r] = 0.0;
    return;
  }
  const double scale = ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma);
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[kRowStride * r]);
    o[r] = f > 0.0 ? dmul(scale, f) : 0.0;
  }
}

void launch_plan_columns(const DevProblem& P, const double* x, int64_t j0, int64_t ncols,
                         double* out, cudaStream_t s) {
  dim3 grid((unsigned)((ncols + 255) / 256), (unsigned)P.L);
  k_plan<<<grid, 256, 0, s>>>(P, x, j0, ncols, out);
}

// ---------------------------------------------------------------- plan diagnostics
// plan_diagnostics(recover_plan(x)) (dual.hpp:116-128, :139-169) without
// storing the plan. One warp per (group l, 32-column chunk c), lane = column:
// the plan entries are k_plan's (bitwise grad_block values); per column the
// block's entry sum (sequential in rows) goes to colpart[l*n + j]; per row the
// chunk's entry sum (fixed xor tree over the 32 lanes) to rowpart[c*m + i];
// blocks whose entries are all exactly 0.0 are counted (the reference's
// all_zero test, dual.hpp:153-162).
__global__ void __launch_bounds__(128) k_plan_diag(DevProblem P, const double* __restrict__ x,
                                                   double* __restrict__ rowpart,
                                                   double* __restrict__ colpart,
                                                   unsigned long long* __restrict__ zero_blocks) {
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.y * 4 + (threadIdx.x >> 5);
  if (l >= P.L) return;  // whole warp
  const int c = blockIdx.x;
  const int64_t j = 32ll * c + lane;
  const bool valid = j < P.n;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const double z = valid ? block_z(P, x, l, j) : 0.0;
  const bool nz = valid && z > P.tau;
  const double scale = nz ? ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma) : 0.0;
  const double bj = valid ? x[P.m + j] : 0.0;
  const double* __restrict__ cp = block_ptr(P, o0, g, valid ? j : 32ll * c);
  double colsum = 0.0;
  bool any = false;
  for (int r = 0; r < g; ++r) {
    double t = 0.0;
    if (nz) {
      const double f = residual(__ldg(x + o0 + r), bj, cp[kRowStride * r]);
      t = f > 0.0 ? dmul(scale, f) : 0.0;
    }
    colsum = dadd(colsum, t);
    any = any || t != 0.0;
    double rs = t;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) rs = dadd(rs, __shfl_xor_sync(0xffffffffu, rs, o));
    if (lane == 0) rowpart[(int64_t)c * P.m + o0 + r] = rs;
  }
  if (valid) colpart[(int64_t)l * P.n + j] = colsum;
  const unsigned zero = __ballot_sync(0xffffffffu, valid && !any);
  if (lane == 0 && zero) atomicAdd(zero_blocks, (unsigned long long)__popc(zero));
}

// primal_objective(recover_plan(x)) (core.hpp:153-180) per block: the plan
// entries of k_plan (bitwise), then sum t c, |t|^2 and the block's norm give
// the block's share <T_b, C_b> + gamma (|T_b|^2 / 2 + mu |T_b|), written to
// colpart[l * n + j]; the fold sums them per column (in group order).
__global__ void __launch_bounds__(128) k_plan_primal(DevProblem P, const double* __restrict__ x,
                                                     double* __restrict__ colpart) {
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.y * 4 + (threadIdx.x >> 5);
  if (l >= P.L) return;
  const int64_t j = 32ll * blockIdx.x + lane;
  if (j >= P.n) return;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const double z = block_z(P, x, l, j);
  double v = 0.0;
  if (z > P.tau) {
    const double scale = ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma);
    const double bj = x[P.m + j];
    const double* __restrict__ cp = block_ptr(P, o0, g, j);
    double tc = 0.0, tt = 0.0;
    for (int r = 0; r < g; ++r) {
      const double c = cp[kRowStride * r];
      const double f = residual(__ldg(x + o0 + r), bj, c);
      const double t = f > 0.0 ? dmul(scale, f) : 0.0;
      tc = dadd(tc, dmul(t, c));
      tt = dadd(tt, dmul(t, t));
    }
    v = dadd(tc, dmul(P.gamma, dadd(dmul(0.5, tt), dmul(P.mu, sqrt(tt)))));
  }
  colpart[(int64_t)l * P.n + j] = v;
}

void launch_plan_primal(const DevProblem& P, const double* x, double* colpart, cudaStream_t s) {
  k_plan_primal<<<dim3((unsigned)P.nw, (unsigned)((P.L + 3) / 4)), 128, 0, s>>>(P, x, colpart);
}

// Plan row sums (over the chunks, in chunk order) into out[0, m) and column
// sums (over the groups, in group order) into out[m, m + n).
__global__ void __launch_bounds__(256) k_plan_diag_fold(DevProblem P,
                                                        const double* __restrict__ rowpart,
                                                        const double* __restrict__ colpart,
                                                        double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < P.m) {
    double s = 0.0;
    for (int c = 0; c < P.nw; ++c) s = dadd(s, rowpart[(int64_t)c * P.m + t]);
    out[t] = s;
  } else if (t < P.m + P.n) {
    const int64_t j = t - P.m;
    double s = 0.0;
    for (int l = 0; l < P.L; ++l) s = dadd(s, colpart[(int64_t)l * P.n + j]);
    out[t] = s;
  }
}

void launch_plan_diag(const DevProblem& P, const double* x, double* rowpart, double* colpart,
                      unsigned long long* zero_blocks, cudaStream_t s) {
  k_plan_diag<<<dim3((unsigned)P.nw, (unsigned)((P.L + 3) / 4)), 128, 0, s>>>(P, x, rowpart, colpart,
                                                                            zero_blocks);
}

void launch_plan_diag_fold(const DevProblem& P, const double* rowpart, const double* colpart,
                           double* sums, cudaStream_t s) {
  k_plan_diag_fold<<<(unsigned)((P.m + P.n + 255) / 256), 256, 0, s>>>(P, rowpart, colpart, sums);
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
  atomicAdd(&sc->counters[0], 1ull);
  if (!(block_z(P, x, l, j) <= P.tau)) {
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
  atomicAdd(&sc->counters[1], 1ull);
  if (!(block_z(P, x, l, j) > P.tau)) {
    if (atomicCAS(&sc->audit_violation, 0, 2) == 0) sc->audit_where = (long long)l * P.n + j;
  }
}

void launch_audit_active(const DevProblem& P, const double* x, const uint32_t* aw,
                         EvalScalars* sc, cudaStream_t s) {
  dim3 grid((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  k_audit_active<<<grid, 256, 0, s>>>(P, x, aw, sc);
}

}  // namespace gsot
