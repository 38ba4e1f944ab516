// gsot_exact2.cu — exact-order mode (GSOT_EVAL_EXACT / GSOT_SOLVE_EXACT) at
// speed: every floating-point operation of the reference's hot path in the
// reference's own order, so a device solve is bitwise the reference's
// trajectory (tests/test_gpu_exact.py), without one-thread sequential loops.
//
//   k_ex_cols     one warp per 32-column chunk, walking the chunk's work
//                 tiles in ascending group order: per block (lane = column)
//                 z = pos_part_norm, the scale (1 - tau/z)/gamma and psi_block
//                 with its dot / sq chains, all sequential over the block rows
//                 (regularizer.hpp:23-91); the column sum of the plan entries
//                 continues across the groups in row order, so
//                 grad_beta_j = b_j - sum_entries(gcol_j) exactly
//                 (dual.hpp:97-98). Nonzero blocks' psi are listed per column.
//   k_ex_rows     one warp per 32-row slab of a group (lane = row), walking
//                 the group's nonzero tiles in ascending column order:
//                 grad_alpha_i = ((a_i - T_i0) - T_i1) - ...   (dual.hpp:91, :96).
//   k_ex_scalars  cluster kernel: psi_sum in (j outer, l inner) order
//                 (dual.hpp:44-50), alpha.a, beta.b (dual.hpp:51) and the
//                 line-search slope grad.d (lbfgs.hpp:89) as four sequential
//                 sums through the gsot_seqsum.cuh engine.
//   k_ex_direction cluster kernel: the curvature pair and its test
//                 (lbfgs.hpp:243-255) and the two-loop recursion (lbfgs.hpp:
//                 109-126), every dot a sequential sum through the engine,
//                 every vector update elementwise in the reference's order.
//
// Skipped and zero blocks contribute literal +0.0 (grad_block's zero fill,
// psi_block's 0.0): adding or subtracting +0.0 leaves every partial sum
// unchanged (they are never -0.0 under round-to-nearest), so the chains visit
// only nonzero terms.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "gsot_device.cuh"
#include "gsot_exact2.cuh"

namespace cg = cooperative_groups;

namespace gsot {

constexpr int kThreads = seq::kT;

// ---------------------------------------------------------------- columns

__global__ void __launch_bounds__(128) k_ex_cols(DevProblem P, const double* __restrict__ x,
                                                 const uint32_t* __restrict__ words,
                                                 uint32_t* __restrict__ cmask, int clear_cmask,
                                                 double* __restrict__ scale_out,
                                                 double* __restrict__ psiT, int* __restrict__ cntj,
                                                 uint32_t* __restrict__ nzw,
                                                 double* __restrict__ grad) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (c >= P.nw) return;
  const int64_t j = static_cast<int64_t>(c) * 32 + lane;
  const bool valid = j < P.n;
  const double bj = valid ? x[P.m + j] : 0.0;
  const int nlw = (P.L + 31) / 32;
  double colacc = 0.0;
  int cnt = 0;
  for (int w = 0; w < nlw; ++w) {
    uint32_t mask = cmask[static_cast<int64_t>(c) * nlw + w];
    if (clear_cmask) {
      __syncwarp();
      if (lane == 0) cmask[static_cast<int64_t>(c) * nlw + w] = 0u;  // consumed
    }
    while (mask) {
      const int l = 32 * w + __ffs(mask) - 1;
      mask &= mask - 1u;
      const uint32_t sw = words[static_cast<int64_t>(l) * P.nw + c];
      if (sw == 0u) continue;
      const bool act = (sw >> lane) & 1u;
      const int o0 = P.off[l], g = P.off[l + 1] - o0;
      const double* __restrict__ al = x + o0;
      const double* __restrict__ tp = P.C + cost_index(P.nw, o0, g, 32ll * c + lane, 0);
      // pos_part_norm: acc += v * v over the rows, ascending (regularizer.hpp:23-30)
      double z2 = 0.0;
      int r = 0;
      for (; r + 8 <= g; r += 8) {
        double cv[8], av[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          cv[q] = act ? tp[kRowStride * (r + q)] : 0.0;
          av[q] = __ldg(al + r + q);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double f = residual(av[q], bj, cv[q]);
          const double v = f > 0.0 ? f : 0.0;
          z2 = dadd(z2, dmul(v, v));
        }
      }
      for (; r < g; ++r) {
        const double f = residual(__ldg(al + r), bj, act ? tp[kRowStride * r] : 0.0);
        const double v = f > 0.0 ? f : 0.0;
        z2 = dadd(z2, dmul(v, v));
      }
      const double z = sqrt(z2);
      const bool nz = act && z > P.tau;
      const uint32_t nzword = __ballot_sync(0xffffffffu, nz);
      if (lane == 0) nzw[static_cast<int64_t>(l) * P.nw + c] = nzword;
      if (nzword == 0u) continue;
      // grad_block / psi_block (regularizer.hpp:64-91): scale, then one more
      // pass for the plan entries, psi's dot / sq chains and the column sum
      const double scale = nz ? ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma) : 0.0;
      double dot = 0.0, sq = 0.0;
      r = 0;
      for (; r + 8 <= g; r += 8) {
        double cv[8], av[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          cv[q] = nz ? tp[kRowStride * (r + q)] : 0.0;
          av[q] = __ldg(al + r + q);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double f = residual(av[q], bj, cv[q]);
          const double gg = f > 0.0 ? dmul(scale, f) : 0.0;
          dot = dadd(dot, dmul(f, gg));
          sq = dadd(sq, dmul(gg, gg));
          if (f > 0.0) colacc = dadd(colacc, gg);
        }
      }
      for (; r < g; ++r) {
        const double f = residual(__ldg(al + r), bj, nz ? tp[kRowStride * r] : 0.0);
        const double gg = f > 0.0 ? dmul(scale, f) : 0.0;
        dot = dadd(dot, dmul(f, gg));
        sq = dadd(sq, dmul(gg, gg));
        if (f > 0.0) colacc = dadd(colacc, gg);
      }
      if (nz) {
        scale_out[static_cast<int64_t>(l) * P.n + j] = scale;
        psiT[j * P.L + cnt] =
            dsub(dot, dmul(P.gamma, dadd(dmul(0.5, sq), dmul(P.mu, sqrt(sq)))));
        ++cnt;
      }
    }
  }
  if (valid) {
    grad[P.m + j] = dsub(P.b[j], colacc);
    cntj[j] = cnt;
  }
}

// k_ex_cols2: the same computation, with each warp streaming its chunk's
// tiles through its own TMA ring (cp.async.bulk of contiguous 32-row tile
// segments and the matching alpha rows into shared memory, mbarrier
// completion; lane 0 issues, every lane waits). A tile of at most kExD
// segments stays resident for pass 2; a taller one is streamed again for
// pass 2 only when it has a nonzero block. One CTA per SM, kExNW warps (4 with
// 5-slot rings, or 12 with 2-slot rings when every tile is tall anyway), each
// an independent chunk owner (the column chains run across the groups of the
// chunk in order). Requires L <= kExG (else k_ex_cols).
constexpr int kExSR = 32;      // rows per segment
constexpr int kExAl = kExSR + 2;  // alpha slot (aligned superset), even
constexpr int kExGmax = 1024;  // groups listed per chunk (largest variant)

// one warp's ring (kExD slots) and its chunk's list of surviving tiles (kExG)
template <int kExD, int kExG>
struct alignas(128) ExColWarp {
  double seg[kExD][kExSR * 32];
  double al[kExD][kExAl];
  uint64_t full[kExD];
  int grp[kExG];
  uint32_t gsw[kExG];
};

template <int kExNW, int kExD, int kExG>
__global__ void __launch_bounds__(32 * kExNW, 1)
    k_ex_cols2(DevProblem P, const double* __restrict__ x, const uint32_t* __restrict__ words,
               uint32_t* __restrict__ cmask, int clear_cmask, double* __restrict__ scale_out,
               double* __restrict__ psiT, int* __restrict__ cntj, uint32_t* __restrict__ nzw,
               double* __restrict__ grad) {
  extern __shared__ __align__(128) unsigned char exc_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ExColWarp<kExD, kExG>& W = reinterpret_cast<ExColWarp<kExD, kExG>*>(exc_smem)[warp];
  if (lane == 0) {
    for (int q = 0; q < kExD; ++q) mbar_init(&W.full[q], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const int nlw = (P.L + 31) / 32;
  uint32_t head = 0, tail = 0;  // ring: segments issued / consumed (this warp)
  // issue segment s of tile (o0, g, c) into the next slot (lane 0)
  auto issue = [&](int c, int o0, int g, int sgi, uint32_t qm) {
    const int slot = head % kExD;
    const int r0 = sgi * kExSR, rows = min(kExSR, g - r0);
    const int64_t a0 = (o0 + r0) & ~1ll;
    const uint32_t abytes = static_cast<uint32_t>(((o0 + r0 + rows - a0) + 1) & ~1ll) * 8u;
    const double* tile = P.C + 32 * (static_cast<int64_t>(P.nw) * o0 + static_cast<int64_t>(c) * g);
    mbar_expect_tx(&W.full[slot],
                   static_cast<uint32_t>(rows) * 64u * static_cast<uint32_t>(__popc(qm)) + abytes);
#pragma unroll
    for (int q = 0; q < 4; ++q)  // one contiguous run per quarter that is read
      if ((qm >> q) & 1u)
        tma_load_1d(W.seg[slot] + q * (kExSR * kPlaneCols),
                    tile + static_cast<int64_t>(q) * kPlaneCols * g +
                        static_cast<int64_t>(r0) * kRowStride,
                    static_cast<uint32_t>(rows) * 64u, &W.full[slot]);
    tma_load_1d(W.al[slot], x + a0, abytes, &W.full[slot]);
    ++head;
  };
  for (int c = blockIdx.x * kExNW + warp; c < P.nw; c += gridDim.x * kExNW) {
    const int64_t j = static_cast<int64_t>(c) * 32 + lane;
    const bool valid = j < P.n;
    const double bj = valid ? x[P.m + j] : 0.0;
    // the chunk's surviving tiles in ascending group order
    int ng = 0;
    for (int w = 0; w < nlw; ++w) {
      const uint32_t mask = cmask[static_cast<int64_t>(c) * nlw + w];
      const int l = 32 * w + lane;
      const uint32_t sw = (mask >> lane) & 1u ? words[static_cast<int64_t>(l) * P.nw + c] : 0u;
      const uint32_t b = __ballot_sync(0xffffffffu, sw != 0u);
      if (sw != 0u) {
        const int pos = ng + __popc(b & ((1u << lane) - 1u));
        W.grp[pos] = l;
        W.gsw[pos] = sw;
      }
      ng += __popc(b);
      if (clear_cmask && lane == 0 && mask) cmask[static_cast<int64_t>(c) * nlw + w] = 0u;  // consumed
    }
    __syncwarp();
    // producer cursor (pt, ps): the next tile / pass-1 segment to issue, in
    // consumption order. It never runs past a tall tile whose pass 1 is fully
    // issued (stop_at) until that tile is done: its pass 2 comes next.
    int pt = 0, ps = 0, stop_at = -1;
    auto tile_geom = [&](int t, int& o0, int& g) {
      const int l = W.grp[t];
      o0 = __ldg(P.off + l);
      g = __ldg(P.off + l + 1) - o0;
    };
    auto pump = [&](int cur) {
      while (pt < ng && head - tail < static_cast<uint32_t>(kExD) && stop_at < cur) {
        if (ps == 0) {  // a tile whose surviving blocks are provably zero is not read
          const int l = W.grp[pt];
          const int64_t jj = static_cast<int64_t>(c) * 32 + lane;
          const bool act = (W.gsw[pt] >> lane) & 1u;
          const bool maybe =
              act && !(dadd(P.amax[l], x[P.m + jj]) <= static_cast<double>(P.cmin[static_cast<int64_t>(l) * P.n + jj]));
          const uint32_t mb = __ballot_sync(0xffffffffu, maybe);
          if (mb == 0u) {
            __syncwarp();
            if (lane == 0) W.grp[pt] = -1 - l;  // marked zero for the walk
            __syncwarp();
            ++pt;
            continue;
          }
          // a surviving column in a quarter without a possibly-nonzero block is
          // provably zero (z = 0: no nonzero block, no psi, no column terms):
          // it leaves the survivor word, and its quarter is not read
          const uint32_t keep = W.gsw[pt] & quarter_lanes(quarter_mask(mb));
          __syncwarp();
          if (lane == 0) W.gsw[pt] = keep;
          __syncwarp();
        }
        int o0, g;
        tile_geom(pt, o0, g);
        const int ns = (g + kExSR - 1) / kExSR;
        if (lane == 0) {
          issue(c, o0, g, ps, quarter_mask(W.gsw[pt]));
        } else {
          ++head;
        }
        if (++ps == ns) {
          ps = 0;
          if (ns > kExD) stop_at = pt;
          ++pt;
        }
      }
    };
    double colacc = 0.0;
    int cnt = 0;
    for (int t = 0; t < ng; ++t) {
      pump(t);  // tile t issued (or marked provably zero) before it is read
      if (W.grp[t] < 0) {  // provably zero: no nonzero block, no psi, no column terms
        if (lane == 0) nzw[static_cast<int64_t>(-1 - W.grp[t]) * P.nw + c] = 0u;
        continue;
      }
      const int l = W.grp[t];
      const uint32_t sw = W.gsw[t];
      const bool act = (sw >> lane) & 1u;
      int o0, g;
      tile_geom(t, o0, g);
      const int ns = (g + kExSR - 1) / kExSR;
      const bool resident = ns <= kExD;
      // pass 1: pos_part_norm, acc += v * v over the rows, ascending
      // (regularizer.hpp:23-30)
      double z2 = 0.0;
      for (int q = 0; q < ns; ++q) {
        pump(t);
        const uint32_t k = resident ? tail + q : tail;
        mbar_wait(&W.full[k % kExD], (k / kExD) & 1u);
        const double* __restrict__ sg = W.seg[k % kExD] + (lane >> 3) * (kExSR * kPlaneCols) + (lane & 7);
        const double* __restrict__ as = W.al[k % kExD] + ((o0 + q * kExSR) & 1);
        const int rows = min(kExSR, g - q * kExSR);
#pragma unroll 8
        for (int r = 0; r < rows; ++r) {
          const double f = residual(as[r], bj, act ? sg[kRowStride * r] : 0.0);
          const double v = f > 0.0 ? f : 0.0;
          z2 = dadd(z2, dmul(v, v));
        }
        if (!resident) {  // a tall tile's segment is released at once
          __syncwarp();
          ++tail;
        }
      }
      const double z = sqrt(z2);
      const bool nz = act && z > P.tau;
      const uint32_t nzword = __ballot_sync(0xffffffffu, nz);
      if (lane == 0) nzw[static_cast<int64_t>(l) * P.nw + c] = nzword;
      if (nzword != 0u) {
        // grad_block / psi_block (regularizer.hpp:64-91): scale, then the plan
        // entries, psi's dot / sq chains and the column sum
        const double scale = nz ? ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma) : 0.0;
        double dot = 0.0, sq = 0.0;
        int issued = 0;  // a tall tile streamed again (the ring is empty here)
        for (int q = 0; q < ns; ++q) {
          uint32_t k = tail + q;
          if (!resident) {
            while (issued < ns && head - tail < static_cast<uint32_t>(kExD)) {
              if (lane == 0) {
                issue(c, o0, g, issued, quarter_mask(sw));
              } else {
                ++head;
              }
              ++issued;
            }
            k = tail;
            mbar_wait(&W.full[k % kExD], (k / kExD) & 1u);
          }
          const double* __restrict__ sg = W.seg[k % kExD] + (lane >> 3) * (kExSR * kPlaneCols) + (lane & 7);
          const double* __restrict__ as = W.al[k % kExD] + ((o0 + q * kExSR) & 1);
          const int rows = min(kExSR, g - q * kExSR);
#pragma unroll 8
          for (int r = 0; r < rows; ++r) {
            const double f = residual(as[r], bj, nz ? sg[kRowStride * r] : 0.0);
            const double gg = f > 0.0 ? dmul(scale, f) : 0.0;
            dot = dadd(dot, dmul(f, gg));
            sq = dadd(sq, dmul(gg, gg));
            if (f > 0.0) colacc = dadd(colacc, gg);
          }
          if (!resident) {
            __syncwarp();
            ++tail;
          }
        }
        if (nz) {
          scale_out[static_cast<int64_t>(l) * P.n + j] = scale;
          psiT[j * P.L + cnt] =
              dsub(dot, dmul(P.gamma, dadd(dmul(0.5, sq), dmul(P.mu, sqrt(sq)))));
          ++cnt;
        }
      }
      if (resident) {
        __syncwarp();
        tail += ns;
      }
    }
    if (valid) {
      grad[P.m + j] = dsub(P.b[j], colacc);
      cntj[j] = cnt;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- rows

constexpr int kRowWin = 1024;  // chunks listed per window (k_ex_rows)

__global__ void __launch_bounds__(128) k_ex_rows(DevProblem P, const double* __restrict__ x,
                                                 const uint32_t* __restrict__ words,
                                                 const uint32_t* __restrict__ gmask,
                                                 const uint32_t* __restrict__ nzw,
                                                 const double* __restrict__ scale,
                                                 const int4* __restrict__ slabs, int nslabs,
                                                 double* __restrict__ grad) {
  extern __shared__ __align__(16) unsigned char rows_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sidx = blockIdx.x * 4 + warp;
  if (sidx >= nslabs) return;
  const int4 sl = slabs[sidx];
  const int l = sl.x, r0 = sl.y, nr = sl.z;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const bool valid = lane < nr;
  const int64_t i = static_cast<int64_t>(o0) + r0 + lane;
  const double ai = valid ? x[i] : 0.0;
  double acc = valid ? P.a[i] : 0.0;  // grad_alpha = a (dual.hpp:91)
  // the group's tiles with a computed nonzero block, ascending: (chunk, word),
  // listed by the whole warp for a window of up to kRowWin chunks at a time,
  // so the walk can load the next tile while it adds the current one
  int2* list = reinterpret_cast<int2*>(rows_smem) + static_cast<size_t>(warp) * kRowWin;
  const int nmw = (P.nw + 31) / 32;
  const double* __restrict__ base =
      P.C + 32 * static_cast<int64_t>(P.nw) * o0 + kRowStride * static_cast<int64_t>(r0 + lane);
  const int64_t plane = static_cast<int64_t>(kPlaneCols) * g;  // quarter planes of a tile
  auto load = [&](int t, double (&cv)[32], double& bk, double& sk, uint32_t& nz) {
    const int2 e = list[t];
    const int c = e.x;
    nz = static_cast<uint32_t>(e.y);
    const int64_t jk = static_cast<int64_t>(c) * 32 + lane;
    const bool mine = (nz >> lane) & 1u;
    bk = mine ? x[P.m + jk] : 0.0;
    sk = mine ? scale[static_cast<int64_t>(l) * P.n + jk] : 0.0;
    const double* __restrict__ row = base + 32 * static_cast<int64_t>(c) * g;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const double2 v = valid ? *reinterpret_cast<const double2*>(row + (q >> 2) * plane + 2 * (q & 3))
                              : make_double2(0.0, 0.0);
      cv[2 * q] = v.x;
      cv[2 * q + 1] = v.y;
    }
  };
  for (int w0 = 0; w0 < nmw; w0 += kRowWin / 32) {
    int n = 0;
    for (int w = w0; w < min(nmw, w0 + kRowWin / 32); ++w) {
      const uint32_t cm = gmask[static_cast<int64_t>(l) * nmw + w];
      const int c = 32 * w + lane;
      uint32_t nz = 0u;
      if ((cm >> lane) & 1u) {
        const int64_t wi = static_cast<int64_t>(l) * P.nw + c;
        nz = words[wi] & nzw[wi];
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, nz != 0u);
      if (nz != 0u) list[n + __popc(bal & ((1u << lane) - 1u))] = make_int2(c, static_cast<int>(nz));
      n += __popc(bal);
    }
    __syncwarp();
    double cv[32], bk = 0.0, sk = 0.0;
    uint32_t nz = 0u;
    if (n > 0) load(0, cv, bk, sk, nz);
    for (int t = 0; t < n; ++t) {
      double cn[32], bn = 0.0, sn = 0.0;
      uint32_t nzn = 0u;
      if (t + 1 < n) load(t + 1, cn, bn, sn, nzn);  // in flight during this tile's chain
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double b = __shfl_sync(0xffffffffu, bk, k);
        const double sc = __shfl_sync(0xffffffffu, sk, k);
        if ((nz >> k) & 1u) {  // grad_alpha -= gcol_j, j ascending (dual.hpp:96)
          const double f = residual(ai, b, cv[k]);
          if (f > 0.0) acc = dsub(acc, dmul(sc, f));
        }
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) cv[k] = cn[k];
      bk = bn;
      sk = sn;
      nz = nzn;
    }
    __syncwarp();
  }
  if (valid) grad[i] = acc;
}

// ---------------------------------------------------------------- scalars

struct ScalarArgs {
  DevProblem P;
  const double* x;
  const double* grad;
  const double* dvec;
  const double* psiT;
  const int* cntj;
  int* lenC;
  int* offC;
  double* flat;
  double* tv;
  int64_t tv_stride;
  EvalScalars* sc;
  unsigned long long* cnt_slots;
};

__global__ void __launch_bounds__(kThreads, 1) k_ex_scalars(ScalarArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  seq::Smem2& sm = *reinterpret_cast<seq::Smem2*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const DevProblem& P = A.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cta = static_cast<int>(cl.block_rank()), ncta = static_cast<int>(cl.num_blocks());
  const int gw = cta * (kThreads / 32) + warp, gnw = ncta * (kThreads / 32);
  const int64_t gt = static_cast<int64_t>(cta) * kThreads + threadIdx.x;
  const int64_t gstride = static_cast<int64_t>(ncta) * kThreads;
  const int64_t dim = P.m + P.n;
  // 1. psi terms per chunk; dot terms (alpha_i * a_i, beta_j * b_j, grad_e * d_e)
  for (int c = gw; c < P.nw; c += gnw) {
    const int64_t j = static_cast<int64_t>(c) * 32 + lane;
    int v = j < P.n ? A.cntj[j] : 0;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) A.lenC[c] = v;
  }
  double* t1 = A.tv;
  double* t2 = A.tv + A.tv_stride;
  double* t3 = A.tv + 2 * A.tv_stride;
  for (int64_t e = gt; e < dim; e += gstride) {
    if (e < P.m)
      t1[e] = dmul(A.x[e], P.a[e]);  // s.alpha.dot(inst.a)
    else
      t2[e - P.m] = dmul(A.x[e], P.b[e - P.m]);  // s.beta.dot(inst.b)
    if (A.dvec) t3[e] = dmul(A.grad[e], A.dvec[e]);  // p.grad.dot(d)
  }
  cl.sync();
  // 2. chunk offsets of the psi chain (CTA 0)
  if (cta == 0) {
    __shared__ int wtot[kThreads / 32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < P.nw; base += kThreads) {
      const int c = base + threadIdx.x;
      const int v = c < P.nw ? __ldcg(A.lenC + c) : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wtot[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const int w = lane < kThreads / 32 ? wtot[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, wi, o);
          if (lane >= o) wi += y;
        }
        if (lane < kThreads / 32) wtot[lane] = wi - w;
      }
      __syncthreads();
      if (c < P.nw) A.offC[c] = carry + wtot[warp] + incl - v;
      __syncthreads();
      if (threadIdx.x == kThreads - 1) carry += wtot[warp] + incl;
      __syncthreads();
    }
    if (threadIdx.x == 0) A.offC[P.nw] = carry;
  }
  cl.sync();
  // 3. the psi chain terms in (j outer, l inner) order
  for (int c = gw; c < P.nw; c += gnw) {
    const int64_t j = static_cast<int64_t>(c) * 32 + lane;
    const int v = j < P.n ? A.cntj[j] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t pos = __ldcg(A.offC + c) + (incl - v);
    const double* __restrict__ src = A.psiT + j * P.L;
#pragma unroll 8
    for (int q = 0; q < v; ++q) A.flat[pos + q] = src[q];
  }
  if (threadIdx.x == 0) {
    const int64_t npsi = __ldcg(A.offC + P.nw);
    sm.ch[0] = seq::Chain2{A.flat, npsi, 0.0};
    sm.ch[1] = seq::Chain2{t1, P.m, 0.0};
    sm.ch[2] = seq::Chain2{t2, P.n, 0.0};
    sm.ch[3] = seq::Chain2{t3, A.dvec ? dim : 0, 0.0};
  }
  cl.sync();
  // 4. the four sequential sums
  seq::engine2(A.dvec ? 4 : 3, sm);
  if (cta == 0) {
    if (warp == 1 && A.cnt_slots) fold_counter_slots(A.cnt_slots, A.sc);  // screen counters
    if (threadIdx.x == 0) {
      const double psi_sum = sm.res[0], da = sm.res[1], db = sm.res[2];
      A.sc->dot_aa = da;
      A.sc->dot_bb = db;
      A.sc->psi_sum = psi_sum;
      A.sc->objective = dsub(dadd(da, db), psi_sum);  // dual.hpp:51
      A.sc->slope = A.dvec ? sm.res[3] : 0.0;
    }
  }
  cl.sync();  // no CTA exits while another may still read its shared memory
}

template <typename T>
static T* dalloc_raw(int64_t count, size_t* tally) {
  T* p = nullptr;
  if (count <= 0) count = 1;
  GSOT_CUDA_CHECK(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(count)));
  if (tally) *tally += sizeof(T) * static_cast<size_t>(count);
  return p;
}

void exact_ws_alloc(ExactWs& w, const DevProblem& P, const std::vector<int32_t>& sizes,
                    size_t* tally) {
  const int64_t Ln = static_cast<int64_t>(P.L) * P.n;
  const int64_t dim = P.m + P.n;
  w.scale = dalloc_raw<double>(Ln, tally);
  w.psiT = dalloc_raw<double>(Ln, tally);
  w.flat = dalloc_raw<double>(Ln, tally);
  w.cntj = dalloc_raw<int>(P.n, tally);
  w.nzw = dalloc_raw<uint32_t>(static_cast<int64_t>(P.L) * P.nw, tally);
  w.lenC = dalloc_raw<int>(P.nw, tally);
  w.offC = dalloc_raw<int>(P.nw + 1, tally);
  w.tv_stride = (dim + 63) / 64 * 64;
  w.tv = dalloc_raw<double>(kTermBufs * w.tv_stride, tally);
  std::vector<int4> sl;
  for (int32_t l = 0; l < P.L; ++l)
    for (int32_t r = 0; r < sizes[l]; r += 32) sl.push_back(make_int4(l, r, std::min(32, sizes[l] - r), 0));
  w.nslabs = static_cast<int>(sl.size());
  w.gmin = *std::min_element(sizes.begin(), sizes.end());
  w.slabs = dalloc_raw<int4>(w.nslabs, tally);
  GSOT_CUDA_CHECK(cudaMemcpy(w.slabs, sl.data(), sizeof(int4) * sl.size(), cudaMemcpyHostToDevice));
}

void exact_ws_free(ExactWs& w) {
  void* ptrs[] = {w.scale, w.psiT, w.flat, w.cntj, w.nzw, w.lenC, w.offC, w.tv, w.slabs};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  w = ExactWs{};
}

// One cluster of kThreads-thread CTAs: 16 CTAs where the device can co-schedule
// a non-portable 16-CTA cluster of the kernel, else 8 (decided once per kernel).
template <typename K, typename Arg>
static void launch_cluster(K kern, const Arg& a, cudaStream_t s) {
  static int ncta = 0;
  const int smem = static_cast<int>(sizeof(seq::Smem2));
  if (ncta == 0) {
    ncta = 8;
    GSOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
        cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = seq::kMaxCtas;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(seq::kMaxCtas);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n >= 1)
        ncta = seq::kMaxCtas;
    }
    (void)cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ncta);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  GSOT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
}

void launch_exact_eval2(const DevProblem& P, const ExactWs& W, const double* x,
                        const uint32_t* words, const uint32_t* gmask, uint32_t* cmask,
                        int clear_cmask, double* grad, const double* dvec, EvalScalars* sc,
                        unsigned long long* cnt_slots, cudaStream_t s) {
  static int nsm = 0;
  if (nsm == 0) {
    int dev = 0;
    GSOT_CUDA_CHECK(cudaGetDevice(&dev));
    GSOT_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  auto run = [&](auto kern, int nwarps, int smem) {
    // the dynamic shared-memory attribute of each kernel variant (a plain
    // function-pointer type is shared by the variants: key by address)
    static std::vector<std::pair<const void*, int>> attrs;
    int* attr = nullptr;
    for (auto& a : attrs)
      if (a.first == reinterpret_cast<const void*>(kern)) attr = &a.second;
    if (!attr) {
      attrs.emplace_back(reinterpret_cast<const void*>(kern), 0);
      attr = &attrs.back().second;
    }
    if (*attr < smem) {
      GSOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      *attr = smem;
    }
    const int grid = std::min(nsm, (P.nw + nwarps - 1) / nwarps);
    kern<<<grid, 32 * nwarps, smem, s>>>(P, x, words, cmask, clear_cmask, W.scale, W.psiT, W.cntj,
                                         W.nzw, grad);
  };
  const char* ev = std::getenv("GSOT_EXACT_COLS");
  const int pick = ev ? std::atoi(ev) : 0;
  // every tile taller than the 5-slot ring anyway (config 5): 12 warps per SM
  // (more chunks in flight) with 2-slot rings
  if (P.L <= 256 && (pick == 2 || (pick == 0 && W.gmin > 5 * kExSR))) {
    run(k_ex_cols2<12, 2, 256>, 12, static_cast<int>(sizeof(ExColWarp<2, 256>) * 12));
  } else if (P.L <= kExGmax) {
    run(k_ex_cols2<4, 5, kExGmax>, 4, static_cast<int>(sizeof(ExColWarp<5, kExGmax>) * 4));
  } else {
    k_ex_cols<<<(P.nw + 3) / 4, 128, 0, s>>>(P, x, words, cmask, clear_cmask, W.scale, W.psiT,
                                              W.cntj, W.nzw, grad);
  }
  {
    static int attr = 0;
    const int rsmem = static_cast<int>(sizeof(int2) * 4 * kRowWin);
    if (attr < rsmem) {
      GSOT_CUDA_CHECK(cudaFuncSetAttribute(k_ex_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem));
      attr = rsmem;
    }
    k_ex_rows<<<(W.nslabs + 3) / 4, 128, rsmem, s>>>(P, x, words, gmask, W.nzw, W.scale, W.slabs,
                                                     W.nslabs, grad);
  }
  ScalarArgs A;
  A.P = P;
  A.x = x;
  A.grad = grad;
  A.dvec = dvec;
  A.psiT = W.psiT;
  A.cntj = W.cntj;
  A.lenC = W.lenC;
  A.offC = W.offC;
  A.flat = W.flat;
  A.tv = W.tv;
  A.tv_stride = W.tv_stride;
  A.sc = sc;
  A.cnt_slots = cnt_slots;
  launch_cluster(k_ex_scalars, A, s);
}

// ---------------------------------------------------------------- direction

struct DirKArgs {
  ExactDirArgs a;
  double* tv;
  int64_t tv_stride;
};

// The pair test and the two-loop recursion on one cluster. Every vector is
// split into CTA slices matching the engine's per-thread blocks (thread g owns
// terms [g b, g b + b), b = ceil(dim / threads)), so the elementwise work of
// a slice and the sequential sums over it need only CTA barriers; the dots'
// terms alternate between two buffer sets (call parity): a remote CTA's
// stitch may still read the previous call's terms.
__global__ void __launch_bounds__(kThreads, 1) k_ex_direction(DirKArgs K) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  seq::Smem2& sm = *reinterpret_cast<seq::Smem2*>(smem_raw);
  __shared__ HistState hs;
  __shared__ double a_loc[kMaxMemory];
  cg::cluster_group cl = cg::this_cluster();
  const ExactDirArgs& A = K.a;
  const int cta = static_cast<int>(cl.block_rank()), ncta = static_cast<int>(cl.num_blocks());
  const int64_t dim = A.dim;
  const int64_t b = seq::block_len(dim, ncta * kThreads);
  const int64_t lo = min(dim, static_cast<int64_t>(cta) * kThreads * b);
  const int64_t hi = min(dim, lo + kThreads * b);
  HistState* H = A.h;
  int call = 0;
  auto buf = [&](int q) { return K.tv + (static_cast<int64_t>(call & 1) * 3 + q) * K.tv_stride; };
  // every CTA works on its own copy of the ring state (CTA 0 writes it back)
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(HistState) / 4); i += kThreads)
    reinterpret_cast<int*>(&hs)[i] = reinterpret_cast<const volatile int*>(H)[i];
  __syncthreads();
  // every vector this CTA's slice will read, prefetched into L2 up front (the
  // evaluation's cost stream evicts them between directions): the elementwise
  // steps between the sequential sums then hit L2 instead of DRAM
  if (threadIdx.x < 32 && hi > lo) {
    auto pf = [&](const double* v) {  // the 16-byte-aligned interior of v[lo, hi)
      const uintptr_t a0 = (reinterpret_cast<uintptr_t>(v + lo) + 15) & ~static_cast<uintptr_t>(15);
      const uintptr_t a1 = reinterpret_cast<uintptr_t>(v + hi) & ~static_cast<uintptr_t>(15);
      if (a1 > a0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0),
                     "r"(static_cast<uint32_t>(a1 - a0))
                     : "memory");
    };
    const int t = threadIdx.x;
    if (t < hs.k) {
      pf(A.S + hs.order[t] * A.stride);
      pf(A.Y + hs.order[t] * A.stride);
    }
    if (t == 31) {
      pf(A.g);
      if (A.pair) {
        pf(A.x);
        pf(A.xprev);
        pf(A.gprev);
        pf(A.S + hs.scratch * A.stride);
        pf(A.Y + hs.scratch * A.stride);
      }
    }
  }

  if (A.pair) {  // s = x_{k+1} - x_k, y = g_k - g_{k+1} (lbfgs.hpp:243-244)
    const int scratch = hs.scratch;
    double* __restrict__ sv = A.S + scratch * A.stride;
    double* __restrict__ yv = A.Y + scratch * A.stride;
    double* t0 = buf(0);
    double* t1 = buf(1);
    double* t2 = buf(2);
    if (threadIdx.x == 0) {
      sm.ch[0] = seq::Chain2{t0, dim, 0.0};
      sm.ch[1] = seq::Chain2{t1, dim, 0.0};
      sm.ch[2] = seq::Chain2{t2, dim, 0.0};
    }
#pragma unroll 4
    for (int64_t e = lo + threadIdx.x; e < hi; e += kThreads) {
      const double s = dsub(A.x[e], A.xprev[e]);
      const double y = dsub(A.gprev[e], A.g[e]);
      sv[e] = s;
      yv[e] = y;
      t0[e] = dmul(s, y);
      t1[e] = dmul(s, s);
      t2[e] = dmul(y, y);
    }
    __syncthreads();
    seq::engine2(3, sm);
    ++call;
    if (threadIdx.x == 0) {  // acceptance test and ring update (lbfgs.hpp:246-255)
      const double sy = sm.res[0], ss = sm.res[1], yy = sm.res[2];
      if (cta == 0) {
        A.sc->extra[0] = sy;
        A.sc->extra[1] = ss;
        A.sc->extra[2] = yy;
      }
      hs.last_sy = sy;
      hs.last_ss = ss;
      hs.last_yy = yy;
      const bool accept = sy > 1e-10 * sqrt(ss) * sqrt(yy);
      hs.accepted = accept ? 1 : 0;
      if (accept) {
        int k = hs.k;
        if (k == hs.mem) {
          const int ev = hs.order[0];
          for (int i = 1; i < k; ++i) {
            hs.order[i - 1] = hs.order[i];
            hs.rho[i - 1] = hs.rho[i];
            hs.sy[i - 1] = hs.sy[i];
            hs.yy[i - 1] = hs.yy[i];
          }
          --k;
          hs.order[k] = scratch;
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
        hs.rho[k] = 1.0 / sy;
        hs.sy[k] = sy;
        hs.yy[k] = yy;
        hs.k = k + 1;
      }
    }
    __syncthreads();
    if (cta == 0) {
      for (int i = threadIdx.x; i < static_cast<int>(sizeof(HistState) / 4); i += kThreads)
        reinterpret_cast<int*>(H)[i] = reinterpret_cast<const int*>(&hs)[i];
    }
  }
  const int k = hs.k;
  double* __restrict__ q = A.d;
  // q = g; for i = k-1 .. 0: a_i = rho_i s_i.q; q -= a_i y_i   (lbfgs.hpp:109-115)
  for (int i = k - 1; i >= 0; --i) {
    const double* __restrict__ si = A.S + hs.order[i] * A.stride;
    const double* __restrict__ yp = i + 1 < k ? A.Y + hs.order[i + 1] * A.stride : nullptr;
    const double ap = i + 1 < k ? a_loc[i + 1] : 0.0;
    double* t0 = buf(0);
    if (threadIdx.x == 0) sm.ch[0] = seq::Chain2{t0, dim, 0.0};
#pragma unroll 8
    for (int64_t e = lo + threadIdx.x; e < hi; e += kThreads) {
      const double qe = yp ? dsub(q[e], dmul(ap, yp[e])) : A.g[e];
      q[e] = qe;
      t0[e] = dmul(si[e], qe);
    }
    __syncthreads();
    seq::engine2(1, sm);
    ++call;
    if (threadIdx.x == 0) a_loc[i] = dmul(hs.rho[i], sm.res[0]);
    __syncthreads();
  }
  // the pending q -= a_0 y_0 and the scaling q *= s.y / y.y (lbfgs.hpp:116-119),
  // then for i = 0 .. k-1: b = rho_i y_i.q; q += (a_i - b) s_i  (lbfgs.hpp:120-124)
  const double cscale = (k > 0 && hs.yy[k - 1] > 0.0) ? ddiv(hs.sy[k - 1], hs.yy[k - 1]) : 1.0;
  const bool do_scale = k > 0 && hs.yy[k - 1] > 0.0;
  double coef_prev = 0.0;
  for (int i = 0; i <= k; ++i) {
    // i < k: round i of the second loop; i == k: the final g.d, d.d
    const double* __restrict__ yi = i < k ? A.Y + hs.order[i] * A.stride : nullptr;
    const double* __restrict__ sp = i > 0 ? A.S + hs.order[i - 1] * A.stride : nullptr;
    const double* __restrict__ y0 = k > 0 ? A.Y + hs.order[0] * A.stride : nullptr;
    const double a0 = k > 0 ? a_loc[0] : 0.0;
    double* t0 = buf(0);
    double* t1 = buf(1);
    if (threadIdx.x == 0) {
      sm.ch[0] = seq::Chain2{t0, dim, 0.0};
      sm.ch[1] = seq::Chain2{t1, dim, 0.0};
    }
#pragma unroll 4
    for (int64_t e = lo + threadIdx.x; e < hi; e += kThreads) {
      double qe;
      if (k == 0) {
        qe = A.g[e];  // d = g
      } else if (i == 0) {
        qe = dsub(q[e], dmul(a0, y0[e]));
        if (do_scale) qe = dmul(qe, cscale);
      } else {
        qe = dadd(q[e], dmul(coef_prev, sp[e]));
      }
      q[e] = qe;
      if (i < k) {
        t0[e] = dmul(yi[e], qe);
      } else {
        t0[e] = dmul(A.g[e], qe);  // res.gradient.dot(d) (lbfgs.hpp:126)
        t1[e] = dmul(qe, qe);      // d.squaredNorm() (d.norm(), lbfgs.hpp:152)
      }
    }
    __syncthreads();
    seq::engine2(i < k ? 1 : 2, sm);
    ++call;
    if (i < k) coef_prev = dsub(a_loc[i], dmul(hs.rho[i], sm.res[0]));
  }
  if (cta == 0 && threadIdx.x == 0) {
    A.out[0] = sm.res[0];
    A.out[1] = sm.res[1];
  }
  cl.sync();  // no CTA exits while another may still read its shared memory
}

void launch_exact_direction(const ExactDirArgs& a, const ExactWs& W, cudaStream_t s) {
  DirKArgs K;
  K.a = a;
  K.tv = W.tv;
  K.tv_stride = W.tv_stride;
  launch_cluster(k_ex_direction, K, s);
}

// ---------------------------------------------------------------- dots / test hook

struct DotArgs {
  const double* a;
  const double* b;  // null: sum of a
  int64_t n;
  double s0;
  double* tv;
  double* out;
};

__global__ void __launch_bounds__(kThreads, 1) k_ex_dot(DotArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  seq::Smem2& sm = *reinterpret_cast<seq::Smem2*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int cta = static_cast<int>(cl.block_rank()), ncta = static_cast<int>(cl.num_blocks());
  const int64_t b = seq::block_len(A.n, ncta * kThreads);
  const int64_t lo = min(A.n, static_cast<int64_t>(cta) * kThreads * b);
  const int64_t hi = min(A.n, lo + kThreads * b);
  const double* terms = A.a;
  if (A.b) {
    for (int64_t e = lo + threadIdx.x; e < hi; e += kThreads) A.tv[e] = dmul(A.a[e], A.b[e]);
    terms = A.tv;
  }
  if (threadIdx.x == 0) sm.ch[0] = seq::Chain2{terms, A.n, A.s0};
  __syncthreads();
  seq::engine2(1, sm);
  if (cta == 0 && threadIdx.x == 0) *A.out = sm.res[0];
  cl.sync();  // no CTA exits while another may still read its shared memory
}

void launch_exact_dot2(const double* a, const double* b, int64_t n, const ExactWs& W,
                       EvalScalars* sc, int slot, cudaStream_t s) {
  DotArgs A{a, b, n, 0.0, W.tv, &sc->extra[slot]};
  launch_cluster(k_ex_dot, A, s);
}

void launch_seqsum(const double* terms, int64_t n, double s0, const ExactWs& W, double* out,
                   cudaStream_t s) {
  DotArgs A{terms, nullptr, n, s0, W.tv, out};
  launch_cluster(k_ex_dot, A, s);
}

// Diagnostic: the engine's phase clocks (-DGSOT_SEQ_PROF builds), 8 values,
// then reset. Returns 0 values in product builds.
void read_seq_prof(unsigned long long* out) {
#ifdef GSOT_SEQ_PROF
  cudaMemcpyFromSymbol(out, seq::g_seq_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(seq::g_seq_prof, z, sizeof(z));
#else
  for (int i = 0; i < 16; ++i) out[i] = 0;
#endif
}

}  // namespace gsot
