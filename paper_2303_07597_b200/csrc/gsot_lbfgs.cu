// gsot_lbfgs.cu — device vector operations of the L-BFGS ascent
// (lbfgs.hpp:61-274). The host keeps the scalar control flow of `maximize`
// exactly; these kernels do every O(m+n) vector operation so that only
// scalars cross PCIe.
//
// The two-loop recursion (lbfgs.hpp:109-124) runs as ONE launch of a
// thread-block cluster (16 CTAs where the device allows non-portable
// clusters, else 8). Each CTA owns a contiguous slice of the vectors and keeps
// its slice of q in shared memory; every dot product is reduced inside the
// CTA (fixed tree), published in shared memory and summed by every CTA over
// the cluster ranks in rank order through distributed shared memory, so all
// CTAs see the same bits and the result is deterministic. Dots are fused with
// the update that precedes them: the recursion makes 2k+1 passes over the
// history instead of 4k+3. Elementwise arithmetic keeps the reference's
// one-rounding-per-operation form (q - a*y, q*c, q + (a-b)*s, x + t*d).
#include <cooperative_groups.h>

#include "gsot_device.cuh"

namespace cg = cooperative_groups;

namespace gsot {

namespace {
constexpr int kTwoLoopThreads = 512;
constexpr int kWarps = kTwoLoopThreads / 32;
int g_cluster = 0;           // chosen cluster size (16 or 8)
size_t g_two_loop_smem = 0;  // dynamic smem configured so far
}  // namespace

// Cluster-wide deterministic sum. `part` is this thread's partial. Uses slot
// `parity` of the per-CTA publication buffer; one cluster barrier.
__device__ __forceinline__ double cluster_sum(cg::cluster_group& cluster, double part,
                                              double* warp_sh, double* pub, double* tot_sh,
                                              int parity, int nranks) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) part = dadd(part, __shfl_xor_sync(0xffffffffu, part, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_sh[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = warp_sh[0];
    for (int w = 1; w < kWarps; ++w) s = dadd(s, warp_sh[w]);
    pub[parity] = s;
  }
  cluster.sync();
  if (warp == 0) {
    double v = 0.0;
    if (lane < nranks) v = cluster.map_shared_rank(pub, lane)[parity];
    // rank-ordered sequential sum on lane 0
    double t = 0.0;
    for (int r = 0; r < nranks; ++r) t = dadd(t, __shfl_sync(0xffffffffu, v, r));
    if (lane == 0) tot_sh[parity] = t;
  }
  __syncthreads();
  return tot_sh[parity];
}

__global__ void __launch_bounds__(kTwoLoopThreads) k_two_loop(const TwoLoopArgs A, int use_smem) {
  extern __shared__ double q_dyn[];
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double warp_sh[kWarps];
  __shared__ double pub[2];
  __shared__ double tot_sh[2];
  __shared__ double a_sh[kMaxMemory];
  const int nranks = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int64_t per = (A.dim + nranks - 1) / nranks;
  const int64_t lo = rank * per;
  const int64_t hi = min(A.dim, lo + per);
  const int64_t len = hi > lo ? hi - lo : 0;
  // q slice: shared memory when it fits, else the output vector itself
  double* __restrict__ q = use_smem ? q_dyn : A.d + lo;
  const double* __restrict__ g = A.g + lo;
  // history snapshot (no CTA writes it during this kernel)
  __shared__ const double* s_ptr[kMaxMemory];
  __shared__ const double* y_ptr[kMaxMemory];
  __shared__ double rho_sh[kMaxMemory];
  __shared__ double scale_sh;
  __shared__ int k_sh, apply_sh;
  if (threadIdx.x == 0) {
    const int kk = A.h->k;
    k_sh = kk;
    for (int i = 0; i < kk; ++i) {
      const int slot = A.h->order[i];
      s_ptr[i] = A.S + slot * A.stride;
      y_ptr[i] = A.Y + slot * A.stride;
      rho_sh[i] = A.h->rho[i];
    }
    // lbfgs.hpp:116-119: q *= s.y / y.y of the newest pair when y.y > 0
    apply_sh = 0;
    scale_sh = 1.0;
    if (kk > 0 && A.h->yy[kk - 1] > 0.0) {
      apply_sh = 1;
      scale_sh = A.h->sy[kk - 1] / A.h->yy[kk - 1];
    }
  }
  __syncthreads();
  const int k = k_sh;
  int parity = 0;

  // Loop 1 (lbfgs.hpp:112-115). Pass i: q -= a_{i+1} y_{i+1} (or q = g for
  // the first pass), then a_i = rho_i * s_i . q.
  for (int i = k - 1; i >= 0; --i) {
    double part = 0.0;
    const double* __restrict__ si = s_ptr[i] + lo;
    if (i == k - 1) {
#pragma unroll 4
      for (int64_t e = threadIdx.x; e < len; e += kTwoLoopThreads) {
        const double qe = g[e];
        q[e] = qe;
        part = dadd(part, dmul(si[e], qe));
      }
    } else {
      const double ap = a_sh[i + 1];
      const double* __restrict__ yp = y_ptr[i + 1] + lo;
#pragma unroll 4
      for (int64_t e = threadIdx.x; e < len; e += kTwoLoopThreads) {
        const double qe = dsub(q[e], dmul(ap, yp[e]));
        q[e] = qe;
        part = dadd(part, dmul(si[e], qe));
      }
    }
    const double dot = cluster_sum(cluster, part, warp_sh, pub, tot_sh, parity, nranks);
    parity ^= 1;
    if (threadIdx.x == 0) a_sh[i] = dmul(rho_sh[i], dot);
    __syncthreads();
  }
  // Close loop 1 (q -= a_0 y_0), scale by s.y / y.y (lbfgs.hpp:116-119), and
  // run loop 2 (lbfgs.hpp:120-123) fused: pass i applies the update of i-1
  // and reduces y_i . q.
  double b_prev = 0.0;
  for (int i = 0; i <= k; ++i) {
    double part = 0.0;
    const bool last = (i == k);
    if (k == 0) {
      for (int64_t e = threadIdx.x; e < len; e += kTwoLoopThreads) q[e] = g[e];  // d = g
    } else if (i == 0) {
      const double a0 = a_sh[0];
      const double* __restrict__ y0 = y_ptr[0] + lo;
#pragma unroll 4
      for (int64_t e = threadIdx.x; e < len; e += kTwoLoopThreads) {
        double qe = dsub(q[e], dmul(a0, y0[e]));
        if (apply_sh) qe = dmul(qe, scale_sh);
        q[e] = qe;
        part = dadd(part, dmul(y0[e], qe));
      }
    } else {
      const double coef = dsub(a_sh[i - 1], b_prev);
      const double* __restrict__ sp = s_ptr[i - 1] + lo;
      const double* __restrict__ yi = last ? nullptr : y_ptr[i] + lo;
#pragma unroll 4
      for (int64_t e = threadIdx.x; e < len; e += kTwoLoopThreads) {
        const double qe = dadd(q[e], dmul(coef, sp[e]));
        q[e] = qe;
        if (!last) part = dadd(part, dmul(yi[e], qe));
      }
    }
    if (last) break;
    const double dot = cluster_sum(cluster, part, warp_sh, pub, tot_sh, parity, nranks);
    parity ^= 1;
    b_prev = dmul(rho_sh[i], dot);
  }
  // d = q; dir_slope = g . d and |d|^2 (lbfgs.hpp:124-126, :152).
  double pg = 0.0, pd = 0.0;
  double* __restrict__ d = A.d + lo;
#pragma unroll 4
  for (int64_t e = threadIdx.x; e < len; e += kTwoLoopThreads) {
    const double de = q[e];
    if (use_smem) d[e] = de;
    pg = dadd(pg, dmul(g[e], de));
    pd = dadd(pd, dmul(de, de));
  }
  const double gd = cluster_sum(cluster, pg, warp_sh, pub, tot_sh, parity, nranks);
  parity ^= 1;
  const double dd = cluster_sum(cluster, pd, warp_sh, pub, tot_sh, parity, nranks);
  if (rank == 0 && threadIdx.x == 0) {
    A.out[0] = gd;
    A.out[1] = dd;
  }
  cluster.sync();  // keep every CTA's shared memory alive until remote reads finish
}

void launch_two_loop(const TwoLoopArgs& a, cudaStream_t s) {
  if (g_cluster == 0) {
    g_cluster = 8;
    if (cudaFuncSetAttribute(k_two_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
        cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = 16;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(kTwoLoopThreads);
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, k_two_loop, &cfg) == cudaSuccess &&
          nclusters > 0)
        g_cluster = 16;
    }
    cudaGetLastError();
  }
  const int64_t per = (a.dim + g_cluster - 1) / g_cluster;
  size_t smem = sizeof(double) * (size_t)per;
  int use_smem = smem <= 200 * 1024 ? 1 : 0;
  if (!use_smem) smem = 0;
  if (smem > g_two_loop_smem) {
    cudaFuncSetAttribute(k_two_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    g_two_loop_smem = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = g_cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.gridDim = dim3(g_cluster);
  cfg.blockDim = dim3(kTwoLoopThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_two_loop, a, use_smem);
}

// trial.x = x + t * d (lbfgs.hpp:86).
__global__ void k_axpy_point(const double* __restrict__ x, const double* __restrict__ tp,
                             const double* __restrict__ d, double* __restrict__ out, int64_t dim) {
  const double t = *tp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = dadd(x[e], dmul(t, d[e]));
}

void launch_axpy_point(const double* x, const double* t, const double* d, double* out,
                       int64_t dim, cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((dim + 255) / 256, 148 * 4);
  k_axpy_point<<<grid, 256, 0, s>>>(x, t, d, out, dim);
}

// Curvature pair (lbfgs.hpp:243-255): s = trial.x - x, y = g - trial.g
// written to the scratch slot, s.y, s.s, y.y (deterministic), then -- in
// the last block -- the acceptance test sy > 1e-10 |s| |y| and the ring
// update: evict the oldest pair when full, append the scratch slot.
__global__ void __launch_bounds__(256) k_pair(const double* __restrict__ xt,
                                              const double* __restrict__ x,
                                              const double* __restrict__ g,
                                              const double* __restrict__ gt,
                                              double* __restrict__ S, double* __restrict__ Y,
                                              int64_t stride, HistState* h, int64_t dim,
                                              double* __restrict__ partials, EvalScalars* sc) {
  const int scratch = h->scratch;  // read by every block before the last one updates h
  double* __restrict__ sv = S + scratch * stride;
  double* __restrict__ yv = Y + scratch * stride;
  double p[3] = {0.0, 0.0, 0.0};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double s = dsub(xt[e], x[e]);
    const double y = dsub(g[e], gt[e]);
    sv[e] = s;
    yv[e] = y;
    p[0] = dadd(p[0], dmul(s, y));
    p[1] = dadd(p[1], dmul(s, s));
    p[2] = dadd(p[2], dmul(y, y));
  }
  double out[3];
  if (last_block_reduce<256, 3>(p, partials, &sc->ticket, out)) {
    const double sy = out[0], ss = out[1], yy = out[2];
    sc->extra[0] = sy;
    sc->extra[1] = ss;
    sc->extra[2] = yy;
    h->last_sy = sy;
    h->last_ss = ss;
    h->last_yy = yy;
    const bool accept = sy > 1e-10 * sqrt(ss) * sqrt(yy);
    h->accepted = accept ? 1 : 0;
    if (accept) {
      int k = h->k;
      if (k == h->mem) {  // erase the oldest (lbfgs.hpp:247-251)
        const int ev = h->order[0];
        for (int i = 1; i < k; ++i) {
          h->order[i - 1] = h->order[i];
          h->rho[i - 1] = h->rho[i];
          h->sy[i - 1] = h->sy[i];
          h->yy[i - 1] = h->yy[i];
        }
        --k;
        h->order[k] = scratch;
        h->scratch = ev;
      } else {
        h->order[k] = scratch;
        // next scratch: the lowest slot not in use
        int next = 0;
        for (;; ++next) {
          bool used = false;
          for (int i = 0; i <= k; ++i) used |= h->order[i] == next;
          if (!used) break;
        }
        h->scratch = next;
      }
      h->rho[k] = 1.0 / sy;
      h->sy[k] = sy;
      h->yy[k] = yy;
      h->k = k + 1;
    }
  }
}

void launch_pair(const double* xt, const double* x, const double* g, const double* gt, double* S,
                 double* Y, int64_t stride, HistState* h, int64_t dim, double* partials,
                 int nblocks, EvalScalars* sc, cudaStream_t s) {
  k_pair<<<nblocks, 256, 0, s>>>(xt, x, g, gt, S, Y, stride, h, dim, partials, sc);
}

// Clear the history (lbfgs.hpp:102-104, :128-130).
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

}  // namespace gsot

// ============================================================ compact L-BFGS
namespace gsot {

namespace {
constexpr int kSlices = 16;  // dim slices per history row in the prepare pass
}

// Multi-dot pass. Row i < k: history pair i (logical) against the new pair
// and the new gradient: s_i.y, y_i.y, s_i.gn, y_i.gn. Row k (pair != 0):
// the new pair itself, written to the scratch slot: s.y, s.s, y.y, s.gn,
// y.gn. Rows beyond are idle (the grid is sized for mem + 1 rows so that a
// captured graph never changes). The last block reduces the partials in
// slice order, applies the acceptance test and ring update, maintains R and
// YY by logical position, and solves for the direction coefficients.
__global__ void __launch_bounds__(256) k_compact_prepare(
    int pair, const double* __restrict__ xt, const double* __restrict__ x,
    const double* __restrict__ gt, const double* __restrict__ g, const double* __restrict__ gn,
    double* __restrict__ S, double* __restrict__ Y, int64_t stride, HistState* h,
    CompactState* cs, int64_t dim, double* __restrict__ partials, EvalScalars* sc) {
  __shared__ double sh[8][5];
  __shared__ bool last;
  const int k = h->k;  // every block reads before the last block updates
  const int scratch = h->scratch;
  const int row = blockIdx.y;
  const int nrows = gridDim.y;
  const int64_t per = (dim + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(dim, lo + per);
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (row < k) {
    const double* __restrict__ si = S + h->order[row] * stride;
    const double* __restrict__ yi = Y + h->order[row] * stride;
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
      const double s = si[e], y = yi[e], gg = gn[e];
      if (pair) {
        const double yn = dsub(g[e], gt[e]);
        acc[0] = dadd(acc[0], dmul(s, yn));
        acc[1] = dadd(acc[1], dmul(y, yn));
      }
      acc[2] = dadd(acc[2], dmul(s, gg));
      acc[3] = dadd(acc[3], dmul(y, gg));
    }
  } else if (row == k && pair) {
    double* __restrict__ sv = S + scratch * stride;
    double* __restrict__ yv = Y + scratch * stride;
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
      const double s = dsub(xt[e], x[e]);
      const double y = dsub(g[e], gt[e]);
      sv[e] = s;
      yv[e] = y;
      const double gg = gn[e];
      acc[0] = dadd(acc[0], dmul(s, y));
      acc[1] = dadd(acc[1], dmul(s, s));
      acc[2] = dadd(acc[2], dmul(y, y));
      acc[3] = dadd(acc[3], dmul(s, gg));
      acc[4] = dadd(acc[4], dmul(y, gg));
    }
  }
  // fixed-tree block reduction of the 5 accumulators
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t base = ((int64_t)row * gridDim.x + blockIdx.x) * 5;
    for (int q = 0; q < 5; ++q) {
      double v = sh[0][q];
      for (int w = 1; w < 8; ++w) v = dadd(v, sh[w][q]);
      partials[base + q] = v;
    }
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // reduce each (row, q) over the slices in slice order (one thread each)
  __shared__ double red[(kMaxMemory + 1) * 5];
  for (int t = threadIdx.x; t < nrows * 5; t += blockDim.x) {
    const int r = t / 5, q = t % 5;
    double pv[kSlices];  // all loads first, then the slice-ordered sum
#pragma unroll
    for (int b = 0; b < kSlices; ++b) pv[b] = __ldcg(partials + ((int64_t)r * kSlices + b) * 5 + q);
    double v = 0.0;
#pragma unroll
    for (int b = 0; b < kSlices; ++b) v = dadd(v, pv[b]);
    red[t] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  sc->ticket = 0u;
  int kk = k;
  double u[kMaxMemory + 1], vv[kMaxMemory + 1];
  for (int i = 0; i < k; ++i) {
    u[i] = red[i * 5 + 2];
    vv[i] = red[i * 5 + 3];
  }
  if (pair) {
    const double sy = red[k * 5 + 0], ss = red[k * 5 + 1], yy = red[k * 5 + 2];
    sc->extra[0] = sy;
    sc->extra[1] = ss;
    sc->extra[2] = yy;
    h->last_sy = sy;
    h->last_ss = ss;
    h->last_yy = yy;
    const bool accept = sy > 1e-10 * sqrt(ss) * sqrt(yy);  // lbfgs.hpp:246
    h->accepted = accept ? 1 : 0;
    if (accept) {
      double sy_new[kMaxMemory], yy_new[kMaxMemory];
      for (int i = 0; i < k; ++i) {
        sy_new[i] = red[i * 5 + 0];  // s_i . y_new
        yy_new[i] = red[i * 5 + 1];  // y_i . y_new
      }
      int first = 0;
      if (k == h->mem) {  // evict the oldest (lbfgs.hpp:247-251)
        first = 1;
        const int ev = h->order[0];
        for (int i = 1; i < k; ++i) {
          h->order[i - 1] = h->order[i];
          h->rho[i - 1] = h->rho[i];
          h->sy[i - 1] = h->sy[i];
          h->yy[i - 1] = h->yy[i];
          for (int j = 1; j < k; ++j) {
            cs->R[(i - 1) * kMaxMemory + (j - 1)] = cs->R[i * kMaxMemory + j];
            cs->YY[(i - 1) * kMaxMemory + (j - 1)] = cs->YY[i * kMaxMemory + j];
          }
        }
        kk = k - 1;
        h->order[kk] = scratch;
        h->scratch = ev;
      } else {
        h->order[k] = scratch;
        int next = 0;
        for (;; ++next) {
          bool used = false;
          for (int i = 0; i <= k; ++i) used |= h->order[i] == next;
          if (!used) break;
        }
        h->scratch = next;
      }
      for (int i = 0; i < kk; ++i) {  // shift u, v and the new column
        u[i] = u[i + first];
        vv[i] = vv[i + first];
        cs->R[i * kMaxMemory + kk] = sy_new[i + first];
        cs->YY[i * kMaxMemory + kk] = yy_new[i + first];
        cs->YY[kk * kMaxMemory + i] = yy_new[i + first];
      }
      cs->R[kk * kMaxMemory + kk] = sy;
      cs->YY[kk * kMaxMemory + kk] = yy;
      u[kk] = red[k * 5 + 3];
      vv[kk] = red[k * 5 + 4];
      h->rho[kk] = 1.0 / sy;
      h->sy[kk] = sy;
      h->yy[kk] = yy;
      kk += 1;
      h->k = kk;
    }
  }
  // gam (lbfgs.hpp:116-119), then w = R^-1 u, z = (D + gam YY) w - gam v,
  // p = R^-T z; d = gam g + S p - gam Y w.
  double gam = 1.0;
  if (kk > 0 && h->yy[kk - 1] > 0.0) gam = h->sy[kk - 1] / h->yy[kk - 1];
  double w[kMaxMemory], p[kMaxMemory];
  for (int i = kk - 1; i >= 0; --i) {
    double t = u[i];
    for (int j = i + 1; j < kk; ++j) t -= cs->R[i * kMaxMemory + j] * w[j];
    w[i] = t / cs->R[i * kMaxMemory + i];
  }
  for (int i = 0; i < kk; ++i) {
    double t = cs->R[i * kMaxMemory + i] * w[i] - gam * vv[i];
    for (int j = 0; j < kk; ++j) t += gam * cs->YY[i * kMaxMemory + j] * w[j];
    for (int j = 0; j < i; ++j) t -= cs->R[j * kMaxMemory + i] * p[j];
    p[i] = t / cs->R[i * kMaxMemory + i];
  }
  for (int i = 0; i < kk; ++i) {
    cs->p[i] = p[i];
    cs->w[i] = gam * w[i];
    cs->u[i] = u[i];
    cs->v[i] = vv[i];
  }
  cs->gam = gam;
  cs->k = kk;
}

void launch_compact_prepare(int pair, const double* xt, const double* x, const double* gt,
                            const double* g, const double* gn, double* S, double* Y,
                            int64_t stride, HistState* h, CompactState* cs, int mem, int64_t dim,
                            double* partials, EvalScalars* sc, cudaStream_t s) {
  // rows: the history capacity + 1, static so that captured graphs never change
  dim3 grid(kSlices, (unsigned)(mem + 1));
  k_compact_prepare<<<grid, 256, 0, s>>>(pair, xt, x, gt, g, gn, S, Y, stride, h, cs, dim,
                                         partials, sc);
}

// d = gam g + sum_i p_i s_i - sum_i w_i y_i (per element, i ascending), the
// slopes g.d and d.d, and the first trial point x + t d.
__global__ void __launch_bounds__(256) k_compact_direction(
    const double* __restrict__ g, const double* __restrict__ S, const double* __restrict__ Y,
    int64_t stride, const HistState* __restrict__ h, const CompactState* __restrict__ cs,
    double* __restrict__ d, const double* __restrict__ x, const double* __restrict__ tp,
    double* __restrict__ xt, int64_t dim, double* __restrict__ partials, EvalScalars* sc,
    double* __restrict__ out) {
  __shared__ const double* sp[kMaxMemory];
  __shared__ const double* yp[kMaxMemory];
  __shared__ double pc[kMaxMemory], wc[kMaxMemory];
  __shared__ int ks;
  __shared__ double gs;
  if (threadIdx.x == 0) {
    ks = cs->k;
    gs = cs->gam;
  }
  __syncthreads();
  const int k = ks;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    sp[i] = S + h->order[i] * stride;
    yp[i] = Y + h->order[i] * stride;
    pc[i] = cs->p[i];
    wc[i] = cs->w[i];
  }
  __syncthreads();
  const double gam = gs;
  const double t = xt ? *tp : 0.0;
  double acc[2] = {0.0, 0.0};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double ge = g[e];
    double de = dmul(gam, ge);
    for (int i = 0; i < k; ++i) de = dadd(de, dmul(pc[i], sp[i][e]));
    for (int i = 0; i < k; ++i) de = dsub(de, dmul(wc[i], yp[i][e]));
    d[e] = de;
    if (xt) xt[e] = dadd(x[e], dmul(t, de));  // lbfgs.hpp:86
    acc[0] = dadd(acc[0], dmul(ge, de));
    acc[1] = dadd(acc[1], dmul(de, de));
  }
  double r[2];
  if (last_block_reduce<256, 2>(acc, partials, &sc->ticket, r)) {
    out[0] = r[0];
    out[1] = r[1];
  }
}

void launch_compact_direction(const double* g, const double* S, const double* Y, int64_t stride,
                              const HistState* h, const CompactState* cs, double* d,
                              const double* x, const double* t, double* xt_out, int64_t dim,
                              double* partials, EvalScalars* sc, double* out, int nblocks,
                              cudaStream_t s) {
  k_compact_direction<<<nblocks, 256, 0, s>>>(g, S, Y, stride, h, cs, d, x, t, xt_out, dim,
                                              partials, sc, out);
}

}  // namespace gsot
