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
