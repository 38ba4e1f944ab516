// gsot_lbfgs.cu — device vector operations of the L-BFGS ascent
// (lbfgs.hpp:61-274). The host keeps the scalar control flow of `maximize`
// exactly; these kernels do every O(m+n) vector operation so that only
// scalars cross PCIe.
//
// The two-loop recursion (lbfgs.hpp:109-124) runs as ONE launch of a
// cluster of kCluster CTAs. Each CTA owns a contiguous slice of the vectors;
// every dot product is reduced inside the CTA (fixed tree), published to
// shared memory and summed by every CTA over the cluster ranks in rank order
// through distributed shared memory, so all CTAs see the same bits and the
// result is deterministic. Dots are fused with the axpy that precedes them,
// so the recursion makes 2k+1 passes over the history instead of 4k+3.
// Elementwise arithmetic keeps the reference's one-rounding-per-operation
// form (q - a*y, q*c, q + (a-b)*s, x + t*d).
#include <cooperative_groups.h>

#include "gsot_internal.cuh"

namespace cg = cooperative_groups;

namespace gsot {

namespace {
constexpr int kCluster = 8;
constexpr int kTwoLoopThreads = 512;

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
}  // namespace

// Cluster-wide deterministic dot reduction. `part` is this thread's partial.
// Uses slot `parity` of the per-CTA publication buffer; one cluster.sync.
__device__ __forceinline__ double cluster_sum(cg::cluster_group& cluster, double part,
                                              double* warp_sh, double* pub, int parity) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) part = dadd(part, __shfl_xor_sync(0xffffffffu, part, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_sh[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kTwoLoopThreads / 32; ++w) s = dadd(s, warp_sh[w]);
    pub[parity] = s;
  }
  cluster.sync();
  double tot = 0.0;
  for (int r = 0; r < kCluster; ++r) {
    const double* remote = cluster.map_shared_rank(pub, r);
    tot = dadd(tot, remote[parity]);
  }
  return tot;
}

__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kTwoLoopThreads)
    k_two_loop(const TwoLoopArgs A) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double warp_sh[kTwoLoopThreads / 32];
  __shared__ double pub[2];
  __shared__ double a_sh[kMaxMemory];
  const int rank = (int)cluster.block_rank();
  const int64_t per = (A.dim + kCluster - 1) / kCluster;
  const int64_t lo = rank * per;
  const int64_t hi = min(A.dim, lo + per);
  double* __restrict__ q = A.d;  // q is built in place in the output vector
  const int k = A.k;
  int parity = 0;

  // q = g; pass for i = k-1: a_{k-1} = rho * s_{k-1}.q
  // Generic pass i (loop 1): q -= a_{i+1} * y_{i+1}; a_i = rho_i * s_i.q
  for (int i = k - 1; i >= 0; --i) {
    double part = 0.0;
    const double* __restrict__ si = A.s[i];
    if (i == k - 1) {
      for (int64_t e = lo + threadIdx.x; e < hi; e += kTwoLoopThreads) {
        const double qe = A.g[e];
        q[e] = qe;
        part = dadd(part, dmul(si[e], qe));
      }
    } else {
      const double ap = a_sh[i + 1];
      const double* __restrict__ yp = A.y[i + 1];
      for (int64_t e = lo + threadIdx.x; e < hi; e += kTwoLoopThreads) {
        const double qe = dsub(q[e], dmul(ap, yp[e]));
        q[e] = qe;
        part = dadd(part, dmul(si[e], qe));
      }
    }
    const double dot = cluster_sum(cluster, part, warp_sh, pub, parity);
    parity ^= 1;
    if (threadIdx.x == 0) a_sh[i] = dmul(A.rho[i], dot);
    __syncthreads();
  }
  // Close loop 1 (q -= a_0 y_0), scale by s.y / y.y (lbfgs.hpp:116-119), and
  // run loop 2 (lbfgs.hpp:120-123) fused: pass i applies the update of i-1
  // and reduces y_i.q.
  double b_prev = 0.0;
  for (int i = 0; i <= k; ++i) {
    double part = 0.0;
    const bool last = (i == k);
    const double* __restrict__ yi = last ? nullptr : A.y[i];
    if (k == 0) {
      // No history: d = g.
      for (int64_t e = lo + threadIdx.x; e < hi; e += kTwoLoopThreads) q[e] = A.g[e];
    } else if (i == 0) {
      const double a0 = a_sh[0];
      const double* __restrict__ y0 = A.y[0];
      for (int64_t e = lo + threadIdx.x; e < hi; e += kTwoLoopThreads) {
        double qe = dsub(q[e], dmul(a0, y0[e]));
        if (A.apply_scale) qe = dmul(qe, A.gamma_scale);
        q[e] = qe;
        part = dadd(part, dmul(yi[e], qe));
      }
    } else {
      const double coef = dsub(a_sh[i - 1], b_prev);
      const double* __restrict__ sp = A.s[i - 1];
      for (int64_t e = lo + threadIdx.x; e < hi; e += kTwoLoopThreads) {
        const double qe = dadd(q[e], dmul(coef, sp[e]));
        q[e] = qe;
        if (!last) part = dadd(part, dmul(yi[e], qe));
      }
    }
    if (last) break;
    const double dot = cluster_sum(cluster, part, warp_sh, pub, parity);
    parity ^= 1;
    b_prev = dmul(A.rho[i], dot);
  }
  // dir_slope = g.d and |d|^2 (lbfgs.hpp:126, :152).
  double pg = 0.0, pd = 0.0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += kTwoLoopThreads) {
    const double de = q[e];
    pg = dadd(pg, dmul(A.g[e], de));
    pd = dadd(pd, dmul(de, de));
  }
  const double gd = cluster_sum(cluster, pg, warp_sh, pub, parity);
  parity ^= 1;
  const double dd = cluster_sum(cluster, pd, warp_sh, pub, parity);
  if (rank == 0 && threadIdx.x == 0) {
    A.out[0] = gd;
    A.out[1] = dd;
  }
  cluster.sync();  // keep every CTA's shared memory alive until remote reads finish
}

void launch_two_loop(const TwoLoopArgs& a, cudaStream_t s) {
  k_two_loop<<<kCluster, kTwoLoopThreads, 0, s>>>(a);
}

// trial.x = x + t * d (lbfgs.hpp:86).
__global__ void k_axpy_point(const double* __restrict__ x, double t, const double* __restrict__ d,
                             double* __restrict__ out, int64_t dim) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = dadd(x[e], dmul(t, d[e]));
}

void launch_axpy_point(const double* x, double t, const double* d, double* out, int64_t dim,
                       cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((dim + 255) / 256, 148 * 4);
  k_axpy_point<<<grid, 256, 0, s>>>(x, t, d, out, dim);
}

namespace {
__device__ __forceinline__ double block_sum256(double v, double* sh) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < 8; ++w) r = dadd(r, sh[w]);
  return r;
}
}  // namespace

// Curvature pair (lbfgs.hpp:243-246): s = trial.x - x, y = g - trial.g
// written to the ring slot, plus s.y, s.s, y.y (deterministic).
__global__ void __launch_bounds__(256) k_pair(const double* __restrict__ xt,
                                              const double* __restrict__ x,
                                              const double* __restrict__ g,
                                              const double* __restrict__ gt,
                                              double* __restrict__ sv, double* __restrict__ yv,
                                              int64_t dim, double* __restrict__ partials,
                                              EvalScalars* sc) {
  __shared__ double sh[8];
  __shared__ bool last;
  double psy = 0.0, pss = 0.0, pyy = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double s = dsub(xt[e], x[e]);
    const double y = dsub(g[e], gt[e]);
    sv[e] = s;
    yv[e] = y;
    psy = dadd(psy, dmul(s, y));
    pss = dadd(pss, dmul(s, s));
    pyy = dadd(pyy, dmul(y, y));
  }
  const double a = block_sum256(psy, sh);
  const double b = block_sum256(pss, sh);
  const double c = block_sum256(pyy, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x * 3 + 0] = a;
    partials[blockIdx.x * 3 + 1] = b;
    partials[blockIdx.x * 3 + 2] = c;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double ta = 0.0, tb = 0.0, tc = 0.0;
    for (unsigned q = 0; q < gridDim.x; ++q) {
      ta = dadd(ta, partials[q * 3 + 0]);
      tb = dadd(tb, partials[q * 3 + 1]);
      tc = dadd(tc, partials[q * 3 + 2]);
    }
    sc->extra[0] = ta;
    sc->extra[1] = tb;
    sc->extra[2] = tc;
    sc->ticket = 0u;
  }
}

void launch_pair(const double* xt, const double* x, const double* g, const double* gt, double* sv,
                 double* yv, int64_t dim, double* partials, int nblocks, EvalScalars* sc,
                 cudaStream_t s) {
  k_pair<<<nblocks, 256, 0, s>>>(xt, x, g, gt, sv, yv, dim, partials, sc);
}

// Plain deterministic dot into sc->extra[slot].
__global__ void __launch_bounds__(256) k_dot(const double* __restrict__ a,
                                             const double* __restrict__ b, int64_t dim,
                                             double* __restrict__ partials, EvalScalars* sc,
                                             int slot) {
  __shared__ double sh[8];
  __shared__ bool last;
  double p = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x)
    p = dadd(p, dmul(a[e], b[e]));
  const double r = block_sum256(p, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = r;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double t = 0.0;
    for (unsigned q = 0; q < gridDim.x; ++q) t = dadd(t, partials[q]);
    sc->extra[slot] = t;
    sc->ticket = 0u;
  }
}

void launch_dot(const double* a, const double* b, int64_t dim, double* partials, int nblocks,
                EvalScalars* sc, int slot, cudaStream_t s) {
  k_dot<<<nblocks, 256, 0, s>>>(a, b, dim, partials, sc, slot);
}

// max |a_e| into sc->extra[slot] (order-independent, exact).
__global__ void __launch_bounds__(256) k_absmax(const double* __restrict__ a, int64_t dim,
                                                double* __restrict__ partials, EvalScalars* sc,
                                                int slot) {
  __shared__ double sh[8];
  __shared__ bool last;
  double p = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dim;
       e += (int64_t)gridDim.x * blockDim.x)
    p = fmax(p, fabs(a[e]));
  for (int o = 16; o >= 1; o >>= 1) p = fmax(p, __shfl_xor_sync(0xffffffffu, p, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < 8; ++w) r = fmax(r, sh[w]);
    partials[blockIdx.x] = r;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double t = 0.0;
    for (unsigned q = 0; q < gridDim.x; ++q) t = fmax(t, partials[q]);
    sc->extra[slot] = t;
    sc->ticket = 0u;
  }
}

void launch_absmax(const double* a, int64_t dim, double* partials, int nblocks, EvalScalars* sc,
                   int slot, cudaStream_t s) {
  k_absmax<<<nblocks, 256, 0, s>>>(a, dim, partials, sc, slot);
}

}  // namespace gsot
