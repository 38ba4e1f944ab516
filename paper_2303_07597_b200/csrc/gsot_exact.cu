// gsot_exact.cu — exact-order mode (GSOT_FLAG_EXACT): every cross-block
// sum in the reference's own association, so a device solve reproduces the
// reference trajectory bit for bit.
//
//   dual_objective  psi_sum += psi_block(f_{l,j}) for j outer, l inner, with
//                   psi_block's dot/sq formula (regularizer.hpp:78-91,
//                   dual.hpp:44-51); a.alpha and b.beta as sequential dots
//   dual_gradient   grad_alpha_i = ((a_i - T_i0) - T_i1) - ...  (dual.hpp:96)
//                   grad_beta_j = b_j - sum_entries(T_.j)      (dual.hpp:97-98)
//   L-BFGS          every dot product sequential in index order (the
//                   oracle's Eigen shim, lbfgs.hpp:89-132, :245-246)
//
// Terms that are exact zeros are skipped in the chains: adding or
// subtracting +0.0 leaves a value unchanged (the partial sums are never -0.0
// under round-to-nearest), so skipping them is exact. This mode exists for
// verification; it runs the sequential chains on one thread.
#include "gsot_device.cuh"

namespace gsot {

// Per block: z, scale (0 when z <= tau) and psi_block exactly as the
// reference (regularizer.hpp:64-91). One thread per (l, j), rows ascending.
__global__ void __launch_bounds__(256) k_exact_blocks(DevProblem P, const double* __restrict__ x,
                                                      double* __restrict__ scale_out,
                                                      double* __restrict__ psi_out) {
  const int l = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const double* __restrict__ al = x + o0;
  const double bj = x[P.m + j];
  const double* __restrict__ cp = block_ptr(P, o0, g, j);
  double z2 = 0.0;
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[32 * r]);
    const double v = f > 0.0 ? f : 0.0;
    z2 = dadd(z2, dmul(v, v));
  }
  const double z = sqrt(z2);
  const int64_t idx = (int64_t)l * P.n + j;
  if (z <= P.tau) {
    scale_out[idx] = 0.0;
    psi_out[idx] = 0.0;
    return;
  }
  const double scale = ddiv(dsub(1.0, ddiv(P.tau, z)), P.gamma);
  double dot = 0.0, sq = 0.0;
  for (int r = 0; r < g; ++r) {
    const double f = residual(__ldg(al + r), bj, cp[32 * r]);
    const double gg = f > 0.0 ? dmul(scale, f) : 0.0;
    dot = dadd(dot, dmul(f, gg));
    sq = dadd(sq, dmul(gg, gg));
  }
  scale_out[idx] = scale;
  psi_out[idx] = dsub(dot, dmul(P.gamma, dadd(dmul(0.5, sq), dmul(P.mu, sqrt(sq)))));
}

// grad_alpha_i = a_i - T_i0 - T_i1 - ... in ascending j (dual.hpp:91, :96).
__global__ void __launch_bounds__(128) k_exact_grad_alpha(DevProblem P, const double* __restrict__ x,
                                                          const double* __restrict__ scale,
                                                          double* __restrict__ grad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P.m) return;
  const int l = P.row_group[i];
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  const int64_t r = i - o0;
  const double ai = x[i];
  const double* __restrict__ sl = scale + (int64_t)l * P.n;
  const double* __restrict__ tile = P.C + 32 * ((int64_t)P.nw * o0) + 32 * r;
  double acc = P.a[i];
  for (int64_t j = 0; j < P.n; ++j) {
    const double s = sl[j];
    if (s == 0.0) continue;  // zero block: T_ij = 0.0
    const double c = tile[(j >> 5) * 32 * (int64_t)g + (j & 31)];
    const double f = residual(ai, x[P.m + j], c);
    if (f > 0.0) acc = dsub(acc, dmul(s, f));
  }
  grad[i] = acc;
}

// grad_beta_j = b_j - sum_entries(gcol_j): the column sum over all m rows in
// ascending order (dual.hpp:97-98, regularizer.hpp:47-51).
__global__ void __launch_bounds__(256) k_exact_grad_beta(DevProblem P, const double* __restrict__ x,
                                                         const double* __restrict__ scale,
                                                         double* __restrict__ grad) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  const double bj = x[P.m + j];
  double acc = 0.0;
  for (int l = 0; l < P.L; ++l) {
    const double s = scale[(int64_t)l * P.n + j];
    if (s == 0.0) continue;
    const int o0 = P.off[l], g = P.off[l + 1] - o0;
    const double* __restrict__ al = x + o0;
    const double* __restrict__ cp = block_ptr(P, o0, g, j);
    for (int r = 0; r < g; ++r) {
      const double f = residual(__ldg(al + r), bj, cp[32 * r]);
      if (f > 0.0) acc = dadd(acc, dmul(s, f));
    }
  }
  grad[P.m + j] = dsub(P.b[j], acc);
}

// objective = a.alpha + b.beta - psi_sum (dual.hpp:51) with the reference's
// association, and the slope grad.d, all sequential on one thread.
__global__ void k_exact_objective(DevProblem P, const double* __restrict__ x,
                                  const double* __restrict__ psi, const double* __restrict__ grad,
                                  const double* __restrict__ dvec, EvalScalars* sc,
                                  unsigned long long* cnt_slots) {
  if (cnt_slots && threadIdx.x < 32) fold_counter_slots(cnt_slots, sc);  // screen counters
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double psi_sum = 0.0;
  for (int64_t j = 0; j < P.n; ++j)
    for (int l = 0; l < P.L; ++l) {
      const double v = psi[(int64_t)l * P.n + j];
      if (v != 0.0) psi_sum = dadd(psi_sum, v);
    }
  double da = 0.0, db = 0.0;
  for (int64_t i = 0; i < P.m; ++i) da = dadd(da, dmul(x[i], P.a[i]));
  for (int64_t j = 0; j < P.n; ++j) db = dadd(db, dmul(x[P.m + j], P.b[j]));
  sc->dot_aa = da;
  sc->dot_bb = db;
  sc->psi_sum = psi_sum;
  sc->objective = dsub(dadd(da, db), psi_sum);
  double sl = 0.0;
  if (dvec)
    for (int64_t e = 0; e < P.m + P.n; ++e) sl = dadd(sl, dmul(grad[e], dvec[e]));
  sc->slope = sl;
}

void launch_exact_eval(const DevProblem& P, const double* x, double* scale, double* psi,
                       double* grad, const double* dvec, EvalScalars* sc,
                       unsigned long long* cnt_slots, cudaStream_t s) {
  dim3 g1((unsigned)((P.n + 255) / 256), (unsigned)P.L);
  k_exact_blocks<<<g1, 256, 0, s>>>(P, x, scale, psi);
  k_exact_grad_alpha<<<(unsigned)((P.m + 127) / 128), 128, 0, s>>>(P, x, scale, grad);
  k_exact_grad_beta<<<(unsigned)((P.n + 255) / 256), 256, 0, s>>>(P, x, scale, grad);
  k_exact_objective<<<1, 32, 0, s>>>(P, x, psi, grad, dvec, sc, cnt_slots);
}

// ---------------------------------------------------------------- L-BFGS

__device__ __forceinline__ double seq_dot(const double* __restrict__ a,
                                          const double* __restrict__ b, int64_t n) {
  double acc = 0.0;
  for (int64_t e = 0; e < n; ++e) acc = dadd(acc, dmul(a[e], b[e]));
  return acc;
}

// Two-loop recursion (lbfgs.hpp:109-126) with sequential dots: one CTA,
// thread 0 reduces, all threads do the elementwise updates.
__global__ void __launch_bounds__(256) k_exact_two_loop(const TwoLoopArgs A) {
  __shared__ double sh;
  const HistState& H = *A.h;
  const int k = H.k;
  double* __restrict__ q = A.d;
  double a_loc[kMaxMemory];
  for (int64_t e = threadIdx.x; e < A.dim; e += blockDim.x) q[e] = A.g[e];
  __syncthreads();
  for (int i = k - 1; i >= 0; --i) {
    const double* si = A.S + H.order[i] * A.stride;
    const double* yi = A.Y + H.order[i] * A.stride;
    if (threadIdx.x == 0) sh = dmul(H.rho[i], seq_dot(si, q, A.dim));
    __syncthreads();
    a_loc[i] = sh;
    for (int64_t e = threadIdx.x; e < A.dim; e += blockDim.x) q[e] = dsub(q[e], dmul(a_loc[i], yi[e]));
    __syncthreads();
  }
  if (k > 0 && H.yy[k - 1] > 0.0) {
    const double c = H.sy[k - 1] / H.yy[k - 1];
    for (int64_t e = threadIdx.x; e < A.dim; e += blockDim.x) q[e] = dmul(q[e], c);
    __syncthreads();
  }
  for (int i = 0; i < k; ++i) {
    const double* si = A.S + H.order[i] * A.stride;
    const double* yi = A.Y + H.order[i] * A.stride;
    if (threadIdx.x == 0) sh = dmul(H.rho[i], seq_dot(yi, q, A.dim));
    __syncthreads();
    const double coef = dsub(a_loc[i], sh);
    for (int64_t e = threadIdx.x; e < A.dim; e += blockDim.x) q[e] = dadd(q[e], dmul(coef, si[e]));
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    A.out[0] = seq_dot(A.g, q, A.dim);
    A.out[1] = seq_dot(q, q, A.dim);
  }
}

void launch_exact_two_loop(const TwoLoopArgs& a, cudaStream_t s) {
  k_exact_two_loop<<<1, 256, 0, s>>>(a);
}

// Curvature pair with sequential dots, then the device-side acceptance test
// and ring update (same logic as k_pair).
__global__ void __launch_bounds__(256) k_exact_pair(const double* __restrict__ xt,
                                                    const double* __restrict__ x,
                                                    const double* __restrict__ g,
                                                    const double* __restrict__ gt,
                                                    double* __restrict__ S, double* __restrict__ Y,
                                                    int64_t stride, HistState* h, int64_t dim,
                                                    EvalScalars* sc) {
  const int scratch = h->scratch;
  double* __restrict__ sv = S + scratch * stride;
  double* __restrict__ yv = Y + scratch * stride;
  for (int64_t e = threadIdx.x; e < dim; e += blockDim.x) {
    sv[e] = dsub(xt[e], x[e]);
    yv[e] = dsub(g[e], gt[e]);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double sy = seq_dot(sv, yv, dim), ss = seq_dot(sv, sv, dim), yy = seq_dot(yv, yv, dim);
  sc->extra[0] = sy;
  sc->extra[1] = ss;
  sc->extra[2] = yy;
  h->last_sy = sy;
  h->last_ss = ss;
  h->last_yy = yy;
  const bool accept = sy > 1e-10 * sqrt(ss) * sqrt(yy);
  h->accepted = accept ? 1 : 0;
  if (!accept) return;
  int k = h->k;
  if (k == h->mem) {
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

void launch_exact_pair(const double* xt, const double* x, const double* g, const double* gt,
                       double* S, double* Y, int64_t stride, HistState* h, int64_t dim,
                       EvalScalars* sc, cudaStream_t s) {
  k_exact_pair<<<1, 256, 0, s>>>(xt, x, g, gt, S, Y, stride, h, dim, sc);
}

__global__ void k_exact_dot(const double* __restrict__ a, const double* __restrict__ b,
                            int64_t dim, EvalScalars* sc, int slot) {
  if (threadIdx.x == 0 && blockIdx.x == 0) sc->extra[slot] = seq_dot(a, b, dim);
}

void launch_exact_dot(const double* a, const double* b, int64_t dim, EvalScalars* sc, int slot,
                      cudaStream_t s) {
  k_exact_dot<<<1, 32, 0, s>>>(a, b, dim, sc, slot);
}

}  // namespace gsot
