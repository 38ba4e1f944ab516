// gsot_data.cu — synthetic instances for the five BASELINE.json configs and
// the on-device cost matrix.
//
// RNG: the reference's pinned Rng (data_io.hpp:32-62): std::mt19937_64,
// uniform01 = (x >> 11) * 2^-53, Box-Muller normals with the spare cached,
// index = engine() % bound. Recipe (pinned here and in
// DESIGN.md §6), draws in this order:
//   1. class means mu_l ~ N(0, 4 I_d): means[l][k] = 2 * normal()
//   2. source rows, class-sorted: x = mu_l + sigma * N(0, I)
//   3. target rows t = 0..n-1 from component t / (n/L): same law
//   4. target transform: cfg1 y <- Q y + 0.5 (Q Haar: MGS-QR of a d x d
//      Gaussian, R diagonal positive); cfg3 y <- (I + 0.1/sqrt(d) G) y + t
//   5. Fisher-Yates shuffle of the target rows (data_io.hpp:93-96)
//   6. cfg4 only: a = Dirichlet(1) weights E_i / sum E, E_i = -log U_i.
// Cost: C_ij = sum_k (x_ik - y_jk)^2, k-sequential, no FMA
// (data_io.hpp:112-121), then C /= max C (data_io.hpp:162-165).
#include <math.h>

#include <algorithm>
#include <random>
#include <vector>

#include "gsot_device.cuh"

namespace gsot {

struct ConfigSpec {
  int64_t m, n;
  int32_t L;
  int64_t d;
  double sigma;
  int transform;  // 0 none, 1 rotation + 0.5 shift, 2 random affine
  bool zipf;      // cfg4 Zipf(1.1) group sizes
  bool dirichlet; // cfg4 Dirichlet(1) source weights
};

static bool config_spec(int cfg, ConfigSpec* s) {
  switch (cfg) {
    case 1: *s = {1000, 1000, 10, 64, 1.0, 1, false, false}; return true;
    case 2: *s = {10000, 10000, 100, 128, 1.0, 0, false, false}; return true;
    case 3: *s = {50000, 20000, 1000, 256, 1.0, 2, false, false}; return true;
    case 4: *s = {40000, 30000, 500, 128, 1.0, 0, true, true}; return true;
    case 5: *s = {100000, 50000, 200, 512, 1.5, 0, false, false}; return true;
    default: return false;
  }
}

class Rng {  // data_io.hpp:32-62
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = uniform01();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    spare_ = r * std::sin(angle);
    has_spare_ = true;
    return r * std::cos(angle);
  }
  uint64_t index(uint64_t bound) { return eng_() % bound; }

 private:
  std::mt19937_64 eng_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// Zipf(1.1) sizes: g_k = clamp(round(c k^-1.1), 2, 4000), k = 1..L, with c
// the smallest value (bisection) whose sizes sum to >= m; any overshoot is
// taken from group 1 (the largest unclamped group).
static std::vector<int32_t> zipf_sizes(int32_t L, int64_t m) {
  auto sizes_for = [&](double c, std::vector<int32_t>* out) {
    int64_t tot = 0;
    for (int k = 1; k <= L; ++k) {
      double v = std::round(c * std::pow(static_cast<double>(k), -1.1));
      v = std::min(4000.0, std::max(2.0, v));
      if (out) (*out)[k - 1] = static_cast<int32_t>(v);
      tot += static_cast<int64_t>(v);
    }
    return tot;
  };
  double lo = 1.0, hi = 1e7;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (sizes_for(mid, nullptr) >= m)
      hi = mid;
    else
      lo = mid;
  }
  std::vector<int32_t> s(static_cast<size_t>(L));
  const int64_t tot = sizes_for(hi, &s);
  s[1] -= static_cast<int32_t>(tot - m);
  return s;
}

static double compensated_sum(const std::vector<double>& v) {  // core.hpp:85-98
  double sum = 0.0, comp = 0.0;
  for (double x : v) {
    const double t = sum + x;
    if (std::abs(sum) >= std::abs(x))
      comp += (sum - t) + x;
    else
      comp += (x - t) + sum;
    sum = t;
  }
  return sum + comp;
}

int config_features(int cfg, uint64_t seed, double* src, double* tgt, int32_t* sizes_out,
                    double* a, double* b) {
  ConfigSpec sp;
  if (!config_spec(cfg, &sp)) throw Error(GSOT_ERR_INVALID_ARGUMENT, "unknown config");
  const int64_t m = sp.m, n = sp.n, d = sp.d;
  const int32_t L = sp.L;
  std::vector<int32_t> sizes;
  if (sp.zipf)
    sizes = zipf_sizes(L, m);
  else
    sizes.assign(static_cast<size_t>(L), static_cast<int32_t>(m / L));
  Rng rng(seed);
  std::vector<double> means(static_cast<size_t>(L * d));
  for (auto& v : means) v = 2.0 * rng.normal();
  int64_t row = 0;
  for (int32_t l = 0; l < L; ++l)
    for (int32_t r = 0; r < sizes[static_cast<size_t>(l)]; ++r, ++row)
      for (int64_t k = 0; k < d; ++k) src[row * d + k] = means[l * d + k] + sp.sigma * rng.normal();
  const int64_t per = n / L;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t comp = t / per;
    for (int64_t k = 0; k < d; ++k) tgt[t * d + k] = means[comp * d + k] + sp.sigma * rng.normal();
  }
  if (sp.transform != 0) {
    std::vector<double> G(static_cast<size_t>(d * d));
    for (auto& v : G) v = rng.normal();
    std::vector<double> A(static_cast<size_t>(d * d));
    std::vector<double> shift(static_cast<size_t>(d), 0.5);
    if (sp.transform == 1) {
      // Modified Gram-Schmidt on the columns of G -> Q with positive R diag.
      std::vector<double> Q(G);
      for (int64_t c = 0; c < d; ++c) {
        for (int64_t p = 0; p < c; ++p) {
          double dot = 0.0;
          for (int64_t r = 0; r < d; ++r) dot += Q[r * d + p] * Q[r * d + c];
          for (int64_t r = 0; r < d; ++r) Q[r * d + c] -= dot * Q[r * d + p];
        }
        double nrm = 0.0;
        for (int64_t r = 0; r < d; ++r) nrm += Q[r * d + c] * Q[r * d + c];
        nrm = std::sqrt(nrm);
        for (int64_t r = 0; r < d; ++r) Q[r * d + c] /= nrm;
      }
      A = Q;
    } else {
      const double sc = 0.1 / std::sqrt(static_cast<double>(d));
      for (int64_t r = 0; r < d; ++r)
        for (int64_t c = 0; c < d; ++c) A[r * d + c] = (r == c ? 1.0 : 0.0) + sc * G[r * d + c];
      for (auto& v : shift) v = rng.normal();
    }
    std::vector<double> y(static_cast<size_t>(d));
    for (int64_t t = 0; t < n; ++t) {
      for (int64_t r = 0; r < d; ++r) {
        double acc = 0.0;
        for (int64_t c = 0; c < d; ++c) acc += A[r * d + c] * tgt[t * d + c];
        y[static_cast<size_t>(r)] = acc + shift[static_cast<size_t>(r)];
      }
      std::copy(y.begin(), y.end(), tgt + t * d);
    }
  }
  for (int64_t i = n - 1; i > 0; --i) {  // data_io.hpp:93-96
    const int64_t j = static_cast<int64_t>(rng.index(static_cast<uint64_t>(i) + 1));
    if (i != j)
      for (int64_t k = 0; k < d; ++k) std::swap(tgt[i * d + k], tgt[j * d + k]);
  }
  if (sp.dirichlet) {
    std::vector<double> e(static_cast<size_t>(m));
    for (auto& v : e) {
      double u = rng.uniform01();
      if (u <= 0.0) u = 0x1.0p-53;
      v = -std::log(u);
    }
    const double s = compensated_sum(e);
    for (int64_t i = 0; i < m; ++i) a[i] = e[static_cast<size_t>(i)] / s;
  } else {
    for (int64_t i = 0; i < m; ++i) a[i] = 1.0 / static_cast<double>(m);
  }
  for (int64_t j = 0; j < n; ++j) b[j] = 1.0 / static_cast<double>(n);
  std::copy(sizes.begin(), sizes.end(), sizes_out);
  return 0;
}

int config_shape(int cfg, int64_t* m, int64_t* n, int32_t* L, int64_t* d) {
  ConfigSpec sp;
  if (!config_spec(cfg, &sp)) throw Error(GSOT_ERR_INVALID_ARGUMENT, "unknown config");
  if (m) *m = sp.m;
  if (n) *n = sp.n;
  if (L) *L = sp.L;
  if (d) *d = sp.d;
  return 0;
}

// ---------------------------------------------------------------- cost matrix
// 64 x 64 output tile per CTA, 16-wide k slabs in shared memory, 4 x 4
// outputs per thread, each a k-sequential sum of rounded squares. fp64 SIMT:
// the recurrence c += (x - y)^2 with one rounding per operation is not a
// contraction the tensor cores can reproduce bit-for-bit.
constexpr int kTile = 64;
constexpr int kSlab = 16;

__global__ void __launch_bounds__(256) k_cost(const double* __restrict__ src, int64_t m,
                                              const double* __restrict__ tgt, int64_t n,
                                              int64_t d, DevProblem T, bool tiled,
                                              double* __restrict__ out) {
  __shared__ double xs[kSlab][kTile + 1];
  __shared__ double ys[kSlab][kTile + 1];
  // tx walks columns (coalesced tiled writes), ty rows
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = blockIdx.x * (int64_t)kTile, j0 = blockIdx.y * (int64_t)kTile;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t k0 = 0; k0 < d; k0 += kSlab) {
    for (int e = threadIdx.x; e < kSlab * kTile; e += 256) {
      const int rr = e / kSlab, kk = e % kSlab;
      const int64_t i = i0 + rr, j = j0 + rr, k = k0 + kk;
      xs[kk][rr] = (i < m && k < d) ? src[i * d + k] : 0.0;
      ys[kk][rr] = (j < n && k < d) ? tgt[j * d + k] : 0.0;
    }
    __syncthreads();
    const int kmax = (d - k0) < kSlab ? (int)(d - k0) : kSlab;
    for (int kk = 0; kk < kmax; ++kk) {
      double xv[4], yv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xv[a] = xs[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) yv[b] = ys[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double diff = __dsub_rn(xv[a], yv[b]);
          acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(diff, diff));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t i = i0 + ty + 16 * a;
    if (i >= m) continue;
    int o0 = 0, g = 0;
    if (tiled) {
      const int l = T.row_group[i];
      o0 = T.off[l];
      g = T.off[l + 1] - o0;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t j = j0 + tx + 16 * b;
      if (j >= n) continue;
      if (tiled)
        out[cost_index(T.nw, o0, g, j, i - o0)] = acc[a][b];
      else
        out[j * m + i] = acc[a][b];
    }
  }
}

void launch_cost_matrix(const double* src, int64_t m, const double* tgt, int64_t n, int64_t d,
                        const DevProblem* tiled, double* out, cudaStream_t s) {
  dim3 grid((unsigned)((m + kTile - 1) / kTile), (unsigned)((n + kTile - 1) / kTile));
  DevProblem T{};
  if (tiled) T = *tiled;
  k_cost<<<grid, 256, 0, s>>>(src, m, tgt, n, d, T, tiled != nullptr, out);
}

__global__ void __launch_bounds__(256) k_max(const double* __restrict__ C, int64_t count,
                                             double* __restrict__ partials, double* out,
                                             unsigned int* ticket) {
  double v[1] = {0.0};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    v[0] = fmax(v[0], C[e]);
  double r[1];
  if (last_block_reduce<256, 1>(v, partials, ticket, r, true)) *out = r[0];
}

void launch_max_reduce(const double* C, int64_t count, double* partials, int nblocks, double* out,
                       unsigned int* ticket, cudaStream_t s) {
  k_max<<<nblocks, 256, 0, s>>>(C, count, partials, out, ticket);
}

__global__ void k_scale_div(double* __restrict__ C, int64_t count, const double* __restrict__ div) {
  const double dv = *div;
  if (!(dv > 0.0)) return;  // data_io.hpp:164: only when max > 0
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    C[e] = __ddiv_rn(C[e], dv);
}

// validate_instance's cost scan (core.hpp:118-123) over the column-tiled
// layout: the first entry in j-major order with !(c >= 0) || !isfinite(c),
// as min(j * m + i) into *first_bad. Thread per (row, chunk): 32 columns.
__global__ void __launch_bounds__(256) k_scan_bad(DevProblem P, unsigned long long* first_bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= P.m) return;
  const int l = P.row_group[i];
  const int o0 = P.off[l], g = P.off[l + 1] - o0;
  unsigned long long bad = ~0ull;
  for (int k = 0; k < 32; ++k) {
    const int64_t j = (int64_t)c * 32 + k;
    if (j >= P.n) break;
    const double v = P.C[cost_index(P.nw, o0, g, j, i - o0)];
    if (!(v >= 0.0) || !isfinite(v)) {
      bad = (unsigned long long)(j * P.m + i);
      break;
    }
  }
  if (bad != ~0ull) atomicMin(first_bad, bad);
}

void launch_scan_bad(const DevProblem& P, unsigned long long* first_bad, cudaStream_t s) {
  dim3 grid((unsigned)((P.m + 255) / 256), (unsigned)P.nw);
  k_scan_bad<<<grid, 256, 0, s>>>(P, first_bad);
}

void launch_scale_div(double* C, int64_t count, const double* div, cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 32);
  k_scale_div<<<grid, 256, 0, s>>>(C, count, div);
}

}  // namespace gsot
