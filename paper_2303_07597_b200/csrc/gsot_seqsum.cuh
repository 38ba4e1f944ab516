// gsot_seqsum.cuh — the reference's SEQUENTIAL floating-point sums, computed
// in parallel and bit for bit (exact-order mode).
//
// The reference accumulates every reduction left to right (`acc += v[i]`,
// Eigen's dot / sum / squaredNorm in the oracle's sequential build,
// regularizer.hpp:23-51, dual.hpp:44-51, lbfgs.hpp:109-132). A sequential
// sum of N terms is N dependent roundings; this header reproduces its exact
// result with O(N / P) + O(P) dependent steps:
//
//  A. approximate start of each of P segments: s^_p = s0 + (any-order sum of
//     the earlier segments' terms);
//  B. speculation, one thread per segment: run the segment's chain from s^_p
//     (run 0) and from s^_p +- ulp (run 1, the other mantissa parity) while
//     the run-0 value stays in one binade [2^E, 2^(E+1)) of one sign. Such a
//     stretch is a "piece": its effect on ANY true start s in the same binade
//     is the translation s -> s + (run end - run start), provided
//       * s - s^ is a multiple of 2u (u = 2^(E-52)) -- the run of the same
//         mantissa parity is used, so the shift between it and s is even;
//       * every exact intermediate sum of the true path stays inside the
//         binade: the run's partial sums, shifted by the same amount, keep a
//         2u margin from both binade bounds (the piece's [lo, hi] range).
//     Then both paths round on the same grid with the same ties-to-even
//     decisions, so they differ by the same shift at every step. A run-0
//     step that leaves the binade (a "crossing") ends the piece; that one
//     term is applied serially in C and a new piece starts after it.
//  C. stitch, one thread: s = s0; for each piece, apply its serial terms,
//     then s += d_parity(s) if s lies in the piece's range, otherwise replay
//     the piece's terms one by one (the reference's own steps).
//
// Every step of C is either the reference's own addition or an exact
// translation, so the result is the sequential sum for any input (the
// fallbacks only cost time). Pinned against sequential sums of adversarial
// inputs (ties, zeros, cancellation, subnormal starts) in
// tests/test_gpu_exact.py and by the bitwise exact-mode solves.
#pragma once

#include <cooperative_groups.h>

#include "gsot_device.cuh"

namespace gsot {
namespace seq {

constexpr int kMaxPieces = 8;   // pieces per segment; later terms are serial in C
constexpr int kWin = 256;       // terms staged in shared memory per warp and window
constexpr int kClusterCtas = 8; // CTAs of the exact-mode cluster kernels
constexpr int kThreads = 512;   // threads per CTA of those kernels
constexpr int kMaxSegs = 512;   // segments per chain (one per thread in the scan)
constexpr int kMaxChains = 4;

struct Piece {
  double s0;                  // run-0 start (the speculative start)
  double d0, d1;              // run end - run start, runs 0 and 1
  double lo0, hi0, lo1, hi1;  // |s| ranges in which each run's translation is exact
  double xpre;                // the serial term right before k0 when npre == 1
  int k0, k1;                 // terms [k0, k1) of the segment
  int npre;                   // serial terms between the previous piece and k0
  int pad;
};

__device__ __forceinline__ unsigned dkey(double s) {  // sign + biased exponent
  return static_cast<unsigned>(static_cast<unsigned long long>(__double_as_longlong(s)) >> 52);
}

// Segment length for a chain of `len` terms: about 2 sqrt(len) (balances the
// speculative runs of B against the pieces of C), at least 128, and at most
// kMaxSegs segments.
__host__ __device__ __forceinline__ int seg_len(int64_t len) {
  int64_t b = 128;
  while (b * b < 4 * len) b += 64;
  while ((len + b - 1) / b > kMaxSegs) b *= 2;
  return static_cast<int>(b);
}

// The speculative run of one segment (one thread).
struct Spec {
  double s;                        // speculative value (run 0 between pieces)
  double st0, st1, t0, t1;         // open piece: run starts and values
  double mn0, mx0, mn1, mx1;       // min / max |value| of each run
  double lowb, highb, u;           // binade bounds of the open piece
  double xpre;
  unsigned key;
  int k0, np, npre;
  bool open, ok1, full;
  Piece* out;

  __device__ void init(double shat, Piece* o) {
    s = shat;
    open = false;
    full = false;
    np = 0;
    npre = 0;
    xpre = 0.0;
    out = o;
  }
  __device__ void serial(double x) {
    if (npre == 0) xpre = x;
    ++npre;
  }
  __device__ bool try_open(int k) {
    const unsigned kk = dkey(s), ex = kk & 0x7ffu;
    if (ex <= 54u || ex >= 0x7feu) return false;  // zero, tiny or huge: serial term
    key = kk;
    lowb = __longlong_as_double(static_cast<long long>(ex) << 52);
    highb = __longlong_as_double(static_cast<long long>(ex + 1) << 52);
    u = __longlong_as_double(static_cast<long long>(ex - 52) << 52);
    const double a0 = fabs(s);
    const double up = dadd(a0, u);
    const double a1 = up < highb ? up : dsub(a0, u);
    st0 = s;
    st1 = s < 0.0 ? -a1 : a1;
    t0 = st0;
    t1 = st1;
    mn0 = mx0 = a0;
    mn1 = mx1 = a1;
    ok1 = true;
    k0 = k;
    open = true;
    return true;
  }
  __device__ void close(int k1) {
    Piece p;
    p.s0 = st0;
    p.d0 = dsub(t0, st0);
    p.d1 = dsub(t1, st1);
    const double u2 = dadd(u, u);
    const double a0 = fabs(st0), a1 = fabs(st1);
    const double m0l = dsub(mn0, lowb), m0h = dsub(highb, mx0);
    const double m1l = dsub(mn1, lowb), m1h = dsub(highb, mx1);
    const bool v0 = m0l >= u2 && m0h >= u2;
    const bool v1 = ok1 && m1l >= u2 && m1h >= u2;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    p.lo0 = v0 ? dadd(dsub(a0, m0l), u2) : inf;
    p.hi0 = v0 ? dsub(dadd(a0, m0h), u2) : -inf;
    p.lo1 = v1 ? dadd(dsub(a1, m1l), u2) : inf;
    p.hi1 = v1 ? dsub(dadd(a1, m1h), u2) : -inf;
    p.xpre = xpre;
    p.k0 = k0;
    p.k1 = k1;
    p.npre = npre;
    p.pad = 0;
    out[np++] = p;
    open = false;
    npre = 0;
    s = t0;
    if (np == kMaxPieces) full = true;
  }
  // One term, with the run state advanced in place.
  __device__ __forceinline__ void step(double x, int k) {
    if (full) return;
    if (!open && !try_open(k)) {
      s = dadd(s, x);
      serial(x);
      return;
    }
    const double n0 = dadd(t0, x);
    if (dkey(n0) != key) {  // crossing: the piece ends, this term is serial
      close(k);
      s = n0;
      serial(x);
      return;
    }
    const double n1 = dadd(t1, x);
    ok1 = ok1 && dkey(n1) == key;
    t0 = n0;
    t1 = n1;
    const double b0 = fabs(n0), b1 = fabs(n1);
    mn0 = fmin(mn0, b0);
    mx0 = fmax(mx0, b0);
    mn1 = fmin(mn1, b1);
    mx1 = fmax(mx1, b1);
  }
  // Four terms: the common no-crossing case runs the two chains without a
  // branch per term; a block with a crossing (or no open piece) is replayed
  // term by term.
  __device__ __forceinline__ void step4(const double* x, int k) {
    if (full) return;
    if (open) {
      double a = t0, b = t1;
      double q0[4], q1[4];
      bool same = true;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a = dadd(a, x[i]);
        b = dadd(b, x[i]);
        q0[i] = a;
        q1[i] = b;
        same = same && dkey(a) == key;
      }
      if (same) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ok1 = ok1 && dkey(q1[i]) == key;
          const double b0 = fabs(q0[i]), b1 = fabs(q1[i]);
          mn0 = fmin(mn0, b0);
          mx0 = fmax(mx0, b0);
          mn1 = fmin(mn1, b1);
          mx1 = fmax(mx1, b1);
        }
        t0 = a;
        t1 = b;
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) step(x[i], k + i);
  }
  __device__ int finish(int len) {
    if (open && !full) close(len);
    return np;
  }
};

// Phase B for one segment by one warp: the segment's terms staged through
// shared memory (`win`, kWin doubles), lane 0 runs the speculation.
__device__ __forceinline__ void spec_segment_warp(const double* __restrict__ v, int len,
                                                  double shat, Piece* __restrict__ out,
                                                  int* __restrict__ np_out, double* win) {
  const int lane = threadIdx.x & 31;
  Spec sp;
  if (lane == 0) sp.init(shat, out);
  for (int w0 = 0; w0 < len; w0 += kWin) {
    const int wl = min(kWin, len - w0);
    __syncwarp();
    for (int i = lane; i < wl; i += 32) win[i] = __ldcg(v + w0 + i);
    __syncwarp();
    if (lane == 0) {
      int i = 0;
      for (; i + 4 <= wl; i += 4) sp.step4(win + i, w0 + i);
      for (; i < wl; ++i) sp.step(win[i], w0 + i);
    }
  }
  if (lane == 0) *np_out = sp.finish(len);
  __syncwarp();
}

// A piece written by another CTA of the cluster (through L2).
__device__ __forceinline__ Piece load_piece(const Piece* q) {
  const double2* d = reinterpret_cast<const double2*>(q);
  const double2 a = __ldcg(d), b = __ldcg(d + 1), c = __ldcg(d + 2), e = __ldcg(d + 3);
  const int4 k = __ldcg(reinterpret_cast<const int4*>(d + 4));
  Piece p;
  p.s0 = a.x;
  p.d0 = a.y;
  p.d1 = b.x;
  p.lo0 = b.y;
  p.hi0 = c.x;
  p.lo1 = c.y;
  p.hi1 = e.x;
  p.xpre = e.y;
  p.k0 = k.x;
  p.k1 = k.y;
  p.npre = k.z;
  p.pad = 0;
  return p;
}

// Phase C for one segment: the exact sequential sum continued from s.
__device__ __forceinline__ double stitch_segment(double s, const double* __restrict__ v, int len,
                                                 const Piece* __restrict__ pcs, int np) {
  int k = 0;
  for (int i = 0; i < np; ++i) {
    const Piece p = load_piece(pcs + i);
    if (p.npre == 1)
      s = dadd(s, p.xpre);
    else
      for (; k < p.k0; ++k) s = dadd(s, __ldcg(v + k));
    const long long bs = __double_as_longlong(s), b0 = __double_as_longlong(p.s0);
    bool done = false;
    if (((bs ^ b0) >> 52) == 0) {  // same sign and binade as the run start
      const bool odd = ((bs ^ b0) & 1) != 0;  // parity of the shift in ulps
      const double as = fabs(s);
      const double lo = odd ? p.lo1 : p.lo0, hi = odd ? p.hi1 : p.hi0;
      if (as >= lo && as <= hi) {
        s = dadd(s, odd ? p.d1 : p.d0);  // exact: the result is the true path's value
        done = true;
      }
    }
    if (!done)
      for (int kk = p.k0; kk < p.k1; ++kk) s = dadd(s, __ldcg(v + kk));
    k = p.k1;
  }
  for (; k < len; ++k) s = dadd(s, __ldcg(v + k));
  return s;
}

// One chain of the engine: `terms` materialised (len doubles), start s_init.
struct Chain {
  const double* terms;
  int64_t len;
  double s_init;
  int B, P;
};

// Per-chain scratch in global memory (kMaxChains x kMaxSegs).
struct Scratch {
  double* segsum;  // [chain][seg]
  Piece* pieces;   // [chain][seg][kMaxPieces]
  int* np;         // [chain][seg]
};

// Warp-level Phase A: segment sums (any order) of segment `p` of chain `c`.
__device__ __forceinline__ double warp_seg_sum(const double* __restrict__ v, int64_t b, int64_t e) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int64_t i = b + lane; i < e; i += 32) acc += __ldcg(v + i);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Shared-memory layout of the engine inside a cluster kernel.
struct EngineSmem {
  double shat[kMaxChains][kMaxSegs];
  double win[kThreads / 32][kWin];
  double res[kMaxChains];
  double wsum[kThreads / 32];
};

// The engine, called by EVERY thread of EVERY CTA of the cluster after the
// chains' terms are written (and visible cluster-wide): phase A (segment
// sums), cluster barrier, the approximate starts (each CTA for itself),
// phase B (one warp per segment over the whole cluster), cluster barrier,
// phase C (every CTA stitches every chain: warp c, lane 0, so no barrier is
// needed afterwards). Results in sm.res[c] after a __syncthreads.
__device__ __forceinline__ void engine(const Chain* ch, int nch, const Scratch& sc, EngineSmem& sm) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int cta = static_cast<int>(cl.block_rank()), ncta = static_cast<int>(cl.num_blocks());
  const int gw = cta * nwarps + warp, gnw = ncta * nwarps;
  // A: segment sums
  int total = 0;
  for (int c = 0; c < nch; ++c) total += ch[c].P;
  for (int job = gw; job < total; job += gnw) {
    int c = 0, p = job;
    while (p >= ch[c].P) p -= ch[c++].P;
    const int64_t b = static_cast<int64_t>(p) * ch[c].B;
    const int64_t e = min(ch[c].len, b + ch[c].B);
    const double s = warp_seg_sum(ch[c].terms, b, e);
    if (lane == 0) sc.segsum[c * kMaxSegs + p] = s;
  }
  cl.sync();
  // approximate starts: exclusive prefix of the segment sums (per CTA)
  for (int c = 0; c < nch; ++c) {
    const int P = ch[c].P;
    double v = threadIdx.x < P ? __ldcg(sc.segsum + c * kMaxSegs + threadIdx.x) : 0.0;
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) sm.wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      double w = lane < nwarps ? sm.wsum[lane] : 0.0;
      double wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < nwarps) sm.wsum[lane] = wi - w;  // exclusive prefix of the warp totals
    }
    __syncthreads();
    if (threadIdx.x < P) sm.shat[c][threadIdx.x] = ch[c].s_init + (sm.wsum[warp] + (incl - v));
    __syncthreads();
  }
  if (threadIdx.x < nch) sm.shat[threadIdx.x][0] = ch[threadIdx.x].s_init;  // exact start
  __syncthreads();
  // B: speculative runs, one warp per segment
  for (int job = gw; job < total; job += gnw) {
    int c = 0, p = job;
    while (p >= ch[c].P) p -= ch[c++].P;
    const int64_t b = static_cast<int64_t>(p) * ch[c].B;
    const int len = static_cast<int>(min(ch[c].len - b, static_cast<int64_t>(ch[c].B)));
    spec_segment_warp(ch[c].terms + b, len, sm.shat[c][p],
                      sc.pieces + (static_cast<int64_t>(c) * kMaxSegs + p) * kMaxPieces,
                      sc.np + c * kMaxSegs + p, sm.win[warp]);
  }
  cl.sync();
  // C: stitch (every CTA, warp c, lane 0)
  if (warp < nch && lane == 0) {
    const Chain& C = ch[warp];
    double s = C.s_init;
    for (int p = 0; p < C.P; ++p) {
      const int64_t b = static_cast<int64_t>(p) * C.B;
      const int len = static_cast<int>(min(C.len - b, static_cast<int64_t>(C.B)));
      s = stitch_segment(s, C.terms + b, len,
                         sc.pieces + (static_cast<int64_t>(warp) * kMaxSegs + p) * kMaxPieces,
                         __ldcg(sc.np + warp * kMaxSegs + p));
    }
    sm.res[warp] = s;
  }
  __syncthreads();
}

__host__ __device__ __forceinline__ Chain make_chain(const double* terms, int64_t len, double s0) {
  Chain c;
  c.terms = terms;
  c.len = len;
  c.s_init = s0;
  c.B = seg_len(len);
  c.P = static_cast<int>((len + c.B - 1) / c.B);
  return c;
}

}  // namespace seq
}  // namespace gsot
