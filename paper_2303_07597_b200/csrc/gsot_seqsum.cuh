// gsot_seqsum.cuh — the reference's SEQUENTIAL floating-point sums, computed
// in parallel and bit for bit (exact-order mode).
//
// The reference accumulates every reduction left to right (`acc += v[i]`,
// Eigen's dot / sum / squaredNorm in the oracle's sequential build,
// regularizer.hpp:23-51, dual.hpp:44-51, lbfgs.hpp:109-132). A sequential sum
// of N terms is N dependent roundings (~14 cycles each on B200); this header
// reproduces its exact result with short dependent chains.
//
// Translation invariance. Let a "run" be the sequential sum of a stretch of
// terms from some start t. If a true start s differs from t by delta, a
// multiple of 2 ulp(t), and at every step both paths' exact sums stay in the
// same binade (same sign, |x| in [2^E, 2^(E+1))), E never above the start
// binade, then both paths round on grids that delta is a multiple of, with
// the same ties-to-even decisions: the true path is the run shifted by delta
// and its end is run_end + delta (exact). Runs start from t and t +- ulp
// (both mantissa parities), so one of them is always an even shift away; a
// run records the shifts of |s| that keep every step 2 ulp(t) inside its
// binade (`dlo`, `dhi`). A step that leaves the allowed binades (upwards, a
// sign change, a tiny value) ends the run; that term is applied serially.
//
//  A. segment sums in any order -> approximate start s^_p of each segment;
//  B. one warp per segment: each lane runs a 1/32 sub-range speculatively
//     from its own approximate start (a warp scan of the lane sub-sums), then
//     lane 0 chains the lanes' runs into the segment's "pieces": a run is
//     continued into the next one when its end lies in the next one's valid
//     shift range (the continued path is again a concrete run of the terms),
//     O(1) per lane instead of one dependent add per term;
//  C. stitch: s = s0, then per piece its serial terms and the translation of
//     the true value when it lies in the piece's range, else the reference's
//     own additions over the piece's terms.
//
// Every step of C is either the reference's own addition or an exact
// translation, so the result is the sequential sum for any input (fallbacks
// only cost time). Pinned against sequential sums of adversarial inputs
// (ties, zeros, cancellation, subnormals) in tests/test_gpu_exact.py and by
// the bitwise exact-mode solves.
#pragma once

#include <cooperative_groups.h>

#include "gsot_device.cuh"

namespace gsot {
namespace seq {

// Diagnostic phase clocks (builds with -DGSOT_SEQ_PROF only): cycles of CTA 0
// in each engine phase, summed over calls; read by gsot_debug_seq_prof.
#ifdef GSOT_SEQ_PROF
__device__ unsigned long long g_seq_prof[16];
#define SEQ_PROF_T(v) unsigned long long v = clock64()
#define SEQ_PROF_ADD(slot, a, b)                                                    \
  do {                                                                              \
    if (threadIdx.x == 0 && cooperative_groups::this_cluster().block_rank() == 0) \
      atomicAdd(&g_seq_prof[slot], (b) - (a));                                      \
  } while (0)
#define SEQ_CNT(slot, v) atomicAdd(&g_seq_prof[slot], (unsigned long long)(v))
#else
#define SEQ_PROF_T(v) \
  do {                \
  } while (0)
#define SEQ_PROF_ADD(slot, a, b) \
  do {                           \
  } while (0)
#define SEQ_CNT(slot, v) \
  do {                   \
  } while (0)
#endif

constexpr int kMaxPieces = 64;  // pieces per segment (later terms: serial)
constexpr int kMaxGPieces = 256; // pieces per group of segments (later terms: serial)
constexpr int kLanePieces = 4;  // runs per lane sub-range in B (later terms: serial)
constexpr int kClusterCtas = 8; // CTAs of the exact-mode cluster kernels
constexpr int kThreads = 256;   // threads per CTA of those kernels
constexpr int kMaxSegs = 512;   // segments per chain
constexpr int kMaxChains = 4;
constexpr int kStage = 4096;    // terms of a segment staged in shared memory (phase B)
constexpr int kBWarps = 4;      // warps per CTA running phases B and C1
constexpr int kGroup = 4;       // segments chained per warp in phase C1
constexpr int kMaxGroups = kMaxSegs / kGroup;

// A run (or a chain of runs) over terms [k0, k1) of a segment.
struct alignas(16) Piece {
  double st[2];           // starts of the two parity runs (st[0]: the speculative start)
  double en[2];           // their ends
  double dlo[2], dhi[2];  // allowed shift of |s| from |st[r]| (empty when dlo > dhi)
  double xpre;            // the nonzero serial term before k0 when npre == 1
  int k0, k1;
  int npre;               // nonzero serial terms between the previous piece and k0
  int pad;
};

__device__ __forceinline__ long long dbits(double s) { return __double_as_longlong(s); }
__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000ll); }

// Segment length for a chain of `len` terms: about len / 64 (multiple of 64,
// at least 256), staged whole in shared memory up to kStage terms; longer
// only when len > kMaxSegs * kStage (then read from L2).
__host__ __device__ __forceinline__ int seg_len(int64_t len) {
  int64_t b = ((len + 63) / 64 + 63) / 64 * 64;
  if (b < 256) b = 256;
  if (b > kStage) b = kStage;
  while ((len + b - 1) / b > kMaxSegs) b *= 2;
  return static_cast<int>(b);
}

// The true value s through piece p when it lies in p's range.
__device__ __forceinline__ bool try_apply(double& s, const Piece& p) {
  const long long bs = dbits(s), b0 = dbits(p.st[0]);
  if (((bs ^ b0) >> 52) != 0) return false;  // not the start binade
  const bool odd = ((bs ^ b0) & 1) != 0;  // the run of s's mantissa parity
  const double delta = dsub(s, odd ? p.st[1] : p.st[0]);  // exact, an even number of ulps
  const double sh = s < 0.0 ? -delta : delta;
  if (!(sh >= (odd ? p.dlo[1] : p.dlo[0]) && sh <= (odd ? p.dhi[1] : p.dhi[0]))) return false;
  s = dadd(odd ? p.en[1] : p.en[0], delta);  // exact: the true path's value
  return true;
}

// One lane's speculative runs over its sub-range (terms streamed in order).
struct LaneSpec {
  double s;                   // speculative value between runs
  double st0, st1, t0, t1;    // open run
  double lo0, hi0, lo1, hi1;  // min distance to the lower / upper bound of the current binade
  double u2;                  // 2 ulp of the run start
  long long bst;              // bits of the run start
  double xpre;
  int k0, np, npre;
  bool open, ok1, full;
  Piece* out;                 // kLanePieces slots

  __device__ void init(double shat, Piece* o) {
    s = shat;
    open = full = false;
    np = npre = 0;
    xpre = 0.0;
    out = o;
  }
  __device__ __forceinline__ void serial(double x) {
    if (npre == 0) xpre = x;
    ++npre;
  }
  // a run value may move to any binade of the start's sign between the
  // start binade and 2^-968 (downwards the grids get finer)
  __device__ __forceinline__ bool inside(double v) const {
    const long long b = dbits(v);
    const int ex = static_cast<int>((b >> 52) & 0x7ff);
    return ((b ^ bst) >= 0) && ex > 54 && ex <= static_cast<int>((bst >> 52) & 0x7ff);
  }
  __device__ __forceinline__ static void margins(double v, double& lo, double& hi) {
    const double a = fabs(v);
    const double lb = __longlong_as_double(dbits(a) & 0x7ff0000000000000ll);
    lo = fmin(lo, dsub(a, lb));            // exact: same binade
    hi = fmin(hi, dsub(dadd(lb, lb), a));  // exact
  }
  __device__ bool try_open(int k) {
    const int ex = static_cast<int>((dbits(s) >> 52) & 0x7ff);
    if (ex <= 54 || ex >= 0x7fe) return false;  // zero, tiny or huge: serial term
    bst = dbits(s);
    const double u = __longlong_as_double(static_cast<long long>(ex - 52) << 52);
    u2 = dadd(u, u);
    const double a0 = fabs(s);
    const double highb = __longlong_as_double(static_cast<long long>(ex + 1) << 52);
    const double up = dadd(a0, u);
    const double a1 = up < highb ? up : dsub(a0, u);
    st0 = s;
    st1 = s < 0.0 ? -a1 : a1;
    t0 = st0;
    t1 = st1;
    lo0 = hi0 = lo1 = hi1 = dinf();
    margins(t0, lo0, hi0);
    margins(t1, lo1, hi1);
    ok1 = true;
    k0 = k;
    open = true;
    return true;
  }
  __device__ void close(int k1) {
    Piece& p = out[np++];
    p.st[0] = st0;
    p.st[1] = st1;
    p.en[0] = t0;
    p.en[1] = t1;
    const double inf = dinf();
    const bool v0 = lo0 >= u2 && hi0 >= u2;
    const bool v1 = ok1 && lo1 >= u2 && hi1 >= u2;
    p.dlo[0] = v0 ? dsub(u2, lo0) : inf;
    p.dhi[0] = v0 ? dsub(hi0, u2) : -inf;
    p.dlo[1] = v1 ? dsub(u2, lo1) : inf;
    p.dhi[1] = v1 ? dsub(hi1, u2) : -inf;
    p.xpre = xpre;
    p.k0 = k0;
    p.k1 = k1;
    p.npre = npre;
    p.pad = 0;
    open = false;
    npre = 0;
    s = t0;
    if (np == kLanePieces) full = true;
  }
  __device__ __forceinline__ void step(double x, int k) {
    // +-0 terms leave every partial sum unchanged (the sums are never -0
    // under round-to-nearest), for the true path as for the runs
    if (full || x == 0.0) return;
    if (!open && !try_open(k)) {
      s = dadd(s, x);
      serial(x);
      return;
    }
    const double n0 = dadd(t0, x);
    if (!inside(n0)) {  // the run ends; this term is serial
      close(k);
      s = n0;
      serial(x);
      return;
    }
    const double n1 = dadd(t1, x);
    ok1 = ok1 && inside(n1);
    t0 = n0;
    t1 = n1;
    margins(n0, lo0, hi0);
    margins(n1, lo1, hi1);
  }
  __device__ int finish(int len) {
    if (open && !full) close(len);
    return np;
  }
};

// Continue `cur` (a piece ending where `nx` starts, no serial term between):
// per parity run of cur whose end lies in nx's range for the matching parity,
// the continued run is concrete (its end is nx's end shifted, exact) and its
// shift range narrows. cur is updated only when at least one parity run
// continues (returns true); otherwise it is left as it was.
__device__ __forceinline__ bool chain_piece(Piece& cur, const Piece& nx) {
  const long long bn0 = dbits(nx.st[0]);
  double en[2], lo[2], hi[2];
  bool any = false;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    en[r] = cur.en[r];
    lo[r] = dinf();
    hi[r] = -dinf();
    if (!(cur.dlo[r] <= cur.dhi[r])) continue;
    const double e = cur.en[r];
    const long long be = dbits(e);
    if (((be ^ bn0) >> 52) != 0) continue;  // not nx's start binade
    const bool odd = ((be ^ bn0) & 1) != 0;
    const double nst = odd ? nx.st[1] : nx.st[0];
    const double nen = odd ? nx.en[1] : nx.en[0];
    const double nlo = odd ? nx.dlo[1] : nx.dlo[0];
    const double nhi = odd ? nx.dhi[1] : nx.dhi[0];
    const double c = dsub(e, nst);  // exact
    const double C = e < 0.0 ? -c : c;
    if (!(C >= nlo && C <= nhi)) continue;
    const double l = fmax(cur.dlo[r], __dsub_ru(nlo, C));
    const double h = fmin(cur.dhi[r], __dsub_rd(nhi, C));
    if (!(l <= h)) continue;
    en[r] = dadd(nen, c);  // exact: the run continued through nx's terms
    lo[r] = l;
    hi[r] = h;
    any = true;
  }
  if (any) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      cur.en[r] = en[r];
      cur.dlo[r] = lo[r];
      cur.dhi[r] = hi[r];
    }
    cur.k1 = nx.k1;
  }
  return any;
}

// Chain a list of units (the lanes of a segment in phase B, the segments of a
// group in phase C1): each unit has `np` pieces (k relative to the list) and
// `tail` nonzero serial terms after them (tail >= 2: unknown, replay; the one
// value in tailx when 1). Consecutive pieces with no serial term between are
// continued (chain_piece). One thread. Writes the list's pieces to out and
// returns their count; the list's own tail in *tail / *tailx.
template <typename Unit>
__device__ __forceinline__ int compose(int nunits, Unit unit, Piece* __restrict__ out, int cap,
                                       int* tail, double* tailx) {
  int no = 0;
  bool have = false, stopped = false;
  Piece cur;
  int pend = 0;        // nonzero serial terms pending before the next piece
  double pendx = 0.0;  // their value when exactly one
  for (int q = 0; q < nunits && !stopped; ++q) {
    int nq, tq;
    double xq;
    const Piece* pq = unit(q, nq, tq, xq);
    for (int t = 0; t < nq; ++t) {
      Piece nx = pq[t];
      const int npre = pend + nx.npre;
      if (npre == 1 && pend == 1) nx.xpre = pendx;
      nx.npre = npre;
      pend = 0;
      if (have && npre == 0 && chain_piece(cur, nx)) continue;
      if (have) {
        out[no++] = cur;
        if (no == cap) {  // out of slots: the rest is serial
          have = false;
          stopped = true;
          break;
        }
      }
      cur = nx;
      have = true;
    }
    if (tq > 0) {
      if (pend == 0 && tq == 1) pendx = xq;
      pend += tq;
    }
  }
  if (have) out[no++] = cur;
  *tail = stopped ? 2 : pend;
  *tailx = pendx;
  return no;
}

// Phase B for one segment by one warp: the segment is staged in shared
// memory (coalesced), each lane runs its sub-range from its approximate start
// (a warp scan of the lane sub-sums), lane 0 chains the lanes' runs.
__device__ __forceinline__ void spec_segment_warp(const double* __restrict__ v, int len,
                                                  double shat, Piece* __restrict__ out,
                                                  int* __restrict__ np_out,
                                                  int* __restrict__ tail_out,
                                                  double* __restrict__ tailx_out, double* stage,
                                                  Piece* lp, int* lnp, int* ltail, double* lxt) {
  const int lane = threadIdx.x & 31;
  const bool staged = len <= kStage;
  if (staged) {
    __syncwarp();
    const int n2 = len / 2;
    const double2* v2 = reinterpret_cast<const double2*>(v);
    double2* s2 = reinterpret_cast<double2*>(stage);
#pragma unroll 4
    for (int i = lane; i < n2; i += 32) s2[i] = __ldcg(v2 + i);
    if ((len & 1) && lane == 0) stage[len - 1] = __ldcg(v + len - 1);
    __syncwarp();
  }
  const double* src = staged ? stage : v;
  const int sb = ((len + 31) / 32) | 1;  // odd stride: no shared-memory bank conflicts
  const int b = min(len, lane * sb), e = min(len, b + sb);
  double sum = 0.0;
  for (int i = b; i < e; ++i) sum += src[i];
  double incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  LaneSpec sp;
  sp.init(lane == 0 ? shat : shat + (incl - sum), lp + lane * kLanePieces);
  int i = b;
  for (; i + 4 <= e; i += 4) {
    const double x0 = src[i], x1 = src[i + 1], x2 = src[i + 2], x3 = src[i + 3];
    sp.step(x0, i);
    sp.step(x1, i + 1);
    sp.step(x2, i + 2);
    sp.step(x3, i + 3);
  }
  for (; i < e; ++i) sp.step(src[i], i);
  lnp[lane] = sp.finish(e);
  ltail[lane] = sp.full ? 2 : sp.npre;  // nonzero serial terms after the lane's last run
  lxt[lane] = sp.xpre;
  __syncwarp();
  if (lane == 0) {
    int t;
    double tx;
    *np_out = compose(
        32,
        [&](int q, int& nq, int& tq, double& xq) -> const Piece* {
          nq = lnp[q];
          tq = ltail[q];
          xq = lxt[q];
          return lp + q * kLanePieces;
        },
        out, kMaxPieces, &t, &tx);
    *tail_out = t;
    *tailx_out = tx;
  }
  __syncwarp();
}

// A piece written by another CTA of the cluster (through L2).
__device__ __forceinline__ Piece load_piece(const Piece* q) {
  const double2* d = reinterpret_cast<const double2*>(q);
  const double2 a = __ldcg(d), b = __ldcg(d + 1), c = __ldcg(d + 2), e = __ldcg(d + 3);
  const double2 f = __ldcg(d + 4);
  const int2 k = __ldcg(reinterpret_cast<const int2*>(d + 5));
  Piece p;
  p.st[0] = a.x;
  p.st[1] = a.y;
  p.en[0] = b.x;
  p.en[1] = b.y;
  p.dlo[0] = c.x;
  p.dlo[1] = c.y;
  p.dhi[0] = e.x;
  p.dhi[1] = e.y;
  p.xpre = f.x;
  p.k0 = __double_as_longlong(f.y) & 0xffffffff;
  p.k1 = static_cast<int>(static_cast<unsigned long long>(__double_as_longlong(f.y)) >> 32);
  p.npre = k.x;
  p.pad = 0;
  return p;
}

// Serial terms v[k0, k1) added to s by a whole warp (loads by all lanes,
// every lane carries the same s; all-zero blocks cost no additions).
__device__ __forceinline__ double serial_warp(double s, const double* __restrict__ v, int k0,
                                              int k1) {
  const int lane = threadIdx.x & 31;
  for (int b = k0; b < k1; b += 32) {
    const double t = b + lane < k1 ? __ldcg(v + b + lane) : 0.0;
    unsigned nzm = __ballot_sync(0xffffffffu, t != 0.0);
    SEQ_CNT(13, lane == 0 ? __popc(nzm) : 0);
    while (nzm) {
      const int q = __ffs(nzm) - 1;
      nzm &= nzm - 1u;
      s = dadd(s, __shfl_sync(0xffffffffu, t, q));
    }
  }
  return s;
}

// The serial terms before a piece (npre nonzero ones in [k, p.k0)).
__device__ __forceinline__ double pre_terms(double s, const Piece& p, const double* v, int k) {
  if (p.npre == 1) return dadd(s, p.xpre);
  if (p.npre > 1) return serial_warp(s, v, k, p.k0);
  return s;
}

// One chain of the engine: `terms` materialised (len doubles), start s_init.
struct Chain {
  const double* terms;
  int64_t len;
  double s_init;
  int B, P;
};

// Per-chain scratch in global memory.
struct Scratch {
  double* segsum;  // [chain][seg]
  Piece* pieces;   // [chain][seg][kMaxPieces]
  int* np;         // [chain][seg]
  int* tail;       // [chain][seg]
  double* tailx;   // [chain][seg]
  Piece* gpieces;  // [chain][group][kMaxGPieces]
  int* gnp;        // [chain][group]
  int* gtail;      // [chain][group]
  double* gtailx;  // [chain][group]
};

// Warp-level Phase A: segment sum (any order, coalesced 16-byte loads).
__device__ __forceinline__ double warp_seg_sum(const double* __restrict__ v, int len) {
  const int lane = threadIdx.x & 31;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
  for (int i = lane; i < len / 2; i += 32) {
    const double2 t = __ldcg(v2 + i);
    a0 += t.x;
    a1 += t.y;
  }
  if ((len & 1) && lane == 0) a0 += __ldcg(v + len - 1);
  double acc = a0 + a1;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Shared-memory layout of the engine inside a cluster kernel.
struct EngineSmem {
  double shat[kMaxChains][kMaxSegs];
  union {
    double stage[kBWarps][kStage];           // phase B: the segment's terms
    Piece gbuf[kBWarps][kGroup * kMaxPieces];  // phase C1: the group's pieces
  } u;
  Piece lp[kBWarps][32 * kLanePieces];  // phase B: the lanes' runs
  int lnp[kBWarps][32];
  int ltail[kBWarps][32];
  double lxt[kBWarps][32];
  int gnp[kBWarps][kGroup], gtl[kBWarps][kGroup];
  double gtx[kBWarps][kGroup];
  Piece pbuf[kMaxChains][32];  // phase C2 batches
  int psg[kMaxChains][32];
  double res[kMaxChains];
  double wsum[kThreads / 32 + 1];
};

// Phase C1 for one group of segments by one warp: the group's pieces are
// loaded into shared memory by all lanes, lane 0 chains them across the
// segment boundaries (k made relative to the group).
__device__ __forceinline__ void chain_group_warp(const Scratch& sc, int c, int g, int P, int B,
                                                 Piece* gbuf, int* gnp, int* gtl, double* gtx) {
  const int lane = threadIdx.x & 31;
  const int p0 = g * kGroup, ns = min(kGroup, P - p0);
  if (lane < ns) {
    gnp[lane] = __ldcg(sc.np + c * kMaxSegs + p0 + lane);
    gtl[lane] = __ldcg(sc.tail + c * kMaxSegs + p0 + lane);
    gtx[lane] = __ldcg(sc.tailx + c * kMaxSegs + p0 + lane);
  }
  __syncwarp();
  for (int t = lane; t < ns * kMaxPieces; t += 32) {
    const int q = t / kMaxPieces, i = t % kMaxPieces;
    if (i < gnp[q]) {
      Piece pc = load_piece(sc.pieces + (static_cast<int64_t>(c) * kMaxSegs + p0 + q) * kMaxPieces + i);
      pc.k0 += q * B;
      pc.k1 += q * B;
      gbuf[t] = pc;
    }
  }
  __syncwarp();
  if (lane == 0) {
    int t;
    double tx;
    sc.gnp[c * kMaxGroups + g] = compose(
        ns,
        [&](int q, int& nq, int& tq, double& xq) -> const Piece* {
          nq = gnp[q];
          tq = gtl[q];
          xq = gtx[q];
          return gbuf + q * kMaxPieces;
        },
        sc.gpieces + (static_cast<int64_t>(c) * kMaxGroups + g) * kMaxGPieces, kMaxGPieces, &t,
        &tx);
    sc.gtail[c * kMaxGroups + g] = t;
    sc.gtailx[c * kMaxGroups + g] = tx;
  }
  __syncwarp();
}

// Phase C2 of one chain by one warp: the groups' pieces, 32 at a time, in one
// round trip into shared memory; every lane applies them in order (the same
// s in every lane). Returns the sum.
__device__ __forceinline__ double stitch_chain_warp(const Chain& C, const Scratch& sc, int c,
                                                    Piece* pbuf, int* psg) {
  const int lane = threadIdx.x & 31;
  const int NG = (C.P + kGroup - 1) / kGroup;
  const int64_t GL = static_cast<int64_t>(kGroup) * C.B;  // terms per group
  double s = C.s_init;
  for (int g0 = 0; g0 < NG; g0 += 32) {
    const int ng = min(32, NG - g0);
    const int npv = lane < ng ? __ldcg(sc.gnp + c * kMaxGroups + g0 + lane) : 0;
    const int tlv = lane < ng ? __ldcg(sc.gtail + c * kMaxGroups + g0 + lane) : 0;
    const double txv = lane < ng ? __ldcg(sc.gtailx + c * kMaxGroups + g0 + lane) : 0.0;
    int incl = npv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - npv;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int cur = 0, k = 0;  // group (within the batch) and term reached in it
    auto finish_group = [&](int gi) {  // the group's tail after its last piece
      const int tl = __shfl_sync(0xffffffffu, tlv, gi);
      const double tx = __shfl_sync(0xffffffffu, txv, gi);
      if (tl == 1) {
        s = dadd(s, tx);
      } else if (tl > 1) {
        const int64_t gb = (g0 + gi) * GL;
        s = serial_warp(s, C.terms + gb, k, static_cast<int>(min(C.len - gb, GL)));
      }
    };
    for (int base = 0; base < total; base += 32) {
      const int t = base + lane;
      int sg = 0;
      for (int q = 0; q < ng; ++q) {
        const int e = __shfl_sync(0xffffffffu, excl, q);
        const int nq = __shfl_sync(0xffffffffu, npv, q);
        if (nq > 0 && e <= t) sg = q;
      }
      const int my_excl = __shfl_sync(0xffffffffu, excl, sg);
      __syncwarp();
      if (t < total) {
        pbuf[lane] = load_piece(sc.gpieces + (static_cast<int64_t>(c) * kMaxGroups + g0 + sg) * kMaxGPieces +
                                (t - my_excl));
        psg[lane] = sg;
      }
      __syncwarp();
      const int mcount = min(32, total - base);
      for (int i = 0; i < mcount; ++i) {
        const int gi = psg[i];
        while (cur < gi) {
          finish_group(cur);
          ++cur;
          k = 0;
        }
        const Piece& p = pbuf[i];
        const double* v = C.terms + (g0 + cur) * GL;
        s = pre_terms(s, p, v, k);
        SEQ_CNT(8, lane == 0);
        if (!try_apply(s, p)) {
          SEQ_CNT(9, lane == 0);
          s = serial_warp(s, v, p.k0, p.k1);
        }
        k = p.k1;
      }
    }
    for (; cur < ng; ++cur) {
      finish_group(cur);
      k = 0;
    }
    __syncwarp();
  }
  return s;
}

// The engine, called by EVERY thread of EVERY CTA of the cluster after the
// chains' terms are written and visible cluster-wide: A (segment sums),
// barrier, the approximate starts (each CTA for itself), B (one warp per
// segment), barrier, C1 (one warp per group of kGroup segments), barrier, C2
// (every CTA stitches every chain, warp c, so no barrier is needed
// afterwards). Results in sm.res[c] after the final __syncthreads.
static __device__ __noinline__ void engine(const Chain* ch, int nch, const Scratch& sc,
                                       EngineSmem& sm) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int cta = static_cast<int>(cl.block_rank()), ncta = static_cast<int>(cl.num_blocks());
  const int gw = cta * nwarps + warp, gnw = ncta * nwarps;
  SEQ_PROF_T(t_a);
  int total = 0, gtotal = 0;
  for (int c = 0; c < nch; ++c) {
    total += ch[c].P;
    gtotal += (ch[c].P + kGroup - 1) / kGroup;
  }
  for (int job = gw; job < total; job += gnw) {  // A: segment sums
    int c = 0, p = job;
    while (p >= ch[c].P) p -= ch[c++].P;
    const int64_t b = static_cast<int64_t>(p) * ch[c].B;
    const int len = static_cast<int>(min(ch[c].len - b, static_cast<int64_t>(ch[c].B)));
    const double s = warp_seg_sum(ch[c].terms + b, len);
    if (lane == 0) sc.segsum[c * kMaxSegs + p] = s;
  }
  SEQ_PROF_T(t_b);
  cl.sync();
  SEQ_PROF_T(t_c);
  for (int c = 0; c < nch; ++c) {  // approximate starts: exclusive prefix (per CTA)
    const int P = ch[c].P;
    double carry = ch[c].s_init;
    for (int base = 0; base < P; base += kThreads) {
      const int p = base + threadIdx.x;
      const double v = p < P ? __ldcg(sc.segsum + c * kMaxSegs + p) : 0.0;
      double incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) sm.wsum[warp] = incl;
      __syncthreads();
      double wtot = 0.0;
      if (warp == 0) {
        const double w = lane < nwarps ? sm.wsum[lane] : 0.0;
        double wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, wi, o);
          if (lane >= o) wi += y;
        }
        if (lane < nwarps) sm.wsum[lane] = wi - w;
        wtot = __shfl_sync(0xffffffffu, wi, 31);
        if (lane == 0) sm.wsum[kThreads / 32] = wtot;
      }
      __syncthreads();
      if (p < P) sm.shat[c][p] = carry + (sm.wsum[warp] + (incl - v));
      carry += sm.wsum[kThreads / 32];
      __syncthreads();
    }
  }
  if (threadIdx.x < nch) sm.shat[threadIdx.x][0] = ch[threadIdx.x].s_init;  // exact start
  __syncthreads();
  SEQ_PROF_T(t_d);
  const int bw = cta * kBWarps + warp, bnw = ncta * kBWarps;  // phase B / C1 warps
  if (warp < kBWarps)
    for (int job = bw; job < total; job += bnw) {  // B: one warp per segment
      int c = 0, p = job;
      while (p >= ch[c].P) p -= ch[c++].P;
      const int64_t b = static_cast<int64_t>(p) * ch[c].B;
      const int len = static_cast<int>(min(ch[c].len - b, static_cast<int64_t>(ch[c].B)));
      const int q = c * kMaxSegs + p;
      spec_segment_warp(ch[c].terms + b, len, sm.shat[c][p],
                        sc.pieces + static_cast<int64_t>(q) * kMaxPieces, sc.np + q, sc.tail + q,
                        sc.tailx + q, sm.u.stage[warp], sm.lp[warp], sm.lnp[warp],
                        sm.ltail[warp], sm.lxt[warp]);
    }
  SEQ_PROF_T(t_e);
  cl.sync();
  SEQ_PROF_T(t_f);
  if (warp < kBWarps)
    for (int job = bw; job < gtotal; job += bnw) {  // C1: one warp per group
      int c = 0, g = job;
      while (g >= (ch[c].P + kGroup - 1) / kGroup) g -= (ch[c++].P + kGroup - 1) / kGroup;
      chain_group_warp(sc, c, g, ch[c].P, ch[c].B, sm.u.gbuf[warp], sm.gnp[warp], sm.gtl[warp],
                       sm.gtx[warp]);
    }
  cl.sync();
  SEQ_PROF_T(t_g0);
  if (warp < nch) {  // C2: stitch
    const double s = stitch_chain_warp(ch[warp], sc, warp, sm.pbuf[warp], sm.psg[warp]);
    if (lane == 0) sm.res[warp] = s;
  }
  SEQ_PROF_T(t_g);
  __syncthreads();
  SEQ_PROF_T(t_h);
  SEQ_PROF_ADD(0, t_a, t_b);    // A
  SEQ_PROF_ADD(1, t_b, t_c);    // barrier after A
  SEQ_PROF_ADD(2, t_c, t_d);    // starts
  SEQ_PROF_ADD(3, t_d, t_e);    // B (CTA 0's own jobs)
  SEQ_PROF_ADD(4, t_e, t_f);    // barrier after B (waits for the slowest CTA)
  SEQ_PROF_ADD(10, t_f, t_g0);  // C1 + barrier
  SEQ_PROF_ADD(5, t_g0, t_g);   // C2 (warp 0 = chain 0's stitch)
  SEQ_PROF_ADD(6, t_g, t_h);    // wait for the other chains' stitches
  SEQ_PROF_ADD(7, 0ull, 1ull);  // engine calls
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
