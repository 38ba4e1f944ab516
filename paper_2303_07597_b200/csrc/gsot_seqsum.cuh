// gsot_seqsum.cuh — the reference's SEQUENTIAL floating-point sums in
// parallel and bit for bit, latency-first (exact-order mode).
//
// A sequential sum of N terms is N dependent roundings. It is computed in
// parallel by speculation on translation invariance: while the partial sums
// of a stretch of terms stay inside binades at or below the binade of the
// stretch's start, the whole path shifted by delta (a multiple of 2 ulp of the
// start) rounds identically, so a "run" computed from an approximate start
// gives the exact result for the true start by one exact addition; runs from
// both mantissa parities of the start cover any delta. Organised for the
// shortest critical path on one thread-block cluster:
//
//   1. every thread of the cluster owns one contiguous block of b terms
//      (b = ceil(len / threads)); approximate block sums, a CTA scan and one
//      cluster barrier give each thread an approximate start s^ (thread 0:
//      the exact start);
//   2. each thread runs its block from s^ ("leaf"): at most kLeafCap runs in
//      both mantissa parities, a run ending where a step leaves the allowed
//      binades (above the start's, or tiny), that term kept inline as a
//      serial term; runs may change sign (signed shift margins);
//   3. lane 0 of each warp composes its 32 leaves into the warp's piece list
//      (runs continued across leaves where the left end is a valid start of
//      the right run), then one lane per chain composes the CTA's warp lists
//      into the CTA's list;
//   4. one more cluster barrier, then EVERY CTA stitches the CTA lists in
//      order from the exact start (an exact translation per piece; inline
//      serial terms: the reference's addition), so the result is in every
//      CTA with no broadcast. A piece that does not apply, and serial terms
//      not kept inline, are replayed with the reference's own additions.
//
// Every step of the stitch is either the reference's addition or an exact
// translation, so the result is the sequential sum for any input; fallbacks
// only cost time. Two cluster barriers per call.
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

// A run (or a chain of runs) over terms [k0, k1).
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


constexpr int kT = 256;            // threads per CTA of the engine's kernels
constexpr int kWarps = kT / 32;    // warps per CTA
constexpr int kMaxCh = 4;          // chains per engine call
constexpr int kMaxCtas = 16;       // cluster size (16 where the device allows, else 8)
constexpr int kLeafCap = 4;        // runs per leaf (later terms of the leaf: replayed)
constexpr int kWarpCap = 16;       // pieces per warp list (later terms of the warp: replayed)
constexpr int kCtaCap = 64;        // pieces per CTA list (else the stitch takes the warp lists)
constexpr int kBatch = 8;          // terms loaded per round trip by one thread
constexpr int kStage = 3328;       // terms of a one-chain call's CTA slice staged in shared memory

struct Chain2 {
  const double* terms;
  int64_t len;
  double s0;
};

// A piece list's tail: nonzero serial terms after its last piece (>= 2:
// replay them from memory; the value when exactly one).
struct Tail {
  int n;
  double x;
};

// Dynamic shared memory of the engine's kernels.
struct Smem2 {
  Chain2 ch[kMaxCh];
  double ctot[kMaxCh];                     // CTA approximate totals (read remotely)
  double wsum[kMaxCh][kWarps];             // scan scratch: warp totals
  Piece lp[kT][kLeafCap];                  // leaf runs (one chain at a time)
  int lnp[kT];
  Tail ltl[kT];
  Piece wl[kMaxCh][kWarps][kWarpCap];      // warp lists
  int wnp[kMaxCh][kWarps];
  Tail wtl[kMaxCh][kWarps];
  Piece cl[kMaxCh][kCtaCap];               // CTA lists (read remotely by the stitch)
  int cnp[kMaxCh];                         // their length; -1: incomplete, use the warp lists
  Tail ctl[kMaxCh];
  Piece st[kMaxCh][kCtaCap];               // stitch: a remote CTA's list, staged
  double res[kMaxCh];
  double stage[kStage];                    // a one-chain call's CTA slice (coalesced copy)
};
static_assert(sizeof(Smem2) <= 227 * 1024, "engine shared memory exceeds the per-CTA limit");

// One thread's block: at most kLeafCap runs, their pieces in shared memory.
// Pieces carry absolute term indices.
struct Leaf {
  double s;                   // speculative value between runs
  double st0, st1, t0, t1;    // open run
  double lo0, hi0, lo1, hi1;  // min distance to the lower / upper bound of the current binade
  double u2;                  // 2 ulp of the run start
  long long bst;              // bits of the run start
  double xpre;
  int k0, np, npre;
  bool open, ok1, full;
  Piece* out;

  __device__ __forceinline__ void init(double shat, Piece* o) {
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
  // a run value may be of either sign and in any binade between 2^-968 and
  // the start's: the true path is the run shifted by delta, and rounding
  // commutes with the shift while both paths' values share a binade (the
  // signed margins below) and delta is a multiple of 2 ulp of that binade
  // (every binade at or below the start's)
  __device__ __forceinline__ bool inside(double v) const {
    const int ex = static_cast<int>((dbits(v) >> 52) & 0x7ff);
    return ex > 54 && ex <= static_cast<int>((bst >> 52) & 0x7ff);
  }
  // the shifts delta keeping v + delta in v's binade: delta > -dneg, < dpos
  __device__ __forceinline__ static void smargins(double v, double& dneg, double& dpos) {
    const double a = fabs(v);
    const double lb = __longlong_as_double(dbits(a) & 0x7ff0000000000000ll);
    const double below = dsub(a, lb), above = dsub(dadd(lb, lb), a);  // exact
    dneg = fmin(dneg, v > 0.0 ? below : above);
    dpos = fmin(dpos, v > 0.0 ? above : below);
  }
  __device__ __forceinline__ bool try_open(int k) {
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
    smargins(t0, lo0, hi0);
    smargins(t1, lo1, hi1);
    ok1 = true;
    k0 = k;
    open = true;
    return true;
  }
  __device__ __forceinline__ void close(int k1) {
    Piece& p = out[np++];
    p.st[0] = st0;
    p.st[1] = st1;
    p.en[0] = t0;
    p.en[1] = t1;
    // lo / hi: allowed negative / positive shift of the start; the piece
    // stores the allowed shift of |s| (sign of the start), 2 ulp kept in reserve
    const double inf = dinf();
    const bool v0 = lo0 >= u2 && hi0 >= u2;
    const bool v1 = ok1 && lo1 >= u2 && hi1 >= u2;
    const bool pos = st0 > 0.0;
    p.dlo[0] = v0 ? dsub(u2, pos ? lo0 : hi0) : inf;
    p.dhi[0] = v0 ? dsub(pos ? hi0 : lo0, u2) : -inf;
    p.dlo[1] = v1 ? dsub(u2, pos ? lo1 : hi1) : inf;
    p.dhi[1] = v1 ? dsub(pos ? hi1 : lo1, u2) : -inf;
    p.xpre = xpre;
    p.k0 = k0;
    p.k1 = k1;
    p.npre = npre;
    p.pad = 0;
    open = false;
    npre = 0;
    s = t0;
    if (np == kLeafCap) full = true;
  }
  __device__ __forceinline__ void step(double x, int k) {
    if (full || x == 0.0) return;  // +-0 terms leave every partial sum unchanged
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
    smargins(n0, lo0, hi0);
    smargins(n1, lo1, hi1);
  }
};

// The reference's additions over v[k0, k1) by a whole warp (every lane
// carries the same s), 128 terms per round trip; zero terms cost nothing.
__device__ __forceinline__ double serial_warp4(double s, const double* __restrict__ v, int k0,
                                               int k1) {
  const int lane = threadIdx.x & 31;
  for (int b = k0; b < k1; b += 128) {
    double t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = b + 32 * j + lane;
      t[j] = k < k1 ? __ldcg(v + k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      unsigned nzm = __ballot_sync(0xffffffffu, t[j] != 0.0);
      while (nzm) {
        const int q = __ffs(nzm) - 1;
        nzm &= nzm - 1u;
        s = dadd(s, __shfl_sync(0xffffffffu, t[j], q));
      }
    }
  }
  return s;
}

// kBatch terms v[kb, kb + kBatch) (zeros past k1), with 16-byte loads where
// the batch is whole (v 16-byte aligned): half the L1 wavefronts of a warp
// whose lanes read distinct blocks.
__device__ __forceinline__ void load_batch(const double* __restrict__ v, int64_t kb, int64_t k1,
                                           double (&x)[kBatch]) {
  if (kb + kBatch <= k1) {
    if ((kb & 1) == 0) {
      const double2* p = reinterpret_cast<const double2*>(v + kb);
#pragma unroll
      for (int q = 0; q < kBatch / 2; ++q) {
        const double2 t = __ldcg(p + q);
        x[2 * q] = t.x;
        x[2 * q + 1] = t.y;
      }
    } else {
      x[0] = __ldcg(v + kb);
      const double2* p = reinterpret_cast<const double2*>(v + kb + 1);
#pragma unroll
      for (int q = 0; q < kBatch / 2 - 1; ++q) {
        const double2 t = __ldcg(p + q);
        x[1 + 2 * q] = t.x;
        x[2 + 2 * q] = t.y;
      }
      x[kBatch - 1] = __ldcg(v + kb + kBatch - 1);
    }
  } else {
#pragma unroll
    for (int q = 0; q < kBatch; ++q) x[q] = kb + q < k1 ? __ldcg(v + kb + q) : 0.0;
  }
}

// Terms per thread of a chain of len terms over P threads: odd, so threads
// reading their blocks from a staged slice hit distinct shared-memory banks.
__host__ __device__ __forceinline__ int64_t block_len(int64_t len, int P) {
  return ((len + P - 1) / P) | 1;
}

// Continue `cur` through `nx` (adjacent, no serial term between): per parity
// run of cur whose end lies in nx's start binade and range, the continued run
// is concrete (its end is nx's end shifted, exact) and its shift range
// narrows. Runs may change sign (the shift ranges are kept relative to each
// piece's start sign, so a sign change between cur's start and nx's start
// mirrors nx's range). cur is updated only when a parity run continues.
__device__ __forceinline__ bool chain2(Piece& cur, const Piece& nx) {
  const long long bn0 = dbits(nx.st[0]);
  const bool same = (cur.st[0] < 0.0) == (nx.st[0] < 0.0);
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
    const double l = fmax(cur.dlo[r], same ? __dsub_ru(nlo, C) : __dsub_ru(C, nhi));
    const double h = fmin(cur.dhi[r], same ? __dsub_rd(nhi, C) : __dsub_rd(C, nlo));
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

// Chain a list of units (the leaves of a warp, the warp lists of a CTA): each
// unit has `np` pieces and `tail` nonzero serial terms after them (tail >= 2:
// unknown, replay; the one value in tailx when 1). Consecutive pieces with no
// serial term between are continued (chain2). One thread. Writes the list's
// pieces to out and returns their count; the list's own tail in *tail / *tailx.
template <typename Unit>
__device__ __forceinline__ int compose2(int nunits, Unit unit, Piece* __restrict__ out, int cap,
                                        int* tail, double* tailx) {
  int no = 0;
  bool have = false, stopped = false;
  Piece cur;
  int pend = 0;
  double pendx = 0.0;
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
      if (have && npre == 0 && chain2(cur, nx)) continue;
      if (have) {
        out[no++] = cur;
        if (no == cap) {
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

// Thread g's block of a chain of len terms over P threads.
__device__ __forceinline__ void block_of(int64_t len, int P, int g, int64_t& k0, int64_t& k1) {
  const int64_t b = block_len(len, P);
  k0 = min(len, static_cast<int64_t>(g) * b);
  k1 = min(len, k0 + b);
}

// ---- engine phases, each a separate (non-inlined) function: the serial parts
// run in one or a few warps, and a compact hot loop stays in the instruction
// cache (an inlined engine is tens of thousands of instructions)

// This thread's approximate block sum of chain c (phase 1).
static __device__ __noinline__ double block_sum(const Smem2& sm, int c, int P, int g, bool staged,
                                                int64_t slo) {
  int64_t k0, k1;
  block_of(sm.ch[c].len, P, g, k0, k1);
  double s = 0.0;
  if (staged) {
#pragma unroll 1
    for (int64_t k = k0; k < k1; ++k) s += sm.stage[k - slo];
  } else {
    const double* __restrict__ v = sm.ch[c].terms;
#pragma unroll 1
    for (int64_t kb = k0; kb < k1; kb += kBatch) {
      double x[kBatch];
      load_batch(v, kb, k1, x);
#pragma unroll
      for (int q = 0; q < kBatch; ++q) s += x[q];
    }
  }
  return s;
}

// This thread's leaf of chain c from the approximate start shat (phase 2).
static __device__ __noinline__ void run_leaf(Smem2& sm, int c, int P, int g, bool staged,
                                             int64_t slo, double shat) {
  int64_t k0, k1;
  block_of(sm.ch[c].len, P, g, k0, k1);
  Leaf lf;
  lf.init(shat, sm.lp[threadIdx.x]);
  if (staged) {
#pragma unroll 1
    for (int64_t k = k0; k < k1; ++k) lf.step(sm.stage[k - slo], static_cast<int>(k));
  } else {
    const double* __restrict__ v = sm.ch[c].terms;
#pragma unroll 1
    for (int64_t kb = k0; kb < k1; kb += kBatch) {
      double x[kBatch];
      load_batch(v, kb, k1, x);
#pragma unroll
      for (int q = 0; q < kBatch; ++q) lf.step(x[q], static_cast<int>(kb + q));
    }
  }
  if (lf.open && !lf.full) lf.close(static_cast<int>(k1));
  sm.lnp[threadIdx.x] = lf.np;
  sm.ltl[threadIdx.x] = Tail{lf.full ? 2 : lf.npre, lf.xpre};
}

// The warp's piece list over its 32 leaves (phase 3, one lane).
static __device__ __noinline__ void compose_warp(Smem2& sm, int c, int warp) {
  int t;
  double tx;
  const int base = warp * 32;
  sm.wnp[c][warp] = compose2(
      32,
      [&](int q, int& nq, int& tq, double& xq) -> const Piece* {
        nq = sm.lnp[base + q];
        tq = sm.ltl[base + q].n;
        xq = sm.ltl[base + q].x;
        return sm.lp[base + q];
      },
      sm.wl[c][warp], kWarpCap, &t, &tx);
  sm.wtl[c][warp] = Tail{t, tx};
}

// The CTA's list over its warp lists (phase 3, one lane per chain); -1 when
// it would not fit (the stitch then takes the warp lists).
static __device__ __noinline__ void compose_cta(Smem2& sm, int c) {
  int tot = 0;
  for (int q = 0; q < kWarps; ++q) tot += sm.wnp[c][q];
  if (tot > kCtaCap) {
    sm.cnp[c] = -1;
    return;
  }
  int t;
  double tx;
  sm.cnp[c] = compose2(
      kWarps,
      [&](int q, int& nq, int& tq, double& xq) -> const Piece* {
        nq = sm.wnp[c][q];
        tq = sm.wtl[c][q].n;
        xq = sm.wtl[c][q].x;
        return sm.wl[c][q];
      },
      sm.cl[c], kCtaCap, &t, &tx);
  sm.ctl[c] = Tail{t, tx};
}

// The reference's additions over v[k0, k1) by a whole warp (every lane
// carries s), 128 terms per round trip; zero terms cost nothing.
static __device__ __noinline__ double serial_terms(double s, const double* __restrict__ v, int k0,
                                                   int k1) {
  return serial_warp4(s, v, k0, k1);
}

// s through np staged pieces over terms [k, kend), then the list's tail (one
// warp, every lane carries s).
static __device__ __noinline__ double apply_list(double s, const Piece* __restrict__ stg, int np,
                                                 Tail tl, int k, int kend,
                                                 const double* __restrict__ terms) {
#pragma unroll 1
  for (int i = 0; i < np; ++i) {
    // every field loaded before s is needed (the loads do not depend on s)
    const Piece& p = stg[i];
    const double st0 = p.st[0], st1 = p.st[1], en0 = p.en[0], en1 = p.en[1];
    const double lo0 = p.dlo[0], lo1 = p.dlo[1], hi0 = p.dhi[0], hi1 = p.dhi[1];
    const double xpre = p.xpre;
    const int npre = p.npre, pk0 = p.k0, pk1 = p.k1;
    if (npre == 1) {
      s = dadd(s, xpre);
    } else if (npre > 1) {
      s = serial_terms(s, terms, k, pk0);
    }
    // the piece applies iff s is in its start binade and its shift in range:
    // then the true path is the run translated (exact)
    const long long bs = dbits(s), b0 = dbits(st0);
    const bool odd = ((bs ^ b0) & 1) != 0;
    const double delta = dsub(s, odd ? st1 : st0);
    const double sh = s < 0.0 ? -delta : delta;
    const bool ok = (((bs ^ b0) >> 52) == 0) && sh >= (odd ? lo1 : lo0) && sh <= (odd ? hi1 : hi0);
    s = ok ? dadd(odd ? en1 : en0, delta) : serial_terms(s, terms, pk0, pk1);
    k = pk1;
  }
  if (tl.n == 1) {
    s = dadd(s, tl.x);
  } else if (tl.n > 1) {
    s = serial_terms(s, terms, k, kend);
  }
  return s;
}

// Phase 4 for chain c (one warp): every CTA's list in order from the exact
// start, each staged into shared memory in one round trip (a CTA whose list
// did not fit: its warp lists).
static __device__ __noinline__ double stitch(Smem2& sm, int c, int P) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31;
  const int ncta = static_cast<int>(cl.num_blocks());
  const Chain2 C = sm.ch[c];
  const int64_t bt = block_len(C.len, P);  // terms per thread
  double s = C.s0;
  Piece* stg = sm.st[c];
#pragma unroll 1
  for (int r = 0; r < ncta; ++r) {
    const int np = *cl.map_shared_rank(&sm.cnp[c], r);
    const int k0 = static_cast<int>(min(C.len, static_cast<int64_t>(r) * kT * bt));
    const int k1 = static_cast<int>(min(C.len, static_cast<int64_t>(r + 1) * kT * bt));
    if (np >= 0) {
      const Tail tl = *cl.map_shared_rank(&sm.ctl[c], r);
      __syncwarp();
      if (lane < np) stg[lane] = *cl.map_shared_rank(&sm.cl[c][lane], r);
      if (lane + 32 < np) stg[lane + 32] = *cl.map_shared_rank(&sm.cl[c][lane + 32], r);
      __syncwarp();
      s = apply_list(s, stg, np, tl, k0, k1, C.terms);
      continue;
    }
    if (cl.block_rank() == 0 && lane == 0) SEQ_CNT(11, 1);
#pragma unroll 1
    for (int w = 0; w < kWarps; ++w) {  // the CTA's list did not fit: its warp lists
      const int wn = *cl.map_shared_rank(&sm.wnp[c][w], r);
      const Tail wt = *cl.map_shared_rank(&sm.wtl[c][w], r);
      __syncwarp();
      if (lane < wn) stg[lane] = *cl.map_shared_rank(&sm.wl[c][w][lane], r);
      __syncwarp();
      const int w0 = static_cast<int>(min(C.len, static_cast<int64_t>(r * kT + w * 32) * bt));
      const int w1 = static_cast<int>(min(C.len, static_cast<int64_t>(r * kT + w * 32 + 32) * bt));
      s = apply_list(s, stg, wn, wt, w0, w1, C.terms);
    }
  }
  return s;
}

// The engine: called by every thread of every CTA of the cluster, with
// sm.ch[0 .. nch) set and every chain's terms written and visible
// cluster-wide. Results in sm.res[c] after the final __syncthreads.
//
// Reuse across calls: a remote CTA reads this CTA's ctot between barrier 1
// and barrier 2 of a call, and its lists after barrier 2 until it arrives at
// barrier 1 of the next call; this CTA rewrites ctot only after barrier 2 and
// its lists only after barrier 1 of the next call. The stitch may replay any
// CTA's terms, so callers alternate term buffers between consecutive calls
// (a buffer is rewritten only after the next call's barrier 1).
static __device__ __noinline__ void engine2(int nch, Smem2& sm) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cta = static_cast<int>(cl.block_rank()), ncta = static_cast<int>(cl.num_blocks());
  const int P = ncta * kT;
  const int g = cta * kT + static_cast<int>(threadIdx.x);
  if (cta == 0 && threadIdx.x == 0) SEQ_CNT(7, 1);
  SEQ_PROF_T(t_a);
  // ---- 1. approximate block sums, CTA scan, CTA totals. A one-chain call
  // whose CTA slice fits is first staged into shared memory with coalesced
  // loads (per-thread blocks read from global memory touch one line per lane)
  const int64_t slo = min(sm.ch[0].len, static_cast<int64_t>(cta) * kT * block_len(sm.ch[0].len, P));
  const int64_t shi = min(sm.ch[0].len, slo + kT * block_len(sm.ch[0].len, P));
  const bool staged = nch == 1 && shi - slo <= kStage;
  if (staged) {
    const double* __restrict__ src = sm.ch[0].terms + slo;
    const int n = static_cast<int>(shi - slo);
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += kT) sm.stage[i] = __ldcg(src + i);
    __syncthreads();
  }
  double excl[kMaxCh];
#pragma unroll
  for (int c = 0; c < kMaxCh; ++c) {
    excl[c] = 0.0;
    if (c >= nch) continue;
    const double s = block_sum(sm, c, P, g, staged, slo);
    double incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) sm.wsum[c][warp] = incl;
    excl[c] = incl - s;
  }
  __syncthreads();
  if (warp < nch) {  // warp c scans chain c's warp totals
    const double w = lane < kWarps ? sm.wsum[warp][lane] : 0.0;
    double wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kWarps) sm.wsum[warp][lane] = wi - w;
    if (lane == kWarps - 1) sm.ctot[warp] = wi;
  }
  SEQ_PROF_T(t_b);
  cl.sync();  // barrier 1: CTA totals visible cluster-wide
  SEQ_PROF_T(t_c);
#ifdef GSOT_SEQ_PROF
  unsigned long long t_runs_end = 0;
#endif
  // ---- 2. leaf runs from the approximate starts; 3. warp lists (lane 0)
#pragma unroll
  for (int c = 0; c < kMaxCh; ++c) {
    if (c >= nch) continue;
    double pre = lane < cta ? *cl.map_shared_rank(&sm.ctot[c], lane) : 0.0;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    const double shat = g == 0 ? sm.ch[c].s0 : sm.ch[c].s0 + (pre + (sm.wsum[c][warp] + excl[c]));
    run_leaf(sm, c, P, g, staged, slo, shat);
    __syncwarp();
    SEQ_PROF_T(t_r);
#ifdef GSOT_SEQ_PROF
    if (c == 0) t_runs_end = t_r;
#endif
    if (lane == 0) {
#ifdef GSOT_SEQ_PROF
      const unsigned long long tw0 = clock64();
      int lsum = 0;
      for (int q = 0; q < 32; ++q) lsum += sm.lnp[warp * 32 + q];
#endif
      compose_warp(sm, c, warp);
#ifdef GSOT_SEQ_PROF
      if (cta == 0 && c == 0) {
        SEQ_CNT(8, lsum);
        SEQ_CNT(9, sm.wnp[c][warp]);
        SEQ_CNT(12, clock64() - tw0);
        SEQ_CNT(13, 1);
      }
#endif
    }
    __syncwarp();
  }
  SEQ_PROF_T(t_d);
  __syncthreads();
  if (warp < nch && lane == 0) compose_cta(sm, warp);
  SEQ_PROF_T(t_e);
  cl.sync();  // barrier 2: CTA lists visible cluster-wide
  SEQ_PROF_T(t_f);
  // ---- 4. stitch (every CTA; warp c: chain c)
  if (warp < nch) {
    const double s = stitch(sm, warp, P);
    if (lane == 0) sm.res[warp] = s;
  }
  SEQ_PROF_T(t_g);
  __syncthreads();
  SEQ_PROF_ADD(0, t_a, t_b);  // block sums + CTA scan
  SEQ_PROF_ADD(1, t_b, t_c);  // barrier 1
  SEQ_PROF_ADD(2, t_c, t_d);  // starts + leaf runs + warp lists
  SEQ_PROF_ADD(15, t_c, t_runs_end);  // starts + leaf runs of chain 0
  SEQ_PROF_ADD(3, t_d, t_e);  // CTA list
  SEQ_PROF_ADD(4, t_e, t_f);  // barrier 2
  SEQ_PROF_ADD(5, t_f, t_g);  // stitch (warp 0: chain 0)
}

}  // namespace seq
}  // namespace gsot
