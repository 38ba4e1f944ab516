// gsot_device.cuh — device helpers shared by the kernel translation units
// (header-only so no relocatable device code is needed).
#pragma once

#include "gsot_internal.cuh"

namespace gsot {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// fused multiply-add (one rounding): fast-mode evaluation only, never on an
// exact-order path
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// f = (alpha_i + beta_j) - c_ij, regularizer.hpp:57.
__device__ __forceinline__ double residual(double alpha_i, double beta_j, double c) {
  return dsub(dadd(alpha_i, beta_j), c);
}

// Address of row 0 of block (l, j); row r is at [kRowStride * r].
__device__ __forceinline__ const double* block_ptr(const DevProblem& P, int o0, int g, int64_t j) {
  return P.C + cost_index(P.nw, o0, g, j, 0);
}

// Quarters (8 columns) of a 32-column word with any bit set, and the lanes of a
// set of quarters.
__device__ __forceinline__ uint32_t quarter_mask(uint32_t word) {
  return ((word & 0xffu) ? 1u : 0u) | ((word & 0xff00u) ? 2u : 0u) | ((word & 0xff0000u) ? 4u : 0u) |
         ((word & 0xff000000u) ? 8u : 0u);
}
__device__ __forceinline__ uint32_t quarter_lanes(uint32_t qm) {
  return ((qm & 1u) ? 0xffu : 0u) | ((qm & 2u) ? 0xff00u : 0u) | ((qm & 4u) ? 0xff0000u : 0u) |
         ((qm & 8u) ? 0xff000000u : 0u);
}

// Warp-wide transpose-reduce of 16 rows: on entry lane t holds v[k] = value of
// row k for column t; on exit lane t holds, in v[0], the sum over all 32
// columns of row (t & 15). The butterfly tree is fixed by lane position, so
// it does not depend on which lanes hold exact zeros.
__device__ __forceinline__ void transpose_reduce16(double (&v)[16], int lane) {
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const double send = up ? v[k] : v[k + o];
      const double keep = up ? v[k + o] : v[k];
      v[k] = dadd(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
  v[0] = dadd(v[0], __shfl_xor_sync(0xffffffffu, v[0], 16));
}

// Last-block-done finalisation: every block writes NV partials; the last
// block to arrive reduces them with all its threads in a fixed order
// (thread t sums partials t, t+NT, ... sequentially, then a fixed tree).
template <int NT, int NV>
__device__ __forceinline__ bool last_block_reduce(const double (&mine)[NV], double* partials,
                                                  unsigned int* ticket, double (&out)[NV],
                                                  bool use_max = false) {
  __shared__ double sh[NT / 32][NV];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    v[q] = mine[q];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v[q], o);
      v[q] = use_max ? fmax(v[q], w) : dadd(v[q], w);
    }
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) sh[warp][q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = sh[0][q];
      for (int w = 1; w < NT / 32; ++w) s = use_max ? fmax(s, sh[w][q]) : dadd(s, sh[w][q]);
      partials[blockIdx.x * NV + q] = s;
    }
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += NT) {
      const double p = __ldcg(partials + b * NV + q);
      s = use_max ? fmax(s, p) : dadd(s, p);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, s, o);
      s = use_max ? fmax(s, w) : dadd(s, w);
    }
    v[q] = s;
  }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) sh[warp][q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = sh[0][q];
      for (int w = 1; w < NT / 32; ++w) s = use_max ? fmax(s, sh[w][q]) : dadd(s, sh[w][q]);
      out[q] = s;
    }
    *ticket = 0u;
  }
  return threadIdx.x == 0;
}


}  // namespace gsot

namespace gsot {

// ---- TMA bulk copies (cp.async.bulk) with mbarrier completion --------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// The same with a suspend-time hint: the waiting warp sleeps in the barrier
// instead of spinning through issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned.
// The proxy fence orders the warp's earlier generic reads of the buffer
// before the async-proxy write.
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// The same with an L2 eviction-priority policy (createpolicy).
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_1d_hint(void* smem_dst, const void* gmem_src,
                                                 uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

}  // namespace gsot

namespace gsot {

// Fold the 64 counter slots into sc->counters etc. and zero them (one warp).
// Programmatic dependent launch: a kernel launched with the PDL attribute may
// start while its predecessor drains; pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible. pdl_trigger()
// lets the successor launch early. Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Diagnostic kernel timeline (builds with -DGSOT_PHASE_CLOCKS only): per
// kernel id, the first block entry and the last block exit of the current
// device sequence (globaltimer ns); k_publish folds them into per-sequence
// offsets. No-ops in the product build.
#ifdef GSOT_PHASE_CLOCKS
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_ENTER(tlp, k) \
  do { if ((tlp) && threadIdx.x == 0) atomicMin(&(tlp)[2 * (k)], gtimer()); } while (0)
#define TL_EXIT(tlp, k) \
  do { if ((tlp) && threadIdx.x == 0) atomicMax(&(tlp)[2 * (k) + 1], gtimer()); } while (0)
#else
#define TL_ENTER(tlp, k) do { } while (0)
#define TL_EXIT(tlp, k) do { } while (0)
#endif
enum TimelineId { TL_SCREEN = 0, TL_EVAL = 1, TL_FINALIZE = 2, TL_PUBLISH = 3, TL_STEP = 4,
                  TL_AXPY = 5, TL_DELTA = 6, TL_SNAPSHOT = 7 };

// max(f, 0) by bit operations (f finite): a negative f, -0 included, -> +0.
// Spelled on the two 32-bit halves (one shift, two and-nots on the integer
// pipe; the 64-bit form compiles to two compares and two selects).
__device__ __forceinline__ double relu(double f) {
  const int hi = __double2hiint(f), lo = __double2loint(f);
  int s;
  asm("shr.s32 %0, %1, 31;" : "=r"(s) : "r"(hi));
  return __hiloint2double(hi & ~s, lo & ~s);
}

// Called by exactly one full warp.
__device__ __forceinline__ void fold_counter_slots(unsigned long long* slots, EvalScalars* sc) {
  const int lane = threadIdx.x & 31;
  unsigned long long v[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    v[k] = slots[lane * 8 + k] + slots[(lane + 32) * 8 + k];
    slots[lane * 8 + k] = 0ull;
    slots[(lane + 32) * 8 + k] = 0ull;
  }
#pragma unroll
  for (int k = 0; k < 7; ++k)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0) {
    sc->counters[0] = v[0];
    sc->counters[1] = v[1];
    sc->counters[2] = v[2];
    sc->counters[3] = v[3];
    sc->surv_rows = v[4];
    sc->task_rows = v[5];
  }
}

}  // namespace gsot
