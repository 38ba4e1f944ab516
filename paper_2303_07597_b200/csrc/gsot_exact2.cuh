// gsot_exact2.cuh — exact-order mode at speed (gsot_exact2.cu): workspace and
// launchers. Exact-order mode reproduces the reference's own order of
// floating-point operations everywhere, so a device solve is
// bitwise the reference's trajectory.
#pragma once

#include "gsot_internal.cuh"
#include "gsot_seqsum.cuh"

namespace gsot {

// Device buffers of the exact-order evaluation and direction (allocated on
// the first exact-mode call of a context).
// term buffers: two call parities x three chains (gsot_exact2.cu)
constexpr int kTermBufs = 6;

struct ExactWs {
  double* scale = nullptr;   // L x n: block scale (1 - tau/z)/gamma of nonzero blocks
  double* psiT = nullptr;    // n x L: per column, its nonzero blocks' psi in group order
  int* cntj = nullptr;       // n: nonzero blocks per column
  uint32_t* nzw = nullptr;   // L x nw: nonzero-block bits of the work tiles
  int* lenC = nullptr;       // nw: psi terms per chunk
  int* offC = nullptr;       // nw + 1: their exclusive prefix
  double* flat = nullptr;    // psi chain terms in (j, l) order (at most L x n)
  double* tv = nullptr;      // kTermBufs x tv_stride: dot-chain terms
  int64_t tv_stride = 0;
  int4* slabs = nullptr;     // 32-row slabs of the groups: {l, first row in group, rows, 0}
  int nslabs = 0;
  int gmin = 0;              // smallest group (kernel variant choice)
};

void exact_ws_alloc(ExactWs& w, const DevProblem& P, const std::vector<int32_t>& sizes,
                    size_t* tally);
void exact_ws_free(ExactWs& w);

// dual_objective + dual_gradient in the reference's order (dual.hpp:38-100)
// over the work tiles of `words` / `gmask` / `cmask` (the screen's, or the
// dense ones): objective, slope grad.d (dvec != null) and the folded screen
// counters into sc; grad [m + n].
void launch_exact_eval2(const DevProblem& P, const ExactWs& W, const double* x,
                        const uint32_t* words, const uint32_t* gmask, uint32_t* cmask,
                        int clear_cmask, double* grad, const double* dvec, EvalScalars* sc,
                        unsigned long long* cnt_slots, cudaStream_t s);

// The exact-order L-BFGS direction (lbfgs.hpp:109-126, and with pair != 0 the
// pending curvature pair and its test first, lbfgs.hpp:243-255): d, out[0] =
// g.d, out[1] = d.d; pair dots into sc->extra[0..2].
struct ExactDirArgs {
  int pair;
  const double *x, *xprev, *g, *gprev;
  double *S, *Y;
  int64_t stride;
  HistState* h;
  double* d;
  int64_t dim;
  double* out;
  EvalScalars* sc;
};
void launch_exact_direction(const ExactDirArgs& a, const ExactWs& W, cudaStream_t s);

// sc->extra[slot] = sequential dot a . b (Eigen's dot in the oracle's order).
void launch_exact_dot2(const double* a, const double* b, int64_t n, const ExactWs& W,
                       EvalScalars* sc, int slot, cudaStream_t s);

// Device-side sequential sum of `terms` from s0 (test hook for the engine).
void launch_seqsum(const double* terms, int64_t n, double s0, const ExactWs& W, double* out,
                   cudaStream_t s);

void read_seq_prof(unsigned long long* out);

}  // namespace gsot
