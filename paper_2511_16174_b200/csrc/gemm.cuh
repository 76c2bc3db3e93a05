// FP64 DMMA GEMM (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) for sm_100a.
// Column-major operands.  C = alpha * op(A) * op(B) + beta * C.
#pragma once
#include "common.cuh"

namespace pevd {

enum AMode : int {
  A_GENERAL = 0,    // op(A) as given
  A_SYM_LOWER = 1,  // A is symmetric m x m, only its lower triangle is valid (transA ignored)
};
enum CMode : int {
  C_ALL = 0,
  C_LOWER_TILES = 1,  // only CTA tiles intersecting the lower triangle (row >= col) are computed
};

struct GemmArgs {
  int64_t m, n, k;
  double alpha, beta;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int transA, transB;
  int amode, cmode;
  const int* amap;  // optional: column j of op(A) is column amap[j] of A (transA == 0 only)
  const int* cmap;  // optional: column j of the product is written to column cmap[j] of C
  int preload = 1;  // beta != 0: start the accumulators at (beta/alpha) C (else read C at the end)
};

// Single GEMM on `stream`; `ws`/`ws_elems` optional split-K workspace (nullptr -> no split-K).
int gemm(cudaStream_t stream, const GemmArgs& g, double* ws = nullptr, int64_t ws_elems = 0);

// Grouped GEMM: `count` problems whose descriptors live in DEVICE memory (may be written by a
// previous kernel on the same stream).  max_m / max_n bound every problem's m / n; CTAs outside
// a problem's tiles exit.  A problem with m, n or k <= 0 is skipped (k <= 0 means C = beta*C).
int gemm_grouped(cudaStream_t stream, const GemmArgs* d_args, int count, int64_t max_m,
                 int64_t max_n);

}  // namespace pevd
