// Internal (C++) interfaces between the translation units of libpevd.so.
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace pevd {

// ---------------- panel QR (panel_qr.cu)
int64_t panel_qr_ws_bytes();
// Householder QR of the m x k panel (col-major, ld ldp): R (k x k, upper, col-major, may be
// null), explicit unit-lower-trapezoidal Y to Y1/Y2 (either may be null; Y1 may alias the
// panel), W = Y T (may be null) and T (k x k col-major, may be null).  Q = I - W Y^T, Q^T P = R.
int panel_qr(cudaStream_t st, int64_t m, int k, const double* panel, int64_t ldp, double* R,
             double* Y1, int64_t ldy1, double* Y2, int64_t ldy2, double* W, int64_t ldw,
             double* T, void* ws);

__host__ __device__ __forceinline__ int64_t bc_slot_offset_dev(int64_t n, int b, int64_t j) {
  return j * (n - 2) - (int64_t)b * j * (j - 1) / 2;
}

// ---------------- SBR (sbr.cu)
// Panel factors: panel x (round x of round_schedule(n, b): c0 = x b, t0 = c0 + b, m = n - t0)
// leaves its explicit unit-lower Y_x in A[t0:, c0:c0+pw] (so after the reduction A holds the
// "Y staircase": zero above the b-th subdiagonal) and T_x at Tall + x*b*b (pw x pw col-major).
int64_t sbr_num_rounds(int64_t n, int b);
int64_t sbr_ws_bytes(int64_t n, int b);
// Dense (lower triangle of A, col-major lda) -> band.  Outputs: bands_ref (C-order (b+1) x n,
// bands[d, j] = A[j+d, j]), Tall (may be null); A becomes the Y staircase.
int sbr_reduce(cudaStream_t st, int64_t n, int b, double* A, int64_t lda, double* bands_ref,
               double* Tall, void* ws);

// ---------------- bulge chasing (bulge.cu)
int64_t bc_num_reflectors(int64_t n, int b);     // fixed slots: sum_j (n - 2 - j b)
int64_t bc_slot_offset(int64_t n, int b, int64_t j);
int64_t bc_ws_bytes(int64_t n, int b);
// band (C-order (b+1) x n, reference layout) -> d (n), e (n-1); reflector slots (tau, V with
// stride vld) in canonical chase-step-major order when tau != null.
int bc_reduce(cudaStream_t st, int64_t n, int b, const double* bands_ref, double* d, double* e,
              double* tau, double* V, int vld, void* ws);
// Partition chase (bulge.py:348-385): sweeps [0, sweep_end) on a band of semi-bandwidth bw <= 2b;
// band_out ((2b+1) x n, may be null) gets the band afterwards, d / e (may be null) its diagonals.
// slot_n / slot_col0 (> 0 / >= 0): the band is the tail [slot_col0, slot_n) of a slot_n problem
// and the reflectors go to that problem's fixed slots (sweep gi is global sweep slot_col0 + gi).
int bc_reduce_range(cudaStream_t st, int64_t n, int b, int bw, const double* bands_ref,
                    int64_t sweep_end, double* d, double* e, double* band_out, double* tau,
                    double* V, int vld, void* ws, int64_t slot_n = 0, int64_t slot_col0 = 0);

// ---------------- tridiagonal divide and conquer (stedc.cu)
int64_t stedc_ws_bytes(int64_t n);
// d (n) in: diagonal, out: eigenvalues ascending; e (n-1) off-diagonal (preserved).
// Q (n x n, ldq) out: eigenvectors.  Sign convention of tridiag.py:325-333 applied.
// (col_lo, col_hi): compute only the columns [col_lo, col_hi) of Q (the rest stays zero); the
// eigenvalues are always complete.
int stedc(cudaStream_t st, int64_t n, double* d, const double* e, double* Q, int64_t ldq,
          void* ws, int* info_host, int64_t col_lo = 0, int64_t col_hi = -1);

// Eigenvalues only (no Q): bisection on Sturm counts, one thread per eigenvalue; lam ascending.
int64_t stebz_ws_bytes(int64_t n);
int stebz(cudaStream_t st, int64_t n, const double* d, const double* e, double* lam, void* ws);

// ---------------- back transformation (backtrans.cu)
// Q_s = prod_x (I - Y_x T_x Y_x^T) formed explicitly into Qs (n x n, ldq).
int64_t sbr_back_ws_bytes(int64_t n, int b);
// (Yfull = the Y staircase left by sbr_reduce in A, leading dimension ldy = lda.)
// Aggregated T factors of every SBR-Back block (depends only on the SBR output); the
// form/apply calls run it themselves unless `prepared` says it already ran on ws.
int sbr_back_prepare(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                     const double* Tall, void* ws);
int sbr_back_form(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                  const double* Tall, double* Qs, int64_t ldq, void* ws, bool prepared = false);
// Apply the SBR reflectors from the left to X (n x ncols): X <- Q_s X (conventional order).
// g_lo/g_hi: only the aggregated blocks [g_lo, g_hi) (all when g_hi < 0); blocks are applied
// from the last backwards, so [k, end) then [0, k) is the full product.
int sbr_back_apply_left(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                        const double* Tall, double* X, int64_t ldx, int64_t ncols, void* ws,
                        bool prepared = false, int64_t g_lo = 0, int64_t g_hi = -1);
// X (nrows x n) <- X Q_s: rows of Q_s from rows of the identity (distributed pipelined order).
int sbr_back_apply_right(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                         const double* Tall, double* X, int64_t ldx, int64_t nrows, void* ws,
                         bool prepared = false);
// Right-apply the bulge reflectors to the rows of X (nrows x n, col-major ldx):
// X <- X Q_b  (== (Q_b^T X^T)^T, the reordered BC-Back, backtrans.py:277-310).
int64_t bc_back_ws_bytes(int64_t n, int64_t nrows, int b);
// the DMMA compact-WY kernels handle b in {8, 16, ..., 64} (reflector stride vld >= b); other b
// use the reflector-by-reflector kernels
bool bc_back_dmma_ok(int b, int vld);
int bc_back_right(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                  double* X, int64_t ldx, int64_t nrows, void* ws);
// Conventional BC-Back on Xt = X^T (nrows x n, column-major), where the bulge kernel's fast
// memory pattern applies: Xt <- Xt Q_b^T.
// (Xt == nullptr: only the preparation (counters, Z of every block), which depends on the chase
//  output alone; prepared = true skips it in the later call on the same ws.)
int bc_back_left_t(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                   double* Xt, int64_t ldx, int64_t nrows, void* ws, bool prepared = false);
// out (cols x rows) = in^T (in: rows x cols)
int transpose(cudaStream_t st, int64_t rows, int64_t cols, const double* in, int64_t ldi,
              double* out, int64_t ldo);
// Left-apply Q_b to X (n x ncols): X <- Q_b X (conventional BC-Back).
int bc_back_left(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                 double* X, int64_t ldx, int64_t ncols, void* ws);

}  // namespace pevd
