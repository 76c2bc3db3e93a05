// Successive band reduction, dense symmetric -> band of half-bandwidth b (sbr.py:155-188).
//
// Single-GPU driver.  The matrix stays in HBM (column-major) but only its lower triangle is ever
// read or written:
//   per round (c0, pw, t0) of round_schedule (sbr.py:54-66), m = n - t0:
//     1. panel QR of A[t0:, c0:c0+pw]             (cooperative kernel, panel_qr.cu)
//        -> R, explicit Y (into the panel itself and into [Y|Z|Y]), W = Y T, T
//     2. band columns [c0, c0+pw) are final: diagonal block of A + R  -> bands
//     3. AW = A22 W        A22 read from its lower triangle only (A_SYM_LOWER DMMA GEMM)
//     4. M  = W^T AW       (split-K DMMA GEMM, deterministic reduction)
//     5. Z  = AW - 1/2 Y M  (sbr.py:119-130)
//     6. A22 -= [Y Z][Z Y]^T on the lower CTA tiles only (rank-2k, sbr.py:133-152)
//     (ragged last round: coupling columns get Q^T from the left first, sbr.py:175-182)
// Afterwards everything above the b-th subdiagonal is zeroed, leaving A = the "Y staircase":
// panel x's explicit Y_x at A[t0:, c0:c0+pw], exactly the compact-WY operand SBR-Back needs.
#include "kernels.cuh"

namespace pevd {

namespace {

// bands[d, c] for the panel columns c in [c0, c0+pw): diagonal block below, R above
__global__ void band_cols_from_panel(int64_t n, int b, int64_t c0, int pw,
                                     const double* __restrict__ A, int64_t lda,
                                     const double* __restrict__ R, double* __restrict__ bands) {
  const int total = (b + 1) * pw;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int d = idx / pw, c = idx % pw;
    const int64_t col = c0 + c, row = col + d;
    double v = 0.0;
    if (row < n) v = (c + d < b) ? A[row + col * lda] : R[(c + d - b) + (int64_t)c * pw];
    bands[(int64_t)d * n + col] = v;
  }
}

// trailing band columns [c_start, n) straight from A's lower triangle
__global__ void band_cols_tail(int64_t n, int b, int64_t c_start, const double* __restrict__ A,
                               int64_t lda, double* __restrict__ bands) {
  const int64_t w = n - c_start;
  const int64_t total = (int64_t)(b + 1) * w;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = idx / w, col = c_start + idx % w;
    bands[d * n + col] = (col + d < n) ? A[col + d + col * lda] : 0.0;
  }
}

// zero A[r, c] for r < c + b: what remains is the Y staircase
__global__ void zero_above_staircase(int64_t n, int b, double* A, int64_t lda) {
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % n, c = idx / n;
    if (r < c + b) A[r + c * lda] = 0.0;
  }
}

}  // namespace

int64_t sbr_num_rounds(int64_t n, int b) {
  if (b < 1 || n <= b) return 0;
  return cdiv(n - b, b);
}

static constexpr int64_t SPLITK_ELEMS = 4 << 20;

int64_t sbr_ws_bytes(int64_t n, int b) {
  // YZY (n x 3b) + W (n x b) + M, R, coupling tmp (b x b each) + split-K + QR
  return (n * 3 * b + n * b + 3 * (int64_t)b * b + SPLITK_ELEMS) * 8 + panel_qr_ws_bytes() + 1024;
}

int sbr_reduce(cudaStream_t st, int64_t n, int b, double* A, int64_t lda, double* bands_ref,
               double* Tall, void* ws) {
  if (b < 1 || n < 2 || b >= n) {
    set_error("sbr_reduce: need 1 <= b < n (n=%lld, b=%d)", (long long)n, b);
    return ERR_VALUE;
  }
  double* YZY = (double*)ws;
  const int64_t ldz = n;
  double* Wb = YZY + n * 3 * b;
  double* Mb = Wb + n * b;
  double* Rb = Mb + (int64_t)b * b;
  double* Cp = Rb + (int64_t)b * b;
  double* sk = Cp + (int64_t)b * b;
  void* qrws = (void*)(sk + SPLITK_ELEMS);

  int64_t x = 0;
  int64_t c_end = 0;
  for (int64_t c0 = 0; c0 < n - b; c0 += b, ++x) {
    const int64_t pw = std::min<int64_t>(b, n - b - c0);
    const int64_t t0 = c0 + b;
    const int64_t m = n - t0;
    double* panel = A + t0 + c0 * lda;
    double* A22 = A + t0 + t0 * lda;
    double* Tx = Tall ? Tall + x * (int64_t)b * b : nullptr;
    double* Yz = YZY;  // [Y | Z | Y], ld = n
    double* Zz = YZY + pw * ldz;
    double* Y3 = YZY + 2 * pw * ldz;
    // 1. panel QR (Y overwrites the panel in A; R kept aside for the band)
    PEVD_TRY(panel_qr(st, m, (int)pw, panel, lda, Rb, panel, lda, Yz, ldz, Wb, n, Tx, qrws));
    // 2. band columns of this panel are final
    band_cols_from_panel<<<1, 256, 0, st>>>(n, b, c0, (int)pw, A, lda, Rb, bands_ref);
    PEVD_LAUNCH_CHECK();
    PEVD_CUDA(cudaMemcpy2DAsync(Y3, ldz * 8, Yz, ldz * 8, m * 8, pw, cudaMemcpyDeviceToDevice, st));
    // ragged final round: coupling columns [c0+pw, t0) rows [t0, n) get Q^T from the left
    if (pw < b) {
      const int64_t nc = b - pw;
      double* cpl = A + t0 + (c0 + pw) * lda;
      GemmArgs g1{pw, nc, m, 1.0, 0.0, Wb, n, cpl, lda, Cp, pw, 1, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g1, sk, SPLITK_ELEMS));
      GemmArgs g2{m, nc, pw, -1.0, 1.0, Yz, ldz, Cp, pw, cpl, lda, 0, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g2, sk, SPLITK_ELEMS));
    }
    // 3. AW = A22 W  (symmetric, lower storage) -> Z slot
    GemmArgs g_aw{m, pw, m, 1.0, 0.0, A22, lda, Wb, n, Zz, ldz, 0, 0, A_SYM_LOWER, C_ALL};
    PEVD_TRY(gemm(st, g_aw, sk, SPLITK_ELEMS));
    // 4. M = W^T AW
    GemmArgs g_m{pw, pw, m, 1.0, 0.0, Wb, n, Zz, ldz, Mb, pw, 1, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g_m, sk, SPLITK_ELEMS));
    // 5. Z = AW - 1/2 Y M
    GemmArgs g_z{m, pw, pw, -0.5, 1.0, Yz, ldz, Mb, pw, Zz, ldz, 0, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g_z, sk, SPLITK_ELEMS));
    // 6. A22 -= [Y Z] [Z Y]^T   (lower tiles)
    GemmArgs g_u{m, m, 2 * pw, -1.0, 1.0, Yz, ldz, Zz, ldz, A22, lda, 0, 1, A_GENERAL,
                 C_LOWER_TILES};
    PEVD_TRY(gemm(st, g_u, nullptr, 0));
    c_end = c0 + pw;
  }
  {
    const int64_t total = (int64_t)(b + 1) * (n - c_end);
    band_cols_tail<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 4096), 256, 0, st>>>(
        n, b, c_end, A, lda, bands_ref);
    PEVD_LAUNCH_CHECK();
  }
  zero_above_staircase<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 16384), 256, 0, st>>>(
      n, b, A, lda);
  PEVD_LAUNCH_CHECK();
  return OK;
}

}  // namespace pevd
