// Back transformation (backtrans.py): SBR-Back (Q_s from the panel factors), BC-Back (the bulge
// reflectors), final GEMM glue lives in api.cu.
//
// SBR-Back: Q_s = H_0 H_1 ... H_{R-1}, H_x = I - Y_x T_x Y_x^T, accumulated backwards from the
// identity (the cheap direction: each step only touches the trailing (n-t0)^2 block).  NB
// consecutive panels are aggregated into one compact-WY block (Y_agg = the panels' columns of the
// explicit-Y staircase left in A by the band reduction, T_agg rebuilt from Y_agg^T Y_agg and the
// panel taus, LAPACK larft recurrence) so the three DMMA GEMMs per block are compute-bound.
//
// BC-Back (reordered, backtrans.py:277-310): X <- X Q_b for a block of rows of X (X = Q_s, so the
// result is Q_s Q_b).  Rows are independent, so one thread owns one row; reflectors are applied in
// the grouped dependency order of the paper's BLAS2 kernel (groups of G sweeps, chase steps
// bottom-to-top, sweeps ascending; backtrans.py:214-236 with group size G).  For b = 32 the
// thread keeps the b+G-1 row entries a reflector group touches in registers while sliding up the
// chase steps, so each entry of X is loaded and stored once per sweep group: arithmetic
// intensity G/4 flop/byte.  The group's reflectors are staged in shared memory (broadcast reads).
#include <cstdlib>
#include "kernels.cuh"

namespace pevd {

namespace {

constexpr int NB_AGG = 4;  // panels per aggregated SBR-Back block

__global__ void set_identity(int64_t n, double* Q, int64_t ldq) {
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    Q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
  }
}

// T_agg (K x K, upper) of the aggregated block reflector I - Y T Y^T from the per-panel T_x
// (diagonal blocks, from the panel QR) and the Gram matrix G = Y^T Y:
//   T[0:c, blk] = -T[0:c, 0:c] G[0:c, blk] T_blk     (blocks of b columns, c = blk * b)
// one CTA, all products in shared memory (K <= NB_AGG * 32 = 128).
__global__ void __launch_bounds__(256)
    larft_kernel(int K, const double* __restrict__ G, int ldg, const double* __restrict__ Tall,
                 int b, int x0, int64_t R, int pw_last, double* __restrict__ T) {
  extern __shared__ double sm[];
  double* Ts = sm;            // K x K (col-major, ld K)
  double* tmp = Ts + K * K;   // K x b
  const int tid = threadIdx.x;
  for (int e = tid; e < K * K; e += blockDim.x) Ts[e] = 0.0;
  __syncthreads();
  const int nblk = (K + b - 1) / b;
  for (int B = 0; B < nblk; ++B) {
    const int x = x0 + B;
    const int pw = (x == R - 1) ? pw_last : b;
    const double* Tx = Tall + (int64_t)x * b * b;  // pw x pw, ld pw
    const int c0 = B * b;
    for (int e = tid; e < pw * pw; e += blockDim.x) {
      const int r = e % pw, c = e / pw;
      Ts[(c0 + r) + (c0 + c) * K] = Tx[r + c * pw];
    }
    __syncthreads();
    if (B == 0) continue;
    // tmp = T[0:c0, 0:c0] G[0:c0, c0:c0+pw]
    for (int e = tid; e < c0 * pw; e += blockDim.x) {
      const int r = e % c0, c = e / c0;
      double s = 0.0;
      for (int t = r; t < c0; ++t) s += Ts[r + t * K] * G[t + (int64_t)(c0 + c) * ldg];
      tmp[r + c * c0] = s;
    }
    __syncthreads();
    // T[0:c0, blk] = -tmp T_blk
    for (int e = tid; e < c0 * pw; e += blockDim.x) {
      const int r = e % c0, c = e / c0;
      double s = 0.0;
      for (int t = 0; t <= c; ++t) s += tmp[r + t * c0] * Ts[(c0 + t) + (c0 + c) * K];
      Ts[r + (c0 + c) * K] = -s;
    }
    __syncthreads();
  }
  for (int e = tid; e < K * K; e += blockDim.x) T[e] = Ts[e];
}

// ------------------------------------------------------------ BC-Back, generic b (slow, tests)

__global__ void bc_back_right_generic(int64_t n, int b, const double* __restrict__ tau,
                                      const double* __restrict__ V, int vld, double* X,
                                      int64_t ldx, int64_t nrows, int G) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  double* x = X + row;
  const int64_t nsw = n - 2;
  for (int64_t i0 = 0; i0 < nsw; i0 += G) {
    const int64_t jmax = (n - 3 - i0) / b;
    for (int64_t j = jmax; j >= 0; --j) {
      const int64_t off = bc_slot_offset_dev(n, b, j);
      for (int64_t i = i0; i < i0 + G && i < nsw; ++i) {
        const int64_t r0 = i + 1 + j * b;
        if (r0 > n - 2) continue;
        const double t = tau[off + i];
        if (t == 0.0) continue;
        const int L = (int)((b < n - r0) ? b : n - r0);
        const double* v = V + (off + i) * vld;
        double dot = 0.0;
        for (int r = 0; r < L; ++r) dot += v[r] * x[(r0 + r) * ldx];
        dot *= t;
        for (int r = 0; r < L; ++r) x[(r0 + r) * ldx] -= dot * v[r];
      }
    }
  }
}

// conventional direction: X <- Q_b X on columns of X (thread per column; used for small n only)
__global__ void bc_back_left_generic(int64_t n, int b, const double* __restrict__ tau,
                                     const double* __restrict__ V, int vld, double* X, int64_t ldx,
                                     int64_t ncols) {
  const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double* x = X + col * ldx;
  const int64_t nsw = n - 2;
  // reverse creation order: sweeps descending, steps descending
  for (int64_t i = nsw - 1; i >= 0; --i) {
    const int64_t jmax = (n - 3 - i) / b;
    for (int64_t j = jmax; j >= 0; --j) {
      const int64_t off = bc_slot_offset_dev(n, b, j);
      const double t = tau[off + i];
      if (t == 0.0) continue;
      const int64_t r0 = i + 1 + j * b;
      const int L = (int)((b < n - r0) ? b : n - r0);
      const double* v = V + (off + i) * vld;
      double dot = 0.0;
      for (int r = 0; r < L; ++r) dot += v[r] * x[r0 + r];
      dot *= t;
      for (int r = 0; r < L; ++r) x[r0 + r] -= dot * v[r];
    }
  }
}

// ------------------------------------------------------------ BC-Back, b = 32 register window

template <int B, int G, int MINB>
__global__ void __launch_bounds__(128, MINB)
    bc_back_right_reg(int64_t n, const double* __restrict__ tau, const double* __restrict__ V,
                      int vld, double* X, int64_t ldx, int64_t nrows) {
  constexpr int WIN = B + G - 1;
  __shared__ __align__(16) double vs[2][G][B];
  __shared__ double ts[2][G];
  const int tid = threadIdx.x;
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + tid;
  const bool active = row < nrows;
  double* x = X + (active ? row : 0);
  const int64_t nsw = n - 2;
  double win[WIN];
  for (int64_t i0 = 0; i0 < nsw; i0 += G) {
    const int64_t jmax = (n - 3 - i0) / B;
    // window for step j covers columns [ws, ws + WIN), ws = i0 + 1 + j*B
    int64_t ws = i0 + 1 + jmax * B;
#pragma unroll
    for (int c = 0; c < WIN; ++c) {
      const int64_t col = ws + c;
      win[c] = (active && col < n) ? x[col * ldx] : 0.0;
    }
    int buf = 0;
    for (int64_t j = jmax; j >= 0; --j) {
      // stage this tile's reflectors (G sweeps x B entries)
      const int64_t off = bc_slot_offset_dev(n, B, j);
      __syncthreads();
      for (int e = tid; e < G * B; e += blockDim.x) {
        const int t = e / B, r = e % B;
        const int64_t i = i0 + t;
        const int64_t r0 = i + 1 + j * B;
        const bool ok = i < nsw && r0 <= n - 2;
        vs[buf][t][r] = ok ? V[(off + i) * vld + r] : 0.0;
        if (r == 0) ts[buf][t] = ok ? tau[off + i] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const double tt = ts[buf][t];
        if (tt != 0.0) {  // uniform across the CTA
          double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int r = 0; r < B; r += 4) {
            const double2 va = *reinterpret_cast<const double2*>(&vs[buf][t][r]);
            const double2 vb = *reinterpret_cast<const double2*>(&vs[buf][t][r + 2]);
            d0 = fma(va.x, win[t + r], d0);
            d1 = fma(va.y, win[t + r + 1], d1);
            d2 = fma(vb.x, win[t + r + 2], d2);
            d3 = fma(vb.y, win[t + r + 3], d3);
          }
          const double dot = tt * ((d0 + d1) + (d2 + d3));
#pragma unroll
          for (int r = 0; r < B; r += 2) {
            const double2 va = *reinterpret_cast<const double2*>(&vs[buf][t][r]);
            win[t + r] = fma(-dot, va.x, win[t + r]);
            win[t + r + 1] = fma(-dot, va.y, win[t + r + 1]);
          }
        }
      }
      buf ^= 1;
      // slide up: store the last B columns, shift the first G-1 to the end, load B new columns
#pragma unroll
      for (int c = G - 1; c < WIN; ++c) {
        const int64_t col = ws + c;
        if (active && col < n) x[col * ldx] = win[c];
      }
      if (j > 0) {
#pragma unroll
        for (int c = G - 2; c >= 0; --c) win[c + B] = win[c];
        ws -= B;
#pragma unroll
        for (int c = 0; c < B; ++c) win[c] = active ? x[(ws + c) * ldx] : 0.0;
      } else {
#pragma unroll
        for (int c = 0; c < G - 1; ++c) {
          const int64_t col = ws + c;
          if (active && col < n) x[col * ldx] = win[c];
        }
      }
    }
  }
}

int launch_larft(cudaStream_t st, int K, const double* G, const double* Tall, int b, int x0,
                 int64_t R, int pw_last, double* T) {
  const size_t smem = (size_t)(K * K + K * b) * 8;
  static int attr_dev = -1;
  int dev;
  PEVD_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    PEVD_CUDA(cudaFuncSetAttribute(larft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   227 * 1024));
    attr_dev = dev;
  }
  larft_kernel<<<1, 256, smem, st>>>(K, G, K, Tall, b, x0, R, pw_last, T);
  PEVD_LAUNCH_CHECK();
  return OK;
}

}  // namespace

int64_t sbr_back_ws_bytes(int64_t n, int b) {
  const int64_t K = (int64_t)NB_AGG * b;
  return (2 * K * n + 2 * K * K + (4 << 20)) * 8 + 1024;
}

int sbr_back_form(cudaStream_t st, int64_t n, int b, const double* Yfull, const double* Tall,
                  double* Qs, int64_t ldq, void* ws) {
  set_identity<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 16384), 256, 0, st>>>(n, Qs, ldq);
  PEVD_LAUNCH_CHECK();
  if (b < 1 || n <= b) return OK;
  const int64_t R = sbr_num_rounds(n, b);
  const int64_t Kmax = (int64_t)NB_AGG * b;
  double* tmp1 = (double*)ws;
  double* tmp2 = tmp1 + Kmax * n;
  double* Gm = tmp2 + Kmax * n;
  double* Tg = Gm + Kmax * Kmax;
  double* sk = Tg + Kmax * Kmax;
  const int64_t skn = 4 << 20;
  const int64_t ngroups = cdiv(R, NB_AGG);
  for (int64_t g = ngroups - 1; g >= 0; --g) {
    const int64_t x0 = g * NB_AGG, x1 = std::min<int64_t>(R, x0 + NB_AGG);
    const int64_t c0 = x0 * b, t0 = c0 + b, m = n - t0;
    int64_t K = 0;
    for (int64_t x = x0; x < x1; ++x) K += std::min<int64_t>(b, n - b - x * b);
    const double* Y = Yfull + t0 + c0 * n;  // m x K, ld n (explicit staircase)
    double* Q22 = Qs + t0 + t0 * ldq;
    // Gram and T_agg
    GemmArgs gg{K, K, m, 1.0, 0.0, Y, n, Y, n, Gm, K, 1, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, gg, sk, skn));
    PEVD_TRY(launch_larft(st, (int)K, Gm, Tall, b, (int)x0, R, (int)(n - b - (R - 1) * b), Tg));
    PEVD_LAUNCH_CHECK();
    // tmp1 = Y^T Q22 (K x m); tmp2 = T tmp1; Q22 -= Y tmp2
    GemmArgs g1{K, m, m, 1.0, 0.0, Y, n, Q22, ldq, tmp1, K, 1, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g1, sk, skn));
    GemmArgs g2{K, m, K, 1.0, 0.0, Tg, K, tmp1, K, tmp2, K, 0, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g2, sk, skn));
    GemmArgs g3{m, m, K, -1.0, 1.0, Y, n, tmp2, K, Q22, ldq, 0, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g3, sk, skn));
  }
  return OK;
}

int sbr_back_apply_left(cudaStream_t st, int64_t n, int b, const double* Yfull, const double* Tall,
                        double* X, int64_t ldx, int64_t ncols, void* ws) {
  // X <- Q_s X = H_0 (H_1 ( ... (H_{R-1} X))): aggregated blocks from the last panel backwards
  if (b < 1 || n <= b) return OK;
  const int64_t R = sbr_num_rounds(n, b);
  const int64_t Kmax = (int64_t)NB_AGG * b;
  double* tmp1 = (double*)ws;
  double* tmp2 = tmp1 + Kmax * n;
  double* Gm = tmp2 + Kmax * n;
  double* Tg = Gm + Kmax * Kmax;
  double* sk = Tg + Kmax * Kmax;
  const int64_t skn = 4 << 20;
  const int64_t ngroups = cdiv(R, NB_AGG);
  for (int64_t g = ngroups - 1; g >= 0; --g) {
    const int64_t x0 = g * NB_AGG, x1 = std::min<int64_t>(R, x0 + NB_AGG);
    const int64_t c0 = x0 * b, t0 = c0 + b, m = n - t0;
    int64_t K = 0;
    for (int64_t x = x0; x < x1; ++x) K += std::min<int64_t>(b, n - b - x * b);
    const double* Y = Yfull + t0 + c0 * n;
    double* X2 = X + t0;
    GemmArgs gg{K, K, m, 1.0, 0.0, Y, n, Y, n, Gm, K, 1, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, gg, sk, skn));
    PEVD_TRY(launch_larft(st, (int)K, Gm, Tall, b, (int)x0, R, (int)(n - b - (R - 1) * b), Tg));
    PEVD_LAUNCH_CHECK();
    for (int64_t c = 0; c < ncols; c += n) {
      const int64_t nc = std::min<int64_t>(n, ncols - c);
      GemmArgs g1{K, nc, m, 1.0, 0.0, Y, n, X2 + c * ldx, ldx, tmp1, K, 1, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g1, sk, skn));
      GemmArgs g2{K, nc, K, 1.0, 0.0, Tg, K, tmp1, K, tmp2, K, 0, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g2, sk, skn));
      GemmArgs g3{m, nc, K, -1.0, 1.0, Y, n, tmp2, K, X2 + c * ldx, ldx, 0, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g3, sk, skn));
    }
  }
  return OK;
}

int bc_back_right(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                  double* X, int64_t ldx, int64_t nrows) {
  if (n < 3 || nrows <= 0 || b < 2) return OK;
  if (b == 32 && vld >= 32) {
    static int g_sel = -1;
    if (g_sel < 0) {
      const char* e = getenv("PEVD_BCBACK_G");
      g_sel = e ? atoi(e) : 32;
    }
    const unsigned grid = (unsigned)cdiv(nrows, 128);
    switch (g_sel) {
      case 8: bc_back_right_reg<32, 8, 4><<<grid, 128, 0, st>>>(n, tau, V, vld, X, ldx, nrows); break;
      case 16: bc_back_right_reg<32, 16, 3><<<grid, 128, 0, st>>>(n, tau, V, vld, X, ldx, nrows); break;
      case 20: bc_back_right_reg<32, 20, 3><<<grid, 128, 0, st>>>(n, tau, V, vld, X, ldx, nrows); break;
      case 32: bc_back_right_reg<32, 32, 2><<<grid, 128, 0, st>>>(n, tau, V, vld, X, ldx, nrows); break;
      case 33: bc_back_right_reg<32, 32, 1><<<grid, 128, 0, st>>>(n, tau, V, vld, X, ldx, nrows); break;
      default: bc_back_right_reg<32, 24, 3><<<grid, 128, 0, st>>>(n, tau, V, vld, X, ldx, nrows); break;
    }
  } else {
    bc_back_right_generic<<<(unsigned)cdiv(nrows, 128), 128, 0, st>>>(n, b, tau, V, vld, X, ldx,
                                                                      nrows, 16);
  }
  PEVD_LAUNCH_CHECK();
  return OK;
}

int bc_back_left(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                 double* X, int64_t ldx, int64_t ncols) {
  if (n < 3 || ncols <= 0 || b < 2) return OK;
  bc_back_left_generic<<<(unsigned)cdiv(ncols, 128), 128, 0, st>>>(n, b, tau, V, vld, X, ldx,
                                                                   ncols);
  PEVD_LAUNCH_CHECK();
  return OK;
}

}  // namespace pevd
