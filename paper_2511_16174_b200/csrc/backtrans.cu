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

constexpr int NB_AGG = 8;  // panels per aggregated SBR-Back block

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
                 int b, int x0, int64_t R, int pw_last, double* T) {
  // T lives in global memory (L2-resident, K <= 256); the per-block product in shared memory
  extern __shared__ double tmp[];  // (K - b) x b
  const int tid = threadIdx.x;
  for (int e = tid; e < K * K; e += blockDim.x) T[e] = 0.0;
  __syncthreads();
  const int nblk = (K + b - 1) / b;
  for (int B = 0; B < nblk; ++B) {
    const int x = x0 + B;
    const int pw = (x == R - 1) ? pw_last : b;
    const double* Tx = Tall + (int64_t)x * b * b;  // pw x pw, ld pw
    const int c0 = B * b;
    for (int e = tid; e < pw * pw; e += blockDim.x) {
      const int r = e % pw, c = e / pw;
      T[(c0 + r) + (c0 + c) * K] = Tx[r + c * pw];
    }
    __syncthreads();
    if (B == 0) continue;
    // tmp = T[0:c0, 0:c0] G[0:c0, c0:c0+pw]
    for (int e = tid; e < c0 * pw; e += blockDim.x) {
      const int r = e % c0, c = e / c0;
      double s = 0.0;
      for (int t = r; t < c0; ++t) s += T[r + t * K] * G[t + (int64_t)(c0 + c) * ldg];
      tmp[r + c * c0] = s;
    }
    __syncthreads();
    // T[0:c0, blk] = -tmp T_blk
    for (int e = tid; e < c0 * pw; e += blockDim.x) {
      const int r = e % c0, c = e / c0;
      double s = 0.0;
      for (int t = 0; t <= c; ++t) s += tmp[r + t * c0] * T[(c0 + t) + (c0 + c) * K];
      T[r + (c0 + c) * K] = -s;
    }
    __syncthreads();
  }
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

template <int B, int G, int MINB, bool LEAN>
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
          const double* vt = &vs[buf][t][0];
          double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int r = 0; r < B; r += 8) {
            // 8-wide chunks with a scheduling fence: keeps only 8 v values live (register
            // budget for 3 CTAs/SM) while each chunk still issues its loads together
            const double2 va = *reinterpret_cast<const double2*>(vt + r);
            const double2 vb = *reinterpret_cast<const double2*>(vt + r + 2);
            const double2 vc = *reinterpret_cast<const double2*>(vt + r + 4);
            const double2 vd = *reinterpret_cast<const double2*>(vt + r + 6);
            d0 = fma(va.x, win[t + r], d0);
            d1 = fma(va.y, win[t + r + 1], d1);
            d2 = fma(vb.x, win[t + r + 2], d2);
            d3 = fma(vb.y, win[t + r + 3], d3);
            d0 = fma(vc.x, win[t + r + 4], d0);
            d1 = fma(vc.y, win[t + r + 5], d1);
            d2 = fma(vd.x, win[t + r + 6], d2);
            d3 = fma(vd.y, win[t + r + 7], d3);
            if (LEAN) asm volatile("" ::: "memory");
          }
          const double dot = tt * ((d0 + d1) + (d2 + d3));
#pragma unroll
          for (int r = 0; r < B; r += 8) {
            const double2 va = *reinterpret_cast<const double2*>(vt + r);
            const double2 vb = *reinterpret_cast<const double2*>(vt + r + 2);
            const double2 vc = *reinterpret_cast<const double2*>(vt + r + 4);
            const double2 vd = *reinterpret_cast<const double2*>(vt + r + 6);
            win[t + r] = fma(-dot, va.x, win[t + r]);
            win[t + r + 1] = fma(-dot, va.y, win[t + r + 1]);
            win[t + r + 2] = fma(-dot, vb.x, win[t + r + 2]);
            win[t + r + 3] = fma(-dot, vb.y, win[t + r + 3]);
            win[t + r + 4] = fma(-dot, vc.x, win[t + r + 4]);
            win[t + r + 5] = fma(-dot, vc.y, win[t + r + 5]);
            win[t + r + 6] = fma(-dot, vd.x, win[t + r + 6]);
            win[t + r + 7] = fma(-dot, vd.y, win[t + r + 7]);
            if (LEAN) asm volatile("" ::: "memory");
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
  const size_t smem = (size_t)(K * b) * 8;
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


// ------------------------------------------------------------ BC-Back, b = 32, 4 lanes per row
// Lane (row r = lane/4, quarter q = lane%4) owns window positions p = 4m + q, m < Q4_WM: a
// 96-wide window (Q4_SG = 64 sweeps + b - 1) costs 24 doubles per lane.  Reflector t touches
// positions [t, t+32): each lane holds 8 of them (9 slots, one padded), the partial dot is
// reduced over the row's 4 lanes with two xor-shuffles.  v is staged per tile in shared memory
// split by phase (v[4k + ph] -> vs[t][ph][k + 2]) with a second copy shifted by one, so every
// lane's 10 consecutive operands start 16-byte aligned (5 LDS.128 per reflector).
// Work units (64-row block, sweep group) are claimed from an atomic counter in group-major
// order by a persistent grid; a per-row-block progress counter orders a block's groups.
constexpr int Q4_SG = 64;
constexpr int Q4_WM = 24;
constexpr int Q4_ROWS = 64;
constexpr int Q4_THREADS = 256;
constexpr int Q4_VR = 12;  // per (t, phase, copy): slots 0..11 (k + 2 in 2..9, zeros around)

struct Q4Smem {
  double v[2][Q4_SG][4][2][Q4_VR];  // [buf][t][phase][copy][slot]
  double tau[2][Q4_SG];
  int unit;
};

__global__ void __launch_bounds__(Q4_THREADS, 2)
    bc_back_q4_kernel(int64_t n, const double* __restrict__ tau, const double* __restrict__ V,
                      int vld, double* X, int64_t ldx, int64_t nrows, int* counter, int* progress,
                      int64_t nunits, int nrb) {
  extern __shared__ __align__(16) unsigned char q4raw[];
  Q4Smem& S = *reinterpret_cast<Q4Smem*>(q4raw);
  constexpr int B = 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3;
  const int rloc = warp * 8 + (lane >> 2);
  const int64_t nsw = n - 2;
  for (int e = tid; e < 2 * Q4_SG * 4 * 2 * Q4_VR; e += Q4_THREADS) (&S.v[0][0][0][0][0])[e] = 0.0;
  __syncthreads();
  for (;;) {
    if (tid == 0) S.unit = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t u = S.unit;
    __syncthreads();
    if (u >= nunits) break;
    const int64_t k = u / nrb;
    const int rb = (int)(u % nrb);
    if (tid == 0) {
      if (ld_acquire(progress + rb) < (int)k) {
        unsigned ns = 64;
        while (ld_acquire(progress + rb) < (int)k) {
          __nanosleep(ns);
          if (ns < 1024) ns <<= 1;
        }
      }
    }
    __syncthreads();
    const int64_t row = (int64_t)rb * Q4_ROWS + rloc;
    const bool active = row < nrows;
    double* x = X + (active ? row : 0);
    const int64_t i0 = k * Q4_SG;
    const int64_t jmax = (n - 3 - i0) / B;
    int64_t ws = i0 + 1 + jmax * B;
    double win[Q4_WM];
#pragma unroll
    for (int m = 0; m < Q4_WM; ++m) {
      const int64_t col = ws + 4 * m + q;
      win[m] = (active && col < n) ? __ldcg(x + col * ldx) : 0.0;
    }
    int buf = 0;
    for (int64_t j = jmax; j >= 0; --j) {
      const int64_t off = bc_slot_offset_dev(n, B, j);
      for (int e = tid; e < Q4_SG * B; e += Q4_THREADS) {
        const int t = e >> 5, r = e & 31;
        const int64_t i = i0 + t;
        const bool ok = i < nsw && i + 1 + j * B <= n - 2;
        const double val = ok ? __ldg(V + (off + i) * vld + r) : 0.0;
        const int ph = r & 3, kk = r >> 2;
        S.v[buf][t][ph][0][kk + 2] = val;  // copy 0: lanes with shift 0 read slots 2..11
        S.v[buf][t][ph][1][kk + 3] = val;  // copy 1: lanes with shift 1 read slots 2..11
        if (r == 0) S.tau[buf][t] = ok ? __ldg(tau + off + i) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < Q4_SG; ++t) {
        const double tt = S.tau[buf][t];
        if (tt != 0.0) {  // uniform across the CTA
          constexpr int dummy = 0;
          (void)dummy;
          const int a = t >> 2, tb = t & 3;
          const int ph = (q - tb) & 3;
          const int sh = (q < tb) ? 1 : 0;
          // operand for m = a + mm is v[4(mm - sh) + ph] -> copy sh, slot (mm - sh + 2 + sh) = mm + 2
          const double* vr = &S.v[buf][t][ph][sh][2];
          double vv[10];
#pragma unroll
          for (int c = 0; c < 10; c += 2) {
            const double2 p2 = *reinterpret_cast<const double2*>(vr + c);
            vv[c] = p2.x;
            vv[c + 1] = p2.y;
          }
          double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
          for (int mm = 0; mm < 9; mm += 3) {
            d0 = fma(win[a + mm], vv[mm], d0);
            d1 = fma(win[a + mm + 1], vv[mm + 1], d1);
            d2 = fma(win[a + mm + 2], vv[mm + 2], d2);
          }
          double dot = (d0 + d1) + d2;
          dot += __shfl_xor_sync(0xffffffffu, dot, 1);
          dot += __shfl_xor_sync(0xffffffffu, dot, 2);
          dot *= tt;
#pragma unroll
          for (int mm = 0; mm < 9; ++mm) win[a + mm] = fma(-dot, vv[mm], win[a + mm]);
        }
      }
      buf ^= 1;
      // slide: positions [64, 96) are final for this group; shift the rest up by b = 32
#pragma unroll
      for (int m = 16; m < Q4_WM; ++m) {
        const int64_t col = ws + 4 * m + q;
        if (active && col < n) x[col * ldx] = win[m];
      }
      if (j > 0) {
#pragma unroll
        for (int m = 15; m >= 0; --m) win[m + 8] = win[m];
        ws -= B;
#pragma unroll
        for (int m = 0; m < 8; ++m) win[m] = active ? __ldcg(x + (ws + 4 * m + q) * ldx) : 0.0;
      } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const int64_t col = ws + 4 * m + q;
          if (active && col < n) x[col * ldx] = win[m];
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(progress + rb, (int)(k + 1));
    }
  }
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

int64_t bc_back_ws_bytes(int64_t nrows) { return (cdiv(nrows, Q4_ROWS) + 64) * 4; }

int bc_back_right(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                  double* X, int64_t ldx, int64_t nrows, void* ws) {
  if (n < 3 || nrows <= 0 || b < 2) return OK;
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("PEVD_BCBACK");
    mode = (e && e[0] == 'q') ? 0 : 1;  // register-window kernel by default
  }
  if (b == 32 && vld >= 32 && mode == 0 && ws) {
    const int nrb = (int)cdiv(nrows, Q4_ROWS);
    const int64_t ngroups = cdiv(n - 2, Q4_SG);
    const int64_t nunits = ngroups * nrb;
    int* counter = (int*)ws;
    int* progress = counter + 32;
    PEVD_CUDA(cudaMemsetAsync(ws, 0, (size_t)(nrb + 32) * 4, st));
    const size_t smem = sizeof(Q4Smem);
    static int attr_dev = -1;
    int dev;
    PEVD_CUDA(cudaGetDevice(&dev));
    if (attr_dev != dev) {
      PEVD_CUDA(cudaFuncSetAttribute(bc_back_q4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
      attr_dev = dev;
    }
    int per_sm = 0;
    PEVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bc_back_q4_kernel, Q4_THREADS,
                                                            smem));
    if (per_sm < 1) {
      set_error("bc_back: persistent kernel cannot be resident");
      return ERR_CUDA;
    }
    const int64_t grid = std::min<int64_t>((int64_t)per_sm * num_sms(), nunits);
    bc_back_q4_kernel<<<(unsigned)grid, Q4_THREADS, smem, st>>>(n, tau, V, vld, X, ldx, nrows,
                                                                counter, progress, nunits, nrb);
    PEVD_LAUNCH_CHECK();
    return OK;
  }
  if (b == 32 && vld >= 32) {
    static int g_sel = -1;
    if (g_sel < 0) {
      const char* e = getenv("PEVD_BCBACK_G");
      g_sel = e ? atoi(e) : 32;
    }
    const unsigned grid = (unsigned)cdiv(nrows, 128);
    (void)g_sel;
    bc_back_right_reg<32, 32, 2, false><<<grid, 128, 0, st>>>(n, tau, V, vld, X, ldx, nrows);
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
