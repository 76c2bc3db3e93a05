// FP64 DMMA GEMM for sm_100a.
//
// Design (B200): FP64 has no tcgen05 kind, so the tensor path is the warp-level DMMA
// (mma.sync.m8n8k4.f64; measured 37.2 TF/s on this pool's B200 vs 34.2 TF/s for DFMA,
// profiles/r01_fp64_peaks.json).  Tiles are staged global->shared with a 3-stage cp.async
// pipeline; each warp owns a WM x WN accumulator block held in registers.  Shared tiles are
// k-major with a 4-double pad so every fragment load is the minimum two wavefronts.
//
// Modes used by the band reduction: A_SYM_LOWER reads a symmetric matrix from its lower
// triangle only (tiles above the diagonal are fetched transposed from below it), and
// C_LOWER_TILES skips CTA tiles strictly above the diagonal (trailing rank-2k update).
#include "gemm.cuh"

namespace pevd {

namespace {

constexpr int PADD = 4;

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct Cfg {
  static constexpr int WARPS_M = BM / WM;
  static constexpr int WARPS_N = BN / WN;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int LDA_S = BM + PADD;
  static constexpr int LDB_S = BN + PADD;
  static constexpr int A_STAGE = BK * LDA_S;
  static constexpr int B_STAGE = BK * LDB_S;
  static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) * 8;
  static constexpr int MI = WM / 8;
  static constexpr int NI = WN / 8;
};

// Load op(A)[i0:i0+BM, k0:k0+BK] into As[kk][i].
template <int BM, int BK, int NT>
__device__ __forceinline__ void load_a_tile(double* As, int lda_s, const GemmArgs& g, int64_t i0,
                                            int64_t k0, int tid) {
  const double* A = g.A;
  const int64_t lda = g.lda;
  int mode;  // 0: contiguous along i (A[i + k*lda]); 1: contiguous along k (A[k + i*lda]); 2: per element sym
  if (g.amode == A_SYM_LOWER) {
    if (k0 + BK - 1 <= i0) mode = 0;          // whole tile on/below the diagonal
    else if (k0 >= i0 + BM - 1) mode = 1;     // whole tile above: read the mirror A[k, i]
    else mode = 2;
  } else {
    mode = g.transA ? 1 : 0;
  }
  const int64_t m = g.m, K = g.k;
  if (mode == 0) {
    const int* amap = g.amap;
#pragma unroll 4
    for (int idx = tid; idx < BM * BK; idx += NT) {
      const int i = idx % BM, kk = idx / BM;
      const int64_t gi = i0 + i, gk = k0 + kk;
      const bool ok = gi < m && gk < K;
      const int64_t col = (amap && ok) ? (int64_t)amap[gk] : gk;
      cp_async8(As + kk * lda_s + i, ok ? A + gi + col * lda : A, ok);
    }
  } else if (mode == 1) {
#pragma unroll 4
    for (int idx = tid; idx < BM * BK; idx += NT) {
      const int kk = idx % BK, i = idx / BK;
      const int64_t gi = i0 + i, gk = k0 + kk;
      const bool ok = gi < m && gk < K;
      cp_async8(As + kk * lda_s + i, ok ? A + gk + gi * lda : A, ok);
    }
  } else {
    for (int idx = tid; idx < BM * BK; idx += NT) {
      const int i = idx % BM, kk = idx / BM;
      const int64_t gi = i0 + i, gk = k0 + kk;
      const bool ok = gi < m && gk < K;
      const double* src = (gi >= gk) ? A + gi + gk * lda : A + gk + gi * lda;
      cp_async8(As + kk * lda_s + i, ok ? src : A, ok);
    }
  }
}

// Load op(B)[k0:k0+BK, j0:j0+BN] into Bs[kk][j].
template <int BN, int BK, int NT>
__device__ __forceinline__ void load_b_tile(double* Bs, int ldb_s, const GemmArgs& g, int64_t k0,
                                            int64_t j0, int tid) {
  const double* B = g.B;
  const int64_t ldb = g.ldb, n = g.n, K = g.k;
  if (!g.transB) {  // B[k + j*ldb]: contiguous along k
#pragma unroll 4
    for (int idx = tid; idx < BN * BK; idx += NT) {
      const int kk = idx % BK, j = idx / BK;
      const int64_t gj = j0 + j, gk = k0 + kk;
      const bool ok = gj < n && gk < K;
      cp_async8(Bs + kk * ldb_s + j, ok ? B + gk + gj * ldb : B, ok);
    }
  } else {  // B[j + k*ldb]: contiguous along j
#pragma unroll 4
    for (int idx = tid; idx < BN * BK; idx += NT) {
      const int j = idx % BN, kk = idx / BN;
      const int64_t gj = j0 + j, gk = k0 + kk;
      const bool ok = gj < n && gk < K;
      cp_async8(Bs + kk * ldb_s + j, ok ? B + gj + gk * ldb : B, ok);
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__device__ __forceinline__ void gemm_tile(const GemmArgs& g, int64_t i0, int64_t j0, int64_t kbeg,
                                          int64_t kend, double* ws_out, int64_t ws_ld,
                                          double* smem) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES>;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  double* As = smem;
  double* Bs = smem + STAGES * C::A_STAGE;

  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int a = 0; a < C::MI; ++a)
#pragma unroll
    for (int b = 0; b < C::NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int64_t KT = (kend - kbeg + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      load_a_tile<BM, BK, C::NT>(As + s * C::A_STAGE, C::LDA_S, g, i0, kbeg + s * BK, tid);
      load_b_tile<BN, BK, C::NT>(Bs + s * C::B_STAGE, C::LDB_S, g, kbeg + s * BK, j0, tid);
    }
    cp_async_commit();
  }
  // the tail of a split-K chunk must not read past kend: clamp via a local K
  for (int64_t kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t pf = kt + STAGES - 1;
      if (pf < KT) {
        const int st = pf % STAGES;
        load_a_tile<BM, BK, C::NT>(As + st * C::A_STAGE, C::LDA_S, g, i0, kbeg + pf * BK, tid);
        load_b_tile<BN, BK, C::NT>(Bs + st * C::B_STAGE, C::LDB_S, g, kbeg + pf * BK, j0, tid);
      }
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * C::A_STAGE + wm * WM + (lane >> 2);
    const double* bs = Bs + (kt % STAGES) * C::B_STAGE + wn * WN + (lane >> 2);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      const int kr = k4 + (lane & 3);
      double af[C::MI], bf[C::NI];
#pragma unroll
      for (int a = 0; a < C::MI; ++a) af[a] = as[kr * C::LDA_S + a * 8];
#pragma unroll
      for (int b = 0; b < C::NI; ++b) bf[b] = bs[kr * C::LDB_S + b * 8];
#pragma unroll
      for (int a = 0; a < C::MI; ++a)
#pragma unroll
        for (int b = 0; b < C::NI; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // epilogue
  const int r_in = lane >> 2, c_in = 2 * (lane & 3);
#pragma unroll
  for (int a = 0; a < C::MI; ++a) {
    const int64_t gi = i0 + wm * WM + a * 8 + r_in;
    if (gi >= g.m) continue;
#pragma unroll
    for (int b = 0; b < C::NI; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gj = j0 + wn * WN + b * 8 + c_in + h;
        if (gj >= g.n) continue;
        if (ws_out) {
          ws_out[gi + gj * ws_ld] = acc[a][b][h];
        } else {
          const int64_t cj = g.cmap ? (int64_t)g.cmap[gj] : gj;
          double* cp = g.C + gi + cj * g.ldc;
          const double v = g.alpha * acc[a][b][h];
          *cp = (g.beta == 0.0) ? v : v + g.beta * *cp;
        }
      }
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, WM, WN, STAGES>::NT)
    gemm_kernel(const __grid_constant__ GemmArgs g, int ksplit, double* ws) {
  extern __shared__ __align__(16) double smem[];
  const int64_t i0 = (int64_t)blockIdx.x * BM, j0 = (int64_t)blockIdx.y * BN;
  if (g.cmode == C_LOWER_TILES && i0 + BM - 1 < j0) return;
  int64_t kbeg = 0, kend = g.k;
  double* wsp = nullptr;
  if (ksplit > 1) {
    const int64_t chunk = ((g.k + ksplit - 1) / ksplit + BK - 1) / BK * BK;
    kbeg = blockIdx.z * chunk;
    kend = kbeg + chunk < g.k ? kbeg + chunk : g.k;
    wsp = ws + (int64_t)blockIdx.z * g.m * g.n;
    if (kbeg >= kend) kbeg = kend;  // empty chunk still writes zeros
  }
  GemmArgs gg = g;
  gg.k = kend;  // loads are bounded by k (absolute index); chunk start via kbeg
  gemm_tile<BM, BN, BK, WM, WN, STAGES>(gg, i0, j0, kbeg, kend, wsp, g.m, smem);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, WM, WN, STAGES>::NT)
    gemm_grouped_kernel(const GemmArgs* __restrict__ args) {
  extern __shared__ __align__(16) double smem[];
  const GemmArgs g = args[blockIdx.z];
  const int64_t i0 = (int64_t)blockIdx.x * BM, j0 = (int64_t)blockIdx.y * BN;
  if (g.m <= 0 || g.n <= 0 || i0 >= g.m || j0 >= g.n) return;
  if (g.cmode == C_LOWER_TILES && i0 + BM - 1 < j0) return;
  gemm_tile<BM, BN, BK, WM, WN, STAGES>(g, i0, j0, 0, g.k > 0 ? g.k : 0, nullptr, 0, smem);
}

__global__ void splitk_reduce(const double* __restrict__ ws, int ksplit, int64_t m, int64_t n,
                              double alpha, double beta, double* C, int64_t ldc,
                              const int* cmap) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    double s = 0.0;
    for (int z = 0; z < ksplit; ++z) s += ws[z * total + idx];  // fixed order: deterministic
    double* cp = C + i + (cmap ? (int64_t)cmap[j] : j) * ldc;
    const double v = alpha * s;
    *cp = (beta == 0.0) ? v : v + beta * *cp;
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
int launch(cudaStream_t st, const GemmArgs& g, int ksplit, double* ws) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = gemm_kernel<BM, BN, BK, WM, WN, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    PEVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  dim3 grid((unsigned)cdiv(g.m, BM), (unsigned)cdiv(g.n, BN), ksplit);
  kern<<<grid, C::NT, C::SMEM, st>>>(g, ksplit, ws);
  PEVD_LAUNCH_CHECK();
  return OK;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
int launch_grouped(cudaStream_t st, const GemmArgs* d_args, int count, int64_t max_m,
                   int64_t max_n) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = gemm_grouped_kernel<BM, BN, BK, WM, WN, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    PEVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  dim3 grid((unsigned)cdiv(max_m, BM), (unsigned)cdiv(max_n, BN), count);
  kern<<<grid, C::NT, C::SMEM, st>>>(d_args);
  PEVD_LAUNCH_CHECK();
  return OK;
}

}  // namespace

int gemm(cudaStream_t st, const GemmArgs& g, double* ws, int64_t ws_elems) {
  if (g.m <= 0 || g.n <= 0) return OK;
  const int sms = num_sms();
  if (g.n <= 32) {
    // skinny (AW = A W, Z = AW - Y M ...): 128 x 32 tiles, split K when the grid is thin
    const int64_t tiles = cdiv(g.m, 128);
    int ks = 1;
    if (ws && g.k >= 1024 && tiles < 2 * sms) {
      ks = (int)std::min<int64_t>(cdiv(3 * sms, tiles), g.k / 256);
      while (ks > 1 && (int64_t)ks * g.m * g.n > ws_elems) --ks;
    }
    if (ks > 1 && g.cmode == C_ALL) {
      PEVD_TRY((launch<128, 32, 16, 32, 32, 3>(st, g, ks, ws)));
      splitk_reduce<<<std::min<int64_t>(cdiv(g.m * g.n, 256), 4 * sms), 256, 0, st>>>(
          ws, ks, g.m, g.n, g.alpha, g.beta, g.C, g.ldc, g.cmap);
      PEVD_LAUNCH_CHECK();
      return OK;
    }
    return launch<128, 32, 16, 32, 32, 3>(st, g, 1, nullptr);
  }
  const int64_t tiles = cdiv(g.m, 128) * cdiv(g.n, 128);
  if (tiles >= sms || g.k < 64) {
    return launch<128, 128, 16, 64, 32, 3>(st, g, 1, nullptr);
  }
  // few output tiles: smaller tiles, then split-K if still thin
  const int64_t tiles64 = cdiv(g.m, 64) * cdiv(g.n, 64);
  int ks = 1;
  if (ws && tiles64 < sms && g.k >= 512) {
    ks = (int)std::min<int64_t>(cdiv(2 * sms, tiles64), g.k / 128);
    while (ks > 1 && (int64_t)ks * g.m * g.n > ws_elems) --ks;
  }
  if (ks > 1 && g.cmode == C_ALL) {
    PEVD_TRY((launch<64, 64, 16, 32, 32, 3>(st, g, ks, ws)));
    splitk_reduce<<<std::min<int64_t>(cdiv(g.m * g.n, 256), 4 * sms), 256, 0, st>>>(
        ws, ks, g.m, g.n, g.alpha, g.beta, g.C, g.ldc, g.cmap);
    PEVD_LAUNCH_CHECK();
    return OK;
  }
  return launch<64, 64, 16, 32, 32, 3>(st, g, 1, nullptr);
}

int gemm_grouped(cudaStream_t st, const GemmArgs* d_args, int count, int64_t max_m,
                 int64_t max_n) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return OK;
  if (max_m * max_n >= (int64_t)128 * 128 * 64)
    return launch_grouped<128, 128, 16, 64, 32, 3>(st, d_args, count, max_m, max_n);
  return launch_grouped<64, 64, 16, 32, 32, 3>(st, d_args, count, max_m, max_n);
}

}  // namespace pevd
