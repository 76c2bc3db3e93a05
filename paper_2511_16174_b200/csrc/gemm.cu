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
#include <cstdlib>
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
    gemm_kernel_generic(const __grid_constant__ GemmArgs g, int ksplit, double* ws) {
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
    gemm_grouped_kernel_generic(const GemmArgs* __restrict__ args) {
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
    // eight interleaved partial sums (loads in flight for deep splits), combined in a fixed
    // order: deterministic
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int z = 0;
    for (; z + 8 <= ksplit; z += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += ws[(int64_t)(z + u) * total + idx];
    }
    for (int u = 0; z < ksplit; ++z, ++u) a[u] += ws[(int64_t)z * total + idx];
    const double s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    double* cp = C + i + (cmap ? (int64_t)cmap[j] : j) * ldc;
    const double v = alpha * s;
    *cp = (beta == 0.0) ? v : v + beta * *cp;
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
int launch_generic(cudaStream_t st, const GemmArgs& g, int ksplit, double* ws) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = gemm_kernel_generic<BM, BN, BK, WM, WN, STAGES>;
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
int launch_grouped_generic(cudaStream_t st, const GemmArgs* d_args, int count, int64_t max_m,
                   int64_t max_n) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = gemm_grouped_kernel_generic<BM, BN, BK, WM, WN, STAGES>;
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


// =====================================================================================
// Fast path (A_GENERAL): compile-time transposes, 16-byte cp.async chunks along each operand's
// contiguous dimension, per-thread base pointers advanced by a constant stride per k-tile.
// Shared layouts keep the contiguous dimension contiguous (so a chunk is one LDGSTS.128); the
// 4-double pads make every DMMA fragment load the minimum two wavefronts in all four cases.
// =====================================================================================

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, bool SYM = false>
struct FCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  // Fragment loads read the k-slot pair (k8 + 2q, k8 + 2q + 1) of lane q for two consecutive
  // k-steps: one LDS.128 from a k-contiguous layout (pitch = 8 mod 16 doubles keeps a quarter
  // warp's 16-byte accesses on distinct banks), two LDS.64 from an m/n-contiguous one (pitch =
  // 2 mod 8 doubles: rows 2q apart land on distinct banks).
  static constexpr int A_LD0 = BM + 2, A_LD1 = BK + 8;   // m-contiguous / k-contiguous layouts
  static constexpr int A_LD = TA ? A_LD1 : A_LD0;
  static constexpr int A_OUT = SYM ? (BK * A_LD0 > BM * A_LD1 ? BK : (BM * A_LD1 + A_LD0 - 1) / A_LD0)
                                   : (TA ? BM : BK);
  static constexpr int B_LD = TB ? BN + 2 : BK + 8;
  static constexpr int B_OUT = TB ? BK : BN;
  static constexpr int A_STAGE = A_OUT * A_LD, B_STAGE = B_OUT * B_LD;
  static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) * 8;
  static constexpr int MI = WM / 8, NI = WN / 8;
};

__device__ __forceinline__ void cp_async_vec(void* smem, const void* gmem, int bytes, bool vec16) {
  if (vec16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(bytes));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(bytes));
}

// One operand tile: rows along the contiguous dimension `c` (length CL), outer dimension `o`
// (length OL).  Global element (c, o) lives at base[c + o*ld]; shared at sm[o*SLD + c].
template <int CL, int OL, int SLD, int NT, int V>
__device__ __forceinline__ void load_tile(double* sm, const double* base, int64_t ld, int64_t c0,
                                          int64_t o0, int64_t c_lim, int64_t o_lim,
                                          const int* omap, int tid) {
  constexpr int CPR = CL / V;             // chunks per outer row
  constexpr int TOT = CPR * OL;
  constexpr int STEP = NT / CPR;          // outer rows covered per pass
  static_assert(NT % CPR == 0 && TOT % NT == 0, "tile/thread mismatch");
  const int cc = (tid % CPR) * V;
  const int orow = tid / CPR;
  const int64_t gc = c0 + cc;
  int vbytes = 0;
  if (gc < c_lim) vbytes = (int)((c_lim - gc >= V ? V : c_lim - gc) * 8);
#pragma unroll
  for (int i = 0; i < TOT / NT; ++i) {
    const int o = orow + i * STEP;
    const int64_t go = o0 + o;
    const bool ok = go < o_lim && vbytes > 0;
    const int64_t col = omap ? (ok ? (int64_t)omap[go] : 0) : go;
    const double* src = ok ? base + gc + col * ld : base;
    cp_async_vec(sm + o * SLD + cc, src, ok ? vbytes : 0, V == 2);
  }
}

// load_tile for a tile known to lie inside the operand (no bounds, no gather, 16-byte chunks)
template <int CL, int OL, int SLD, int NT>
__device__ __forceinline__ void load_tile_inner(double* sm, const double* base, int64_t ld,
                                                int64_t c0, int64_t o0, int tid) {
  constexpr int CPR = CL / 2;
  constexpr int TOT = CPR * OL;
  constexpr int STEP = NT / CPR;
  static_assert(NT % CPR == 0 && TOT % NT == 0, "tile/thread mismatch");
  const int cc = (tid % CPR) * 2;
  const int orow = tid / CPR;
  const double* src = base + (c0 + cc) + (o0 + orow) * ld;
  const int64_t sstep = (int64_t)STEP * ld;
#pragma unroll
  for (int i = 0; i < TOT / NT; ++i)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                     smem_u32(sm + (orow + i * STEP) * SLD + cc)),
                 "l"(src + i * sstep));
}

// load_tile_inner with the outer (k) index gathered through omap (the D&C merge's column map)
template <int CL, int OL, int SLD, int NT>
__device__ __forceinline__ void load_tile_inner_map(double* sm, const double* base, int64_t ld,
                                                    int64_t c0, int64_t o0, const int* omap,
                                                    int tid) {
  constexpr int CPR = CL / 2;
  constexpr int TOT = CPR * OL;
  constexpr int STEP = NT / CPR;
  const int cc = (tid % CPR) * 2;
  const int orow = tid / CPR;
  const double* src = base + (c0 + cc);
#pragma unroll
  for (int i = 0; i < TOT / NT; ++i) {
    const int o = orow + i * STEP;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                     smem_u32(sm + o * SLD + cc)),
                 "l"(src + (int64_t)__ldg(omap + o0 + o) * ld));
  }
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, int V,
          bool SYM = false>
__device__ __forceinline__ void fast_tile(const GemmArgs& g, int64_t i0, int64_t j0, int64_t kbeg,
                                          int64_t kend, double* ws_out, int64_t ws_ld,
                                          double* smem) {
  using C = FCfg<TA, TB, BM, BN, BK, WM, WN, STAGES, SYM>;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  double* As = smem;
  double* Bs = smem + STAGES * C::A_STAGE;
  double acc[C::MI][C::NI][2];
  // beta != 0: start the accumulators at (beta/alpha) C, so the epilogue is a plain store and the
  // C reads overlap the pipeline prologue instead of trailing the (short-K) main loop
  const bool preload = (ws_out == nullptr) && g.beta != 0.0 && g.alpha != 0.0 && g.preload;
  {
    const double sc = preload ? g.beta / g.alpha : 0.0;
    const int r_in = lane >> 2, c_in = 2 * (lane & 3);
#pragma unroll
    for (int a = 0; a < C::MI; ++a) {
      const int64_t gi = i0 + wm * WM + a * 8 + r_in;
#pragma unroll
      for (int b = 0; b < C::NI; ++b) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double v = 0.0;
          const int64_t gj = j0 + wn * WN + b * 8 + c_in + h;
          if (preload && gi < g.m && gj < g.n) {
            const int64_t cj = g.cmap ? (int64_t)g.cmap[gj] : gj;
            v = sc * g.C[gi + cj * g.ldc];
          }
          acc[a][b][h] = v;
        }
      }
    }
  }

  // symmetric-lower A (A_SYM_LOWER): per k-tile, tiles on/below the diagonal are read as stored
  // (m-contiguous), tiles above it from their mirror below the diagonal (k-contiguous layout),
  // and the few tiles crossing the diagonal element by element.
  auto sym_mode = [&](int64_t k0) { return (k0 + BK - 1 <= i0) ? 0 : (k0 >= i0 + BM ? 1 : 2); };
  auto load_stage = [&](int st, int64_t k0) {
    double* as = As + st * C::A_STAGE;
    double* bs = Bs + st * C::B_STAGE;
    if (SYM) {
      const int md = sym_mode(k0);
      if (md == 0)
        load_tile<BM, BK, C::A_LD0, C::NT, V>(as, g.A, g.lda, i0, k0, g.m, kend, nullptr, tid);
      else if (md == 1)
        load_tile<BK, BM, C::A_LD1, C::NT, V>(as, g.A, g.lda, k0, i0, kend, g.m, nullptr, tid);
      else
        for (int idx = tid; idx < BM * BK; idx += C::NT) {
          const int i = idx % BM, kk = idx / BM;
          const int64_t gi = i0 + i, gk = k0 + kk;
          const bool ok = gi < g.m && gk < kend;
          const double* src = (gi >= gk) ? g.A + gi + gk * g.lda : g.A + gk + gi * g.lda;
          cp_async8(as + kk * C::A_LD0 + i, ok ? src : g.A, ok);
        }
    } else if (!TA)  // A[m + k*lda]: contiguous m, outer k (optionally gathered by amap)
      load_tile<BM, BK, C::A_LD, C::NT, V>(as, g.A, g.lda, i0, k0, g.m, kend, g.amap, tid);
    else      // A[k + m*lda]: contiguous k, outer m
      load_tile<BK, BM, C::A_LD, C::NT, V>(as, g.A, g.lda, k0, i0, kend, g.m, nullptr, tid);
    if (!TB)  // B[k + n*ldb]: contiguous k, outer n
      load_tile<BK, BN, C::B_LD, C::NT, V>(bs, g.B, g.ldb, k0, j0, kend, g.n, nullptr, tid);
    else      // B[n + k*ldb]: contiguous n, outer k
      load_tile<BN, BK, C::B_LD, C::NT, V>(bs, g.B, g.ldb, j0, k0, g.n, kend, nullptr, tid);
  };

  // interior tiles (the bulk of every large GEMM): unpredicated 16-byte copies
  const bool inner = V == 2 && (g.amap == nullptr || !TA) && i0 + BM <= g.m && j0 + BN <= g.n;
  const int64_t kfull = kbeg + (kend - kbeg) / BK * BK;  // k-tiles below this are complete
  auto load_stage_any = [&](int st, int64_t k0) {
    if (inner && k0 + BK <= kfull && (!SYM || sym_mode(k0) != 2)) {
      double* as = As + st * C::A_STAGE;
      double* bs = Bs + st * C::B_STAGE;
      if (SYM) {  // a whole tile below (as stored) or above (its mirror) the diagonal
        if (sym_mode(k0) == 0) load_tile_inner<BM, BK, C::A_LD0, C::NT>(as, g.A, g.lda, i0, k0, tid);
        else load_tile_inner<BK, BM, C::A_LD1, C::NT>(as, g.A, g.lda, k0, i0, tid);
      } else if (!TA) {
        if (g.amap)
          load_tile_inner_map<BM, BK, C::A_LD, C::NT>(as, g.A, g.lda, i0, k0, g.amap, tid);
        else
          load_tile_inner<BM, BK, C::A_LD, C::NT>(as, g.A, g.lda, i0, k0, tid);
      } else {
        load_tile_inner<BK, BM, C::A_LD, C::NT>(as, g.A, g.lda, k0, i0, tid);
      }
      if (!TB) load_tile_inner<BK, BN, C::B_LD, C::NT>(bs, g.B, g.ldb, k0, j0, tid);
      else     load_tile_inner<BN, BK, C::B_LD, C::NT>(bs, g.B, g.ldb, j0, k0, tid);
    } else {
      load_stage(st, k0);
    }
  };
  const int64_t KT = (kend - kbeg + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage_any(s, kbeg + s * BK);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t pf = kt + STAGES - 1;
      if (pf < KT) load_stage_any((int)(pf % STAGES), kbeg + pf * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * C::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * C::B_STAGE;
    const int r8 = lane >> 2, c4 = lane & 3;
    const bool a_kc = SYM ? (sym_mode(kbeg + kt * BK) == 1) : TA;  // k-contiguous A layout
#pragma unroll
    for (int k8 = 0; k8 < BK; k8 += 8) {
      const int kr = k8 + 2 * c4;  // k-step h of this pair uses k = kr + h in lane c4's slot
      double af[2][C::MI], bf[2][C::NI];
#pragma unroll
      for (int a = 0; a < C::MI; ++a) {
        const int r = wm * WM + a * 8 + r8;
        if (a_kc) {
          const double2 t = *reinterpret_cast<const double2*>(as + r * C::A_LD1 + kr);
          af[0][a] = t.x;
          af[1][a] = t.y;
        } else {
          af[0][a] = as[kr * C::A_LD0 + r];
          af[1][a] = as[(kr + 1) * C::A_LD0 + r];
        }
      }
#pragma unroll
      for (int b = 0; b < C::NI; ++b) {
        const int c = wn * WN + b * 8 + r8;
        if (TB) {
          bf[0][b] = bs[kr * C::B_LD + c];
          bf[1][b] = bs[(kr + 1) * C::B_LD + c];
        } else {
          const double2 t = *reinterpret_cast<const double2*>(bs + c * C::B_LD + kr);
          bf[0][b] = t.x;
          bf[1][b] = t.y;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int a = 0; a < C::MI; ++a)
#pragma unroll
          for (int b = 0; b < C::NI; ++b)
            dmma884(acc[a][b][0], acc[a][b][1], af[h][a], bf[h][b]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  const int r_in = lane >> 2, c_in = 2 * (lane & 3);
  constexpr int LDC = BM + 2;  // staged tile pitch: 8 rows x 4 column pairs hit distinct banks
  if (ws_out == nullptr && !preload && BN * LDC <= STAGES * (C::A_STAGE + C::B_STAGE)) {
    // Epilogue through shared memory: the accumulators are staged as a column-major tile, then
    // every warp streams whole columns (BM contiguous rows) of C with 16-byte accesses, reading
    // C (beta != 0) and writing the result in full lines.
    double* Cs = smem;
#pragma unroll
    for (int a = 0; a < C::MI; ++a)
#pragma unroll
      for (int b = 0; b < C::NI; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          Cs[(wn * WN + b * 8 + c_in + h) * LDC + wm * WM + a * 8 + r_in] = acc[a][b][h];
    __syncthreads();
    const bool vec = ((uintptr_t)g.C % 16 == 0) && (g.ldc % 2 == 0);
    constexpr int PAIRS = BM / 2;
    constexpr int TOT = BN * PAIRS;
    constexpr int EB = 8;  // C reads issued together: one memory round trip per 8 pairs
    const bool full = vec && i0 + BM <= g.m && j0 + BN <= g.n;
    for (int e0 = tid; e0 < TOT; e0 += EB * C::NT) {
      if (full) {
        double* cps[EB];
        double2 cv[EB];
#pragma unroll
        for (int u = 0; u < EB; ++u) {
          const int e = e0 + u * C::NT;
          const int col = e / PAIRS, rp = (e % PAIRS) * 2;
          const int64_t gj = j0 + col;
          const int64_t cj = g.cmap ? (int64_t)g.cmap[gj] : gj;
          cps[u] = g.C + (i0 + rp) + cj * g.ldc;
          cv[u] = (e < TOT && g.beta != 0.0) ? *reinterpret_cast<const double2*>(cps[u])
                                             : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < EB; ++u) {
          const int e = e0 + u * C::NT;
          if (e >= TOT) continue;
          const int col = e / PAIRS, rp = (e % PAIRS) * 2;
          double2 o;
          o.x = g.alpha * Cs[col * LDC + rp] + g.beta * cv[u].x;
          o.y = g.alpha * Cs[col * LDC + rp + 1] + g.beta * cv[u].y;
          *reinterpret_cast<double2*>(cps[u]) = o;
        }
        continue;
      }
      for (int u = 0; u < EB; ++u) {
        const int e = e0 + u * C::NT;
        if (e >= TOT) break;
        const int col = e / PAIRS, rp = (e % PAIRS) * 2;
        const int64_t gj = j0 + col, gi = i0 + rp;
        if (gj >= g.n || gi >= g.m) continue;
        const int64_t cj = g.cmap ? (int64_t)g.cmap[gj] : gj;
        double* cp = g.C + gi + cj * g.ldc;
        const double v0 = g.alpha * Cs[col * LDC + rp], v1 = g.alpha * Cs[col * LDC + rp + 1];
        if (vec && gi + 1 < g.m) {
          double2 o;
          if (g.beta != 0.0) {
            const double2 c = *reinterpret_cast<const double2*>(cp);
            o.x = v0 + g.beta * c.x;
            o.y = v1 + g.beta * c.y;
          } else {
            o.x = v0;
            o.y = v1;
          }
          *reinterpret_cast<double2*>(cp) = o;
        } else {
          cp[0] = (g.beta == 0.0) ? v0 : v0 + g.beta * cp[0];
          if (gi + 1 < g.m) cp[1] = (g.beta == 0.0) ? v1 : v1 + g.beta * cp[1];
        }
      }
    }
    return;
  }
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
          *cp = (g.beta == 0.0 || preload) ? v : v + g.beta * *cp;
        }
      }
    }
  }
}

// 16-byte chunks need every chunk start 16B aligned: base aligned, ld even, tile origins even
__device__ __host__ __forceinline__ bool vec_ok(const GemmArgs& g) {
  return ((uintptr_t)g.A % 16 == 0) && ((uintptr_t)g.B % 16 == 0) && (g.lda % 2 == 0) &&
         (g.ldb % 2 == 0);
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, bool SYM>
__global__ void __launch_bounds__(FCfg<TA, TB, BM, BN, BK, WM, WN, STAGES, SYM>::NT)
    gemm_fast_kernel(const __grid_constant__ GemmArgs g, int ksplit, double* ws) {
  extern __shared__ __align__(16) double smem[];
  int64_t i0 = (int64_t)blockIdx.x * BM, j0 = (int64_t)blockIdx.y * BN;
  if (g.cmode == C_LOWER_TILES) {
    // 1-D grid over the tiles intersecting the lower triangle, column by column
    const int64_t RT = (g.m + BM - 1) / BM;
    int64_t idx = blockIdx.x, tj = 0;
    for (;; ++tj) {
      const int64_t lo = tj * BN - BM + 1;
      const int64_t tmin = lo <= 0 ? 0 : (lo + BM - 1) / BM;
      const int64_t cnt = RT > tmin ? RT - tmin : 0;
      if (idx < cnt) {
        i0 = (tmin + idx) * BM;
        break;
      }
      idx -= cnt;
    }
    j0 = tj * BN;
  }
  int64_t kbeg = 0, kend = g.k;
  double* wsp = nullptr;
  if (ksplit > 1) {
    const int64_t chunk = ((g.k + ksplit - 1) / ksplit + BK - 1) / BK * BK;
    kbeg = blockIdx.z * chunk;
    kend = kbeg + chunk < g.k ? kbeg + chunk : g.k;
    if (kbeg > kend) kbeg = kend;
    wsp = ws + (int64_t)blockIdx.z * g.m * g.n;
  }
  if (vec_ok(g))
    fast_tile<TA, TB, BM, BN, BK, WM, WN, STAGES, 2, SYM>(g, i0, j0, kbeg, kend, wsp, g.m, smem);
  else
    fast_tile<TA, TB, BM, BN, BK, WM, WN, STAGES, 1, SYM>(g, i0, j0, kbeg, kend, wsp, g.m, smem);
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(FCfg<TA, TB, BM, BN, BK, WM, WN, STAGES>::NT)
    gemm_fast_grouped_kernel(const GemmArgs* __restrict__ args) {
  extern __shared__ __align__(16) double smem[];
  const GemmArgs g = args[blockIdx.z];
  const int64_t i0 = (int64_t)blockIdx.x * BM, j0 = (int64_t)blockIdx.y * BN;
  if (g.m <= 0 || g.n <= 0 || i0 >= g.m || j0 >= g.n) return;
  if (g.cmode == C_LOWER_TILES && i0 + BM - 1 < j0) return;
  const int64_t k = g.k > 0 ? g.k : 0;
  if (vec_ok(g))
    fast_tile<TA, TB, BM, BN, BK, WM, WN, STAGES, 2>(g, i0, j0, 0, k, nullptr, 0, smem);
  else
    fast_tile<TA, TB, BM, BN, BK, WM, WN, STAGES, 1>(g, i0, j0, 0, k, nullptr, 0, smem);
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, bool SYM = false>
int launch_fast(cudaStream_t st, const GemmArgs& g, int ksplit, double* ws) {
  using C = FCfg<TA, TB, BM, BN, BK, WM, WN, STAGES, SYM>;
  auto kern = gemm_fast_kernel<TA, TB, BM, BN, BK, WM, WN, STAGES, SYM>;
  static int attr_dev = -1;
  int dev;
  PEVD_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    PEVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_dev = dev;
  }
  dim3 grid((unsigned)cdiv(g.m, BM), (unsigned)cdiv(g.n, BN), ksplit);
  if (g.cmode == C_LOWER_TILES) {  // only the tiles intersecting the lower triangle
    int64_t cnt = 0;
    const int64_t RT = cdiv(g.m, BM);
    for (int64_t tj = 0; tj < cdiv(g.n, BN); ++tj) {
      const int64_t lo = tj * BN - BM + 1;
      const int64_t tmin = lo <= 0 ? 0 : (lo + BM - 1) / BM;
      cnt += RT > tmin ? RT - tmin : 0;
    }
    if (cnt == 0) return OK;
    grid = dim3((unsigned)cnt, 1, ksplit);
  }
  kern<<<grid, C::NT, C::SMEM, st>>>(g, ksplit, ws);
  PEVD_LAUNCH_CHECK();
  return OK;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
int launch_fast_t(cudaStream_t st, const GemmArgs& g, int ksplit, double* ws) {
  if (!g.transA && !g.transB) return launch_fast<false, false, BM, BN, BK, WM, WN, STAGES>(st, g, ksplit, ws);
  if (g.transA && !g.transB) return launch_fast<true, false, BM, BN, BK, WM, WN, STAGES>(st, g, ksplit, ws);
  if (!g.transA && g.transB) return launch_fast<false, true, BM, BN, BK, WM, WN, STAGES>(st, g, ksplit, ws);
  return launch_fast<true, true, BM, BN, BK, WM, WN, STAGES>(st, g, ksplit, ws);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
int launch_fast_grouped(cudaStream_t st, const GemmArgs* d_args, int count, int64_t max_m,
                        int64_t max_n) {
  // grouped problems of the D&C merge: A column-gathered, not transposed; B not transposed
  using C = FCfg<false, false, BM, BN, BK, WM, WN, STAGES>;
  auto kern = gemm_fast_grouped_kernel<false, false, BM, BN, BK, WM, WN, STAGES>;
  static int attr_dev = -1;
  int dev;
  PEVD_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    PEVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_dev = dev;
  }
  dim3 grid((unsigned)cdiv(max_m, BM), (unsigned)cdiv(max_n, BN), count);
  kern<<<grid, C::NT, C::SMEM, st>>>(d_args);
  PEVD_LAUNCH_CHECK();
  return OK;
}

int splitk_finish(cudaStream_t st, const GemmArgs& g, int ks, double* ws) {
  splitk_reduce<<<(unsigned)std::min<int64_t>(cdiv(g.m * g.n, 256), 4 * num_sms()), 256, 0, st>>>(
      ws, ks, g.m, g.n, g.alpha, g.beta, g.C, g.ldc, g.cmap);
  PEVD_LAUNCH_CHECK();
  return OK;
}

}  // namespace

// Split-K factor for a grid of `tiles` CTA tiles when `slots` CTAs are resident at once: the
// number of chunks (each >= min_chunk deep) whose wave count wastes the least of the last wave,
// with a 1.5% charge per extra chunk for the partial-sum traffic and the reduction.
static int pick_ks(int64_t tiles, int64_t k, int64_t slots, int64_t min_chunk, int64_t mn,
                   int64_t ws_elems) {
  if (tiles >= 8 * slots || k < 2 * min_chunk) return 1;
  if (tiles * (k / min_chunk) < slots / 2) {
    // a tiny output with a long K (W^T AW of the band reduction: 32 x 32, K = m): even the
    // deepest split below leaves most SMs idle and each CTA latency-bound on a long K loop, so
    // split to 128-deep chunks across the whole GPU (one reduction pass sums them in order)
    int64_t ks = std::min<int64_t>(k / 128, slots / tiles);
    while (ks > 1 && ks * mn > ws_elems) --ks;
    return (int)std::max<int64_t>(ks, 1);
  }
  const int64_t kmax = std::min<int64_t>(k / min_chunk, 32);
  int best = 1;
  double best_eff = 0.0;
  for (int64_t ks = 1; ks <= kmax; ++ks) {
    if (ks > 1 && ks * mn > ws_elems) break;
    const int64_t ctas = tiles * ks;
    const double eff = (double)ctas / (double)(slots * cdiv(ctas, slots)) * (1.0 - 0.015 * (ks - 1));
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = (int)ks;
    }
  }
  return best;
}

// executed flops of the grouped problems (sizes live on the device), into this thread's counter
__global__ void grouped_flops_kernel(const GemmArgs* __restrict__ a, int count, int stage,
                                     unsigned long long* __restrict__ acc) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const GemmArgs& g = a[i];
    if (g.m > 0 && g.n > 0 && g.k > 0) s += 2ull * g.m * g.n * g.k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(acc + stage, s);
}

static void count_gemm_flops(const GemmArgs& g) {
  double f = 2.0 * (double)g.m * (double)g.n * (double)g.k;
  if (g.cmode == C_LOWER_TILES && g.m == g.n) f *= 0.5 * (1.0 + 64.0 / (double)g.m);
  flops_add(f);
}

int gemm(cudaStream_t st, const GemmArgs& g0, double* ws, int64_t ws_elems) {
  if (g0.m <= 0 || g0.n <= 0) return OK;
  count_gemm_flops(g0);
  static int pre = -1;
  if (pre < 0) {
    const char* e = getenv("PEVD_PRELOAD");
    pre = e ? atoi(e) : 0;
  }
  GemmArgs g = g0;
  g.preload = pre;
  const int sms = num_sms();
  if (g.amode == A_SYM_LOWER) {
    // symmetric operand read from its lower triangle (A W of the band reduction): N is small
    const int64_t tiles = cdiv(g.m, 128) * cdiv(g.n, 32);
    const int ks = ws ? pick_ks(tiles, g.k, 2 * sms, 512, g.m * g.n, ws_elems) : 1;
    if (g.n <= 32) {
      // 4 warps of 32 x 32, BK = 16, 3 stages: 79 KB of shared memory -> 2 CTAs/SM; 8 LDS per
      // 16 DMMA (27-28 TF/s at m = 24576-49152 vs 23-24 for 8 warps of 16 x 32; 64-row tiles
      // with 2 warps lose at every m from 4096 to 32768, e.g. 27.5 vs 28.8 TF/s at 16384)
      if (g.transB) PEVD_TRY((launch_fast<false, true, 128, 32, 16, 32, 32, 3, true>(st, g, ks, ks > 1 ? ws : nullptr)));
      else PEVD_TRY((launch_fast<false, false, 128, 32, 16, 32, 32, 3, true>(st, g, ks, ks > 1 ? ws : nullptr)));
      if (ks > 1) PEVD_TRY(splitk_finish(st, g, ks, ws));
      return OK;
    }
    if (g.n <= 64) {
      // panels of 33..64 columns (b > 32): 128 x 64 tiles, 8 warps of 32 x 32
      const int ks64 = ws ? pick_ks(cdiv(g.m, 128), g.k, 2 * sms, 512, g.m * g.n, ws_elems) : 1;
      if (g.transB) PEVD_TRY((launch_fast<false, true, 128, 64, 16, 32, 32, 3, true>(st, g, ks64, ks64 > 1 ? ws : nullptr)));
      else PEVD_TRY((launch_fast<false, false, 128, 64, 16, 32, 32, 3, true>(st, g, ks64, ks64 > 1 ? ws : nullptr)));
      if (ks64 > 1) PEVD_TRY(splitk_finish(st, g, ks64, ws));
      return OK;
    }
    return launch_generic<128, 128, 16, 64, 32, 3>(st, g, 1, nullptr);
  }
  if (g.n <= 32) {
    // skinny: 128 x 32 tiles, split K when the grid is thin
    const int64_t tiles = cdiv(g.m, 128);
    static int chunk = -1;  // PEVD_SKINNY_CHUNK: smallest split-K chunk (tuning knob)
    if (chunk < 0) {
      const char* e = getenv("PEVD_SKINNY_CHUNK");
      chunk = e ? std::max(64, atoi(e)) : 512;
    }
    const int ks = (ws && g.cmode == C_ALL) ? pick_ks(tiles, g.k, 2 * sms, chunk, g.m * g.n, ws_elems)
                                            : 1;
    // 8 warps of 16 x 32, BK = 16, 3 stages (<= 92 KB: 2 CTAs/SM); 31 TF/s at 49152 x 32 x 49152
    PEVD_TRY((launch_fast_t<128, 32, 16, 16, 32, 3>(st, g, ks, ks > 1 ? ws : nullptr)));
    if (ks > 1) PEVD_TRY(splitk_finish(st, g, ks, ws));
    return OK;
  }
  const int64_t tiles = cdiv(g.m, 64) * cdiv(g.n, 128);
  // lower-triangle updates (the band reduction's rank-2K): 64 x 64 tiles, 4 stages, 3 CTAs/SM --
  // half the diagonal-tile waste and finer balance: 2.40 s vs 2.48 s per n = 49152 SBR (plain
  // GEMMs stay on 64 x 128, which is 5% faster there: 33.4 vs 31.8 TF/s at 24576^2 x 1024)
  if (g.cmode == C_LOWER_TILES && tiles >= sms)
    return launch_fast_t<64, 64, 16, 32, 32, 4>(st, g, 1, nullptr);
  if (tiles >= sms || g.k < 64) {
    // 64 x 128 CTA tiles, 4 warps of 32 x 64, BK = 16, 3 stages: 87.5 KB of shared memory and
    // <= 224 registers, so two CTAs share an SM and one's barrier/epilogue hides under the
    // other's DMMAs (the cuBLAS d884 configuration; 32.5 TF/s on 8192^3 vs 30.8 for 128 x 128)
    return launch_fast_t<64, 128, 16, 32, 64, 3>(st, g, 1, nullptr);
  }
  const int64_t tiles64 = cdiv(g.m, 64) * cdiv(g.n, 64);
  int ks = 1;
  if (ws && tiles64 < sms && g.k >= 512 && g.cmode == C_ALL) {
    ks = (int)std::min<int64_t>(cdiv(2 * sms, tiles64), g.k / 128);
    while (ks > 1 && (int64_t)ks * g.m * g.n > ws_elems) --ks;
  }
  PEVD_TRY((launch_fast_t<64, 64, 16, 32, 32, 4>(st, g, ks, ks > 1 ? ws : nullptr)));
  if (ks > 1) PEVD_TRY(splitk_finish(st, g, ks, ws));
  return OK;
}

int gemm_grouped(cudaStream_t st, const GemmArgs* d_args, int count, int64_t max_m,
                 int64_t max_n) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return OK;
  if (unsigned long long* acc = flops_dev()) {
    grouped_flops_kernel<<<1, 256, 0, st>>>(d_args, count, flops_stage(), acc);
    PEVD_LAUNCH_CHECK();
  }
  if (max_m * max_n >= (int64_t)128 * 128 * 64)
    return launch_fast_grouped<64, 128, 16, 32, 64, 3>(st, d_args, count, max_m, max_n);
  return launch_fast_grouped<64, 64, 16, 32, 32, 4>(st, d_args, count, max_m, max_n);
}

}  // namespace pevd
