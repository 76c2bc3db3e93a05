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
#include <cstdio>
#include <cstdlib>
#include <vector>
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

static constexpr int64_t SPLITK_ELEMS = 16 << 20;  // A W at m = 49152 wants 3-4 K chunks (1.6 M each)
static constexpr int64_t SPLITK2_ELEMS = 1 << 20;  // split-K of the side stream's P2^T W
static constexpr int NBB_MAX = 16;  // workspace bound on the panels per double-blocked update

// panels per double-blocked trailing update (rank 2 * nbb * b); PEVD_NBB overrides (tuning)
static int sbr_nbb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PEVD_NBB");
    v = e ? atoi(e) : 16;
    if (v < 1) v = 1;
    if (v > NBB_MAX) v = NBB_MAX;
  }
  return v;
}

int64_t sbr_ws_bytes(int64_t n, int b) {
  // P1, P2 (n x 2*NBB*b each) + W (n x b) + M, R, coupling (b x b) + t (2*NBB*b x b) + split-K + QR
  const int64_t K = (int64_t)NBB_MAX * b;
  return (n * 4 * K + n * b + 3 * (int64_t)b * b + 2 * K * b + SPLITK_ELEMS + SPLITK2_ELEMS) * 8 +
         panel_qr_ws_bytes() + 1024;
}

namespace {

struct SbrWs {
  double *YZY, *Wb, *Mb, *Rb, *Cp, *tZ, *tY, *sk, *sk2;
  void* qrws;
  int64_t ldz;
};

// the single-panel round (used for the ragged last round, sbr.py:175-182 coupling)
int sbr_single_round(cudaStream_t st, int64_t n, int b, double* A, int64_t lda, double* bands,
                     double* Tall, const SbrWs& W, int64_t x) {
  const int64_t c0 = x * b;
  const int64_t pw = std::min<int64_t>(b, n - b - c0);
  const int64_t t0 = c0 + b;
  const int64_t m = n - t0;
  const int64_t ldz = W.ldz;
  double* panel = A + t0 + c0 * lda;
  double* A22 = A + t0 + t0 * lda;
  double* Tx = Tall ? Tall + x * (int64_t)b * b : nullptr;
  double* Yz = W.YZY;
  double* Zz = W.YZY + pw * ldz;
  double* Y3 = W.YZY + 2 * pw * ldz;
  PEVD_TRY(panel_qr(st, m, (int)pw, panel, lda, W.Rb, panel, lda, Yz, ldz, W.Wb, n, Tx, W.qrws));
  band_cols_from_panel<<<1, 256, 0, st>>>(n, b, c0, (int)pw, A, lda, W.Rb, bands);
  PEVD_LAUNCH_CHECK();
  PEVD_CUDA(cudaMemcpy2DAsync(Y3, ldz * 8, Yz, ldz * 8, m * 8, pw, cudaMemcpyDeviceToDevice, st));
  if (pw < b) {
    const int64_t nc = b - pw;
    double* cpl = A + t0 + (c0 + pw) * lda;
    GemmArgs g1{pw, nc, m, 1.0, 0.0, W.Wb, n, cpl, lda, W.Cp, pw, 1, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g1, W.sk, SPLITK_ELEMS));
    GemmArgs g2{m, nc, pw, -1.0, 1.0, Yz, ldz, W.Cp, pw, cpl, lda, 0, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g2, W.sk, SPLITK_ELEMS));
  }
  GemmArgs g_aw{m, pw, m, 1.0, 0.0, A22, lda, W.Wb, n, Zz, ldz, 0, 0, A_SYM_LOWER, C_ALL};
  PEVD_TRY(gemm(st, g_aw, W.sk, SPLITK_ELEMS));
  GemmArgs g_m{pw, pw, m, 1.0, 0.0, W.Wb, n, Zz, ldz, W.Mb, pw, 1, 0, A_GENERAL, C_ALL};
  PEVD_TRY(gemm(st, g_m, W.sk, SPLITK_ELEMS));
  GemmArgs g_z{m, pw, pw, -0.5, 1.0, Yz, ldz, W.Mb, pw, Zz, ldz, 0, 0, A_GENERAL, C_ALL};
  PEVD_TRY(gemm(st, g_z, W.sk, SPLITK_ELEMS));
  GemmArgs g_u{m, m, 2 * pw, -1.0, 1.0, Yz, ldz, Zz, ldz, A22, lda, 0, 1, A_GENERAL, C_LOWER_TILES};
  PEVD_TRY(gemm(st, g_u, nullptr, 0));
  return OK;
}

// A high-priority side stream for the work of a panel that is off the critical path
// (QR -> A W -> Z -> next panel): the copy of Y_i into P2, the panel's band columns and
// t = P2^T W_i.  They run under the symmetric A W GEMM (its CTAs are scheduled first, ahead of
// the A W tail wave) and are joined before the correction AW_i -= P1 t.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool joined = false;  // every side task is ordered before later work on the main stream
  int init() {
    int lo, hi;
    PEVD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    PEVD_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
    PEVD_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    PEVD_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    return OK;
  }
  ~SideStream() {
    if (s && !joined) cudaStreamSynchronize(s);  // error path: nothing may run on after return
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (s) cudaStreamDestroy(s);
  }
};

// PEVD_SBR_PROF=1: CUDA events between the phases on the main stream, summed per phase and
// printed to stderr at the end (a measurement mode: it synchronises once at the end).
struct SbrProf {
  enum { MEMSET, G1, QR, AW, GC, GM, GZ, ZCOPY, RANK2K, TAIL, NCAT };
  bool on = false;
  std::vector<std::pair<int, cudaEvent_t>> ev;
  SbrProf() {
    const char* e = getenv("PEVD_SBR_PROF");
    on = e && atoi(e) != 0;
  }
  void mark(cudaStream_t st, int cat) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.emplace_back(cat, e);
  }
  void report() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    static const char* names[NCAT] = {"memset", "g1_pending", "panel_qr", "aw_symm",
                                      "gc_correct", "gm_wtaw", "gz_form", "z_copy", "rank2k",
                                      "tail"};
    double ms[NCAT] = {0};
    for (size_t k = 1; k < ev.size(); ++k) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[k - 1].second, ev[k].second);
      ms[ev[k].first] += t;
    }
    fprintf(stderr, "{\"sbr_prof_ms\": {");
    for (int c = 0; c < NCAT; ++c) fprintf(stderr, "%s\"%s\": %.2f", c ? ", " : "", names[c], ms[c]);
    fprintf(stderr, "}}\n");
    for (auto& p : ev) cudaEventDestroy(p.second);
    ev.clear();
  }
};

}  // namespace

// Double-blocked band reduction.  A block of nbl <= NBB full panels (c0, t0 = c0 + b, m0 = n - t0)
// keeps Y_p and Z_p (block-relative rows [0, m0), zero above their own start) interleaved in
// P1 = [Y_0 Z_0 Y_1 Z_1 ...] and P2 = [Z_0 Y_0 Z_1 Y_1 ...]; for panel i of the block:
//   1. its columns (rows from the panel's diagonal block down) receive the pending updates of
//      panels 0..i-1:  C -= Y_p Z_p^T + Z_p Y_p^T = P1 P2^T   (one skinny GEMM)
//   2. panel QR; its band columns are now final
//   3. AW_i = A_blockstart[t_i:, t_i:] W_i  - P1 (P2^T W_i)
//   4. Z_i = AW_i - 1/2 Y_i (W_i^T AW_i)
// then one rank-2*nbl*b update of the remaining trailing matrix (lower tiles):
//   A[t0+(nbl-1)b:, same] -= P1 P2^T.
int sbr_reduce(cudaStream_t st, int64_t n, int b, double* A, int64_t lda, double* bands_ref,
               double* Tall, void* ws) {
  if (b < 1 || n < 2 || b >= n) {
    set_error("sbr_reduce: need 1 <= b < n (n=%lld, b=%d)", (long long)n, b);
    return ERR_VALUE;
  }
  const int NBB = sbr_nbb();
  const int64_t Kmax = (int64_t)NBB * b;
  SbrWs W;
  W.ldz = n;
  W.YZY = (double*)ws;
  W.Wb = W.YZY + n * 4 * Kmax;
  W.Mb = W.Wb + n * b;
  W.Rb = W.Mb + (int64_t)b * b;
  W.Cp = W.Rb + (int64_t)b * b;
  W.tZ = W.Cp + (int64_t)b * b;
  W.tY = W.tZ + Kmax * b;
  W.sk = W.tY + Kmax * b;
  W.sk2 = W.sk + SPLITK_ELEMS;
  W.qrws = (void*)(W.sk2 + SPLITK2_ELEMS);
  const int64_t ldz = W.ldz;
  const int64_t R = sbr_num_rounds(n, b);
  int64_t c_end = 0;
  SideStream side;
  PEVD_TRY(side.init());
  const cudaStream_t ss = side.s;
  SbrProf prof;
  prof.mark(st, SbrProf::TAIL);
  for (int64_t x = 0; x < R;) {
    const int64_t c0 = x * b;
    const int64_t pw0 = std::min<int64_t>(b, n - b - c0);
    if (pw0 < b) {  // ragged last round
      PEVD_TRY(sbr_single_round(st, n, b, A, lda, bands_ref, Tall, W, x));
      c_end = c0 + pw0;
      ++x;
      continue;
    }
    int nbl = 1;
    while (nbl < NBB && x + nbl < R && (n - b - (x + nbl) * b) >= b) ++nbl;
    const int64_t t0 = c0 + b, m0 = n - t0;
    const int64_t K = (int64_t)nbl * b;
    // P1 = [Y_0 Z_0 Y_1 Z_1 ...], P2 = [Z_0 Y_0 Z_1 Y_1 ...] (block-relative rows [0, m0)):
    // every sum over the block's panels, sum_q Y_q Z_q^T + Z_q Y_q^T, is then ONE GEMM
    // P1[:, 0:2r] P2[:, 0:2r]^T with contiguous operands
    double* P1 = W.YZY;
    double* P2 = W.YZY + 2 * Kmax * ldz;
    // rows above each panel's start must read as zero
    PEVD_CUDA(cudaMemset2DAsync(P1, ldz * 8, 0, (size_t)K * 8, (size_t)(2 * K), st));
    PEVD_CUDA(cudaMemset2DAsync(P2, ldz * 8, 0, (size_t)K * 8, (size_t)(2 * K), st));
    prof.mark(st, SbrProf::MEMSET);
    for (int i = 0; i < nbl; ++i) {
      const int64_t ci = c0 + (int64_t)i * b, ti = t0 + (int64_t)i * b, mi = n - ti;
      const int64_t ri = (int64_t)i * b;
      double* Yi = P1 + ri + (2 * ri) * ldz;      // Y_i slot of P1, from its start row
      double* Zi = P1 + ri + (2 * ri + b) * ldz;  // Z_i slot of P1
      if (i >= 1) {
        // 1. pending updates on the panel columns, rows [ci, n) = block rows [ri - b, m0):
        //    C -= sum_{q<i} Y_q Z_q^T + Z_q Y_q^T
        double* Cpan = A + ci + ci * lda;
        GemmArgs g1{mi + b, b, 2 * ri, -1.0, 1.0, P1 + (ri - b), ldz, P2 + (ri - b), ldz, Cpan,
                    lda, 0, 1, A_GENERAL, C_ALL};
        PEVD_TRY(gemm(st, g1, W.sk, SPLITK_ELEMS));
        prof.mark(st, SbrProf::G1);
      }
      // 2. panel QR (explicit Y into the staircase and into P1; P2 gets a copy)
      double* panel = A + ti + ci * lda;
      double* Tx = Tall ? Tall + (x + i) * (int64_t)b * b : nullptr;
      PEVD_TRY(panel_qr(st, mi, b, panel, lda, W.Rb, panel, lda, Yi, ldz, W.Wb, n, Tx, W.qrws));
      prof.mark(st, SbrProf::QR);
      // side stream: Y_i into P2, the band columns, t = P2^T W_i (all read only QR outputs and
      // columns of P2 before Y_i's; the next QR rewrites W.Wb / W.Rb only after the join below)
      PEVD_CUDA(cudaEventRecord(side.fork, st));
      PEVD_CUDA(cudaStreamWaitEvent(ss, side.fork, 0));
      PEVD_CUDA(cudaMemcpy2DAsync(P2 + ri + (2 * ri + b) * ldz, ldz * 8, Yi, ldz * 8, mi * 8, b,
                                  cudaMemcpyDeviceToDevice, ss));
      band_cols_from_panel<<<1, 256, 0, ss>>>(n, b, ci, b, A, lda, W.Rb, bands_ref);
      PEVD_LAUNCH_CHECK();
      if (i >= 1) {
        GemmArgs gt{2 * ri, b, mi, 1.0, 0.0, P2 + ri, ldz, W.Wb, n, W.tZ, 2 * ri, 1, 0,
                    A_GENERAL, C_ALL};                              // t = P2^T W_i
        PEVD_TRY(gemm(ss, gt, W.sk2, SPLITK2_ELEMS));
      }
      PEVD_CUDA(cudaEventRecord(side.join, ss));
      // 3. AW_i into the Z slot: A_blockstart W_i - sum_{q<i} (Y_q Z_q^T + Z_q Y_q^T) W_i
      GemmArgs g_aw{mi, b, mi, 1.0, 0.0, A + ti + ti * lda, lda, W.Wb, n, Zi, ldz, 0, 0,
                    A_SYM_LOWER, C_ALL};
      PEVD_TRY(gemm(st, g_aw, W.sk, SPLITK_ELEMS));
      PEVD_CUDA(cudaStreamWaitEvent(st, side.join, 0));
      prof.mark(st, SbrProf::AW);
      if (i >= 1) {
        GemmArgs gc{mi, b, 2 * ri, -1.0, 1.0, P1 + ri, ldz, W.tZ, 2 * ri, Zi, ldz, 0, 0,
                    A_GENERAL, C_ALL};                              // AW_i -= P1 t
        PEVD_TRY(gemm(st, gc, W.sk, SPLITK_ELEMS));
        prof.mark(st, SbrProf::GC);
      }
      // 4. Z_i = AW_i - 1/2 Y_i (W_i^T AW_i), then its copy in P2
      GemmArgs g_m{b, b, mi, 1.0, 0.0, W.Wb, n, Zi, ldz, W.Mb, b, 1, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g_m, W.sk, SPLITK_ELEMS));
      prof.mark(st, SbrProf::GM);
      GemmArgs g_z{mi, b, b, -0.5, 1.0, Yi, ldz, W.Mb, b, Zi, ldz, 0, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g_z, W.sk, SPLITK_ELEMS));
      prof.mark(st, SbrProf::GZ);
      PEVD_CUDA(cudaMemcpy2DAsync(P2 + ri + (2 * ri) * ldz, ldz * 8, Zi, ldz * 8, mi * 8, b,
                                  cudaMemcpyDeviceToDevice, st));
      prof.mark(st, SbrProf::ZCOPY);
    }
    // the block's rank-2K trailing update (lower tiles)
    const int64_t ru = (int64_t)(nbl - 1) * b;
    const int64_t mu = m0 - ru;
    double* Cu = A + (t0 + ru) + (t0 + ru) * lda;
    GemmArgs g_u{mu, mu, 2 * K, -1.0, 1.0, P1 + ru, ldz, P2 + ru, ldz, Cu, lda, 0, 1, A_GENERAL,
                 C_LOWER_TILES};
    PEVD_TRY(gemm(st, g_u, nullptr, 0));
    prof.mark(st, SbrProf::RANK2K);
    c_end = c0 + K;
    x += nbl;
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
  side.joined = true;  // the main stream waited on the last panel's side work
  prof.mark(st, SbrProf::TAIL);
  prof.report();
  return OK;
}

}  // namespace pevd
