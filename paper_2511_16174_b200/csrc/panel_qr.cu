// Tall-skinny Householder panel QR (the SBR panel factorisation, sbr.py:69-116).
//
// One cooperative launch per panel.  Each CTA keeps a contiguous chunk of the m x k panel rows
// resident in shared memory for the whole factorisation (m <= ~65k, k <= 32 -> <= ~120 KB), so
// the panel is read from HBM once and written once.  Per column there is exactly one grid-wide
// reduction: every CTA contributes, for its rows, the tail dot products x_tail^T a_c of the pivot
// column with all remaining columns (which yields ||x_tail||^2 and v^T a_c = a_c[j] +
// x_tail^T a_c,tail / (x0 - alpha) without a second pass) and, lagged by one column, the dot
// products Y(:,0:j-1)^T v_{j-1} that build the T factor (W = Y T, Q = I - W Y^T = I - Y T Y^T).
// Partials are reduced in a fixed order by every CTA, so all CTAs derive bit-identical alpha,
// tau and T, and reruns are bitwise reproducible (no atomics on data).
//
// Householder convention (core.py:238-255): v[0] = 1, alpha = -sign(x0) ||x||, sign(0) = +,
// zero tail -> tau = 0, alpha = x0.
#include <cstdlib>
#include "common.cuh"
#include "kernels.cuh"

namespace pevd {

namespace {

constexpr int QR_THREADS = 512;
constexpr int KMAX = 64;        // widest panel (b <= 64); 32-wide panels run the KM = 32 build

struct QrWork {
  double* part;     // [2][MAXCTA][2 KMAX], double-buffered by step parity
  double* piv;      // [2][KMAX]
  unsigned* bar;    // [2] barrier count / generation
};
constexpr int MAXCTA = 1024;

// Grid barrier on a monotonic arrival counter: every CTA's thread 0 adds 1 with release
// semantics (after the CTA barrier, so the release covers the whole CTA's writes) and polls the
// count relaxed until it reaches (barriers passed) x (CTAs); one acquire re-read then pairs with
// every arrival (each add continues the release sequences before it).  No last-arriver hop: an
// arrival is fire-and-forget and the last add releases everybody directly.  (The previous
// count + generation barrier cost an atomic round trip plus a second release per barrier: the
// grid-barrier wait was 24% of the kernel's stall samples, the poll's ld.acquire an L1
// invalidate per iteration.)  The count starts at 0 per launch (panel_qr's memset).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& gen) {
  __syncthreads();
  if (nblocks == 1) return;  // one CTA: the CTA barrier is the whole barrier
  if (threadIdx.x == 0) {
    ++gen;
    const unsigned target = gen * nblocks;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
  }
  __syncthreads();
}

template <int KM>
__global__ void __launch_bounds__(QR_THREADS)
    panel_qr_kernel(int64_t m, int k, const double* panel, int64_t ldp, double* Rout,
                    double* Y1, int64_t ldy1, double* Y2, int64_t ldy2,
                    double* __restrict__ W, int64_t ldw, double* __restrict__ Tout,
                    QrWork wk, int64_t rows_per_cta) {
  constexpr int LDP = KM + 1;            // smem panel row stride (doubles)
  constexpr int NVAL = 2 * KM;           // partial values per CTA per step: h[0..KM), g[0..KM)
  constexpr int NG = QR_THREADS / NVAL;  // thread groups splitting the rows of a partial
  extern __shared__ __align__(16) double sm[];
  double* P = sm;                                      // [rows_per_cta][LDP]
  double* red = P + rows_per_cta * LDP;                // [4][NVAL]
  double* hv = red + NG * NVAL;                        // [NVAL] reduced values
  double* T = hv + NVAL;                               // [KM][KM] col-major T
  double* coef = T + KM * KM;                      // [KM]
  double* scal = coef + KM;                          // [4]: denom, tau, alpha, flag
  double* taus = scal + 4;                             // [KM]

  const int tid = threadIdx.x;
  const unsigned ncta = gridDim.x;
  unsigned bar_gen = 0;  // barriers passed (thread 0's count; the word starts at 0 per launch)
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = r0 + rows_per_cta < m ? r0 + rows_per_cta : m;
  const int nr = (int)(r1 > r0 ? r1 - r0 : 0);

  // load the row chunk (coalesced along rows, column by column)
  for (int c = 0; c < k; ++c)
    for (int lr = tid; lr < nr; lr += QR_THREADS) P[lr * LDP + c] = panel[r0 + lr + c * ldp];
  for (int i = tid; i < KM * KM; i += QR_THREADS) T[i] = 0.0;
  __syncthreads();

  for (int j = 0; j <= k; ++j) {
    // ---- partial sums for this CTA's rows
    {
      const int vi = tid % NVAL, grp = tid / NVAL;  // NG groups
      double s = 0.0;
      if (vi < KM) {
        const int c = vi;
        if (j < k && c >= j && c < k) {
          double s1 = 0.0;
          int lr = grp;
          for (; lr + NG < nr; lr += 2 * NG) {
            const int64_t r = r0 + lr;
            if (r > j) s += P[lr * LDP + j] * P[lr * LDP + c];
            if (r + NG > j) s1 += P[(lr + NG) * LDP + j] * P[(lr + NG) * LDP + c];
          }
          for (; lr < nr; lr += NG) {
            const int64_t r = r0 + lr;
            if (r > j) s += P[lr * LDP + j] * P[lr * LDP + c];
          }
          s += s1;
        }
      } else {
        const int q = vi - KM;
        const int jp = j - 1;  // previous reflector
        if (jp >= 1 && q < jp) {
          for (int lr = grp; lr < nr; lr += NG) {
            const int64_t r = r0 + lr;
            if (r >= jp) {
              const double v = (r == jp) ? 1.0 : P[lr * LDP + jp];
              s += P[lr * LDP + q] * v;
            }
          }
        }
      }
      red[grp * NVAL + vi] = s;
    }
    // the CTA holding the pivot row publishes it
    // (buffers alternate by step parity: a CTA can run at most one barrier ahead, so it never
    //  overwrites values a slower CTA has yet to read)
    double* part = wk.part + (j & 1) * (MAXCTA * NVAL);
    double* piv = wk.piv + (j & 1) * KM;
    if (j < k && j >= r0 && j < r1 && tid < k) {
      piv[tid] = P[(j - r0) * LDP + tid];
    }
    __syncthreads();
    if (tid < NVAL) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NG; ++q) s += red[q * NVAL + tid];
      part[(int64_t)blockIdx.x * NVAL + tid] = s;
    }
    grid_barrier(wk.bar, ncta, bar_gen);
    // ---- deterministic reduction of all CTA partials (identical in every CTA)
    {
      const int vi = tid % NVAL, grp = tid / NVAL;
      // all of this thread's partials (CTAs grp, grp+NG, ...) are loaded before any is summed:
      // one L2 round trip per 40 CTAs instead of one per 16, in a fixed order
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
      for (unsigned base = grp; base < ncta; base += NG * 40) {
        double v[40];
#pragma unroll
        for (int q = 0; q < 40; ++q) {
          const unsigned p = base + NG * q;
          v[q] = p < ncta ? __ldcg(part + (int64_t)p * NVAL + vi) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 40; ++q) acc[q & 7] += v[q];
      }
      red[grp * NVAL + vi] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) +
                             ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    }
    __syncthreads();
    if (tid < NVAL) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NG; ++q) s += red[q * NVAL + tid];
      hv[tid] = s;
    }
    if (tid < KM) coef[tid] = (j < k && tid >= j && tid < k) ? __ldcg(piv + tid) : 0.0;
    __syncthreads();
    // ---- T column j-1: T[0:jp, jp] = -tau_jp * T[0:jp, 0:jp] * g[0:jp]  (row q per thread;
    //      column jp only reads columns < jp, so all rows are independent)
    //      one warp per row, warps 1.. only: warp 0's thread 0 computes the next reflector's
    //      scalars meanwhile (a serial row loop on thread 0 was ~0.5 us of every column step)
    if (j >= 1 && tid >= 32) {
      const int jp = j - 1, lane = tid & 31;
      const double tj = taus[jp];
      for (int q = (tid >> 5) - 1; q <= jp; q += QR_THREADS / 32 - 1) {
        double s = 0.0;
        for (int t = q + lane; t < jp; t += 32) s += T[q + t * KM] * hv[KM + t];
        s = warp_sum(s);
        if (lane == 0) T[q + jp * KM] = (q == jp) ? tj : -tj * s;
      }
    }
    if (j == k) break;
    // ---- reflector j (thread 0 computes scalars; everyone reads them)
    if (tid == 0) {
      const double x0 = coef[j];
      const double tail2 = hv[j];
      if (tail2 == 0.0) {
        scal[0] = 1.0; scal[1] = 0.0; scal[2] = x0; scal[3] = 0.0;
      } else {
        const double nrm = sqrt(x0 * x0 + tail2);
        const double alpha = (x0 >= 0.0) ? -nrm : nrm;
        const double denom = x0 - alpha;
        const double tau = 2.0 / (1.0 + tail2 / (denom * denom));
        scal[0] = denom; scal[1] = tau; scal[2] = alpha; scal[3] = 1.0;
      }
      taus[j] = scal[1];
    }
    __syncthreads();
    const double denom = scal[0], tau = scal[1], alpha = scal[2];
    const bool active = scal[3] != 0.0;
    // coefficients tau * v^T a_c for c > j
    if (tid < KM) {
      const int c = tid;
      double cf = 0.0;
      if (active && c > j && c < k) cf = tau * (coef[c] + hv[c] / denom);
      red[c] = cf;  // reuse red[0..31] (all reads of red are done)
    }
    __syncthreads();
    // ---- column j becomes v (rows > j) and alpha (row j); then apply H_j to columns > j
    for (int lr = tid; lr < nr; lr += QR_THREADS) {
      const int64_t r = r0 + lr;
      if (r > j) P[lr * LDP + j] = active ? P[lr * LDP + j] / denom : 0.0;
    }
    __syncthreads();
    if (active) {
      for (int idx = tid; idx < nr * KM; idx += QR_THREADS) {
        const int lr = idx / KM, c = idx % KM;
        const int64_t r = r0 + lr;
        if (r < j || c <= j || c >= k) continue;
        const double v = (r == j) ? 1.0 : P[lr * LDP + j];
        P[lr * LDP + c] -= red[c] * v;
      }
    }
    __syncthreads();
    if (j >= r0 && j < r1 && tid == 0) P[(j - r0) * LDP + j] = alpha;
    __syncthreads();
  }
  __syncthreads();

  // ---- outputs: R (k x k upper), explicit unit-lower Y (may overwrite the input panel), W, T
  for (int c = 0; c < k; ++c) {
    for (int lr = tid; lr < nr; lr += QR_THREADS) {
      const int64_t r = r0 + lr;
      const double pv = P[lr * LDP + c];
      const double y = (r > c) ? pv : (r == c ? 1.0 : 0.0);
      if (Rout && r < k) Rout[r + c * k] = (r <= c) ? pv : 0.0;
      if (Y1) Y1[r + c * ldy1] = y;
      if (Y2) Y2[r + c * ldy2] = y;
    }
  }
  if (W) {
    for (int idx = tid; idx < nr * k; idx += QR_THREADS) {
      const int lr = idx % nr, c = idx / nr;
      const int64_t r = r0 + lr;
      double s = 0.0;
      for (int q = 0; q <= c; ++q) {
        const double y = (r > q) ? P[lr * LDP + q] : (r == q ? 1.0 : 0.0);
        s += y * T[q + c * KM];
      }
      W[r + c * ldw] = s;
    }
  }
  if (Tout && blockIdx.x == 0) {
    for (int i = tid; i < k * k; i += QR_THREADS) {
      const int q = i % k, c = i / k;
      Tout[q + c * k] = T[q + c * KM];
    }
  }
}

// ---- panels of at most 32 columns: lane = column, one shared-memory pass per column step.
// Warp w takes rows w, w + 16, ... of the CTA's chunk and lane c its column c.  At step j the
// pass applies reflector j-1 (the lane holding column j-1 forms v = x / denom and shuffles it to
// the warp; every lane updates its own column) and, with the updated values, accumulates the
// partials of step j: the tail dots x_j^T a_c (c >= j, x_j shuffled from lane j) and the T
// column of reflector j-1, Y^T v (c < j-1).  The two column ranges are disjoint, so every lane
// carries ONE partial.  Per column: the pass, a cross-warp sum, the grid barrier, the fixed-order
// reduction over CTAs, the scalars (thread 0) beside the T column (warps 1..15) -- five CTA
// barriers instead of ten, and the panel read once per step instead of three times.
__global__ void __launch_bounds__(QR_THREADS, 1)
    panel_qr32_kernel(int64_t m, int k, const double* panel, int64_t ldp, double* Rout,
                      double* Y1, int64_t ldy1, double* Y2, int64_t ldy2,
                      double* __restrict__ W, int64_t ldw, double* __restrict__ Tout,
                      QrWork wk, int64_t rows_per_cta) {
  constexpr int KM = 32, LDP = KM + 1, NWARP = QR_THREADS / 32;
  extern __shared__ __align__(16) double sm[];
  double* P = sm;                          // [rows_per_cta][LDP]
  double* red = P + rows_per_cta * LDP;    // [NWARP][KM]
  double* hv = red + NWARP * KM;           // [KM] reduced partials
  double* T = hv + KM;                     // [KM][KM] col-major T
  double* scal = T + KM * KM;              // [4]: denom, tau, alpha, active
  double* taus = scal + 4;                 // [KM]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned ncta = gridDim.x;
  unsigned bar_gen = 0;  // barriers passed (thread 0's count; the word starts at 0 per launch)
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = r0 + rows_per_cta < m ? r0 + rows_per_cta : m;
  const int nr = (int)(r1 > r0 ? r1 - r0 : 0);

  for (int c = 0; c < KM; ++c)
    for (int lr = tid; lr < nr; lr += QR_THREADS)
      P[lr * LDP + c] = c < k ? panel[r0 + lr + c * ldp] : 0.0;
  for (int i = tid; i < KM * KM; i += QR_THREADS) T[i] = 0.0;
  __syncthreads();

  double cf = 0.0;                         // tau (v^T a_lane) of the reflector being applied
  double denom = 1.0, rdenom = 1.0, alpha = 0.0;  // v = x * (1 / denom): one DMUL per row, not
                                                  // a DDIV subroutine on every row's path
  bool active = false;
  for (int j = 0; j <= k; ++j) {
    const int jp = j - 1;
    double* part = wk.part + (j & 1) * (MAXCTA * 2 * KMAX);
    double* piv = wk.piv + (j & 1) * KMAX;
    // ---- the pass: apply reflector jp, accumulate step j's partial
    double acc = 0.0;
    // four rows per iteration (independent chains: the shuffles and the division of one row no
    // longer serialise the next)
    // rows below the pivot (all but a few rows of CTA 0): branch-free.  cf is 0 on the lanes
    // < jp, so those keep a; lane jp takes v; the partial's multiplier is v (T column, lanes
    // < jp), x_j (tail dots, lanes >= j) or 0 (lane jp)
    const bool tdot = lane < jp, hdot = lane >= j && j < k;
    auto row_fast = [&](int lr, double& ac) {
      double a = P[lr * LDP + lane];
      if (jp >= 0) {
        const double vj = active ? __shfl_sync(0xffffffffu, a, jp) * rdenom : 0.0;
        a = (lane == jp) ? vj : fma(-cf, vj, a);
        P[lr * LDP + lane] = a;
        if (tdot) ac = fma(a, vj, ac);
      }
      if (j < k) {
        const double xj = __shfl_sync(0xffffffffu, a, j);
        if (hdot) ac = fma(xj, a, ac);
      }
    };
    auto row_pass = [&](int lr, double& ac) {
      const int64_t r = r0 + lr;
      if (r > j) {
        row_fast(lr, ac);
        return;
      }
      double a = P[lr * LDP + lane];
      if (jp >= 0 && r >= jp) {
        double vj = 1.0;
        if (r > jp) vj = active ? __shfl_sync(0xffffffffu, a, jp) * rdenom : 0.0;
        if (lane == jp) a = (r > jp) ? vj : alpha;
        else if (lane > jp) a -= cf * vj;
        if (lane < jp) ac += a * vj;      // T column jp: Y[r, lane] v_jp[r]   (r >= jp > lane)
        P[lr * LDP + lane] = a;
      }
      if (j < k) {
        const double xj = __shfl_sync(0xffffffffu, a, j);
        if (r > j && lane >= j) ac += xj * a;   // tail dots x_j^T a_lane
        if (r == j) piv[lane] = a;              // the pivot row, for every CTA
      }
    };
    {
      double ac1 = 0.0, ac2 = 0.0, ac3 = 0.0;
      int lr = warp;
      for (; lr + 3 * NWARP < nr; lr += 4 * NWARP) {
        row_pass(lr, acc);
        row_pass(lr + NWARP, ac1);
        row_pass(lr + 2 * NWARP, ac2);
        row_pass(lr + 3 * NWARP, ac3);
      }
      for (; lr < nr; lr += NWARP) row_pass(lr, acc);
      acc = (acc + ac1) + (ac2 + ac3);
    }
    red[warp * KM + lane] = acc;
    __syncthreads();
    if (tid < KM) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) s += red[w * KM + tid];
      part[(int64_t)blockIdx.x * KM + tid] = s;
    }
    grid_barrier(wk.bar, ncta, bar_gen);
    // ---- fixed-order reduction over the CTAs (identical in every CTA)
    {
      double v[10];
      double s = 0.0;
      for (unsigned base = warp; base < ncta; base += NWARP * 10) {
#pragma unroll
        for (int q = 0; q < 10; ++q) {
          const unsigned p = base + NWARP * q;
          v[q] = p < ncta ? __ldcg(part + (int64_t)p * KM + lane) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 10; ++q) s += v[q];
      }
      red[warp * KM + lane] = s;
    }
    const double pv = (j < k) ? __ldcg(piv + lane) : 0.0;  // pivot row entry of this lane
    __syncthreads();
    if (tid < KM) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) s += red[w * KM + tid];
      hv[tid] = s;
    }
    __syncthreads();
    // ---- T column jp (warps 1..: one row per warp) beside the next reflector's scalars
    if (jp >= 0 && warp >= 1) {
      const double tj = taus[jp];
      for (int q = warp - 1; q <= jp; q += NWARP - 1) {
        double s2 = 0.0;
        for (int t = q + lane; t < jp; t += 32) s2 += T[q + t * KM] * hv[t];
        s2 = warp_sum(s2);
        if (lane == 0) T[q + jp * KM] = (q == jp) ? tj : -tj * s2;
      }
    }
    if (j == k) break;
    if (tid == 0) {
      const double xj = __ldcg(piv + j);
      const double tail2 = hv[j];
      if (tail2 == 0.0) {
        scal[0] = 1.0; scal[1] = 0.0; scal[2] = xj; scal[3] = 0.0;
      } else {
        const double nrm = sqrt(xj * xj + tail2);
        const double al = (xj >= 0.0) ? -nrm : nrm;
        const double dn = xj - al;
        scal[0] = dn; scal[1] = 2.0 / (1.0 + tail2 / (dn * dn)); scal[2] = al; scal[3] = 1.0;
      }
      taus[j] = scal[1];
    }
    __syncthreads();
    denom = scal[0];
    rdenom = 1.0 / denom;
    alpha = scal[2];
    active = scal[3] != 0.0;
    const double tau = scal[1];
    // tau v^T a_c = tau (a_c[j] + x_tail^T a_c,tail / denom)  for c > j
    cf = (active && lane > j && lane < k) ? tau * (pv + hv[lane] * rdenom) : 0.0;
  }
  __syncthreads();

  // ---- outputs: R (k x k upper), explicit unit-lower Y, W = Y T, T
  for (int c = 0; c < k; ++c) {
    for (int lr = tid; lr < nr; lr += QR_THREADS) {
      const int64_t r = r0 + lr;
      const double pvv = P[lr * LDP + c];
      const double y = (r > c) ? pvv : (r == c ? 1.0 : 0.0);
      if (Rout && r < k) Rout[r + c * k] = (r <= c) ? pvv : 0.0;
      if (Y1) Y1[r + c * ldy1] = y;
      if (Y2) Y2[r + c * ldy2] = y;
    }
  }
  if (W) {
    for (int idx = tid; idx < nr * k; idx += QR_THREADS) {
      const int lr = idx % nr, c = idx / nr;
      const int64_t r = r0 + lr;
      double s = 0.0;
      for (int q = 0; q <= c; ++q) {
        const double y = (r > q) ? P[lr * LDP + q] : (r == q ? 1.0 : 0.0);
        s += y * T[q + c * KM];
      }
      W[r + c * ldw] = s;
    }
  }
  if (Tout && blockIdx.x == 0) {
    for (int i = tid; i < k * k; i += QR_THREADS) {
      const int q = i % k, c = i / k;
      Tout[q + c * k] = T[q + c * KM];
    }
  }
}

}  // namespace

// PEVD_QR_FUSED=0 selects the two-pass kernel for 32-column panels (comparison runs)
static bool fused_qr() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PEVD_QR_FUSED");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v != 0;
}

int64_t panel_qr_ws_bytes() { return (int64_t)(2 * MAXCTA * 2 * KMAX + 2 * KMAX + 16) * 8; }

int panel_qr(cudaStream_t st, int64_t m, int k, const double* panel, int64_t ldp, double* R,
             double* Y1, int64_t ldy1, double* Y2, int64_t ldy2, double* W, int64_t ldw,
             double* T, void* ws) {
  if (k < 1 || k > KMAX) {
    set_error("panel_qr: panel width %d outside [1, %d]", k, KMAX);
    return ERR_VALUE;
  }
  if (m < k) {
    set_error("panel_qr: panel must be at least as tall as wide (m=%lld, k=%d)", (long long)m, k);
    return ERR_VALUE;
  }
  // Householder QR 2 m k^2 - 2/3 k^3 flops, plus the Y^T v column of T and W = Y T: 2 m k^2
  flops_add(4.0 * (double)m * k * k - 2.0 / 3.0 * (double)k * k * k);
  const int sms = num_sms();
  // fewer, fatter CTAs for short panels: every grid step pays one arrival + one partial per CTA
  // (one CTA per 192 rows: a single CTA for a short panel measured slower -- 304 vs 158 us at
  //  m = 768 -- its per-column pass grows faster than the grid barrier it saves)
  int ncta = (int)std::min<int64_t>(sms, cdiv(m, 192));
  if (ncta < 1) ncta = 1;
  int64_t rows = cdiv(m, ncta);
  ncta = (int)cdiv(m, rows);
  const int KM = k <= 32 ? 32 : 64;
  const int NVAL = 2 * KM, NG = QR_THREADS / NVAL;
  const bool fused = KM == 32 && fused_qr();
  const size_t smem = fused
      ? (size_t)(rows * 33 + (QR_THREADS / 32) * 32 + 32 + 32 * 32 + 4 + 32) * 8
      : (size_t)(rows * (KM + 1) + NG * NVAL + NVAL + KM * KM + KM + 4 + KM) * 8;
  if (smem > 227 * 1024) {
    set_error("panel_qr: panel too tall for the resident-panel kernel (m=%lld, k=%d)",
              (long long)m, k);
    return ERR_VALUE;
  }
  const void* kern = fused ? (const void*)panel_qr32_kernel
                   : KM == 32 ? (const void*)panel_qr_kernel<32> : (const void*)panel_qr_kernel<64>;
  static int attr_dev[3] = {-1, -1, -1};
  const int ki = fused ? 2 : (KM == 64);
  int dev;
  PEVD_CUDA(cudaGetDevice(&dev));
  if (attr_dev[ki] != dev) {
    PEVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_dev[ki] = dev;
  }
  QrWork wk;
  wk.part = (double*)ws;
  wk.piv = wk.part + 2 * MAXCTA * 2 * KMAX;
  wk.bar = (unsigned*)(wk.piv + 2 * KMAX);
  PEVD_CUDA(cudaMemsetAsync(wk.bar, 0, 2 * sizeof(unsigned), st));
  void* args[] = {&m, &k, &panel, &ldp, &R, &Y1, &ldy1, &Y2, &ldy2, &W, &ldw, &T, &wk, &rows};
  PEVD_CUDA(cudaLaunchCooperativeKernel(kern, dim3(ncta), dim3(QR_THREADS), args, smem, st));
  count_launch();
  return OK;
}

}  // namespace pevd
