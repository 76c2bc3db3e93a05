// Divide-and-conquer symmetric tridiagonal eigensolver on the device (replaces the reference's
// QL/QR `_steqr`, tridiag.py:133-295; output convention of `tridiag_eig`, tridiag.py:298-334).
//
// Cuppen tearing T = diag(T1, T2) + rho u u^T (rho = |e_k| >= 0, u = [e_last; sign(e_k) e_first])
// over a balanced binary tree whose 2^L leaves all have <= 32 rows.  Every level is batched:
// one launch per phase covers all merges of the level.
//   leaves : warp-per-leaf implicit QL/QR (same iteration as the reference solver), lane = column.
//   merge  : z from the children's boundary rows; merge-sort of the two spectra; deflation scan
//            (small |z_i| and Givens for near-equal poles, LAPACK dlaed2 rules; one thread per
//            merge, rotations then applied row-parallel); secular roots (one thread per root,
//            shifted to the nearer pole, rational two-pole "middle way" steps inside a bisection
//            bracket); Gu-Eisenstat/Loewner recomputation of z so the eigenvectors are
//            numerically orthogonal; eigenvector matrix U written in [top | mixed | bottom]
//            row order; and the merge itself as two grouped DMMA GEMMs per merge
//            Q_top = Q1[:, top|mixed] U_top,  Q_bot = Q2[:, mixed|bottom] U_bot,
//            written straight into sorted column positions (GEMM column maps).
// Values are scaled by max|T| first (LAPACK dstedc) and scaled back at the end.  Finally every
// eigenvector gets the reference's sign convention: largest-magnitude entry positive
// (earliest index on ties).
#include <vector>
#include <cmath>
#include <algorithm>
#include "kernels.cuh"

namespace pevd {

namespace {

constexpr int LEAF = 32;
constexpr double DEPS = 1.1102230246251565e-16;  // 0.5 * DBL_EPSILON (unit roundoff)
constexpr double SAFMIN = 2.2250738585072014e-308;

struct Level {
  int count;      // merges at this level (or leaves)
  int smax;       // max node size
  int n1max;      // max child size
  int64_t off;    // offset into node arrays
  int64_t uoff;   // unused
};

// per-merge scalar block (device), 16 ints / doubles
enum { M_K = 0, M_ND, M_NROT, M_K1, M_K2, M_K3, M_NINT };

// U layout of a merge with K roots: a zero row after the first k1 rows when k1 is odd, an even
// leading dimension, so the two merge GEMMs' B operands are 16-byte aligned (see merge_gemm_args)
__host__ __device__ __forceinline__ int u_pad(int k1) { return k1 & 1; }
__host__ __device__ __forceinline__ int64_t u_ld(int K, int k1) { return (K + u_pad(k1) + 1) & ~1; }
// elements reserved for a merge of size s (K <= s roots), even so the next offset stays aligned
__host__ __device__ __forceinline__ int64_t u_elems(int64_t s) { return (s * (s + 2) + 1) & ~1LL; }

// ---------------------------------------------------------------- helpers

__global__ void scale_kernel(int64_t n, const double* d, const double* e, double* dw, double* ew,
                             const double* scal) {
  const double s = 1.0 / scal[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    dw[i] = d[i] * s;
    if (i + 1 < n) ew[i] = e[i] * s;
  }
}

__global__ void tear_kernel(double* dw, const double* ew, const int* cuts, int ncuts) {
  // cut k splits between rows k-1 and k: d[k-1] -= |e[k-1]|, d[k] -= |e[k-1]| (LAPACK dlaed0).
  // A row can be touched by two cuts (size-1 leaves), so apply them serially.
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int c = 0; c < ncuts; ++c) {
      const int k = cuts[c];
      const double a = fabs(ew[k - 1]);
      dw[k - 1] -= a;
      dw[k] -= a;
    }
  }
}

__global__ void absmax_kernel(int64_t n, const double* d, const double* e, double* out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    m = fmax(m, fabs(d[i]));
    if (i + 1 < n) m = fmax(m, fabs(e[i]));
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0] > 0.0 ? red[0] : 1.0;
}

__global__ void zero_fill(double* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

// ---------------------------------------------------------------- leaves

__device__ void d_lartg(double f, double g, double& c, double& s, double& r) {
  if (g == 0.0) { c = 1.0; s = 0.0; r = f; return; }
  if (f == 0.0) { c = 0.0; s = 1.0; r = g; return; }
  double rr = sqrt(f * f + g * g);
  if (rr == 0.0) {
    const double scl = 1.0 / SAFMIN;
    const double fs = f * scl, gs = g * scl;
    rr = sqrt(fs * fs + gs * gs) * SAFMIN;
  }
  double cc = f / rr, ss = g / rr;
  if (fabs(f) > fabs(g) && cc < 0.0) { cc = -cc; ss = -ss; rr = -rr; }
  c = cc; s = ss; r = rr;
}

__device__ void d_laev2(double a, double b, double c, double& rt1, double& rt2, double& cs1,
                        double& sn1) {
  const double sm = a + c, df = a - c, adf = fabs(df), tb = b + b, ab = fabs(tb);
  double acmx, acmn, rt, sgn1, sgn2, cs;
  if (fabs(a) > fabs(c)) { acmx = a; acmn = c; } else { acmx = c; acmn = a; }
  if (adf > ab) { const double q = ab / adf; rt = adf * sqrt(1.0 + q * q); }
  else if (adf < ab) { const double q = adf / ab; rt = ab * sqrt(1.0 + q * q); }
  else rt = ab * sqrt(2.0);
  if (sm < 0.0) { rt1 = 0.5 * (sm - rt); sgn1 = -1.0; rt2 = (acmx / rt1) * acmn - (b / rt1) * b; }
  else if (sm > 0.0) { rt1 = 0.5 * (sm + rt); sgn1 = 1.0; rt2 = (acmx / rt1) * acmn - (b / rt1) * b; }
  else { rt1 = 0.5 * rt; rt2 = -0.5 * rt; sgn1 = 1.0; }
  if (df >= 0.0) { cs = df + rt; sgn2 = 1.0; } else { cs = df - rt; sgn2 = -1.0; }
  double c1, s1;
  if (fabs(cs) > ab) { const double ct = -tb / cs; s1 = 1.0 / sqrt(1.0 + ct * ct); c1 = ct * s1; }
  else if (ab == 0.0) { c1 = 1.0; s1 = 0.0; }
  else { const double tn = -cs / tb; c1 = 1.0 / sqrt(1.0 + tn * tn); s1 = tn * c1; }
  if (sgn1 == sgn2) { const double tn = c1; c1 = -s1; s1 = tn; }
  cs1 = c1; sn1 = s1;
}

// One warp per leaf.  zt (s x s) in smem, row i = eigenvector candidate of d[i]; lane = column.
// The scalar recurrence is executed redundantly (and identically) by every lane.
__global__ void __launch_bounds__(128)
    leaf_kernel(const int* __restrict__ leaf_lo, const int* __restrict__ leaf_hi, int nleaves,
                double* __restrict__ dw, const double* __restrict__ ew, double* __restrict__ Q,
                int64_t ldq, int* __restrict__ info) {
  __shared__ double zts[4][LEAF * (LEAF + 1)];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int leaf = blockIdx.x * 4 + w;
  if (leaf >= nleaves) return;
  const int lo = leaf_lo[leaf], hi = leaf_hi[leaf];
  const int n = hi - lo;
  double* zt = zts[w];
  // every lane runs the scalar recurrence on its own private copy of (d, e): identical inputs
  // and operations give identical rotations in all lanes, and no lane can observe another
  // lane's partial update.  Lane k applies the rotations to column k of zt.
  double d[LEAF], e[LEAF];
  constexpr int LDZ = LEAF + 1;
  for (int i = 0; i < n; ++i) zt[i * LDZ + lane] = (i == lane) ? 1.0 : 0.0;
  for (int i = 0; i < n; ++i) {
    d[i] = dw[lo + i];
    e[i] = (i + 1 < n) ? ew[lo + i] : 0.0;
  }
  __syncwarp();
  const double ulp = DEPS, eps2 = ulp * ulp;
  const int cap = 30 * n;
  int total = 0;
  int l1 = 0;
  bool failed = false;
  // rotation of rows p, q of zt: ql=1: a'=c a - s b, b' = s a + c b;  ql=0: a'=c a + s b, b'=c b - s a
  auto rot = [&](int p, int q, double c, double s, int ql) {
    if (lane < n) {
      const double za = zt[p * LDZ + lane], zb = zt[q * LDZ + lane];
      if (ql) { zt[p * LDZ + lane] = c * za - s * zb; zt[q * LDZ + lane] = s * za + c * zb; }
      else { zt[p * LDZ + lane] = c * za + s * zb; zt[q * LDZ + lane] = c * zb - s * za; }
    }
  };
  while (l1 < n && !failed) {
    if (l1 > 0) e[l1 - 1] = 0.0;
    int m = n - 1;
    for (int mm = l1; mm < n - 1; ++mm) {
      const double tst = fabs(e[mm]);
      if (tst == 0.0) { m = mm; break; }
      if (tst <= (sqrt(fabs(d[mm])) * sqrt(fabs(d[mm + 1]))) * ulp) { e[mm] = 0.0; m = mm; break; }
    }
    int l = l1, lend = m;
    l1 = m + 1;
    if (lend == l) continue;
    if (fabs(d[lend]) < fabs(d[l])) { const int t = l; l = lend; lend = t; }
    if (lend > l) {
      for (;;) {
        m = lend;
        for (int mm = l; mm < lend; ++mm) {
          const double tst = e[mm] * e[mm];
          if (tst <= (eps2 * fabs(d[mm])) * fabs(d[mm + 1]) + SAFMIN) { m = mm; break; }
        }
        if (m < lend) e[m] = 0.0;
        double p = d[l];
        if (m == l) { ++l; if (l <= lend) continue; break; }
        if (m == l + 1) {
          double rt1, rt2, cc, ss;
          d_laev2(d[l], e[l], d[l + 1], rt1, rt2, cc, ss);
          rot(l, l + 1, cc, ss, 0);
          d[l] = rt1; d[l + 1] = rt2; e[l] = 0.0;
          l += 2;
          if (l <= lend) continue;
          break;
        }
        if (total == cap) { failed = true; break; }
        ++total;
        double g = (d[l + 1] - p) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[m] - p + e[l] / (g + (g >= 0.0 ? r : -r));
        double s = 1.0, c = 1.0;
        p = 0.0;
        for (int i = m - 1; i >= l; --i) {
          const double f = s * e[i], bb = c * e[i];
          d_lartg(g, f, c, s, r);
          if (i != m - 1) e[i + 1] = r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * bb;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - bb;
          rot(i, i + 1, c, s, 1);
        }
        d[l] = d[l] - p;
        e[l] = g;
      }
    } else {
      for (;;) {
        m = lend;
        for (int mm = l; mm > lend; --mm) {
          const double tst = e[mm - 1] * e[mm - 1];
          if (tst <= (eps2 * fabs(d[mm])) * fabs(d[mm - 1]) + SAFMIN) { m = mm; break; }
        }
        if (m > lend) e[m - 1] = 0.0;
        double p = d[l];
        if (m == l) { --l; if (l >= lend) continue; break; }
        if (m == l - 1) {
          double rt1, rt2, cc, ss;
          d_laev2(d[l - 1], e[l - 1], d[l], rt1, rt2, cc, ss);
          rot(l - 1, l, cc, ss, 0);
          d[l - 1] = rt1; d[l] = rt2; e[l - 1] = 0.0;
          l -= 2;
          if (l >= lend) continue;
          break;
        }
        if (total == cap) { failed = true; break; }
        ++total;
        double g = (d[l - 1] - p) / (2.0 * e[l - 1]);
        double r = hypot(g, 1.0);
        g = d[m] - p + e[l - 1] / (g + (g >= 0.0 ? r : -r));
        double s = 1.0, c = 1.0;
        p = 0.0;
        for (int i = m; i < l; ++i) {
          const double f = s * e[i], bb = c * e[i];
          d_lartg(g, f, c, s, r);
          if (i != m) e[i - 1] = r;
          g = d[i] - p;
          r = (d[i + 1] - g) * s + 2.0 * c * bb;
          p = s * r;
          d[i] = g + p;
          g = c * r - bb;
          rot(i, i + 1, c, s, 0);
        }
        d[l] = d[l] - p;
        e[l - 1] = g;
      }
    }
    __syncwarp();
  }
  __syncwarp();
  if (failed) {
    if (lane == 0) atomicExch(info, lo + 1);
    return;
  }
  // stable ascending sort; Q block column rank <- zt row lane
  if (lane < n) {
    const double v = d[lane];
    int rank = 0;
    for (int i = 0; i < n; ++i) rank += (d[i] < v) || (d[i] == v && i < lane);
    dw[lo + rank] = v;
    for (int k = 0; k < n; ++k) Q[(lo + k) + (int64_t)(lo + rank) * ldq] = zt[lane * LDZ + k];
  }
}

// ---------------------------------------------------------------- merge phases
// Node arrays per level: lo, mid, hi (ints).  Per-element arrays are indexed by absolute row.

struct MergeBufs {
  const int* lo; const int* mid; const int* hi;
  double* Dcur;     // children's eigenvalues, each child sorted ascending
  double* Dnext;    // merged eigenvalues, sorted ascending
  const double* ew; // torn off-diagonals (scaled): rho = |ew[mid-1]|
  double* Ds; double* zs; int* colid; int* ctype;   // merged-sorted arrays
  double* dl; double* zl; int* ncol; int* ntype;    // non-deflated (sorted)
  double* dv; int* dcol;                            // deflated (scan order)
  double* dvs; int* dcols;                          // deflated sorted
  int* rp; int* rq; double* rc; double* rs;         // rotations
  int* org; double* tau; double* lam; double* zhat; // roots
  int* rpos;                                        // non-deflated sorted idx -> U row
  int* amapT; int* amapB; int* cmap;
  int* mint;                                        // per-merge ints [M_NINT]
  double* rho;                                      // per-merge rho (scaled, after z normalisation)
  GemmArgs* gargs;
  double* U;                                        // U workspace
  const int64_t* uoff;                              // per-merge U offsets (elements)
};

__global__ void merge_prep(MergeBufs B, const double* __restrict__ X, int64_t ldx) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi], mid = B.mid[mi], hi = B.hi[mi];
  const int n1 = mid - lo, n2 = hi - mid, s = n1 + n2;
  const double beta = B.ew[mid - 1];
  const double sgn = (beta < 0.0) ? -1.0 : 1.0;
  const double isq2 = 0.70710678118654752440;
  if (blockIdx.x == 0 && threadIdx.x == 0) B.rho[mi] = 2.0 * fabs(beta);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < s; t += gridDim.x * blockDim.x) {
    double val, z;
    int pos, type;
    if (t < n1) {
      val = B.Dcur[lo + t];
      z = X[(mid - 1) + (int64_t)(lo + t) * ldx] * isq2;
      // # of D2 strictly below val
      int a = 0, b = n2;
      while (a < b) { const int c = (a + b) >> 1; if (B.Dcur[mid + c] < val) a = c + 1; else b = c; }
      pos = t + a;
      type = 1;
    } else {
      const int u = t - n1;
      val = B.Dcur[mid + u];
      z = sgn * X[mid + (int64_t)(mid + u) * ldx] * isq2;
      int a = 0, b = n1;  // # of D1 <= val
      while (a < b) { const int c = (a + b) >> 1; if (B.Dcur[lo + c] <= val) a = c + 1; else b = c; }
      pos = u + a;
      type = 3;
    }
    B.Ds[lo + pos] = val;
    B.zs[lo + pos] = z;
    B.colid[lo + pos] = t;
    B.ctype[lo + pos] = type;
  }
}

// one warp per merge: reductions in parallel, the deflation scan itself sequential in lane 0
__global__ void merge_deflate(MergeBufs B) {
  const int mi = blockIdx.x;
  const int lane = threadIdx.x;
  const int lo = B.lo[mi], mid = B.mid[mi], hi = B.hi[mi];
  const int s = hi - lo, n1 = mid - lo;
  double dmax = 0.0, zmax = 0.0;
  for (int t = lane; t < s; t += 32) {
    dmax = fmax(dmax, fabs(B.Ds[lo + t]));
    zmax = fmax(zmax, fabs(B.zs[lo + t]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
  }
  const double rho = B.rho[mi];
  const double tol = 8.0 * DEPS * fmax(dmax, zmax);  // LAPACK dlaed2
  int K = 0, nd = 0, nrot = 0;
  double* Ds = B.Ds + lo;
  double* zs = B.zs + lo;
  int* colid = B.colid + lo;
  int* ctype = B.ctype + lo;
  if (rho * zmax <= tol) {
    if (lane != 0) return;
    for (int p = 0; p < s; ++p) { B.dv[lo + nd] = Ds[p]; B.dcol[lo + nd] = colid[p]; ++nd; }
  } else {
    // The scan is sequential (a Givens deflation changes the pole it chains to), so lane 0 runs
    // it; the whole warp stages the next 32 entries in shared memory first, and the current
    // pole pj lives in registers, so no iteration waits on an L2 round trip.
    __shared__ double sD[32], sZ[32];
    __shared__ int sC[32], sT[32];
    int pj = -1;
    double dpj = 0.0, zpj = 0.0;
    int cpj = 0, tpj = 0;
    for (int base = 0; base < s; base += 32) {
      __syncwarp();
      if (base + lane < s) {
        sD[lane] = Ds[base + lane];
        sZ[lane] = zs[base + lane];
        sC[lane] = colid[base + lane];
        sT[lane] = ctype[base + lane];
      }
      __syncwarp();
      if (lane == 0) {
        const int cnt = s - base < 32 ? s - base : 32;
        for (int q = 0; q < cnt; ++q) {
          const int p = base + q;
          double dp = sD[q], zp = sZ[q];
          const int cp = sC[q];
          int tp = sT[q];
          if (rho * fabs(zp) <= tol) {
            B.dv[lo + nd] = dp; B.dcol[lo + nd] = cp; ++nd;
            continue;
          }
          if (pj < 0) { pj = p; dpj = dp; zpj = zp; cpj = cp; tpj = tp; continue; }
          double S = zpj, C = zp;
          const double tau = hypot(C, S);
          const double t = dp - dpj;
          C /= tau;
          S = -S / tau;
          if (fabs(t * C * S) <= tol) {
            zp = tau;
            zs[p] = tau;
            zs[pj] = 0.0;
            B.rp[lo + nrot] = cpj; B.rq[lo + nrot] = cp;
            B.rc[lo + nrot] = C; B.rs[lo + nrot] = S; ++nrot;
            if (tp != tpj) { tp = 2; ctype[p] = 2; }
            const double tmp = dpj * C * C + dp * S * S;
            dp = dpj * S * S + dp * C * C;
            Ds[p] = dp;
            Ds[pj] = tmp;
            B.dv[lo + nd] = tmp; B.dcol[lo + nd] = cpj; ++nd;
          } else {
            B.dl[lo + K] = dpj; B.zl[lo + K] = zpj;
            B.ncol[lo + K] = cpj; B.ntype[lo + K] = tpj; ++K;
          }
          pj = p; dpj = dp; zpj = zp; cpj = cp; tpj = tp;
        }
      }
    }
    if (lane != 0) return;
    if (pj >= 0) {
      B.dl[lo + K] = dpj; B.zl[lo + K] = zpj;
      B.ncol[lo + K] = cpj; B.ntype[lo + K] = tpj; ++K;
    }
  }
  // U row order [top-only | mixed | bottom-only]; column maps of the two merge GEMMs
  int k1 = 0, k2 = 0, k3 = 0;
  for (int k = 0; k < K; ++k) {
    const int ty = B.ntype[lo + k];
    k1 += ty == 1; k2 += ty == 2; k3 += ty == 3;
  }
  int i1 = 0, i2 = 0, i3 = 0;
  for (int k = 0; k < K; ++k) {
    const int ty = B.ntype[lo + k];
    const int r = (ty == 1) ? i1++ : (ty == 2) ? k1 + i2++ : k1 + k2 + i3++;
    B.rpos[lo + k] = r;
    if (r < k1 + k2) B.amapT[lo + r] = B.ncol[lo + k];
    if (r >= k1) B.amapB[lo + (r - k1)] = B.ncol[lo + k];
  }
  int* mint = B.mint + mi * M_NINT;
  mint[M_K] = K; mint[M_ND] = nd; mint[M_NROT] = nrot;
  mint[M_K1] = k1; mint[M_K2] = k2; mint[M_K3] = k3;
  (void)n1;
}

// rotations act on columns; every row is independent -> row-parallel, sequential per row
__global__ void merge_rotate(MergeBufs B, double* X, int64_t ldx) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi], hi = B.hi[mi];
  const int nrot = B.mint[mi * M_NINT + M_NROT];
  if (nrot == 0) return;
  for (int r = lo + blockIdx.x * blockDim.x + threadIdx.x; r < hi; r += gridDim.x * blockDim.x) {
    for (int t = 0; t < nrot; ++t) {
      const int64_t p = lo + B.rp[lo + t], q = lo + B.rq[lo + t];
      const double c = B.rc[lo + t], s = B.rs[lo + t];
      double* xp = X + r + p * ldx;
      double* xq = X + r + q * ldx;
      const double x = *xp, y = *xq;
      *xp = c * x + s * y;
      *xq = c * y - s * x;
    }
  }
}

// secular equation 1/rho + sum z_i^2 / (d_i - lambda) = 0, root j in (d_j, d_{j+1})
// (last root in (d_{K-1}, d_{K-1} + rho |z|^2]); result stored as origin index + offset tau.
// SEC_G lanes per root: every lane sums a strided slice of the K terms (psi over i <= j, phi over
// i > j) and an xor butterfly gives every lane of the group the same totals (a + b == b + a at
// each level), so all lanes take identical steps and exit together.  One thread per root left
// a K = 49152 merge with ~10 warps per SM running dependent division chains (198 ms of secular
// solves per n = 49152 EVD).
constexpr int SEC_G = 8;

__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = SEC_G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, SEC_G);
  return v;
}

__global__ void merge_secular(MergeBufs B, int* info) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi];
  const int K = B.mint[mi * M_NINT + M_K];
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = gt / SEC_G, sub = gt % SEC_G;
  if (j >= K) return;  // whole groups leave together (blockDim is a multiple of SEC_G)
  const unsigned mask = ((1u << SEC_G) - 1u) << ((threadIdx.x & 31) / SEC_G * SEC_G);
  const double* dl = B.dl + lo;
  const double* zl = B.zl + lo;
  const double rho = B.rho[mi];
  const double rhoinv = 1.0 / rho;
  if (K == 1) {
    if (sub == 0) {
      B.org[lo] = 0;
      B.tau[lo] = rho * zl[0] * zl[0];
      B.lam[lo] = dl[0] + rho * zl[0] * zl[0];
    }
    return;
  }
  const bool last = (j == K - 1);
  int org;
  double lo_t, hi_t, tau;
  if (!last) {
    const double gap = dl[j + 1] - dl[j];
    const double midp = 0.5 * gap;
    const double dj0 = dl[j];
    double f = 0.0;
    for (int i = sub; i < K; i += SEC_G) f += zl[i] * zl[i] / ((dl[i] - dj0) - midp);
    f = rhoinv + group_sum(f, mask);
    if (f >= 0.0) { org = j; lo_t = 0.0; hi_t = midp; tau = midp; }
    else { org = j + 1; lo_t = -(gap - midp); hi_t = 0.0; tau = -(gap - midp); }
  } else {
    double zz = 0.0;
    for (int i = sub; i < K; i += SEC_G) zz += zl[i] * zl[i];
    zz = group_sum(zz, mask);
    org = K - 1;
    lo_t = 0.0;
    hi_t = rho * zz * (1.0 + 8.0 * DEPS) + SAFMIN;
    tau = 0.5 * hi_t;
  }
  const double dorg = dl[org];
  // first phi index of this lane's slice: the smallest i > j with i = sub (mod SEC_G)
  const int i_phi = j + 1 + ((sub - (j + 1)) % SEC_G + SEC_G) % SEC_G;
  bool conv = false;
  for (int it = 0; it < 200; ++it) {
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
    for (int i = sub; i <= j; i += SEC_G) {
      const double tmp = zl[i] / ((dl[i] - dorg) - tau);
      psi += zl[i] * tmp;
      dpsi += tmp * tmp;
    }
    for (int i = i_phi; i < K; i += SEC_G) {
      const double tmp = zl[i] / ((dl[i] - dorg) - tau);
      phi += zl[i] * tmp;
      dphi += tmp * tmp;
    }
    psi = group_sum(psi, mask);
    dpsi = group_sum(dpsi, mask);
    phi = group_sum(phi, mask);
    dphi = group_sum(dphi, mask);
    const double w = rhoinv + psi + phi;
    const double errb = 8.0 * (2.0 * DEPS) * (rhoinv + phi - psi) + 2.0 * DEPS * fabs(w);
    if (fabs(w) <= errb) { conv = true; break; }
    if (w > 0.0) hi_t = tau; else lo_t = tau;
    const double dj = (dl[j] - dorg) - tau;  // d_j - lambda  (< 0)
    double eta;
    if (!last) {
      const double dj1 = (dl[j + 1] - dorg) - tau;  // > 0
      const double s1 = dj * dj * dpsi, s2 = dj1 * dj1 * dphi;
      const double c = w - dj * dpsi - dj1 * dphi;
      const double a1 = c * (dj + dj1) + s1 + s2;
      const double a0 = dj * dj1 * w;
      double disc = a1 * a1 - 4.0 * c * a0;
      if (disc < 0.0) disc = 0.0;
      const double den = a1 + copysign(sqrt(disc), a1);
      eta = (den != 0.0) ? 2.0 * a0 / den : 0.0;
    } else {
      const double s1 = dj * dj * dpsi;
      const double c = w - dj * dpsi;
      eta = (c > 0.0) ? dj + s1 / c : 0.5 * (hi_t - tau);
    }
    double tn = tau + eta;
    if (!(tn > lo_t && tn < hi_t)) tn = 0.5 * (lo_t + hi_t);
    if (tn == tau) { conv = true; break; }
    tau = tn;
    if (hi_t - lo_t <= 4.0 * DEPS * fmax(fabs(lo_t), fabs(hi_t))) { conv = true; break; }
  }
  if (sub != 0) return;
  if (!conv) atomicExch(info, -(lo + j + 1));
  B.org[lo + j] = org;
  B.tau[lo + j] = tau;
  B.lam[lo + j] = dorg + tau;
}

__device__ __forceinline__ double delta_ij(const double* dl, const int* org, const double* tau,
                                           int i, int j) {
  return (dl[i] - dl[org[j]]) - tau[j];  // d_i - lambda_j, accurate
}

// Loewner / Gu-Eisenstat: zhat_i^2 = prod_j (d_i - lambda_j) / prod_{j != i} (d_i - d_j) (sign < 0)
__global__ void merge_zhat(MergeBufs B) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi];
  const int K = B.mint[mi * M_NINT + M_K];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const double* dl = B.dl + lo;
  const int* org = B.org + lo;
  const double* tau = B.tau + lo;
  double w = delta_ij(dl, org, tau, i, i);
  for (int j = 0; j < K; ++j) {
    if (j == i) continue;
    w *= delta_ij(dl, org, tau, i, j) / (dl[i] - dl[j]);
  }
  const double zi = B.zl[lo + i];
  B.zhat[lo + i] = copysign(sqrt(fabs(w)), zi);
}

// deflated values: stable rank sort (values were appended in nearly sorted order)
__global__ void merge_sort_deflated(MergeBufs B) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi];
  const int nd = B.mint[mi * M_NINT + M_ND];
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nd) return;
  const double v = B.dv[lo + q];
  int rank = 0;
  for (int t = 0; t < nd; ++t) {
    const double u = B.dv[lo + t];
    rank += (u < v) || (u == v && t < q);
  }
  B.dvs[lo + rank] = v;
  B.dcols[lo + rank] = B.dcol[lo + q];
}

// one warp per root j: U[rpos(i), j] = zhat_i / (d_i - lambda_j) / ||.||; output column map
__global__ void merge_vectors(MergeBufs B) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi];
  const int K = B.mint[mi * M_NINT + M_K];
  const int nd = B.mint[mi * M_NINT + M_ND];
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= K) return;
  const double* dl = B.dl + lo;
  const int* org = B.org + lo;
  const double* tau = B.tau + lo;
  const double* zh = B.zhat + lo;
  double ss = 0.0;
  for (int i = lane; i < K; i += 32) {
    const double u = zh[i] / delta_ij(dl, org, tau, i, j);
    ss += u * u;
  }
  ss = warp_sum(ss);
  const double inv = 1.0 / sqrt(ss);
  double* U = B.U + B.uoff[mi];
  const int k1 = B.mint[mi * M_NINT + M_K1];
  const int pad = u_pad(k1);
  const int64_t ldu = u_ld(K, k1);
  for (int i = lane; i < K; i += 32) {
    const double u = zh[i] / delta_ij(dl, org, tau, i, j);
    const int r = B.rpos[lo + i];
    U[r + (r >= k1 ? pad : 0) + (int64_t)j * ldu] = u * inv;
  }
  if (pad && lane == 0) U[k1 + (int64_t)j * ldu] = 0.0;
  if (lane == 0) {
    const double lj = B.lam[lo + j];
    int a = 0, b = nd;  // deflated strictly below lambda_j
    while (a < b) { const int c = (a + b) >> 1; if (B.dvs[lo + c] < lj) a = c + 1; else b = c; }
    B.cmap[lo + j] = j + a;
    B.Dnext[lo + j + a] = lj;
  }
}

// (clo, chi): only the output columns [clo, chi) are wanted (the columns of a rank in the
// distributed conventional order).  cmap is increasing (roots ascending, deflated values merged
// in), so the U columns landing there are one contiguous range [ja, jb).
__global__ void merge_gemm_args(MergeBufs B, const double* X, int64_t ldx, double* Y, int64_t ldy,
                                int nm, int64_t clo, int64_t chi) {
  // (X here is the compacted operand buffer of merge_gather_cols: no column maps)
  const int mi = blockIdx.x * blockDim.x + threadIdx.x;
  if (mi >= nm) return;
  const int lo = B.lo[mi], mid = B.mid[mi], hi = B.hi[mi];
  const int* mint = B.mint + mi * M_NINT;
  const int K = mint[M_K], k1 = mint[M_K1], k2 = mint[M_K2], k3 = mint[M_K3];
  double* U = B.U + B.uoff[mi];
  const int* cm = B.cmap + lo;
  auto lower = [&](int64_t v) {  // first j with cmap[j] >= v - lo
    int a = 0, b2 = K;
    while (a < b2) {
      const int c = (a + b2) >> 1;
      if (cm[c] < v - lo) a = c + 1; else b2 = c;
    }
    return a;
  };
  const int ja = lower(clo), jb = lower(chi);
  // U (and the top block of X) carry a zero row (column) after the k1 block when k1 is odd, and
  // U's leading dimension is even: both GEMMs' B operands start 16-byte aligned with an even
  // stride, so they take the 16-byte cp.async path (vec_ok) whatever the deflation left
  const int pad = u_pad(k1);
  const int64_t ldu = u_ld(K, k1);
  GemmArgs t{};
  t.m = mid - lo; t.n = jb - ja; t.k = k1 + pad + k2; t.alpha = 1.0; t.beta = 0.0;
  t.A = X + lo + (int64_t)lo * ldx; t.lda = ldx; t.amap = nullptr;
  t.B = U + (int64_t)ja * ldu; t.ldb = ldu;
  t.C = Y + lo + (int64_t)lo * ldy; t.ldc = ldy; t.cmap = cm + ja;
  t.transA = 0; t.transB = 0; t.amode = A_GENERAL; t.cmode = C_ALL;
  GemmArgs bt = t;
  bt.m = hi - mid; bt.k = k2 + k3;
  bt.A = X + mid + (int64_t)lo * ldx; bt.amap = nullptr;
  bt.B = U + k1 + pad + (int64_t)ja * ldu;
  bt.C = Y + mid + (int64_t)lo * ldy;
  if (K == 0) { t.m = 0; bt.m = 0; }
  B.gargs[2 * mi] = t;
  B.gargs[2 * mi + 1] = bt;
}

// The merge GEMMs' A operands, compacted: the k1 + k2 columns of Q1 the top GEMM reads (through
// amapT) and the k2 + k3 columns of Q2 the bottom one reads (amapB) are copied next to each
// other, so the GEMMs stream plain column blocks (a gathered operand made every cp.async wait on
// an index load: 10% of the grouped GEMM's stall samples).  Xc has X's block structure: the
// top block at rows [lo, mid), the bottom one at rows [mid, hi), both from column lo.
__global__ void merge_gather_cols(MergeBufs B, const double* __restrict__ X, int64_t ldx,
                                  double* __restrict__ Xc, int64_t ldc) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi], mid = B.mid[mi], hi = B.hi[mi];
  const int* mint = B.mint + mi * M_NINT;
  const int K = mint[M_K], k1 = mint[M_K1], k2 = mint[M_K2], k3 = mint[M_K3];
  const int c = blockIdx.x;
  if (K == 0) return;
  const int pad = u_pad(k1);
  if (c < k1 + pad + k2) {  // top block, with the zero column at k1 when k1 is odd
    double* dst = Xc + (int64_t)(lo + c) * ldc;
    if (pad && c == k1) {
      for (int r = lo + threadIdx.x; r < mid; r += blockDim.x) dst[r] = 0.0;
    } else {
      const int cs = (c < k1) ? c : c - pad;
      const double* src = X + (int64_t)(lo + B.amapT[lo + cs]) * ldx;
      for (int r = lo + threadIdx.x; r < mid; r += blockDim.x) dst[r] = src[r];
    }
  }
  if (c < k2 + k3) {
    const double* src = X + (int64_t)(lo + B.amapB[lo + c]) * ldx;
    double* dst = Xc + (int64_t)(lo + c) * ldc;
    for (int r = mid + threadIdx.x; r < hi; r += blockDim.x) dst[r] = src[r];
  }
}

// deflated eigenpairs: copy the (rotated) column of X into its sorted output position
__global__ void merge_deflated_copy(MergeBufs B, const double* X, int64_t ldx, double* Y,
                                    int64_t ldy, int64_t clo, int64_t chi) {
  const int mi = blockIdx.y;
  const int lo = B.lo[mi], hi = B.hi[mi];
  const int K = B.mint[mi * M_NINT + M_K];
  const int nd = B.mint[mi * M_NINT + M_ND];
  const int q = blockIdx.x;
  if (q >= nd) return;
  const double v = B.dvs[lo + q];
  int a = 0, b = K;  // roots <= v
  while (a < b) { const int c = (a + b) >> 1; if (B.lam[lo + c] <= v) a = c + 1; else b = c; }
  const int pos = q + a;
  if (threadIdx.x == 0) B.Dnext[lo + pos] = v;
  if (lo + pos < clo || lo + pos >= chi) return;  // column not wanted (eigenvalue kept above)
  const int64_t src = lo + B.dcols[lo + q];
  for (int r = lo + threadIdx.x; r < hi; r += blockDim.x)
    Y[r + (int64_t)(lo + pos) * ldy] = X[r + src * ldx];
}

__global__ void finalize_kernel(int64_t n, const double* dw, double* d, const double* scal) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = dw[i] * scal[0];
}

// sign convention: largest |q_ij| in each column positive, earliest index on ties
__global__ void sign_fix(int64_t n, double* Q, int64_t ldq, int64_t j0) {
  const int64_t j = j0 + blockIdx.x;
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(Q[i + j * ldq]);
    if (a > best) { best = a; bidx = i; }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = bv[threadIdx.x + s];
      const int64_t oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const bool neg = Q[bi[0] + j * ldq] < 0.0;
  if (!neg) return;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) Q[i + j * ldq] = -Q[i + j * ldq];
}

// ---------------------------------------------------------------- host plan

struct Plan {
  int L = 0;
  std::vector<int> leaf_lo, leaf_hi;
  std::vector<std::vector<int>> mlo, mmid, mhi;  // per level (0 = just above leaves)
  std::vector<int> cuts;
};

Plan make_plan(int64_t n) {
  Plan p;
  int L = 0;
  while ((n >> L) > LEAF) ++L;
  // ceil(n / 2^L) <= LEAF
  while ((n + (1LL << L) - 1) / (1LL << L) > LEAF) ++L;
  p.L = L;
  // node boundaries at each depth: recursive halving, sizes differ by <= 1
  std::vector<std::vector<int64_t>> bounds(L + 1);
  bounds[0] = {0, n};
  for (int dpt = 1; dpt <= L; ++dpt) {
    auto& prev = bounds[dpt - 1];
    auto& cur = bounds[dpt];
    cur.push_back(0);
    for (size_t i = 0; i + 1 < prev.size(); ++i) {
      const int64_t a = prev[i], b = prev[i + 1];
      cur.push_back(a + (b - a) / 2);
      cur.push_back(b);
    }
  }
  auto& lb = bounds[L];
  for (size_t i = 0; i + 1 < lb.size(); ++i) {
    p.leaf_lo.push_back((int)lb[i]);
    p.leaf_hi.push_back((int)lb[i + 1]);
  }
  // merges: level t (t = 0 first processed) combines depth L-t children into depth L-t-1 nodes
  for (int dpt = L - 1; dpt >= 0; --dpt) {
    std::vector<int> lo, mid, hi;
    auto& b = bounds[dpt];
    auto& c = bounds[dpt + 1];
    for (size_t i = 0; i + 1 < b.size(); ++i) {
      lo.push_back((int)b[i]);
      mid.push_back((int)c[2 * i + 1]);
      hi.push_back((int)b[i + 1]);
      p.cuts.push_back((int)c[2 * i + 1]);
    }
    p.mlo.push_back(lo);
    p.mmid.push_back(mid);
    p.mhi.push_back(hi);
  }
  return p;
}

struct WsLayout {
  int64_t total = 0;
  int64_t add(int64_t bytes) {
    const int64_t o = total;
    total += (bytes + 255) / 256 * 256;
    return o;
  }
};

int64_t u_elems_for(const Plan& p) {
  int64_t mx = 0;
  for (size_t l = 0; l < p.mlo.size(); ++l) {
    int64_t t = 0;
    for (size_t i = 0; i < p.mlo[l].size(); ++i) {
      const int64_t s = p.mhi[l][i] - p.mlo[l][i];
      t += u_elems(s);
    }
    mx = std::max(mx, t);
  }
  return mx;
}

}  // namespace

int64_t stedc_ws_bytes(int64_t n) {
  Plan p = make_plan(n);
  const int64_t nm_total = std::max<int64_t>(1, (int64_t)p.cuts.size());
  WsLayout w;
  w.add(n * n * 8);                 // second ping-pong buffer
  w.add((n * n + n) * 8);           // compacted merge-GEMM operands (+ the pad column)
  w.add(u_elems_for(p) * 8);        // U
  w.add(24 * n * 8);                // per-element arrays
  w.add(nm_total * (M_NINT * 4 + 8 + 2 * (int64_t)sizeof(GemmArgs) + 8) + 4 * n * 4 + 4096);
  return w.total + 1024;
}

int stedc(cudaStream_t st, int64_t n, double* d, const double* e, double* Q, int64_t ldq,
          void* ws, int* info_host, int64_t col_lo, int64_t col_hi) {
  if (col_hi < 0 || col_hi > n) col_hi = n;
  if (col_lo < 0) col_lo = 0;
  if (col_lo > col_hi) col_lo = col_hi;
  if (info_host) *info_host = 0;
  if (n < 1) return OK;
  if (n > (int64_t)1 << 30) {
    set_error("stedc: n too large");
    return ERR_VALUE;
  }
  Plan p = make_plan(n);
  const int nlev = (int)p.mlo.size();
  const int64_t nm_total = std::max<int64_t>(1, (int64_t)p.cuts.size());
  // ---- workspace carve-up
  char* base = (char*)ws;
  WsLayout w;
  double* W2 = (double*)(base + w.add(n * n * 8));
  double* Xc = (double*)(base + w.add((n * n + n) * 8));
  double* Ubuf = (double*)(base + w.add(u_elems_for(p) * 8));
  double* arr = (double*)(base + w.add(24 * n * 8));
  char* misc = base + w.add(nm_total * (M_NINT * 4 + 8 + 2 * (int64_t)sizeof(GemmArgs) + 8) +
                            4 * n * 4 + 4096);
  double* dw = arr;            // working d
  double* ew = arr + n;        // scaled e
  double* dn = arr + 2 * n;    // next d
  MergeBufs B;
  B.Ds = arr + 3 * n; B.zs = arr + 4 * n; B.dl = arr + 5 * n; B.zl = arr + 6 * n;
  B.dv = arr + 7 * n; B.dvs = arr + 8 * n; B.rc = arr + 9 * n; B.rs = arr + 10 * n;
  B.tau = arr + 11 * n; B.lam = arr + 12 * n; B.zhat = arr + 13 * n;
  double* scal = arr + 14 * n;
  int* iarr = (int*)(arr + 15 * n);  // 9n doubles = 18n ints available
  B.colid = iarr; B.ctype = iarr + n; B.ncol = iarr + 2 * n; B.ntype = iarr + 3 * n;
  B.dcol = iarr + 4 * n; B.dcols = iarr + 5 * n; B.rp = iarr + 6 * n; B.rq = iarr + 7 * n;
  B.org = iarr + 8 * n; B.rpos = iarr + 9 * n; B.amapT = iarr + 10 * n; B.amapB = iarr + 11 * n;
  B.cmap = iarr + 12 * n;
  int* d_info = iarr + 13 * n;
  // misc: node arrays (lo/mid/hi for all levels + leaves + cuts), per-merge ints, rho, gargs, uoff
  int64_t mo = 0;
  auto take = [&](int64_t bytes) { char* r = misc + mo; mo += (bytes + 15) / 16 * 16; return r; };
  const int64_t nleaves = (int64_t)p.leaf_lo.size();
  int* d_nodes = (int*)take((3 * nm_total + 2 * nleaves + nm_total) * 4 + 64);
  B.mint = (int*)take(nm_total * M_NINT * 4);
  B.rho = (double*)take(nm_total * 8);
  B.gargs = (GemmArgs*)take(2 * nm_total * sizeof(GemmArgs));
  int64_t* d_uoff = (int64_t*)take(nm_total * 8);
  B.U = Ubuf;

  // ---- host node tables -> device (one copy)
  std::vector<int> hnodes;
  std::vector<int64_t> lev_off(nlev);
  for (int l = 0; l < nlev; ++l) {
    lev_off[l] = (int64_t)hnodes.size();
    for (int v : p.mlo[l]) hnodes.push_back(v);
    for (int v : p.mmid[l]) hnodes.push_back(v);
    for (int v : p.mhi[l]) hnodes.push_back(v);
  }
  const int64_t leaf_off = (int64_t)hnodes.size();
  for (int v : p.leaf_lo) hnodes.push_back(v);
  for (int v : p.leaf_hi) hnodes.push_back(v);
  const int64_t cut_off = (int64_t)hnodes.size();
  for (int v : p.cuts) hnodes.push_back(v);
  // U offsets per level (merges of one level share the U buffer)
  std::vector<int64_t> huoff;
  std::vector<int64_t> lev_uoff(nlev);
  for (int l = 0; l < nlev; ++l) {
    lev_uoff[l] = (int64_t)huoff.size();
    int64_t o = 0;
    for (size_t i = 0; i < p.mlo[l].size(); ++i) {
      const int64_t s = p.mhi[l][i] - p.mlo[l][i];
      huoff.push_back(o);
      o += u_elems(s);
    }
  }
  PEVD_CUDA(cudaMemcpyAsync(d_nodes, hnodes.data(), hnodes.size() * 4, cudaMemcpyHostToDevice, st));
  if (!huoff.empty())
    PEVD_CUDA(cudaMemcpyAsync(d_uoff, huoff.data(), huoff.size() * 8, cudaMemcpyHostToDevice, st));
  PEVD_CUDA(cudaMemsetAsync(d_info, 0, 4, st));

  // ---- scale, tear
  absmax_kernel<<<1, 256, 0, st>>>(n, d, e, scal);
  scale_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 4096), 256, 0, st>>>(n, d, e, dw, ew,
                                                                                scal);
  PEVD_LAUNCH_CHECK();
  if (!p.cuts.empty()) {
    tear_kernel<<<1, 32, 0, st>>>(dw, ew, d_nodes + cut_off, (int)p.cuts.size());
    PEVD_LAUNCH_CHECK();
  }
  // ---- ping-pong buffers: leaves go where the last level ends up in Q
  double* bufs[2] = {Q, W2};
  int64_t lds[2] = {ldq, n};
  int cur = (nlev % 2 == 0) ? 0 : 1;
  for (int b = 0; b < 2; ++b) {
    if (lds[b] == n) {
      zero_fill<<<4096, 256, 0, st>>>(bufs[b], n * n);
    } else {
      PEVD_CUDA(cudaMemset2DAsync(bufs[b], lds[b] * 8, 0, n * 8, n, st));
    }
    PEVD_LAUNCH_CHECK();
  }
  leaf_kernel<<<(unsigned)cdiv(nleaves, 4), 128, 0, st>>>(d_nodes + leaf_off,
                                                          d_nodes + leaf_off + nleaves,
                                                          (int)nleaves, dw, ew, bufs[cur],
                                                          lds[cur], d_info);
  PEVD_LAUNCH_CHECK();
  B.ew = ew;
  for (int l = 0; l < nlev; ++l) {
    const int nm = (int)p.mlo[l].size();
    int smax = 0, hmax = 0;
    for (int i = 0; i < nm; ++i) {
      smax = std::max(smax, p.mhi[l][i] - p.mlo[l][i]);
      hmax = std::max(hmax, std::max(p.mmid[l][i] - p.mlo[l][i], p.mhi[l][i] - p.mmid[l][i]));
    }
    B.lo = d_nodes + lev_off[l];
    B.mid = B.lo + nm;
    B.hi = B.mid + nm;
    B.uoff = d_uoff + lev_uoff[l];
    B.Dcur = dw;
    B.Dnext = dn;
    double* X = bufs[cur];
    const int64_t ldx = lds[cur];
    double* Y = bufs[cur ^ 1];
    const int64_t ldy = lds[cur ^ 1];
    const unsigned gx = (unsigned)cdiv(smax, 256);
    merge_prep<<<dim3(gx, nm), 256, 0, st>>>(B, X, ldx);
    PEVD_LAUNCH_CHECK();
    merge_deflate<<<nm, 32, 0, st>>>(B);
    PEVD_LAUNCH_CHECK();
    merge_rotate<<<dim3(gx, nm), 256, 0, st>>>(B, X, ldx);
    PEVD_LAUNCH_CHECK();
    merge_secular<<<dim3((unsigned)cdiv((int64_t)smax * SEC_G, 256), nm), 256, 0, st>>>(B, d_info);
    PEVD_LAUNCH_CHECK();
    merge_zhat<<<dim3((unsigned)cdiv(smax, 128), nm), 128, 0, st>>>(B);
    PEVD_LAUNCH_CHECK();
    merge_sort_deflated<<<dim3((unsigned)cdiv(smax, 128), nm), 128, 0, st>>>(B);
    PEVD_LAUNCH_CHECK();
    merge_vectors<<<dim3((unsigned)cdiv(smax, 8), nm), 256, 0, st>>>(B);
    PEVD_LAUNCH_CHECK();
    // only the last level writes Q: it alone is restricted to the wanted columns
    const int64_t clo = (l == nlev - 1) ? col_lo : 0, chi = (l == nlev - 1) ? col_hi : n;
    merge_gather_cols<<<dim3((unsigned)smax + 1, nm), 256, 0, st>>>(B, X, ldx, Xc, n);
    PEVD_LAUNCH_CHECK();
    merge_gemm_args<<<(unsigned)cdiv(nm, 128), 128, 0, st>>>(B, Xc, n, Y, ldy, nm, clo, chi);
    PEVD_LAUNCH_CHECK();
    PEVD_TRY(gemm_grouped(st, B.gargs, 2 * nm, hmax, smax));
    merge_deflated_copy<<<dim3((unsigned)smax, nm), 256, 0, st>>>(B, X, ldx, Y, ldy, clo, chi);
    PEVD_LAUNCH_CHECK();
    std::swap(dw, dn);
    cur ^= 1;
  }
  // cur now indexes Q
  finalize_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 4096), 256, 0, st>>>(n, dw, d, scal);
  PEVD_LAUNCH_CHECK();
  if (col_hi > col_lo) {
    sign_fix<<<(unsigned)(col_hi - col_lo), 256, 0, st>>>(n, Q, ldq, col_lo);
  }
  PEVD_LAUNCH_CHECK();
  if (info_host) {
    PEVD_CUDA(cudaMemcpyAsync(info_host, d_info, 4, cudaMemcpyDeviceToHost, st));
  }
  return OK;
}

}  // namespace pevd

// ------------------------------------------------------------------ eigenvalues only: bisection
// With want_vectors = 0 nothing needs the eigenvector matrix, so instead of the divide and
// conquer (whose merges are O(n^3) eigenvector GEMMs) every eigenvalue is found independently by
// bisection on the Sturm count of T - x I (LAPACK dstebz's recurrence with its pivmin guard):
// one thread per eigenvalue, O(n) per count, ~ 64 counts each; the k-th thread converges to the
// k-th smallest eigenvalue, so the output is ascending.  Accuracy: an interval of relative width
// ~ 2 eps around each eigenvalue, well inside the north star's 10 n eps ||A||_2.
namespace pevd {
namespace {

__global__ void stebz_bounds_kernel(int64_t n, const double* __restrict__ d,
                                    const double* __restrict__ e, double* out) {
  // out[0] = gershgorin lower, out[1] = upper, out[2] = pivmin (block-reduced by one CTA)
  __shared__ double slo[256], shi[256], sem[256];
  double lo = INFINITY, hi = -INFINITY, em = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double el = i > 0 ? fabs(e[i - 1]) : 0.0, er = i + 1 < n ? fabs(e[i]) : 0.0;
    lo = fmin(lo, d[i] - el - er);
    hi = fmax(hi, d[i] + el + er);
    em = fmax(em, er * er);
  }
  slo[threadIdx.x] = lo;
  shi[threadIdx.x] = hi;
  sem[threadIdx.x] = em;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      slo[threadIdx.x] = fmin(slo[threadIdx.x], slo[threadIdx.x + s]);
      shi[threadIdx.x] = fmax(shi[threadIdx.x], shi[threadIdx.x + s]);
      sem[threadIdx.x] = fmax(sem[threadIdx.x], sem[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tnorm = fmax(fabs(slo[0]), fabs(shi[0]));
    const double eps = 2.220446049250313e-16, safmin = 2.2250738585072014e-308;
    const double pad = 2.0 * eps * tnorm * (double)n + 2.0 * safmin;
    out[0] = slo[0] - pad;
    out[1] = shi[0] + pad;
    out[2] = fmax(safmin, safmin * sem[0]);  // dstebz's pivmin
  }
}

// number of eigenvalues of T strictly less than x
__device__ __forceinline__ int64_t sturm_count(int64_t n, const double* __restrict__ d,
                                               const double* __restrict__ e2, double x,
                                               double pivmin) {
  int64_t cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int64_t i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

__global__ void stebz_e2_kernel(int64_t n, const double* __restrict__ e, double* __restrict__ e2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < n;
       i += (int64_t)gridDim.x * blockDim.x)
    e2[i] = e[i] * e[i];
}

__global__ void __launch_bounds__(128)
    stebz_kernel(int64_t n, const double* __restrict__ d, const double* __restrict__ e2,
                 const double* __restrict__ bnd, double* __restrict__ lam) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // wanted: k-th smallest
  if (k >= n) return;
  double lo = bnd[0], hi = bnd[1];
  const double pivmin = bnd[2];
  const double eps = 2.220446049250313e-16;
  for (int it = 0; it < 128; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) + pivmin || mid <= lo || mid >= hi) break;
    if (sturm_count(n, d, e2, mid, pivmin) > k) hi = mid;
    else lo = mid;
  }
  lam[k] = 0.5 * (lo + hi);
}

}  // namespace

int64_t stebz_ws_bytes(int64_t n) { return (n + 8) * 8; }

int stebz(cudaStream_t st, int64_t n, const double* d, const double* e, double* lam, void* ws) {
  if (n < 1) return OK;
  double* bnd = (double*)ws;
  double* e2 = bnd + 4;
  stebz_e2_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4096)), 256, 0,
                    st>>>(n, e, e2);
  PEVD_LAUNCH_CHECK();
  stebz_bounds_kernel<<<1, 256, 0, st>>>(n, d, e, bnd);
  PEVD_LAUNCH_CHECK();
  stebz_kernel<<<(unsigned)cdiv(n, 128), 128, 0, st>>>(n, d, e2, bnd, lam);
  PEVD_LAUNCH_CHECK();
  return OK;
}

}  // namespace pevd
