/*
 * pevd_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, scalar, single thread) of the three scalar
 * kernels of the reference `pipeevd` package, used as the parity checker for
 * the CUDA path and as the CPU baseline leg of bench.py.  Nothing in the
 * product path links or calls this library; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may.
 *
 * Restated functions (reference paths relative to /root/reference/pkg/src/pipeevd):
 *   orc_chase      <- bulge.py:170-252   (_chase, numba njit)
 *   orc_steqr      <- tridiag.py:133-295 (_steqr, with _lartg :47-67, _laev2 :70-130)
 *   orc_rank1_seq  <- backtrans.py:252-274 (_rank1_seq)
 *
 * Compiled with -ffp-contract=off so that no multiply-add is fused: the
 * arithmetic then rounds operation by operation exactly like the numba
 * kernels, and the golden fixtures in tests/golden/ pin it bit-for-bit.
 *
 * Matrices are row-major (C order) like the numpy arrays the reference
 * kernels receive.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <float.h>

#define S(r, c) s[(int64_t)(r) * lds + (c)]

/* Householder bulge chase over sweeps [i0, min(i1, n-2)) on a dense
 * row-major window `s` (leading dimension lds) whose row/col 0 is global
 * index col0.  Records one reflector per non-trivial step.  Returns the
 * number of recorded reflectors; *macs receives the MAC count.  */
int64_t orc_chase(double* s, int64_t lds, int64_t col0, int64_t n, int64_t b,
                  int64_t i0, int64_t i1, int64_t* i_arr, int64_t* j_arr,
                  int64_t* row0_arr, int64_t* len_arr, double* tau_arr,
                  double* v_arr, int64_t v_stride, int64_t* macs) {
  double ubuf[4096], wbuf[4096];
  int64_t cnt = 0, mac = 0;
  int64_t hi = i1 < n - 2 ? i1 : n - 2;
  for (int64_t gi = i0; gi < hi; ++gi) {
    for (int64_t j = 0; gi + 1 + j * b <= n - 2; ++j) {
      const int64_t cg = (j == 0) ? gi : gi + 1 + (j - 1) * b;
      const int64_t w0 = gi + 1 + j * b;
      const int64_t L = (b < n - w0) ? b : n - w0;
      const int64_t wl = w0 - col0, cl = cg - col0;
      double tail = 0.0;
      for (int64_t r = 1; r < L; ++r) tail += S(wl + r, cl) * S(wl + r, cl);
      if (tail == 0.0) continue;
      const double x0 = S(wl, cl);
      const double nrm = sqrt(x0 * x0 + tail);
      const double alpha = (x0 >= 0.0) ? -nrm : nrm;
      const double denom = x0 - alpha;
      double* v = v_arr + cnt * v_stride;
      v[0] = 1.0;
      double vsq = 1.0;
      for (int64_t r = 1; r < L; ++r) {
        v[r] = S(wl + r, cl) / denom;
        vsq += v[r] * v[r];
      }
      const double tau = 2.0 / vsq;
      i_arr[cnt] = gi; j_arr[cnt] = j; row0_arr[cnt] = w0; len_arr[cnt] = L;
      tau_arr[cnt] = tau;
      /* annihilate the column below its pivot, mirrored */
      S(wl, cl) = alpha;
      S(cl, wl) = alpha;
      for (int64_t r = 1; r < L; ++r) { S(wl + r, cl) = 0.0; S(cl, wl + r) = 0.0; }
      /* H applied from the left to the bulge columns strictly between */
      for (int64_t c = cl + 1; c < wl; ++c) {
        double dot = 0.0;
        for (int64_t r = 0; r < L; ++r) dot += v[r] * S(wl + r, c);
        dot *= tau;
        for (int64_t r = 0; r < L; ++r) {
          S(wl + r, c) -= dot * v[r];
          S(c, wl + r) = S(wl + r, c);
        }
        mac += 2 * L;
      }
      /* H A H on the window square */
      for (int64_t r = 0; r < L; ++r) {
        double acc = 0.0;
        for (int64_t c = 0; c < L; ++c) acc += S(wl + r, wl + c) * v[c];
        ubuf[r] = tau * acc;
      }
      double gam = 0.0;
      for (int64_t r = 0; r < L; ++r) gam += v[r] * ubuf[r];
      gam *= 0.5 * tau;
      for (int64_t r = 0; r < L; ++r) wbuf[r] = ubuf[r] - gam * v[r];
      for (int64_t r = 0; r < L; ++r)
        for (int64_t c = 0; c < L; ++c)
          S(wl + r, wl + c) -= v[r] * wbuf[c] + wbuf[r] * v[c];
      mac += 3 * L * L + 3 * L;
      /* H from the right on the next b rows (creates the next bulge) */
      int64_t t_end = (w0 + L + b < n ? w0 + L + b : n) - col0;
      for (int64_t t = wl + L; t < t_end; ++t) {
        double dot = 0.0;
        for (int64_t r = 0; r < L; ++r) dot += S(t, wl + r) * v[r];
        dot *= tau;
        for (int64_t r = 0; r < L; ++r) {
          S(t, wl + r) -= dot * v[r];
          S(wl + r, t) = S(t, wl + r);
        }
        mac += 2 * L;
      }
      ++cnt;
    }
  }
  if (macs) *macs = mac;
  return cnt;
}

/* plane rotation with c*f + s*g = r, c*g - s*f = 0 (tridiag.py:47-67) */
static void orc_lartg(double f, double g, double* c, double* s, double* r) {
  if (g == 0.0) { *c = 1.0; *s = 0.0; *r = f; return; }
  if (f == 0.0) { *c = 0.0; *s = 1.0; *r = g; return; }
  double rr = sqrt(f * f + g * g);
  if (rr == 0.0) {
    const double scl = 1.0 / DBL_MIN;
    const double fs = f * scl, gs = g * scl;
    rr = sqrt(fs * fs + gs * gs) * DBL_MIN;
  }
  double cc = f / rr, ss = g / rr;
  if (fabs(f) > fabs(g) && cc < 0.0) { cc = -cc; ss = -ss; rr = -rr; }
  *c = cc; *s = ss; *r = rr;
}

/* closed-form 2x2 symmetric eigenproblem (tridiag.py:70-130) */
static void orc_laev2(double a, double b, double c, double* rt1, double* rt2,
                      double* cs1, double* sn1) {
  const double sm = a + c, df = a - c, adf = fabs(df), tb = b + b, ab = fabs(tb);
  double acmx, acmn, rt, sgn1, sgn2, cs;
  if (fabs(a) > fabs(c)) { acmx = a; acmn = c; } else { acmx = c; acmn = a; }
  if (adf > ab) { double q = ab / adf; rt = adf * sqrt(1.0 + q * q); }
  else if (adf < ab) { double q = adf / ab; rt = ab * sqrt(1.0 + q * q); }
  else rt = ab * sqrt(2.0);
  if (sm < 0.0) { *rt1 = 0.5 * (sm - rt); sgn1 = -1.0; *rt2 = (acmx / *rt1) * acmn - (b / *rt1) * b; }
  else if (sm > 0.0) { *rt1 = 0.5 * (sm + rt); sgn1 = 1.0; *rt2 = (acmx / *rt1) * acmn - (b / *rt1) * b; }
  else { *rt1 = 0.5 * rt; *rt2 = -0.5 * rt; sgn1 = 1.0; }
  if (df >= 0.0) { cs = df + rt; sgn2 = 1.0; } else { cs = df - rt; sgn2 = -1.0; }
  const double acs = fabs(cs);
  double c1, s1;
  if (acs > ab) { double ct = -tb / cs; s1 = 1.0 / sqrt(1.0 + ct * ct); c1 = ct * s1; }
  else if (ab == 0.0) { c1 = 1.0; s1 = 0.0; }
  else { double tn = -cs / tb; c1 = 1.0 / sqrt(1.0 + tn * tn); s1 = tn * c1; }
  if (sgn1 == sgn2) { double tn = c1; c1 = -s1; s1 = tn; }
  *cs1 = c1; *sn1 = s1;
}

/* rotate rows p, q of the row-major eigenvector-candidate matrix zt */
static inline void rot_rows(double* zt, int64_t nrow, int64_t p, int64_t q,
                            double c, double s, int ql) {
  double* a = zt + p * nrow;
  double* b = zt + q * nrow;
  if (ql) {  /* QL chase: a' = c a - s b, b' = s a + c b */
    for (int64_t k = 0; k < nrow; ++k) {
      const double za = a[k], zb = b[k];
      a[k] = c * za - s * zb;
      b[k] = s * za + c * zb;
    }
  } else {   /* QR chase / 2x2: a' = c a + s b, b' = c b - s a */
    for (int64_t k = 0; k < nrow; ++k) {
      const double za = a[k], zb = b[k];
      a[k] = c * za + s * zb;
      b[k] = c * zb - s * za;
    }
  }
}

/* Implicit-shift QL/QR (tridiag.py:133-295).  d (n), e (n, e[n-1]=0) are
 * overwritten; zt is n x nrow row-major (nrow = 0 for values only).
 * Returns failed index (-1 on success); *total / *rots receive the shift
 * and rotation counts.  */
int64_t orc_steqr(double* d, double* e, int64_t n, double* zt, int64_t nrow,
                  int64_t cap, int64_t* total_out, int64_t* rots_out) {
  const double ulp = 0.5 * DBL_EPSILON, eps2 = ulp * ulp;
  int64_t total = 0, rots = 0, l1 = 0;
  while (l1 < n) {
    if (l1 > 0) e[l1 - 1] = 0.0;
    int64_t m = n - 1;
    for (int64_t mm = l1; mm < n - 1; ++mm) {
      const double tst = fabs(e[mm]);
      if (tst == 0.0) { m = mm; break; }
      if (tst <= (sqrt(fabs(d[mm])) * sqrt(fabs(d[mm + 1]))) * ulp) { e[mm] = 0.0; m = mm; break; }
    }
    int64_t l = l1, lend = m;
    l1 = m + 1;
    if (lend == l) continue;
    if (fabs(d[lend]) < fabs(d[l])) { int64_t t = l; l = lend; lend = t; }
    if (lend > l) {
      for (;;) {  /* QL */
        m = lend;
        for (int64_t mm = l; mm < lend; ++mm) {
          const double tst = e[mm] * e[mm];
          if (tst <= (eps2 * fabs(d[mm])) * fabs(d[mm + 1]) + DBL_MIN) { m = mm; break; }
        }
        if (m < lend) e[m] = 0.0;
        double p = d[l];
        if (m == l) { ++l; if (l <= lend) continue; break; }
        if (m == l + 1) {
          double rt1, rt2, cc, ss;
          orc_laev2(d[l], e[l], d[l + 1], &rt1, &rt2, &cc, &ss);
          ++rots;
          if (nrow) rot_rows(zt, nrow, l, l + 1, cc, ss, 0);
          d[l] = rt1; d[l + 1] = rt2; e[l] = 0.0;
          l += 2;
          if (l <= lend) continue;
          break;
        }
        if (total == cap) { *total_out = total; *rots_out = rots; return l; }
        ++total;
        double g = (d[l + 1] - p) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[m] - p + e[l] / (g + (g >= 0.0 ? r : -r));
        double s = 1.0, c = 1.0;
        p = 0.0;
        for (int64_t i = m - 1; i >= l; --i) {
          const double f = s * e[i], bb = c * e[i];
          orc_lartg(g, f, &c, &s, &r);
          if (i != m - 1) e[i + 1] = r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * bb;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - bb;
          ++rots;
          if (nrow) rot_rows(zt, nrow, i, i + 1, c, s, 1);
        }
        d[l] = d[l] - p;
        e[l] = g;
      }
    } else {
      for (;;) {  /* QR */
        m = lend;
        for (int64_t mm = l; mm > lend; --mm) {
          const double tst = e[mm - 1] * e[mm - 1];
          if (tst <= (eps2 * fabs(d[mm])) * fabs(d[mm - 1]) + DBL_MIN) { m = mm; break; }
        }
        if (m > lend) e[m - 1] = 0.0;
        double p = d[l];
        if (m == l) { --l; if (l >= lend) continue; break; }
        if (m == l - 1) {
          double rt1, rt2, cc, ss;
          orc_laev2(d[l - 1], e[l - 1], d[l], &rt1, &rt2, &cc, &ss);
          ++rots;
          if (nrow) rot_rows(zt, nrow, l - 1, l, cc, ss, 0);
          d[l - 1] = rt1; d[l] = rt2; e[l - 1] = 0.0;
          l -= 2;
          if (l >= lend) continue;
          break;
        }
        if (total == cap) { *total_out = total; *rots_out = rots; return l; }
        ++total;
        double g = (d[l - 1] - p) / (2.0 * e[l - 1]);
        double r = hypot(g, 1.0);
        g = d[m] - p + e[l - 1] / (g + (g >= 0.0 ? r : -r));
        double s = 1.0, c = 1.0;
        p = 0.0;
        for (int64_t i = m; i < l; ++i) {
          const double f = s * e[i], bb = c * e[i];
          orc_lartg(g, f, &c, &s, &r);
          if (i != m) e[i - 1] = r;
          g = d[i] - p;
          r = (d[i + 1] - g) * s + 2.0 * c * bb;
          p = s * r;
          d[i] = g + p;
          g = c * r - bb;
          ++rots;
          if (nrow) rot_rows(zt, nrow, i, i + 1, c, s, 0);
        }
        d[l] = d[l] - p;
        e[l - 1] = g;
      }
    }
  }
  *total_out = total; *rots_out = rots;
  return -1;
}

/* Rank-1 reflector replay (backtrans.py:252-274): for each position p in
 * `order`, X[r0:r0+l, :] -= tau v (v^T X[r0:r0+l, :]).  X is row-major
 * (nrows x m).  Returns the MAC count.  */
int64_t orc_rank1_seq(double* q, int64_t m, const int64_t* order, int64_t norder,
                      const int64_t* row0, const int64_t* length,
                      const double* tau, const double* v, int64_t v_stride,
                      double* dots) {
  int64_t mac = 0;
  for (int64_t oo = 0; oo < norder; ++oo) {
    const int64_t p = order[oo];
    const int64_t r0 = row0[p], ell = length[p];
    const double t = tau[p];
    const double* vp = v + p * v_stride;
    for (int64_t k = 0; k < m; ++k) dots[k] = 0.0;
    for (int64_t r = 0; r < ell; ++r) {
      const double vr = vp[r];
      const double* row = q + (r0 + r) * m;
      for (int64_t k = 0; k < m; ++k) dots[k] += vr * row[k];
    }
    for (int64_t k = 0; k < m; ++k) dots[k] *= t;
    for (int64_t r = 0; r < ell; ++r) {
      const double vr = vp[r];
      double* row = q + (r0 + r) * m;
      for (int64_t k = 0; k < m; ++k) row[k] -= vr * dots[k];
    }
    mac += 2 * ell * m;
  }
  return mac;
}
