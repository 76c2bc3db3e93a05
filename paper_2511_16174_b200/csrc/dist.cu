// Blockwise multi-GPU pipelined EVD: the per-rank orchestrator (pipeline.py:170-508 restated for
// one GPU per rank, driven by a C++ host thread instead of Python).
//
// Distribution (the paper's blockwise columns, schedule.py:21-33): rank r owns the column block
// [col_lo[r], col_lo[r+1]) with ALL n rows ("full storage").  Per SBR round
// (c0, pw, t0 = c0 + b) of round_schedule:
//   * the panel's owner factors it (straddling pieces arrive by an all-gather) and broadcasts
//     the factor [W | Y | T | R] (C4 of SURVEY §2.3; the reference ships (W, Y), pipeline.py:236);
//   * every rank forms the rows of A W that belong to its own columns BY SYMMETRY from those
//     columns (the off-diagonal row blocks from the full columns, its own diagonal block from its
//     lower triangle), and the row blocks are all-gathered (C5, pipeline.py:251-271);
//   * Z = A W - 1/2 Y (W^T A W) on every rank; each rank updates only its own columns.
// Panels are double-blocked 16 at a time exactly as on one GPU (sbr.cu): a panel's
// columns take the group's pending updates P1 P2^T just before its QR, A W_i is corrected by
// -P1 (P2^T W_i), and each rank's trailing columns receive ONE rank-2K update per group, split in
// three: the rows above the rank's diagonal block and below it (full storage) and the diagonal
// block itself on its lower tiles only -- so one rank does exactly the single-GPU flops.
// Lookahead: the trailing update runs on its own stream; the next group's first panel columns
// are updated first on the compute stream, so that panel's QR and broadcast proceed while the
// rank-2K update of the rest of the trailing matrix is still running.
// Collectives run on a comm stream ordered by events, and every collective is a trace span of
// stage "Comm" with the words it moved.
//
// BC and the solver: the band (13 MB at n = 49152) is all-gathered and every rank runs the
// deterministic wavefront chase (bitwise identical everywhere).  The chase's critical path is
// ~3n step slots whatever the GPU count, so the reference's relay (bulge.py:348-385, serial across
// workers by design, README.md:117-121) would add hand-offs and a 10 GB reflector all-gather
// without shortening it.  The divide and conquer forms only the rank's back-transform columns in
// conventional order (pevd_stedc_cols); eigenvalues-only runs use bisection (stebz).
//
// Back transformation, per order (pipeline.py:367-413):
//   conventional: Q[:, cols] = Q_s Q_b Q_d[:, cols] for the rank's columns (back_lo): BC-Back on
//     the transpose, then the aggregated SBR-Back from the left; no communication at all.
//   pipelined: on a back stream, right after the SBR: the rank's rows of Q_s (RowAccumulator,
//     backtrans.py:149-183) -- overlapping the band gather, the chase and the D&C -- then
//     BC-Back on those rows once the chase is done, then Q[rows, :] = (Q_s Q_b)[rows, :] Q_d.
//   sequential: the same stages on one stream.
#include <time.h>
#include <cstring>
#include <string>
#include <thread>
#include "comm.h"
#include "kernels.cuh"
#include "../../include/pevd.h"

namespace pevd {

namespace {

constexpr int NBB = 16;  // panels per double-blocked group (as sbr.cu)
constexpr int64_t SKN = 4 << 20;

// trace stages (pevd.h PEVD_TRACE_*)
enum : int { TR_SBR = 0, TR_BC = 1, TR_SBR_BACK = 2, TR_BC_BACK = 3, TR_SOLVER = 4, TR_FINAL = 5,
             TR_COMM = 6 };

double mono_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e9 + (double)ts.tv_nsec;
}

// own band diagonals, packed per column: out[(c - lo) (b + 1) + d] = A[c + d, c]
__global__ void band_pack_kernel(int64_t n, int b, int64_t lo, int64_t w,
                                 const double* __restrict__ blk, int64_t ldb,
                                 double* __restrict__ out) {
  const int64_t total = w * (b + 1);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / (b + 1);
    const int d = (int)(idx % (b + 1));
    const int64_t c = lo + j;
    out[idx] = (c + d < n) ? blk[(c + d) + j * ldb] : 0.0;
  }
}

// the factored panel's columns become [R; 0] below the panel's row t0, for own columns
// [c_lo, c_hi) of the panel [ci, ci + pw) (blk column j = global column lo + j)
__global__ void write_r_kernel(int64_t m, int pw, int64_t t0, int64_t ci, int64_t c_lo,
                               int64_t c_hi, int64_t lo, const double* __restrict__ R,
                               double* __restrict__ blk, int64_t ldb) {
  const int64_t nc = c_hi - c_lo;
  const int64_t total = nc * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % m, c = c_lo + idx / m;
    const int64_t pc = c - ci;
    blk[(t0 + r) + (c - lo) * ldb] = (r < pw && r <= pc) ? R[r + pc * pw] : 0.0;
  }
}

// M (r x n, ld r) = rows [r0, r0 + r) of the identity
__global__ void rows_of_identity(int64_t r, int64_t n, int64_t r0, double* __restrict__ M) {
  const int64_t total = r * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % r, c = idx / r;
    M[idx] = (c == r0 + i) ? 1.0 : 0.0;
  }
}

unsigned grid_for(int64_t total, int64_t cap = 8192) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), cap));
}

struct Arena {
  char* base = nullptr;
  int64_t off = 0, cap = 0;
  template <class T>
  T* take(int64_t elems) {
    T* p = base ? (T*)(base + off) : nullptr;
    off += (elems * (int64_t)sizeof(T) + 255) / 256 * 256;
    return p;
  }
};

struct Span {
  int stage, block, lane;  // lane: the worker, or -1 (HOST) for the concurrent back stream
  cudaEvent_t a, b;
  int64_t words;
};
constexpr int TR_SBR_ALL = 100;  // whole-SBR span for the stage times (not a trace event: the
                                 // trace's SBR event of a rank spans the rounds it owns)

// per-rank state of one distributed EVD
struct Rank {
  Comm& C;
  int r, G;
  int64_t n;
  int b, want_vectors, order;
  const int64_t *col_lo, *back_lo;
  int64_t lo, hi, w;  // own SBR columns
  cudaStream_t cs, ms, ts, bs;
  // buffers
  double *blk, *Ystair, *Tall, *P[2][2], *BUF, *gbuf, *AWt, *piece, *Mb, *tv, *sk, *bandT, *bands;
  double *d, *e, *tau, *V, *Qd, *Mrows, *dl, *el, *band_out, *tailbuf, *ovbuf, *ugather;
  int64_t* uprefix;
  void *qrws, *ws_bc, *ws_dc, *ws_back, *ws_bcb;
  int vld;
  int64_t ldb;
  std::vector<Span> spans;
  std::vector<cudaEvent_t> evpool;
  cudaEvent_t base = nullptr;
  int64_t sbr_span = -1;

  Rank(Comm& c, int64_t n_, int b_, int wv, int ord, const int64_t* cl, const int64_t* bl)
      : C(c), r(c.rank()), G(c.size()), n(n_), b(b_), want_vectors(wv), order(ord), col_lo(cl),
        back_lo(bl) {
    lo = col_lo[r];
    hi = col_lo[r + 1];
    w = hi - lo;
  }

  int owner_of(int64_t col) const {
    for (int x = 0; x < G; ++x)
      if (col >= col_lo[x] && col < col_lo[x + 1]) return x;
    return G - 1;
  }

  cudaEvent_t new_event() {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    evpool.push_back(e);
    return e;
  }
  // e recorded on `from`, waited on by `to`
  int link(cudaStream_t from, cudaStream_t to) {
    if (from == to) return OK;
    cudaEvent_t e = nullptr;
    PEVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    evpool.push_back(e);
    PEVD_CUDA(cudaEventRecord(e, from));
    PEVD_CUDA(cudaStreamWaitEvent(to, e, 0));
    return OK;
  }
  size_t open(int stage, int block, cudaStream_t st, int64_t words = 0, int lane = -2) {
    spans.push_back(Span{stage, block, lane == -2 ? r : lane, new_event(), new_event(), words});
    cudaEventRecord(spans.back().a, st);
    return spans.size() - 1;
  }
  void close(size_t idx, cudaStream_t st) { cudaEventRecord(spans[idx].b, st); }

  // collectives on the comm stream, ordered after `after` and before later work on `after`
  int bcast(void* buf, int64_t bytes, int root, cudaStream_t after, int block) {
    if (G == 1) return OK;
    PEVD_TRY(link(after, ms));
    const size_t sp = open(TR_COMM, block, ms, bytes / 8);
    PEVD_TRY(C.bcast(buf, bytes, root, ms));
    close(sp, ms);
    return link(ms, after);
  }
  int allgatherv(const void* send, const int64_t* counts, void* recv, cudaStream_t after,
                 int block, int stage) {
    if (G > 1 && counts[r] > 0) C.record(r, DST_BROADCAST, stage, counts[r] / 8);
    if (G == 1) {
      if (counts[0] > 0 && send != recv)
        PEVD_CUDA(cudaMemcpyAsync(recv, send, counts[0], cudaMemcpyDeviceToDevice, after));
      return OK;
    }
    int64_t tot = 0;
    for (int x = 0; x < G; ++x) tot += counts[x];
    PEVD_TRY(link(after, ms));
    const size_t sp = open(TR_COMM, block, ms, tot / 8);
    PEVD_TRY(C.allgatherv(send, counts, recv, ms));
    close(sp, ms);
    return link(ms, after);
  }

  int p2p(const void* send, void* recv, int64_t words, int src, int dst, cudaStream_t after,
          int stage) {
    if (G == 1 || words <= 0 || src == dst) return OK;
    if (r == src) C.record(src, dst, stage, words);
    PEVD_TRY(link(after, ms));
    const size_t sp = open(TR_COMM, src, ms, words);
    PEVD_TRY(C.p2p(send, recv, words * 8, src, dst, ms));
    close(sp, ms);
    return link(ms, after);
  }

  int gemm_(cudaStream_t st, GemmArgs g) { return gemm(st, g, sk, SKN); }
  int relay_chase();

  int sbr();
  int panel(int64_t x, int64_t ci, int pw, int64_t ti, double* P1, double* P2, int64_t t0, int i,
            cudaEvent_t trail_done);
  int trailing(int64_t t0, int64_t tl, int64_t K2, const double* P1, const double* P2,
               int64_t ru, int64_t strip_hi, cudaStream_t st_strip, cudaStream_t st_rest);
};

// one panel of a double-blocked group (i = index in the group, t0 = group's trailing start).
// P1 / P2 hold the group's [Y Z ...] / [Z Y ...] (block-relative rows from t0).
int Rank::panel(int64_t x, int64_t ci, int pw, int64_t ti, double* P1, double* P2, int64_t t0,
                int i, cudaEvent_t trail_done) {
  const int64_t m = n - ti;
  const int64_t ri = (int64_t)i * b;
  const int owner = owner_of(ci);
  const int64_t plo = std::max(ci, lo), phi = std::min<int64_t>(ci + pw, hi);  // own panel cols
  // 1. the group's pending updates on our part of the panel columns (rows ci..n)
  flops_set_stage(ST_SBR);
  if (i >= 1 && plo < phi) {
    GemmArgs g{n - ci, phi - plo, 2 * ri, -1.0, 1.0, P1 + (ri - b), n, P2 + (plo - t0), n,
               blk + ci + (plo - lo) * ldb, ldb, 0, 1, A_GENERAL, C_ALL};
    PEVD_TRY(gemm_(cs, g));
  }
  // 2. straddling panel: the pieces go to every rank (only the owner factors)
  bool straddle = col_lo[owner + 1] < ci + pw;
  const double* P = blk + ti + (ci - lo) * ldb;
  int64_t ldp = ldb;
  if (straddle) {
    std::vector<int64_t> cnt(G, 0);
    for (int y = 0; y < G; ++y) {
      const int64_t a = std::max(ci, col_lo[y]), z = std::min<int64_t>(ci + pw, col_lo[y + 1]);
      if (a < z) cnt[y] = (z - a) * m * 8;
    }
    if (plo < phi)
      PEVD_CUDA(cudaMemcpy2DAsync(gbuf + (plo - ci) * m, m * 8, blk + ti + (plo - lo) * ldb,
                                  ldb * 8, m * 8, phi - plo, cudaMemcpyDeviceToDevice, cs));
    PEVD_TRY(allgatherv(plo < phi ? gbuf + (plo - ci) * m : gbuf, cnt.data(), gbuf, cs, (int)x,
                        LS_SBR_PANEL));
    P = gbuf;
    ldp = m;
  }
  // 3. panel QR at the owner: BUF = [W (m x pw) | Y (m x pw) | T (pw^2) | R (pw^2)]
  double* Wb = BUF;
  double* Yb = BUF + m * pw;
  double* Tb = Yb + m * pw;
  double* Rb = Tb + (int64_t)pw * pw;
  if (r == owner) {
    if (sbr_span < 0) sbr_span = (int64_t)open(TR_SBR, r, cs);  // first round this rank owns
    PEVD_TRY(panel_qr(cs, m, pw, P, ldp, Rb, Yb, m, nullptr, 0, Wb, m, Tb, qrws));
    if (G > 1) {  // one physical broadcast, booked as the reference books it
      C.record(owner, DST_BROADCAST, LS_SBR, 2 * m * pw);                  // (W, Y): pipeline.py:236
      C.record(owner, DST_BROADCAST, LS_SBR_PANEL, 2 * (int64_t)pw * pw);  // T and R
    }
  }
  // 4. broadcast the factor
  PEVD_TRY(bcast(BUF, (2 * m * pw + 2 * (int64_t)pw * pw) * 8, owner, cs, (int)x));
  if (r == owner) PEVD_CUDA(cudaEventRecord(spans[sbr_span].b, cs));  // ... to its last
  // 5. keep Y (staircase) and T for the back transformation; our panel columns become [R; 0];
  //    Y_i into P1 / P2
  if (want_vectors) {
    PEVD_CUDA(cudaMemcpy2DAsync(Ystair + ti + ci * n, n * 8, Yb, m * 8, m * 8, pw,
                                cudaMemcpyDeviceToDevice, cs));
    PEVD_CUDA(cudaMemcpyAsync(Tall + x * (int64_t)b * b, Tb, (int64_t)pw * pw * 8,
                              cudaMemcpyDeviceToDevice, cs));
  }
  if (plo < phi) {
    write_r_kernel<<<grid_for((phi - plo) * m), 256, 0, cs>>>(m, pw, ti, ci, plo, phi, lo, Rb, blk,
                                                             ldb);
    PEVD_LAUNCH_CHECK();
  }
  PEVD_CUDA(cudaMemcpy2DAsync(P1 + ri + (2 * ri) * n, n * 8, Yb, m * 8, m * 8, pw,
                              cudaMemcpyDeviceToDevice, cs));
  PEVD_CUDA(cudaMemcpy2DAsync(P2 + ri + (2 * ri + pw) * n, n * 8, Yb, m * 8, m * 8, pw,
                              cudaMemcpyDeviceToDevice, cs));
  // 6. our rows of A W (rows [a, hi) of the trailing part), by symmetry from our columns; the
  //    previous group's trailing update must be complete
  if (trail_done) PEVD_CUDA(cudaStreamWaitEvent(cs, trail_done, 0));
  const int64_t a = std::max(ti, lo);
  const int64_t c = std::max<int64_t>(0, hi - a);
  if (c > 0) {
    // diagonal block from its lower triangle
    GemmArgs g1{c, pw, c, 1.0, 0.0, blk + a + (a - lo) * ldb, ldb, Wb + (a - ti), m, piece, c, 0,
                0, A_SYM_LOWER, C_ALL};
    PEVD_TRY(gemm_(cs, g1));
    if (hi < n) {  // rows below our block: A[hi:, a:hi]^T W[hi:]
      GemmArgs g2{c, pw, n - hi, 1.0, 1.0, blk + hi + (a - lo) * ldb, ldb, Wb + (hi - ti), m,
                  piece, c, 1, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm_(cs, g2));
    }
    if (ti < lo) {  // rows above our block (full storage): A[ti:lo, a:hi]^T W[:lo-ti]
      GemmArgs g3{c, pw, lo - ti, 1.0, 1.0, blk + ti + (a - lo) * ldb, ldb, Wb, m, piece, c, 1,
                  0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm_(cs, g3));
    }
    if (i >= 1) {  // pending updates: -P1[a:hi] (P2^T W_i)
      GemmArgs gt{2 * ri, pw, m, 1.0, 0.0, P2 + ri, n, Wb, m, tv, 2 * ri, 1, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm_(cs, gt));
      GemmArgs gc{c, pw, 2 * ri, -1.0, 1.0, P1 + (a - t0), n, tv, 2 * ri, piece, c, 0, 0,
                  A_GENERAL, C_ALL};
      PEVD_TRY(gemm_(cs, gc));
    }
    // transposed into our slot of AW^T (pw x m): rows of AW in rank order == row order
    PEVD_TRY(transpose(cs, c, pw, piece, c, AWt + (a - ti) * pw, pw));
  }
  {
    std::vector<int64_t> cnt(G, 0);
    for (int y = 0; y < G; ++y) {
      const int64_t ay = std::max(ti, col_lo[y]);
      if (ay < col_lo[y + 1]) cnt[y] = (col_lo[y + 1] - ay) * pw * 8;
    }
    PEVD_TRY(allgatherv(c > 0 ? AWt + (a - ti) * pw : AWt, cnt.data(), AWt, cs, (int)x, LS_SBR));
  }
  // 7. Z_i = A W - 1/2 Y (W^T A W) into P1 / P2
  GemmArgs gm{pw, pw, m, 1.0, 0.0, Wb, m, AWt, pw, Mb, pw, 1, 1, A_GENERAL, C_ALL};
  PEVD_TRY(gemm_(cs, gm));
  double* Zi = P1 + ri + (2 * ri + pw) * n;
  PEVD_TRY(transpose(cs, pw, m, AWt, pw, Zi, n));
  GemmArgs gz{m, pw, pw, -0.5, 1.0, Yb, m, Mb, pw, Zi, n, 0, 0, A_GENERAL, C_ALL};
  PEVD_TRY(gemm_(cs, gz));
  PEVD_CUDA(cudaMemcpy2DAsync(P2 + ri + (2 * ri) * n, n * 8, Zi, n * 8, m * 8, pw,
                              cudaMemcpyDeviceToDevice, cs));
  return OK;
}

// The group's rank-K2 update (K2 = 2K columns of P1 / P2, block-relative rows from t0) of our
// columns >= tl: first the strip [tl, strip_hi) (the next panel's columns, on st_strip), then the
// rest on st_rest -- the rows above our diagonal block and below it in full, the diagonal block
// on its lower tiles.
int Rank::trailing(int64_t t0, int64_t tl, int64_t K2, const double* P1, const double* P2,
                   int64_t ru, int64_t strip_hi, cudaStream_t st_strip, cudaStream_t st_rest) {
  (void)ru;
  const int64_t s_lo = std::max(tl, lo), s_hi = std::min(strip_hi, hi);
  if (s_lo < s_hi) {
    GemmArgs g{n - tl, s_hi - s_lo, K2, -1.0, 1.0, P1 + (tl - t0), n, P2 + (s_lo - t0), n,
               blk + tl + (s_lo - lo) * ldb, ldb, 0, 1, A_GENERAL, C_ALL};
    PEVD_TRY(gemm_(st_strip, g));
  }
  const int64_t a2 = std::max(strip_hi, lo);
  if (a2 >= hi) return OK;
  const int64_t nc = hi - a2;
  if (tl < lo) {  // rows [tl, lo)
    GemmArgs g{lo - tl, nc, K2, -1.0, 1.0, P1 + (tl - t0), n, P2 + (a2 - t0), n,
               blk + tl + (a2 - lo) * ldb, ldb, 0, 1, A_GENERAL, C_ALL};
    PEVD_TRY(gemm_(st_rest, g));
  }
  {  // diagonal block [a2, hi)^2, lower tiles
    GemmArgs g{nc, nc, K2, -1.0, 1.0, P1 + (a2 - t0), n, P2 + (a2 - t0), n,
               blk + a2 + (a2 - lo) * ldb, ldb, 0, 1, A_GENERAL, C_LOWER_TILES};
    PEVD_TRY(gemm(st_rest, g, nullptr, 0));
  }
  if (hi < n) {  // rows [hi, n)
    GemmArgs g{n - hi, nc, K2, -1.0, 1.0, P1 + (hi - t0), n, P2 + (a2 - t0), n,
               blk + hi + (a2 - lo) * ldb, ldb, 0, 1, A_GENERAL, C_ALL};
    PEVD_TRY(gemm_(st_rest, g));
  }
  return OK;
}

// sweeps of rank x's partition present at chase step j: global sweeps [c0_x, c0_x + count)
static int64_t part_count(int64_t n, int b, int64_t c0, int64_t npiv, int64_t j) {
  return std::max<int64_t>(0, std::min<int64_t>(npiv, n - c0 - 2 - j * b));
}

// reflectors of the runs of one rank (prefix[j] = packed index of step j's first reflector)
// between the fixed-slot arrays and a packed buffer of (1 + vld) words per reflector
template <bool PACK>
__global__ void uset_pack_kernel(int64_t n, int b, int64_t c0, int64_t J,
                                 const int64_t* __restrict__ prefix, int vld, double* tau,
                                 double* V, double* packed) {
  const int64_t total = prefix[J];
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total;
       p += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = J;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (prefix[mid] <= p) lo = mid; else hi = mid;
    }
    const int64_t j = lo;
    const int64_t slot = bc_slot_offset_dev(n, b, j) + c0 + (p - prefix[j]);
    double* q = packed + p * (1 + vld);
    if (PACK) {
      q[0] = tau[slot];
      for (int k = 0; k < vld; ++k) q[1 + k] = V[slot * vld + k];
    } else {
      tau[slot] = q[0];
      for (int k = 0; k < vld; ++k) V[slot * vld + k] = q[1 + k];
    }
  }
}

// the 2b x b overlap block rows [pend, pend + 2b) x columns [pend - b, pend) of the band after
// the partition's sweeps (band_out: (2b+1) x m reference layout of the tail from c0)
__global__ void overlap_kernel(int64_t m, int b, int64_t c0, int64_t pend, int64_t n,
                               const double* __restrict__ band_out, double* __restrict__ vals) {
  for (int idx = threadIdx.x; idx < 2 * b * b; idx += blockDim.x) {
    const int rr = idx % (2 * b), cc = idx / (2 * b);
    const int64_t gr = pend + rr, gc = pend - b + cc;
    double v = 0.0;
    if (gr < n && gc >= c0 && gr - gc >= 0 && gr - gc <= 2 * b) v = band_out[(gr - gc) * m + (gc - c0)];
    vals[rr + cc * 2 * b] = v;
  }
}

int Rank::relay_chase() {
  // partitions: rank x chases sweeps with pivot in [col_lo[x], col_lo[x+1]) (the last: all
  // remaining), on the band tail [col_lo[x], n) it received
  const int64_t J = (n - 3) / b + 1;  // chase steps
  int64_t* hprefix_all = nullptr;
  std::vector<int64_t> pref((size_t)G * (J + 1));
  for (int x = 0; x < G; ++x) {
    const int64_t c0 = col_lo[x], np = (x == G - 1) ? n - c0 : col_lo[x + 1] - c0;
    int64_t acc = 0;
    for (int64_t j = 0; j < J; ++j) {
      pref[(size_t)x * (J + 1) + j] = acc;
      acc += part_count(n, b, c0, np, j);
    }
    pref[(size_t)x * (J + 1) + J] = acc;
  }
  (void)hprefix_all;
  if (want_vectors && b < 2) {  // no chase at all: every reflector slot is the identity
    PEVD_CUDA(cudaMemsetAsync(tau, 0, bc_num_reflectors(n, b) * 8, cs));
    PEVD_CUDA(cudaMemsetAsync(V, 0, bc_num_reflectors(n, b) * vld * 8, cs));
  }
  if (want_vectors && G > 1)
    PEVD_CUDA(cudaMemcpyAsync(uprefix, pref.data(), pref.size() * 8, cudaMemcpyHostToDevice, cs));
  for (int x = 0; x < G; ++x) {
    const int64_t c0 = col_lo[x];
    const bool last = (x == G - 1);
    const int64_t pend = last ? n : col_lo[x + 1];
    const int64_t m = n - c0, npiv = pend - c0;
    const int64_t mr = n - pend;
    const int bwo = (int)std::min<int64_t>(2 * b, std::max<int64_t>(mr - 1, 0));
    if (r == x) {
      const double* in = (x == 0) ? bands : tailbuf;
      const int bw_in = (x == 0) ? b : (int)std::min<int64_t>(2 * b, m - 1);
      const size_t sp = open(TR_BC, r, cs);
      PEVD_TRY(bc_reduce_range(cs, m, b, bw_in, in, npiv, dl, el, last ? nullptr : band_out, tau, V,
                               vld, ws_bc, n, c0));
      close(sp, cs);
      if (!last) {
        overlap_kernel<<<1, 256, 0, cs>>>(m, b, c0, pend, n, band_out, ovbuf);
        PEVD_LAUNCH_CHECK();
        // the tail [pend, n) for the successor, semi-bandwidth <= 2b
        if (mr > 0)
          PEVD_CUDA(cudaMemcpy2DAsync(tailbuf, mr * 8, band_out + (pend - c0), m * 8, mr * 8,
                                      bwo + 1, cudaMemcpyDeviceToDevice, cs));
      }
    }
    if (!last) {
      PEVD_TRY(p2p(ovbuf, ovbuf, 2 * (int64_t)b * b, x, x + 1, cs, LS_BC));
      PEVD_TRY(p2p(tailbuf, tailbuf, (int64_t)(bwo + 1) * mr, x, x + 1, cs, LS_BANDSTAGE));
    }
  }
  // the tridiagonal pieces (final for the rank's columns) to every rank
  {
    const int64_t c0 = lo, pend = (r == G - 1) ? n : hi;
    std::vector<int64_t> cd(G), ce(G);
    for (int x = 0; x < G; ++x) {
      const int64_t a = col_lo[x], z = (x == G - 1) ? n : col_lo[x + 1];
      cd[x] = (z - a) * 8;
      ce[x] = (std::min<int64_t>(z, n - 1) - a) * 8;
    }
    (void)c0;
    (void)pend;
    PEVD_TRY(allgatherv(dl, cd.data(), d, cs, -1, LS_GATHER));
    PEVD_TRY(allgatherv(el, ce.data(), e, cs, -1, LS_GATHER));
  }
  // the reflector sets of all partitions to every rank (U-gather, pipeline.py:464-466)
  if (want_vectors && G > 1) {
    std::vector<int64_t> cnt(G), base(G + 1, 0);
    for (int x = 0; x < G; ++x) {
      const int64_t tot = pref[(size_t)x * (J + 1) + J];
      cnt[x] = tot * (1 + vld) * 8;
      base[x + 1] = base[x] + tot;
    }
    const int64_t np_r = (r == G - 1) ? n - lo : hi - lo;
    (void)np_r;
    double* mine = ugather + base[r] * (1 + vld);
    uset_pack_kernel<true><<<grid_for(base[r + 1] - base[r], 16384), 256, 0, cs>>>(
        n, b, lo, J, uprefix + (size_t)r * (J + 1), vld, tau, V, mine);
    PEVD_LAUNCH_CHECK();
    PEVD_TRY(allgatherv(mine, cnt.data(), ugather, cs, -1, LS_UGATHER));
    for (int x = 0; x < G; ++x) {
      if (x == r || base[x + 1] == base[x]) continue;
      uset_pack_kernel<false><<<grid_for(base[x + 1] - base[x], 16384), 256, 0, cs>>>(
          n, b, col_lo[x], J, uprefix + (size_t)x * (J + 1), vld, tau, V,
          ugather + base[x] * (1 + vld));
      PEVD_LAUNCH_CHECK();
    }
  }
  return OK;
}

int Rank::sbr() {
  const int64_t R = sbr_num_rounds(n, b);
  cudaEvent_t trail_done = nullptr;
  int set = 0;
  for (int64_t x = 0; x < R;) {
    const int64_t c0 = x * b;
    const int pw0 = (int)std::min<int64_t>(b, n - b - c0);
    const int64_t t0 = c0 + b, m0 = n - t0;
    double* P1 = P[set][0];
    double* P2 = P[set][1];
    if (pw0 < b) {
      // ---- ragged last round (sbr.py:175-182): one panel, coupling columns, full update
      PEVD_CUDA(cudaMemset2DAsync(P1, n * 8, 0, (size_t)m0 * 8, 2 * pw0, cs));
      PEVD_CUDA(cudaMemset2DAsync(P2, n * 8, 0, (size_t)m0 * 8, 2 * pw0, cs));
      PEVD_TRY(panel(x, c0, pw0, t0, P1, P2, t0, 0, trail_done));
      trail_done = nullptr;
      // coupling columns [c0 + pw, t0) of ours get Q^T from the left: cp -= Y (W^T cp)
      const int64_t klo = std::max<int64_t>(c0 + pw0, lo), khi = std::min(t0, hi);
      if (klo < khi) {
        double* cp = blk + t0 + (klo - lo) * ldb;
        GemmArgs g1{pw0, khi - klo, m0, 1.0, 0.0, BUF, m0, cp, ldb, tv, pw0, 1, 0, A_GENERAL,
                    C_ALL};
        PEVD_TRY(gemm_(cs, g1));
        GemmArgs g2{m0, khi - klo, pw0, -1.0, 1.0, BUF + m0 * pw0, m0, tv, pw0, cp, ldb, 0, 0,
                    A_GENERAL, C_ALL};
        PEVD_TRY(gemm_(cs, g2));
      }
      PEVD_TRY(trailing(t0, t0, 2 * pw0, P1, P2, 0, t0, cs, cs));
      ++x;
      continue;
    }
    int nbl = 1;
    while (nbl < NBB && x + nbl < R && (n - b - (x + nbl) * b) >= b) ++nbl;
    const int64_t K = (int64_t)nbl * b;
    PEVD_CUDA(cudaMemset2DAsync(P1, n * 8, 0, (size_t)K * 8, (size_t)(2 * K), cs));
    PEVD_CUDA(cudaMemset2DAsync(P2, n * 8, 0, (size_t)K * 8, (size_t)(2 * K), cs));
    for (int i = 0; i < nbl; ++i) {
      const int64_t ci = c0 + (int64_t)i * b, ti = t0 + (int64_t)i * b;
      PEVD_TRY(panel(x + i, ci, b, ti, P1, P2, t0, i, i == 0 ? trail_done : nullptr));
    }
    // the group's trailing update: the next panel's columns first (compute stream), the rest on
    // the trailing stream so the next panel's QR and broadcast overlap it
    const int64_t ru = (int64_t)(nbl - 1) * b;
    const int64_t tl = t0 + ru;
    int64_t strip_hi = tl;
    if (x + nbl < R) strip_hi = tl + std::min<int64_t>(b, n - b - tl);
    PEVD_TRY(link(cs, ts));
    // (the trailing update is a trace event of the helper lane: it runs beside the next panel's
    //  QR and broadcast, whose Comm spans it overlaps)
    const size_t tsp = open(TR_SBR, r, ts, 0, -1);
    PEVD_TRY(trailing(t0, tl, 2 * K, P1, P2, ru, strip_hi, cs, ts));
    close(tsp, ts);
    trail_done = new_event();
    PEVD_CUDA(cudaEventRecord(trail_done, ts));
    set ^= 1;
    x += nbl;
  }
  if (trail_done) PEVD_CUDA(cudaStreamWaitEvent(cs, trail_done, 0));
  return OK;
}

}  // namespace

// One rank of the distributed EVD.  Q: conventional -> n x (back cols) col-major (ldq);
// pipelined / sequential -> the rank's rows as an n x (back rows) col-major block (= the rows
// of Q in C order).
int dist_syevd(Comm& C, int64_t n, int b, double* blk, int64_t ldb, const int64_t* col_lo,
               const int64_t* back_lo, double* lam, double* Q, int64_t ldq, int want_vectors,
               int order, cudaStream_t user_stream, pevd_dist_stats* out) {
  const int G = C.size(), r = C.rank();
  if (n < 3 || b < 1 || b >= n || b > 64 || col_lo[0] != 0 || col_lo[G] != n ||
      back_lo[0] != 0 || back_lo[G] != n) {
    set_error("dist_syevd: bad arguments (n=%lld, b=%d; need 3 <= n, 1 <= b <= 64, b < n, "
              "partitions covering [0, n))", (long long)n, b);
    return ERR_VALUE;
  }
  for (int x = 0; x < G; ++x)
    if (col_lo[x + 1] <= col_lo[x] || back_lo[x + 1] < back_lo[x]) {
      set_error("dist_syevd: empty column block or decreasing partition");
      return ERR_VALUE;
    }
  Rank K(C, n, b, want_vectors, order, col_lo, back_lo);
  K.blk = blk;
  K.ldb = ldb;
  const int64_t R = sbr_num_rounds(n, b);
  const int64_t Kmax = (int64_t)NBB * b;
  const int64_t bl0 = back_lo[r], bl1 = back_lo[r + 1], nbk = bl1 - bl0;
  const bool bisect = !want_vectors;
  const int64_t nref = bc_num_reflectors(n, b);
  K.vld = (int)pad8(b);
  // ---- workspace
  Arena ar;
  auto carve = [&](Arena& A) {
    K.Ystair = want_vectors ? A.take<double>(n * n) : nullptr;
    K.Tall = A.take<double>(std::max<int64_t>(R, 1) * b * b);
    for (int s = 0; s < 2; ++s)
      for (int q = 0; q < 2; ++q) K.P[s][q] = A.take<double>(n * 2 * Kmax);
    K.BUF = A.take<double>(2 * n * b + 2 * b * b);
    K.gbuf = A.take<double>(n * b);
    K.AWt = A.take<double>(n * b);
    K.piece = A.take<double>(n * b);
    K.Mb = A.take<double>(b * b);
    K.tv = A.take<double>(2 * Kmax * b + n * b);
    K.sk = A.take<double>(SKN);
    K.bandT = A.take<double>((b + 1) * n);
    K.bands = A.take<double>((b + 1) * n);
    K.d = A.take<double>(n);
    K.e = A.take<double>(n);
    K.dl = A.take<double>(n);
    K.el = A.take<double>(n);
    K.band_out = A.take<double>((2 * b + 1) * n);
    K.tailbuf = A.take<double>((2 * b + 1) * n);
    K.ovbuf = A.take<double>(2 * b * b);
    K.ugather = (want_vectors && G > 1) ? A.take<double>(nref * (1 + K.vld)) : nullptr;
    K.uprefix = A.take<int64_t>((int64_t)G * ((n - 3) / b + 2));
    K.tau = want_vectors ? A.take<double>(nref) : nullptr;
    K.V = want_vectors ? A.take<double>(nref * K.vld) : nullptr;
    K.Qd = bisect ? nullptr : A.take<double>(n * n);
    K.Mrows = (want_vectors && order != PEVD_ORDER_CONVENTIONAL) ? A.take<double>(nbk * n) : nullptr;
    K.qrws = A.take<char>(panel_qr_ws_bytes());
    K.ws_bc = A.take<char>(bc_ws_bytes(n, b));
    K.ws_dc = A.take<char>(bisect ? stebz_ws_bytes(n) : stedc_ws_bytes(n));
    K.ws_back = want_vectors ? A.take<char>(sbr_back_ws_bytes(n, b)) : nullptr;
    K.ws_bcb = want_vectors ? A.take<char>(bc_back_ws_bytes(n, std::max<int64_t>(nbk, 1), b)) : nullptr;
  };
  carve(ar);  // sizes
  Arena real;
  real.cap = ar.off;
  if (cudaMalloc(&real.base, real.cap) != cudaSuccess) {
    cudaGetLastError();
    set_error("dist_syevd: rank %d cannot allocate %.2f GB of workspace", r, real.cap / 1e9);
    return ERR_NOMEM;
  }
  carve(real);
  int rc = OK, info = 0;
  cudaStream_t cs = user_stream;
  cudaStreamCreateWithFlags(&K.ms, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&K.ts, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&K.bs, cudaStreamNonBlocking);
  K.cs = cs;
  // spans on the back stream run beside the worker's own chain: the helper lane (HOST), as the
  // single-GPU run() reports its back stream
  auto stage_span = [&](int stage, cudaStream_t s) -> size_t {
    return K.open(stage, r, s, 0, s == K.bs ? -1 : r);
  };
  double t0_ns = 0.0;
  flops_reset();
  do {
    // common time base: every rank records it right after a barrier
    K.base = K.new_event();
    if ((rc = (cudaStreamSynchronize(cs) == cudaSuccess) ? OK : ERR_CUDA)) break;
    if ((rc = C.barrier())) break;
    K.base = C.time_base(K.base, cs, t0_ns);
    if (want_vectors)
      if ((rc = cudaMemsetAsync(K.Ystair, 0, n * n * 8, cs) == cudaSuccess ? OK : ERR_CUDA)) break;
    // ---------------- SBR
    size_t sp = stage_span(TR_SBR_ALL, cs);
    flops_set_stage(ST_SBR);
    if ((rc = K.sbr())) break;
    K.close(sp, cs);
    cudaEvent_t sbr_done = K.new_event();
    cudaEventRecord(sbr_done, cs);
    // ---------------- pipelined: the rank's rows of Q_s on the back stream, under BC and D&C
    cudaStream_t back = (order == PEVD_ORDER_PIPELINED) ? K.bs : cs;
    if (want_vectors && order != PEVD_ORDER_CONVENTIONAL && nbk > 0) {
      cudaStreamWaitEvent(back, sbr_done, 0);
      flops_set_stage(ST_SBR_BACK);
      sp = stage_span(TR_SBR_BACK, back);
      rows_of_identity<<<grid_for(nbk * n, 16384), 256, 0, back>>>(nbk, n, bl0, K.Mrows);
      count_launch();
      if ((rc = sbr_back_apply_right(back, n, b, K.Ystair, n, K.Tall, K.Mrows, nbk, nbk,
                                     K.ws_back, false)))
        break;
      K.close(sp, back);
    }
    // ---------------- band pieces to rank 0, then the relayed chase (bulge.py:348-385):
    //      rank x chases the sweeps with pivot in its columns down the whole remaining band and
    //      hands the 2b x b overlap block and the band tail to rank x + 1
    flops_set_stage(ST_BC);
    band_pack_kernel<<<grid_for(K.w * (b + 1)), 256, 0, cs>>>(n, b, K.lo, K.w, blk, ldb,
                                                               K.bandT + K.lo * (b + 1));
    count_launch();
    for (int y = 1; y < G && rc == OK; ++y)
      rc = K.p2p(K.bandT + col_lo[y] * (b + 1), K.bandT + col_lo[y] * (b + 1),
                 (col_lo[y + 1] - col_lo[y]) * (b + 1), y, 0, cs, LS_BANDSTAGE);
    if (rc) break;
    if (r == 0 && (rc = transpose(cs, b + 1, n, K.bandT, b + 1, K.bands, n))) break;
    if ((rc = K.relay_chase())) break;
    cudaEvent_t bc_done = K.new_event();
    cudaEventRecord(bc_done, cs);
    // ---------------- back-transform preparations / BC-Back on the back stream
    if (want_vectors && order == PEVD_ORDER_CONVENTIONAL) {
      cudaStreamWaitEvent(K.bs, bc_done, 0);
      flops_set_stage(ST_SBR_BACK);
      if ((rc = sbr_back_prepare(K.bs, n, b, K.Ystair, n, K.Tall, K.ws_back))) break;
      flops_set_stage(ST_BC_BACK);
      if (nbk > 0 && bc_back_dmma_ok(b, K.vld) &&
          (rc = bc_back_left_t(K.bs, n, b, K.tau, K.V, K.vld, nullptr, nbk, nbk, K.ws_bcb, false)))
        break;
    } else if (want_vectors && nbk > 0) {
      cudaStreamWaitEvent(back, bc_done, 0);
      flops_set_stage(ST_BC_BACK);
      sp = stage_span(TR_BC_BACK, back);
      if ((rc = bc_back_right(back, n, b, K.tau, K.V, K.vld, K.Mrows, nbk, nbk, K.ws_bcb))) break;
      K.close(sp, back);
    }
    cudaEvent_t back_done = K.new_event();
    cudaEventRecord(back_done, want_vectors ? (order == PEVD_ORDER_CONVENTIONAL ? K.bs : back) : cs);
    // ---------------- solver
    flops_set_stage(ST_SOLVER);
    sp = stage_span(TR_SOLVER, cs);
    if (bisect) {
      if ((rc = stebz(cs, n, K.d, K.e, lam, K.ws_dc))) break;
    } else {
      const int64_t c_lo = (order == PEVD_ORDER_CONVENTIONAL) ? bl0 : 0;
      const int64_t c_hi = (order == PEVD_ORDER_CONVENTIONAL) ? bl1 : n;
      if ((rc = stedc(cs, n, K.d, K.e, K.Qd, n, K.ws_dc, &info, c_lo, c_hi))) break;
      if ((rc = cudaMemcpyAsync(lam, K.d, n * 8, cudaMemcpyDeviceToDevice, cs) == cudaSuccess
                    ? OK : ERR_CUDA))
        break;
    }
    K.close(sp, cs);
    // ---------------- back transformation of our columns / rows
    if (want_vectors && nbk > 0) {
      cudaStreamWaitEvent(cs, back_done, 0);
      if (order == PEVD_ORDER_CONVENTIONAL) {
        double* Xt = (double*)K.ws_dc;  // the D&C's ping-pong buffer is free now
        flops_set_stage(ST_BC_BACK);
        sp = stage_span(TR_BC_BACK, cs);
        if (bc_back_dmma_ok(b, K.vld)) {  // the DMMA kernel on the transpose (its coalesced pattern)
          if ((rc = transpose(cs, n, nbk, K.Qd + bl0 * n, n, Xt, nbk))) break;
          if ((rc = bc_back_left_t(cs, n, b, K.tau, K.V, K.vld, Xt, nbk, nbk, K.ws_bcb, true)))
            break;
          if ((rc = transpose(cs, nbk, n, Xt, nbk, Q, ldq))) break;
        } else {
          if (cudaMemcpy2DAsync(Q, ldq * 8, K.Qd + bl0 * n, n * 8, n * 8, nbk,
                                cudaMemcpyDeviceToDevice, cs) != cudaSuccess) {
            rc = ERR_CUDA;
            break;
          }
          if ((rc = bc_back_left(cs, n, b, K.tau, K.V, K.vld, Q, ldq, nbk, K.ws_bcb))) break;
        }
        K.close(sp, cs);
        flops_set_stage(ST_SBR_BACK);
        sp = stage_span(TR_SBR_BACK, cs);
        if ((rc = sbr_back_apply_left(cs, n, b, K.Ystair, n, K.Tall, Q, ldq, nbk, K.ws_back, true)))
          break;
        K.close(sp, cs);
      } else {
        // Q_d is complete on every rank before any final multiply (the reference broadcasts it
        // from the host's solver thread, pipeline.py:497-500)
        if (G > 1) {
          if ((rc = K.link(cs, K.ms))) break;
          if ((rc = C.device_barrier(K.ms))) break;
          if ((rc = K.link(K.ms, cs))) break;
        }
        flops_set_stage(ST_FINAL);
        sp = stage_span(TR_FINAL, cs);
        // Q[rows, :]^T = Q_d^T (Q_s Q_b)[rows, :]^T: the rows of Q in C order
        GemmArgs g{n, nbk, n, 1.0, 0.0, K.Qd, n, K.Mrows, nbk, Q, ldq, 1, 1, A_GENERAL, C_ALL};
        if ((rc = gemm(cs, g, K.sk, SKN))) break;
        K.close(sp, cs);
      }
    }
    if (cudaStreamSynchronize(cs) != cudaSuccess || cudaStreamSynchronize(K.bs) != cudaSuccess ||
        cudaStreamSynchronize(K.ts) != cudaSuccess || cudaStreamSynchronize(K.ms) != cudaSuccess) {
      set_error("rank %d: device failure: %s", r, cudaGetErrorString(cudaGetLastError()));
      rc = ERR_CUDA;
      break;
    }
    if (info != 0) {
      set_error("rank %d: tridiagonal divide and conquer did not converge (info=%d)", r, info);
      rc = ERR_CONVERGE;
      break;
    }
  } while (0);
  // ---- stats (also on failure paths where the events exist)
  if (rc == OK && out) {
    auto el = [&](cudaEvent_t e) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, K.base, e);
      return (double)ms;
    };
    pevd_stats& S = out->stages;
    memset(&S, 0, sizeof(S));
    for (auto& s : K.spans) {
      double* slot = nullptr;
      switch (s.stage) {
        case TR_SBR_ALL: slot = S.sbr_ms; break;
        case TR_BC: slot = S.bc_ms; break;
        case TR_SOLVER: slot = S.solver_ms; break;
        case TR_SBR_BACK: slot = S.sbr_back_ms; break;
        case TR_BC_BACK: slot = S.bc_back_ms; break;
        case TR_FINAL: slot = S.final_ms; break;
        default: break;
      }
      if (slot) {
        slot[0] = el(s.a);
        slot[1] = el(s.b);
      }
    }
    S.total_ms = 0.0;
    for (auto& s : K.spans) S.total_ms = std::max(S.total_ms, el(s.b));
    S.n_reflectors = nref;
    S.n_rounds = R;
    flops_read(S.flops);
    out->t0_mono_ns = t0_ns;
    int64_t ne = 0;
    for (auto& s : K.spans) {
      if (s.stage == TR_SBR_ALL) continue;
      if (ne < out->events_cap && out->events) {
        pevd_trace_event& E = out->events[ne];
        E.worker = s.lane;
        E.stage = s.stage;
        E.block = s.block;
        E.pad = 0;
        E.t_start_ms = el(s.a);
        E.t_end_ms = el(s.b);
        E.words = s.words;
      }
      ++ne;
    }
    out->n_events = ne;
    int64_t nm = 0;
    for (auto& m : C.messages()) {
      if (nm < out->msgs_cap && out->msgs) {
        pevd_message& M = out->msgs[nm];
        M.src = m.src;
        M.dst = m.dst;
        M.stage = m.stage;
        M.pad = 0;
        M.words = m.words;
      }
      ++nm;
    }
    out->n_msgs = nm;
  }
  C.messages().clear();
  cudaStreamSynchronize(cs);
  if (K.bs) { cudaStreamSynchronize(K.bs); cudaStreamDestroy(K.bs); }
  if (K.ts) { cudaStreamSynchronize(K.ts); cudaStreamDestroy(K.ts); }
  if (K.ms) { cudaStreamSynchronize(K.ms); cudaStreamDestroy(K.ms); }
  for (cudaEvent_t e : K.evpool) cudaEventDestroy(e);
  cudaFree(real.base);
  return rc;
}

}  // namespace pevd

using namespace pevd;

extern "C" {

int pevd_nccl_unique_id(char* out128) { return NcclComm::unique_id(out128); }

int pevd_comm_nccl_create(int rank, int size, const char* id128, void** comm) {
  if (!comm || rank < 0 || rank >= size) {
    set_error("pevd_comm_nccl_create: bad arguments");
    return ERR_VALUE;
  }
  NcclComm* c = NcclComm::create(rank, size, id128);
  if (!c) return ERR_CUDA;
  *comm = c;
  return OK;
}

void pevd_comm_destroy(void* comm) { delete (Comm*)comm; }

int pevd_dist_syevd(void* comm, int64_t n, int b, double* blk, int64_t ldb, const int64_t* col_lo,
                    const int64_t* back_lo, double* lam, double* Q, int64_t ldq, int want_vectors,
                    int order, void* stream, pevd_dist_stats* stats) {
  if (!comm || !blk || !lam || !col_lo || !back_lo || (want_vectors && !Q) || order < 0 ||
      order > 2) {
    set_error("pevd_dist_syevd: bad arguments");
    return ERR_VALUE;
  }
  return dist_syevd(*(Comm*)comm, n, b, blk, ldb, col_lo, back_lo, lam, Q, ldq, want_vectors, order,
                    (cudaStream_t)stream, stats);
}

int pevd_syevd_multi(int G, const int* devs, int64_t n, int b, const double* A, int64_t lda,
                     const int64_t* col_lo, const int64_t* back_lo, double* lam, double* Q,
                     int want_vectors, int order, pevd_dist_stats* stats) {
  if (G < 1 || !devs || !A || !lam || lda < n || (want_vectors && !Q) || !col_lo || !back_lo ||
      order < 0 || order > 2) {
    set_error("pevd_syevd_multi: bad arguments");
    return ERR_VALUE;
  }
  PeerWorld world(G, devs);
  std::vector<int> rcs(G, OK);
  std::vector<std::string> errs(G);
  auto worker = [&](int x) {
    int rc = OK;
    double *dblk = nullptr, *dlam = nullptr, *dQ = nullptr;
    cudaStream_t st = nullptr;
    do {
      if (cudaSetDevice(devs[x]) != cudaSuccess) {
        set_error("worker %d: cannot use device %d", x, devs[x]);
        rc = ERR_CUDA;
        break;
      }
      PeerComm comm(&world, x);
      const int64_t lo = col_lo[x], w = col_lo[x + 1] - col_lo[x];
      const int64_t bl0 = back_lo[x], nbk = back_lo[x + 1] - back_lo[x];
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
          cudaMalloc(&dblk, std::max<int64_t>(n * w, 1) * 8) != cudaSuccess ||
          cudaMalloc(&dlam, n * 8) != cudaSuccess ||
          (want_vectors && cudaMalloc(&dQ, std::max<int64_t>(n * nbk, 1) * 8) != cudaSuccess)) {
        cudaGetLastError();
        set_error("worker %d: device allocation failed", x);
        rc = ERR_NOMEM;
        break;
      }
      if (cudaMemcpy2D(dblk, n * 8, A + lo * lda, lda * 8, n * 8, w, cudaMemcpyHostToDevice) !=
          cudaSuccess) {
        set_error("worker %d: H2D copy failed", x);
        rc = ERR_CUDA;
        break;
      }
      rc = dist_syevd(comm, n, b, dblk, n, col_lo, back_lo, dlam, dQ, n, want_vectors, order, st,
                      stats ? &stats[x] : nullptr);
      if (rc != OK) break;
      // the result slab: Fortran-order columns (conventional) or C-order rows (pipelined /
      // sequential) are both one contiguous n * nbk block of the host Q
      if (want_vectors && nbk > 0 &&
          cudaMemcpy(Q + bl0 * n, dQ, n * nbk * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
        set_error("worker %d: D2H copy failed", x);
        rc = ERR_CUDA;
        break;
      }
      if (x == 0 && cudaMemcpy(lam, dlam, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
        set_error("worker 0: D2H copy failed");
        rc = ERR_CUDA;
        break;
      }
      if (stats && want_vectors && nbk > 0) {  // the result gather (pipeline.py:491-502)
        pevd_dist_stats& S = stats[x];
        if (S.n_msgs < S.msgs_cap && S.msgs)
          S.msgs[S.n_msgs] = pevd_message{x, DST_HOST, LS_RESULT, 0, n * nbk};
        ++S.n_msgs;
      }
    } while (0);
    if (rc != OK) {
      errs[x] = last_error();
      world.abort();
    }
    rcs[x] = rc;
    if (st) cudaStreamDestroy(st);
    cudaFree(dblk);
    cudaFree(dlam);
    cudaFree(dQ);
  };
  std::vector<std::thread> th;
  for (int x = 1; x < G; ++x) th.emplace_back(worker, x);
  int cur = 0;
  cudaGetDevice(&cur);
  worker(0);
  for (auto& t : th) t.join();
  cudaSetDevice(cur);
  for (int x = 0; x < G; ++x)
    if (rcs[x] != OK && !(errs[x].find("another worker failed") != std::string::npos)) {
      set_error("worker %d failed: %s", x, errs[x].c_str());
      return rcs[x];
    }
  for (int x = 0; x < G; ++x)
    if (rcs[x] != OK) {
      set_error("worker %d failed: %s", x, errs[x].c_str());
      return rcs[x];
    }
  return OK;
}

}  // extern "C"
