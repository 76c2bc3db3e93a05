// Back transformation (backtrans.py): SBR-Back (Q_s from the panel factors), BC-Back (the bulge
// reflectors), final GEMM glue lives in api.cu.
//
// SBR-Back: Q_s = H_0 H_1 ... H_{R-1}, H_x = I - Y_x T_x Y_x^T, accumulated backwards from the
// identity (the cheap direction: each step only touches the trailing (n-t0)^2 block).  NB
// consecutive panels are aggregated into one compact-WY block (Y_agg = the panels' columns of the
// explicit-Y staircase left in A by the band reduction, T_agg merged from the panel T's and
// Y_agg^T Y_agg by the recursive larft recurrence, all groups batched up front) so the three
// DMMA GEMMs per block are compute-bound.
//
// BC-Back (backtrans.py:277-310): the bulge reflectors applied to the rows of X (X <- X Q_b,
// reordered) or, on the transpose, to its columns (X <- Q_b X, conventional), in the grouped
// dependency order of the paper's BLAS2 kernel (sweep groups of 64, chase steps in order, sweeps
// within a step).  b = 32 runs the DMMA compact-WY kernel (bc_back_wy_kernel, below); any other
// band width the reflector-by-reflector generic kernels.
#include <cstdlib>
#include "kernels.cuh"

namespace pevd {

namespace {

constexpr int NB_AGG_MAX = 32;  // workspace bound on the panels per aggregated SBR-Back block

// panels per aggregated SBR-Back block (K = nb * b reflectors per compact-WY GEMM pass);
// PEVD_NBAGG overrides the default for tuning probes
int nb_agg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PEVD_NBAGG");
    v = e ? atoi(e) : 32;
    if (v < 1) v = 1;
    if (v > NB_AGG_MAX) v = NB_AGG_MAX;
    while (v & (v - 1)) v &= v - 1;  // the recursive T merge pairs sibling blocks
  }
  return v;
}

__global__ void set_identity(int64_t n, double* Q, int64_t ldq) {
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    Q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
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

// conventional direction on the transpose: Xt <- Xt Q_b^T, i.e. X <- Q_b X with X = Xt^T, one
// thread per row of Xt (a column of X), reflectors in reverse creation order (sweeps
// descending, steps descending): consecutive threads touch consecutive addresses of Xt
__global__ void bc_back_left_t_generic(int64_t n, int b, const double* __restrict__ tau,
                                       const double* __restrict__ V, int vld, double* Xt,
                                       int64_t ldx, int64_t nrows) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  double* x = Xt + row;
  const int64_t nsw = n - 2;
  for (int64_t i = nsw - 1; i >= 0; --i) {
    const int64_t jmax = (n - 3 - i) / b;
    for (int64_t j = jmax; j >= 0; --j) {
      const int64_t off = bc_slot_offset_dev(n, b, j);
      const double t = tau[off + i];
      if (t == 0.0) continue;
      const int64_t r0 = i + 1 + j * b;
      const int L = (int)((b < n - r0) ? b : n - r0);
      const double* v = V + (off + i) * vld;
      double* xr = x + r0 * ldx;
      double dot = 0.0;
      for (int r = 0; r < L; ++r) dot = fma(v[r], xr[r * ldx], dot);
      dot *= t;
      for (int r = 0; r < L; ++r) xr[r * ldx] -= dot * v[r];
    }
  }
}

// ------------------------------------------------------------ BC-Back, b = 32 work units
// Work units (64-row block, sweep group of Q4_SG sweeps) are claimed from an atomic counter in
// group-major order by a persistent grid; a per-row-block progress counter orders a block's groups.
constexpr int Q4_SG = 64;

// ------------------------------------------------------------ BC-Back, b = 32, DMMA compact WY
// A warp owns 8 rows of X and a 96-column window (Q4_SG = 64 sweeps + b) kept as 12 DMMA
// accumulator tiles (lane l holds X[l/4][8c + 2(l%4) + h]).  The 64 reflectors of a tile
// (sweeps i0..i0+63 at chase step j) are applied as 8 blocks of 8 with the compact WY form
// (forward T, LAPACK larft):  X_slice <- X_slice (I - V T V^T),  slice = window columns
// [8s, 8s+40):
//   P  = X_slice V        10 DMMA   (A operand = the accumulator tiles themselves)
//   P2 = P (-T)            2 DMMA
//   X_slice += P2 V^T     10 DMMA
// The accumulator layout gives lane l the columns {2(l%4), 2(l%4)+1} of each 8-column tile; by
// reading the k-index of every B operand through that permutation (k-slot l%4 of k-step h is
// column/reflector 2(l%4)+h) the C fragments ARE the A fragments: no shuffles, no conversion.
// The T factors of all blocks are computed up front (wy_tfactor_kernel); each step's V and -T
// are prefetched into registers during the previous step and staged double-buffered.
constexpr int WY_ROWS = 64;  // 8 warps x 8 rows
constexpr int WY_THREADS = 256;
// Per-bandwidth layout constants (B = b, a multiple of 8 up to 32).  A block of 8 staggered
// reflectors spans 8 + B window columns.
//  * V part vb[h][tl][s] (pitch PA): element p = 2 s + h of local reflector tl; the lanes of a
//    half warp read PA r8 + qd: PA = 4 or 12 mod 16 makes them 16 distinct 8-byte banks
//  * Z part zb[s][p] (pitch PB = 8 + B + 2): lanes read 2 qd PB + r8 (2 PB = 4 mod 16)
constexpr int wy_pitch(int need) {  // smallest pitch >= need with pitch % 16 in {4, 12}
  return (need % 16 == 4 || need % 16 == 12) ? need : wy_pitch(need + 1);
}

template <int B>
struct WyB {
  static_assert(B % 8 == 0 && B >= 8 && B <= 64, "BC-Back DMMA kernel: b a multiple of 8 <= 64");
  static constexpr int SPAN = 8 + B;                       // window columns of one block
  static constexpr int PA = wy_pitch(SPAN / 2);
  static constexpr int PB = SPAN + 2;
  static constexpr int VB = 2 * 8 * PA;
  static constexpr int ZB = 8 * PB;
  static constexpr int BLK = VB + ZB;                      // doubles per record
  static constexpr int STEP = 8 * BLK;                     // doubles per (group, step)
  static constexpr int NBT = SPAN / 8;                     // accumulator tiles per block
  static constexpr int NWT = (Q4_SG + B) / 8;              // tiles of the window
  static constexpr int SLT = B / 8;                        // tiles the window slides per step
};
static_assert(WyB<32>::PA == 20 && WyB<32>::BLK == 656, "b = 32 layout");
static_assert(WyB<16>::PA % 16 == 12 || WyB<16>::PA % 16 == 4, "pitch");
static_assert(WyB<8>::PA >= 8 && WyB<24>::PA >= 16 && WyB<64>::PA >= 36, "pitch covers the span");

template <int B>
struct WySmem {
  double vz[2][WyB<B>::STEP];  // [buf][blk][V | Z]
  uint64_t full[2];            // bulk copy of buffer landed
  int cnt[2];                  // warps done with buffer
  int unit;
};

// sum_{i < cnt} floor((a i + b) / m) for a, b >= 0, m > 0 (Euclid-like, O(log))
__host__ __device__ __forceinline__ int64_t floor_sum(int64_t cnt, int64_t m, int64_t a, int64_t b) {
  int64_t ans = 0;
  while (true) {
    if (a >= m) {
      ans += (cnt - 1) * cnt / 2 * (a / m);
      a %= m;
    }
    if (b >= m) {
      ans += cnt * (b / m);
      b %= m;
    }
    const int64_t y_max = a * cnt + b;
    if (y_max < m) break;
    cnt = y_max / m;
    b = y_max % m;
    const int64_t t = m;
    m = a;
    a = t;
  }
  return ans;
}

// records (padded 8-sweep blocks) before chase step j: sum_{j' < j} 8 ceil(nb(j') / 8) with
// nb(j') = ceil((n - 2 - B j') / 8) = c - (B / 8) j'; every step's block count is padded to a
// multiple of 8 (zero records) so the 8 blocks of a 64-sweep group are one contiguous record
template <int B>
__host__ __device__ __forceinline__ int64_t vz_block0(int64_t n, int64_t j) {
  if (j <= 0) return 0;
  const int64_t c = (n - 2 + 7) / 8, g = B / 8;
  if (B == 32) {  // ceil((c - 4 j') / 8) alternates between two arithmetic series
    const int64_t A = (c + 7) / 8, Bo = (c + 3) / 8;
    const int64_t E = (j + 1) / 2, O = j / 2;
    return 8 * (E * A - E * (E - 1) / 2 + O * Bo - O * (O - 1) / 2);
  }
  // sum_{i'=0}^{j-1} floor((c + 7 - g (j - 1) + g i') / 8), i' = j - 1 - j'
  return 8 * floor_sum(j, 8, g, c + 7 - g * (j - 1));
}

// records of chase step j (its 8-sweep block count padded to a multiple of 8)
template <int B>
__host__ __device__ __forceinline__ int64_t vz_step_records(int64_t n, int64_t j) {
  const int64_t nb = (n - 2 + 7) / 8 - (B / 8) * j;
  return 8 * ((nb + 7) / 8);
}

// Z = V (-T)^T of every block of 8 consecutive sweeps at every chase step, so that a block
// acts as X <- X (I - V T V^T) = X + (X V) Z^T; written with the block's V into its record
// (record id = vz_block0(n, j) + q for block q of step j; padding records are zero).
template <int B, bool BACKWARD>
__global__ void wy_tfactor_kernel(int64_t n, const double* __restrict__ tau,
                                  const double* __restrict__ V, int vld, int64_t jcount,
                                  double* __restrict__ VZ) {
  // forward:  H_0 H_1 ... H_7 = I - V T V^T, T upper (LAPACK larft 'F')
  // backward: H_7 H_6 ... H_0 = I - V T V^T, T lower (larft 'B')
  using C = WyB<B>;
  const int64_t total = vz_block0<B>(n, jcount);
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = jcount;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (vz_block0<B>(n, mid) <= id) lo = mid; else hi = mid;
    }
    const int64_t j = lo, q = id - vz_block0<B>(n, j);
    const int64_t off = bc_slot_offset_dev(n, B, j);
    const int64_t nsw_j = n - 2 - j * B;
    double tv[8];
    const double* v[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int64_t i = 8 * q + s;
      const bool ok = i < nsw_j;
      tv[s] = ok ? tau[off + i] : 0.0;
      v[s] = V + (ok ? (off + i) : off) * vld;
    }
    double* rec = VZ + id * C::BLK;
    // V part: vb[h][tl][s] = v_tl[2 s + h - tl] inside the support, 0 outside (and for absent
    // reflectors, whose tau is 0)
#pragma unroll 1
    for (int e = 0; e < C::VB; ++e) {
      const int h = e / (8 * C::PA), tl = (e / C::PA) % 8, ss = e % C::PA;
      const int idx = 2 * ss + h - tl;
      rec[e] = (tv[tl] != 0.0 && idx >= 0 && idx < B) ? v[tl][idx] : 0.0;
    }
    // Gram entries g[u][t] = v_u^T v_t for u < t (v_u starts t - u rows above v_t)
    double G[8][8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        double acc = 0.0;
        if (u < t && tv[u] != 0.0 && tv[t] != 0.0) {
          const int d = t - u;
          for (int r = 0; r < B - d; ++r) acc = fma(v[u][r + d], v[t][r], acc);
        }
        G[u][t] = acc;
      }
    double T[8][8];
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int t = 0; t < 8; ++t) T[s][t] = 0.0;
    if (!BACKWARD) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        T[t][t] = tv[t];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          if (s < t) {
            double acc = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (u >= s && u < t) acc = fma(T[s][u], G[u][t], acc);
            T[s][t] = -tv[t] * acc;
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        T[i][i] = tv[i];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          if (s > i) {
            double acc = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (u > i && u <= s) acc = fma(T[s][u], G[i][u], acc);  // v_u^T v_i = G[i][u]
            T[s][i] = -tv[i] * acc;
          }
        }
      }
    }
    // Z[p][s] = sum_t v_t[p - t] * (-T)[s][t]
    double* out = rec + C::VB;
#pragma unroll 1
    for (int p = 0; p < C::PB; ++p) {
      double vp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t)
        vp[t] = (tv[t] != 0.0 && p - t >= 0 && p - t < B) ? v[t][p - t] : 0.0;
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) acc = fma(vp[t], -T[s2][t], acc);
        out[s2 * C::PB + p] = (p < C::SPAN) ? acc : 0.0;
      }
    }
  }
}

// LEFT = false: X <- X Q_b on the rows of X (element (row, col) at X[row + col*ldx]), reflectors
//   in creation-compatible grouped order (groups ascending, steps bottom-to-top, sweeps
//   ascending), forward T.
// LEFT = true:  X <- Q_b X, done as Y <- Y Q_b^T on the rows of Y = X^T: groups descending,
//   steps top-to-bottom, sweeps descending, backward T (the conventional grouped order of
//   backtrans.py:232-235).  X column-major (X[row + col*ldx], rows contiguous down a column:
//   64-byte segments per 8-row tile): the conventional application runs on the transpose.
// Staging: each (group, step) record (V and Z of its 8 blocks, 42 KB at b = 32) is ONE bulk copy
// on the TMA engine into a double buffer, completing on an mbarrier.  No __syncthreads per step:
// every warp waits only for the bytes of the step it is about to apply, and the LAST warp to
// finish with a buffer (a shared counter) launches the copy of the step after next into it, so
// warps drift freely within the one-step slack the double buffer gives.
template <int B, bool LEFT>
__global__ void __launch_bounds__(WY_THREADS, (B <= 40 ? 2 : 1))
    bc_back_wy_kernel(int64_t n, const double* __restrict__ VZ, double* X, int64_t ldx,
                      int64_t nrows, int* counter, int* progress, int64_t nunits, int nrb,
                      int l2hint) {
  using C = WyB<B>;
  // L2 policies: X streams through once per group (evict first), the group's records are
  // re-read by every row block (evict last); l2hint = 0 leaves both at the normal priority
  const uint64_t pol_x = l2hint ? l2_policy_evict_first() : l2_policy_evict_normal();
  const uint64_t pol_r = l2hint ? l2_policy_evict_last() : l2_policy_evict_normal();
  extern __shared__ __align__(128) unsigned char wyraw[];
  WySmem<B>& S = *reinterpret_cast<WySmem<B>*>(wyraw);
  constexpr int NW = WY_THREADS / 32;
  constexpr int NWT = C::NWT, SLT = C::SLT, NBT = C::NBT;
  constexpr uint32_t STEP_BYTES = C::STEP * 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qd = lane & 3, r8 = lane >> 2;
  const int64_t nsw = n - 2;
  const int64_t ngroups = (nsw + Q4_SG - 1) / Q4_SG;
  if (tid == 0) {
    mbar_init(&S.full[0], 1);
    mbar_init(&S.full[1], 1);
    S.cnt[0] = S.cnt[1] = 0;
    mbar_init_fence();
  }
  __syncthreads();
  uint32_t gstep = 0;  // steps this CTA has consumed (buffer = gstep & 1, parity = (gstep >> 1) & 1)
  // record of group k at the step whose padded block prefix is `off`
  auto rec = [&](int64_t k, int64_t off) { return VZ + (off + 8 * k) * C::BLK; };
  for (;;) {
    if (tid == 0) S.unit = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t u = S.unit;
    __syncthreads();
    if (u >= nunits) break;
    const int64_t seq = u / nrb;                       // groups this row block has done before
    const int64_t k = LEFT ? ngroups - 1 - seq : seq;
    const int rb = (int)(u % nrb);
    const int64_t i0 = k * Q4_SG;
    const int64_t jmax = (n - 3 - i0) / B;
    const int64_t jfirst = LEFT ? 0 : jmax;
    // block prefix of the step two ahead of the current one, advanced by one step per step
    // (uniform over the CTA; the refilling warp uses it)
    const int64_t dj = LEFT ? 1 : -1;
    int64_t off2 = (jmax >= 2) ? vz_block0<B>(n, jfirst + 2 * dj) : 0;
    if (tid == 0) {
      // the unit's first two steps (the buffers are free: every warp passed the barrier above)
      for (int64_t s2 = 0; s2 < 2 && s2 <= jmax; ++s2) {
        const uint32_t g = gstep + (uint32_t)s2;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&S.full[g & 1], STEP_BYTES);
        bulk_g2s_hint(S.vz[g & 1], rec(k, vz_block0<B>(n, jfirst + s2 * dj)), STEP_BYTES,
                      &S.full[g & 1], pol_r);
      }
      if (ld_acquire(progress + rb) < (int)seq) {
        unsigned ns = 64;
        while (ld_acquire(progress + rb) < (int)seq) {
          __nanosleep(ns);
          if (ns < 1024) ns <<= 1;
        }
      }
    }
    const int64_t row = (int64_t)rb * WY_ROWS + warp * 8 + r8;
    const bool active = row < nrows;
    double* x = X + (active ? row : 0);
    int64_t ws = i0 + 1 + jfirst * B;
    __syncthreads();  // progress acquired by tid 0 before anyone reads X
    double w[NWT][2];
#pragma unroll
    for (int c = 0; c < NWT; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = ws + 8 * c + 2 * qd + h;
        w[c][h] = (active && col < n) ? ld_cg_hint(x + col * ldx, pol_x) : 0.0;
      }
    for (int64_t jj = 0; jj <= jmax; ++jj, ++gstep) {
      const bool more = jj < jmax;
      const int buf = gstep & 1;
      const int64_t off2_now = off2;  // prefix of step jj + 2 (used by the refill below)
      {  // ... and of step jj + 3 for the next iteration
        const int64_t j2 = jfirst + (jj + 2) * dj;
        off2 += LEFT ? vz_step_records<B>(n, j2) : -vz_step_records<B>(n, j2 - 1);
      }
      // prefetch the next step's new window columns (registers)
      double nx[SLT][2];
      const int64_t nbase = LEFT ? ws + 8 * NWT : ws - B;
#pragma unroll
      for (int c = 0; c < SLT; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = nbase + 8 * c + 2 * qd + h;
          nx[c][h] = (more && active && col < n) ? ld_cg_hint(x + col * ldx, pol_x) : 0.0;
        }
      mbar_wait(&S.full[buf], (gstep >> 1) & 1);  // this step's V and Z have landed
      const double* vz = S.vz[buf];
      // ---- apply the 8 blocks of this step: P = X V (2 NBT DMMA), X += P Z^T (2 NBT DMMA)
#pragma unroll
      for (int bb = 0; bb < Q4_SG / 8; ++bb) {
        const int blk = LEFT ? Q4_SG / 8 - 1 - bb : bb;
        const double* vb = vz + blk * C::BLK;
        double p0 = 0.0, p1 = 0.0;
        const double* v0 = vb + r8 * C::PA + qd;
        const double* v1 = v0 + 8 * C::PA;
        // two interleaved chains (k-step parities) merged by a DADD: 26.0 TF/s at n = 32768
        // against 25.5 for one chain of 10 dependent DMMAs (b = 32)
        double e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int cc = 0; cc < NBT; ++cc) {
          const double a = v0[4 * cc], c = v1[4 * cc];
          dmma884(p0, p1, w[blk + cc][0], a);
          dmma884(e0, e1, w[blk + cc][1], c);
        }
        p0 += e0;
        p1 += e1;
        const double* z0 = vb + C::VB + (2 * qd) * C::PB + r8;
        const double* z1 = z0 + C::PB;
        // all tiles' first k-step, then the second: two updates of a tile are NBT DMMAs apart
#pragma unroll
        for (int cc = 0; cc < NBT; ++cc) dmma884(w[blk + cc][0], w[blk + cc][1], p0, z0[8 * cc]);
#pragma unroll
        for (int cc = 0; cc < NBT; ++cc) dmma884(w[blk + cc][0], w[blk + cc][1], p1, z1[8 * cc]);
      }
      // ---- done with this buffer: the last warp refills it with the step after next
      __syncwarp();
      if (lane == 0) {
        const int prev = atomicAdd(&S.cnt[buf], 1);
        if (prev == NW - 1) {
          S.cnt[buf] = 0;
          if (jj + 2 <= jmax) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&S.full[buf], STEP_BYTES);
            bulk_g2s_hint(S.vz[buf], rec(k, off2_now), STEP_BYTES, &S.full[buf], pol_r);
          }
        }
      }
      // ---- slide by b (SLT tiles): the trailing SLT tiles (right) / leading SLT tiles (left)
      //      are final for this group
#pragma unroll
      for (int c = 0; c < SLT; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cw = LEFT ? c : c + NWT - SLT;
          const int64_t col = ws + 8 * cw + 2 * qd + h;
          if (active && col < n) st_hint(x + col * ldx, w[cw][h], pol_x);
        }
      if (more) {
        if (!LEFT) {
#pragma unroll
          for (int c = NWT - 1; c >= SLT; --c) {
            w[c][0] = w[c - SLT][0];
            w[c][1] = w[c - SLT][1];
          }
#pragma unroll
          for (int c = 0; c < SLT; ++c) {
            w[c][0] = nx[c][0];
            w[c][1] = nx[c][1];
          }
        } else {
#pragma unroll
          for (int c = 0; c < NWT - SLT; ++c) {
            w[c][0] = w[c + SLT][0];
            w[c][1] = w[c + SLT][1];
          }
#pragma unroll
          for (int c = 0; c < SLT; ++c) {
            w[NWT - SLT + c][0] = nx[c][0];
            w[NWT - SLT + c][1] = nx[c][1];
          }
        }
        ws += LEFT ? B : -B;
      } else {
#pragma unroll
        for (int c = 0; c < NWT; ++c) {
          if (LEFT ? c < SLT : c >= NWT - SLT) continue;  // already stored above
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t col = ws + 8 * c + 2 * qd + h;
            if (active && col < n) st_hint(x + col * ldx, w[c][h], pol_x);
          }
        }
      }
    }
    __syncthreads();  // every warp is done with the unit (and its buffers) before the next
    if (tid == 0) {
      __threadfence();
      st_release(progress + rb, (int)(seq + 1));
    }
  }
}

}  // namespace

// ---------------------------------------------------------------- SBR-Back (compact WY)
// Panels are aggregated NB = nb_agg() at a time (K = NB b reflectors):
//   H_x0 ... H_x0+NB-1 = I - Y T Y^T,  Y = the strided staircase view A[t0:, c0:c0+K]
// The aggregated T factors of ALL groups are built up front (sbr_back_prepare), batched over the
// groups: G = Y^T Y per group, then the recursive larft merge (LAPACK dlarft, recursive form)
//   T12 = -T11 (G12 T22)  for pairs of sibling blocks of s = b, 2b, 4b, ... columns,
// each level two grouped DMMA GEMM launches over every (group, pair).  Every group is padded to
// K = NB b columns (absent panels: zero T blocks, zero Gram), so all groups share one layout:
// T of group g at Tagg + g K^2 (ld K).  The prep depends only on the SBR output, so the
// orchestrator runs it on a side stream under the bulge chase / divide and conquer.
struct SbrBackWs {
  double *tmp1, *tmp2, *sk, *Tagg, *G, *Tmp;
  GemmArgs* dargs;
  int64_t ngroups, K, skn;
  int NB;
};

static int64_t sbr_back_ngroups(int64_t n, int b, int NB) {
  return (b < 1 || n <= b) ? 0 : cdiv(sbr_num_rounds(n, b), NB);
}

static SbrBackWs sbr_back_carve(int64_t n, int b, void* ws, int NB) {
  SbrBackWs W;
  W.NB = NB;
  W.K = (int64_t)NB * b;
  W.ngroups = sbr_back_ngroups(n, b, NB);
  const int64_t Km = (int64_t)NB_AGG_MAX * b;
  const int64_t gmax = sbr_back_ngroups(n, b, 1);  // bound for any NB >= 1
  W.tmp1 = (double*)ws;
  W.tmp2 = W.tmp1 + Km * n;
  W.skn = 4 << 20;
  W.sk = W.tmp2 + Km * n;
  // groups * K^2 <= cdiv(R, NB) * NB^2 b^2 <= (R + NB) * NB * b^2
  const int64_t tsz = (gmax + NB_AGG_MAX) * (int64_t)NB_AGG_MAX * b * b;
  W.Tagg = W.sk + W.skn;
  W.G = W.Tagg + tsz;
  W.Tmp = W.G + tsz;
  W.dargs = (GemmArgs*)(W.Tmp + tsz);
  return W;
}

__global__ void tagg_init_kernel(int64_t ngroups, int NB, int b, int64_t R, int pw_last,
                                 const double* __restrict__ Tall, double* __restrict__ Tagg,
                                 double* __restrict__ G) {
  const int64_t K = (int64_t)NB * b;
  const int64_t total = ngroups * K * K;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = idx / (K * K), e = idx % (K * K);
    const int r = (int)(e % K), c = (int)(e / K);
    double v = 0.0;
    if (r / b == c / b) {
      const int64_t x = g * NB + r / b;
      if (x < R) {
        const int pw = (x == R - 1) ? pw_last : b;
        const int lr = r % b, lc = c % b;
        if (lr < pw && lc < pw) v = Tall[x * b * b + lr + (int64_t)lc * pw];
      }
    }
    Tagg[idx] = v;
    G[idx] = 0.0;
  }
}

// descriptors of one merge level: entries [0, cnt) Tmp12 = G12 T22, [cnt, 2 cnt) T12 = -T11 Tmp12
// for every (group g, pair p) with o = 2 p s
__global__ void tagg_args_kernel(int64_t ngroups, int64_t K, int64_t s, double* G, double* Tagg,
                                 double* Tmp, GemmArgs* out) {
  const int64_t pairs = K / (2 * s), cnt = ngroups * pairs;
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= 2 * cnt) return;
  const int pass = (int)(id / cnt);
  const int64_t g = (id % cnt) / pairs, p = (id % cnt) % pairs;
  const int64_t o = p * 2 * s, K2 = K * K, blk12 = o + (o + s) * K;
  double* Tg = Tagg + g * K2;
  GemmArgs a{};
  a.m = a.n = a.k = s;
  a.beta = 0.0;
  a.lda = a.ldb = a.ldc = K;
  a.transA = a.transB = 0;
  a.amode = A_GENERAL;
  a.cmode = C_ALL;
  a.amap = a.cmap = nullptr;
  if (pass == 0) {
    a.alpha = 1.0;
    a.A = G + g * K2 + blk12;
    a.B = Tg + (o + s) + (o + s) * K;
    a.C = Tmp + g * K2 + blk12;
  } else {
    a.alpha = -1.0;
    a.A = Tg + o + o * K;
    a.B = Tmp + g * K2 + blk12;
    a.C = Tg + blk12;
  }
  out[id] = a;
}

int64_t sbr_back_ws_bytes(int64_t n, int b) {
  const int64_t Km = (int64_t)NB_AGG_MAX * b;
  const int64_t gmax = sbr_back_ngroups(n, b, 1);
  const int64_t tsz = (gmax + NB_AGG_MAX) * (int64_t)NB_AGG_MAX * b * b;
  const int64_t nargs = 2 * (gmax + 1) * NB_AGG_MAX;
  return (2 * Km * n + (4 << 20) + 3 * tsz) * 8 + nargs * (int64_t)sizeof(GemmArgs) + 4096;
}

// group g: panels [g NB, min(R, g NB + NB)), rows from t0 = g NB b + b, K_g reflectors
static void group_dims(int64_t n, int b, int NB, int64_t R, int64_t g, int64_t* t0, int64_t* c0,
                       int64_t* Kg) {
  const int64_t x0 = g * NB, x1 = std::min<int64_t>(R, x0 + NB);
  *c0 = x0 * b;
  *t0 = *c0 + b;
  int64_t K = 0;
  for (int64_t x = x0; x < x1; ++x) K += std::min<int64_t>(b, n - b - x * b);
  *Kg = K;
}

int sbr_back_prepare(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                     const double* Tall, void* ws) {
  if (b < 1 || n <= b) return OK;
  const int NB = nb_agg();
  SbrBackWs W = sbr_back_carve(n, b, ws, NB);
  const int64_t R = sbr_num_rounds(n, b);
  const int64_t K = W.K, K2 = K * K;
  tagg_init_kernel<<<(unsigned)std::min<int64_t>(cdiv(W.ngroups * K2, 256), 16384), 256, 0, st>>>(
      W.ngroups, NB, b, R, (int)(n - b - (R - 1) * b), Tall, W.Tagg, W.G);
  PEVD_LAUNCH_CHECK();
  // Gram matrices (the staircase is zero above each panel, so Y^T Y over rows [t0, n) is exact)
  for (int64_t g = 0; g < W.ngroups; ++g) {
    int64_t t0, c0, Kg;
    group_dims(n, b, NB, R, g, &t0, &c0, &Kg);
    const double* Y = Yfull + t0 + c0 * ldy;
    GemmArgs gg{Kg, Kg, n - t0, 1.0, 0.0, Y, ldy, Y, ldy, W.G + g * K2, K, 1, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, gg, W.sk, W.skn));
  }
  if (NB == 1) return OK;
  // recursive merge, one level per doubling of the block size; descriptors written on the
  // device (no host synchronisation, so the prep can be enqueued on a side stream)
  int64_t off = 0;
  for (int64_t s = b; s < K; s *= 2) {
    const int64_t cnt = W.ngroups * (K / (2 * s));
    tagg_args_kernel<<<(unsigned)cdiv(2 * cnt, 128), 128, 0, st>>>(W.ngroups, K, s, W.G, W.Tagg,
                                                                   W.Tmp, W.dargs + off);
    PEVD_LAUNCH_CHECK();
    PEVD_TRY(gemm_grouped(st, W.dargs + off, (int)cnt, s, s));
    PEVD_TRY(gemm_grouped(st, W.dargs + off + cnt, (int)cnt, s, s));
    off += 2 * cnt;
  }
  return OK;
}

int sbr_back_form(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                  const double* Tall, double* Qs, int64_t ldq, void* ws, bool prepared) {
  set_identity<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 16384), 256, 0, st>>>(n, Qs, ldq);
  PEVD_LAUNCH_CHECK();
  if (b < 1 || n <= b) return OK;
  if (!prepared) PEVD_TRY(sbr_back_prepare(st, n, b, Yfull, ldy, Tall, ws));
  const int NB = nb_agg();
  SbrBackWs W = sbr_back_carve(n, b, ws, NB);
  const int64_t R = sbr_num_rounds(n, b);
  for (int64_t g = W.ngroups - 1; g >= 0; --g) {
    int64_t t0, c0, K;
    group_dims(n, b, NB, R, g, &t0, &c0, &K);
    const int64_t m = n - t0;
    const double* Y = Yfull + t0 + c0 * ldy;  // m x K, ld ldy (explicit staircase)
    const double* Tg = W.Tagg + g * W.K * W.K;
    double* Q22 = Qs + t0 + t0 * ldq;
    // tmp1 = Y^T Q22 (K x m); tmp2 = T tmp1; Q22 -= Y tmp2
    GemmArgs g1{K, m, m, 1.0, 0.0, Y, ldy, Q22, ldq, W.tmp1, K, 1, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g1, W.sk, W.skn));
    GemmArgs g2{K, m, K, 1.0, 0.0, Tg, W.K, W.tmp1, K, W.tmp2, K, 0, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g2, W.sk, W.skn));
    GemmArgs g3{m, m, K, -1.0, 1.0, Y, ldy, W.tmp2, K, Q22, ldq, 0, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g3, W.sk, W.skn));
  }
  return OK;
}

int sbr_back_apply_left(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                        const double* Tall, double* X, int64_t ldx, int64_t ncols, void* ws,
                        bool prepared, int64_t g_lo, int64_t g_hi) {
  // X <- Q_s X = H_0 (H_1 ( ... (H_{R-1} X))): aggregated blocks from the last panel backwards
  if (b < 1 || n <= b) return OK;
  if (!prepared) PEVD_TRY(sbr_back_prepare(st, n, b, Yfull, ldy, Tall, ws));
  const int NB = nb_agg();
  SbrBackWs W = sbr_back_carve(n, b, ws, NB);
  const int64_t R = sbr_num_rounds(n, b);
  if (g_hi < 0 || g_hi > W.ngroups) g_hi = W.ngroups;
  for (int64_t g = g_hi - 1; g >= std::max<int64_t>(g_lo, 0); --g) {
    int64_t t0, c0, K;
    group_dims(n, b, NB, R, g, &t0, &c0, &K);
    const int64_t m = n - t0;
    const double* Y = Yfull + t0 + c0 * ldy;
    const double* Tg = W.Tagg + g * W.K * W.K;
    double* X2 = X + t0;
    for (int64_t c = 0; c < ncols; c += n) {
      const int64_t nc = std::min<int64_t>(n, ncols - c);
      GemmArgs g1{K, nc, m, 1.0, 0.0, Y, ldy, X2 + c * ldx, ldx, W.tmp1, K, 1, 0, A_GENERAL,
                  C_ALL};
      PEVD_TRY(gemm(st, g1, W.sk, W.skn));
      GemmArgs g2{K, nc, K, 1.0, 0.0, Tg, W.K, W.tmp1, K, W.tmp2, K, 0, 0, A_GENERAL, C_ALL};
      PEVD_TRY(gemm(st, g2, W.sk, W.skn));
      GemmArgs g3{m, nc, K, -1.0, 1.0, Y, ldy, W.tmp2, K, X2 + c * ldx, ldx, 0, 0, A_GENERAL,
                  C_ALL};
      PEVD_TRY(gemm(st, g3, W.sk, W.skn));
    }
  }
  return OK;
}

// X (nrows x n, col-major ldx) <- X Q_s = X B_0 B_1 ... (aggregated blocks in creation order):
// the RowAccumulator of backtrans.py:149-183 for a block of rows (the distributed pipelined
// order forms only its rows of Q_s, starting from X = the rows of the identity).
int sbr_back_apply_right(cudaStream_t st, int64_t n, int b, const double* Yfull, int64_t ldy,
                         const double* Tall, double* X, int64_t ldx, int64_t nrows, void* ws,
                         bool prepared) {
  if (b < 1 || n <= b || nrows <= 0) return OK;
  if (nrows > n) {
    set_error("sbr_back_apply_right: %lld rows > n", (long long)nrows);
    return ERR_VALUE;
  }
  if (!prepared) PEVD_TRY(sbr_back_prepare(st, n, b, Yfull, ldy, Tall, ws));
  const int NB = nb_agg();
  SbrBackWs W = sbr_back_carve(n, b, ws, NB);
  const int64_t R = sbr_num_rounds(n, b);
  for (int64_t g = 0; g < W.ngroups; ++g) {
    int64_t t0, c0, K;
    group_dims(n, b, NB, R, g, &t0, &c0, &K);
    const int64_t m = n - t0;
    const double* Y = Yfull + t0 + c0 * ldy;  // m x K
    const double* Tg = W.Tagg + g * W.K * W.K;
    double* X2 = X + t0 * ldx;                // nrows x m
    // tmp1 = X2 Y (nrows x K); tmp2 = tmp1 T; X2 -= tmp2 Y^T
    GemmArgs g1{nrows, K, m, 1.0, 0.0, X2, ldx, Y, ldy, W.tmp1, nrows, 0, 0, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g1, W.sk, W.skn));
    GemmArgs g2{nrows, K, K, 1.0, 0.0, W.tmp1, nrows, Tg, W.K, W.tmp2, nrows, 0, 0, A_GENERAL,
                C_ALL};
    PEVD_TRY(gemm(st, g2, W.sk, W.skn));
    GemmArgs g3{nrows, m, K, -1.0, 1.0, W.tmp2, nrows, Y, ldy, X2, ldx, 0, 1, A_GENERAL, C_ALL};
    PEVD_TRY(gemm(st, g3, W.sk, W.skn));
  }
  return OK;
}

// out (cols x rows, ld ldo) = in^T (in: rows x cols, ld ldi); 32 x 32 tiles through shared memory
__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* __restrict__ in,
                                 int64_t ldi, double* __restrict__ out, int64_t ldo) {
  __shared__ double t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < rows && c < cols) t[k][threadIdx.x] = in[r + c * ldi];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + k;
    if (r < rows && c < cols) out[c + r * ldo] = t[threadIdx.x][k];
  }
}

int transpose(cudaStream_t st, int64_t rows, int64_t cols, const double* in, int64_t ldi,
              double* out, int64_t ldo) {
  if (rows <= 0 || cols <= 0) return OK;
  if (cdiv(cols, 32) > 65535) {
    set_error("transpose: %lld columns exceed the grid", (long long)cols);
    return ERR_VALUE;
  }
  transpose_kernel<<<dim3((unsigned)cdiv(rows, 32), (unsigned)cdiv(cols, 32)), dim3(32, 8), 0,
                     st>>>(rows, cols, in, ldi, out, ldo);
  PEVD_LAUNCH_CHECK();
  return OK;
}

static int64_t wy_counter_bytes(int64_t nrows) { return ((nrows / 32 + 64) * 4 + 255) / 256 * 256; }

bool bc_back_dmma_ok(int b, int vld) { return b % 8 == 0 && b >= 8 && b <= 64 && vld >= b; }

template <int B>
static int64_t wy_records(int64_t n) {
  return n >= 3 ? vz_block0<B>(n, (n - 3) / B + 1) * (int64_t)WyB<B>::BLK : 0;
}

int64_t bc_back_ws_bytes(int64_t n, int64_t nrows, int b) {
  // counters + the (V, Z) record of every padded block of 8 sweeps at every chase step
  int64_t rec = 0;
  switch (b) {
    case 8: rec = wy_records<8>(n); break;
    case 16: rec = wy_records<16>(n); break;
    case 24: rec = wy_records<24>(n); break;
    case 32: rec = wy_records<32>(n); break;
    case 40: rec = wy_records<40>(n); break;
    case 48: rec = wy_records<48>(n); break;
    case 56: rec = wy_records<56>(n); break;
    case 64: rec = wy_records<64>(n); break;
    default: rec = n * nrows;  // the reflector-by-reflector kernels: room for X^T
  }
  return wy_counter_bytes(nrows) + rec * 8 + 256;
}

// The DMMA compact-WY BC-Back: X <- X Q_b (LEFT = false) or Xt <- Xt Q_b^T (LEFT = true, the
// conventional application on the transpose).  `prepared`: the counters and the (V, Z) records
// of ws were already built by a call with X == nullptr (they depend on the chase output only,
// so the orchestrators run that beside the divide and conquer).
template <int B, bool LEFT>
static int bc_back_wy_launch(cudaStream_t st, int64_t n, const double* tau, const double* V,
                             int vld, double* X, int64_t ldx, int64_t nrows, void* ws,
                             bool prepared) {
  using C = WyB<B>;
  const int nrb = (int)cdiv(nrows, WY_ROWS);
  const int64_t ngroups = cdiv(n - 2, Q4_SG);
  const int64_t nunits = ngroups * nrb;
  int* counter = (int*)ws;
  int* progress = counter + 32;
  const int64_t jcount = (n - 3) / B + 1;
  double* VZ = (double*)((char*)ws + wy_counter_bytes(nrows));
  const int64_t nrec = vz_block0<B>(n, jcount);
  if (!prepared) {
    PEVD_CUDA(cudaMemsetAsync(ws, 0, (size_t)(nrb + 32) * 4, st));
    wy_tfactor_kernel<B, LEFT><<<(unsigned)std::min<int64_t>(cdiv(nrec, 128), 16384), 128, 0, st>>>(
        n, tau, V, vld, jcount, VZ);
    PEVD_LAUNCH_CHECK();
  }
  if (X == nullptr) return OK;  // preparation only
  // executed: 4 NBT DMMA (512 flops each) per 8 rows per (unpadded) block of 8 reflectors
  {
    int64_t nblk = 0;
    for (int64_t j = 0; j < jcount; ++j) nblk += cdiv(n - 2 - j * B, 8);
    flops_add(4.0 * C::NBT * 512.0 / 8.0 * (double)nrows * (double)nblk);
  }
  auto kfn = bc_back_wy_kernel<B, LEFT>;
  const size_t smem = sizeof(WySmem<B>);
  static int attr_dev = -1;
  int dev;
  PEVD_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    PEVD_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_dev = dev;
  }
  int per_sm = 0;
  PEVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, WY_THREADS, smem));
  if (per_sm < 1) {
    set_error("bc_back: persistent kernel cannot be resident");
    return ERR_CUDA;
  }
  const int64_t grid = std::min<int64_t>((int64_t)per_sm * num_sms(), nunits);
  static int l2hint = -1;
  if (l2hint < 0) {
    // on by default: X evict-first, records evict-last: DRAM reads 3.19 -> 2.87 TB and
    // 2.697 -> 2.684 s at n = 32768 (PEVD_BCB_L2HINT=0 turns it off)
    const char* e = getenv("PEVD_BCB_L2HINT");
    l2hint = e ? atoi(e) : 1;
  }
  kfn<<<(unsigned)grid, WY_THREADS, smem, st>>>(n, VZ, X, ldx, nrows, counter, progress, nunits,
                                               nrb, l2hint);
  PEVD_LAUNCH_CHECK();
  return OK;
}

template <bool LEFT>
static int bc_back_wy_dispatch(cudaStream_t st, int64_t n, int b, const double* tau,
                               const double* V, int vld, double* X, int64_t ldx, int64_t nrows,
                               void* ws, bool prepared) {
  switch (b) {
    case 8: return bc_back_wy_launch<8, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
    case 16: return bc_back_wy_launch<16, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
    case 24: return bc_back_wy_launch<24, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
    case 40: return bc_back_wy_launch<40, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
    case 48: return bc_back_wy_launch<48, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
    case 56: return bc_back_wy_launch<56, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
    case 64: return bc_back_wy_launch<64, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
    default: return bc_back_wy_launch<32, LEFT>(st, n, tau, V, vld, X, ldx, nrows, ws, prepared);
  }
}

int bc_back_right(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                  double* X, int64_t ldx, int64_t nrows, void* ws) {
  if (n < 3 || nrows <= 0 || b < 2) return OK;
  if (bc_back_dmma_ok(b, vld) && ws)  // DMMA compact-WY kernel (fully asynchronous)
    return bc_back_wy_dispatch<false>(st, n, b, tau, V, vld, X, ldx, nrows, ws, false);
  // any other b (or a padded reflector stride): one thread per row, reflector by reflector
  flops_add(4.0 * b * (double)bc_num_reflectors(n, b) * (double)nrows);
  bc_back_right_generic<<<(unsigned)cdiv(nrows, 128), 128, 0, st>>>(n, b, tau, V, vld, X, ldx,
                                                                    nrows, 16);
  PEVD_LAUNCH_CHECK();
  return OK;
}

// X (n x ncols, column-major) <- Q_b X: the DMMA kernel for b a multiple of 8 (up to 64) on the
// transpose; any other b one reflector at a time, also on the transpose (held in ws), so that
// the per-thread columns of X become coalesced rows
int bc_back_left(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                 double* X, int64_t ldx, int64_t ncols, void* ws) {
  if (n < 3 || ncols <= 0 || b < 2) return OK;
  if (!ws) {
    set_error("bc_back_left: needs the workspace (pevd_bc_back_workspace_bytes)");
    return ERR_VALUE;
  }
  if (bc_back_dmma_ok(b, vld)) {
    // the records live in ws too: the transpose goes to a separate allocation
    double* Xt = nullptr;
    PEVD_CUDA(cudaMallocAsync(&Xt, (size_t)n * ncols * 8, st));
    int rc = transpose(st, n, ncols, X, ldx, Xt, ncols);
    if (rc == OK) rc = bc_back_wy_dispatch<true>(st, n, b, tau, V, vld, Xt, ncols, ncols, ws, false);
    if (rc == OK) rc = transpose(st, ncols, n, Xt, ncols, X, ldx);
    cudaFreeAsync(Xt, st);
    return rc;
  }
  flops_add(4.0 * b * (double)bc_num_reflectors(n, b) * (double)ncols);
  double* Xt = (double*)((char*)ws + wy_counter_bytes(ncols));
  PEVD_TRY(transpose(st, n, ncols, X, ldx, Xt, ncols));
  bc_back_left_t_generic<<<(unsigned)cdiv(ncols, 128), 128, 0, st>>>(n, b, tau, V, vld, Xt, ncols,
                                                                     ncols);
  PEVD_LAUNCH_CHECK();
  return transpose(st, ncols, n, Xt, ncols, X, ldx);
}

int bc_back_left_t(cudaStream_t st, int64_t n, int b, const double* tau, const double* V, int vld,
                   double* Xt, int64_t ldx, int64_t nrows, void* ws, bool prepared) {
  if (!(bc_back_dmma_ok(b, vld) && ws)) {  // only the DMMA kernel has the transposed layout
    set_error("bc_back_left_t: needs b a multiple of 8 up to 64 and a workspace");
    return ERR_VALUE;
  }
  if (n < 3 || nrows <= 0) return OK;
  return bc_back_wy_dispatch<true>(st, n, b, tau, V, vld, Xt, ldx, nrows, ws, prepared);
}

}  // namespace pevd
