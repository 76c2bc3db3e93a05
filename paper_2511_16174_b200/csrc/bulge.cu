// Bulge chasing, band -> symmetric tridiagonal (bulge.py:170-252), as a wavefront over sweeps.
//
// One warp executes one chase step (sweep gi, step j) at a time; the band (2b+1 stored
// subdiagonals, ~25 MB at n=49152, b=32: L2-resident) lives in global memory, column-major with
// leading dimension LDB: Bd[c*LDB + d] = S[c+d, c].  A persistent grid of warps takes sweeps
// round-robin.  Sweep gi may run step j once sweep gi-1 has COMPLETED step j+2 (progress
// counter >= j+3): the regions of (gi, j) and of (gi-1, >= j+3) are then column-disjoint, so the
// wavefront performs exactly the sequential chase's operations (SURVEY.md §7 hard part 1).
// Warps wait on each other, so the kernel is launched COOPERATIVELY: the runtime makes the whole
// grid co-resident or refuses the launch, and no CTA can spin on a CTA that never gets an SM
// (e.g. beside another EVD on another stream).  Sweeps are assigned round-robin (sweep gi to
// warp gi mod total): consecutive sweeps land on consecutive CTAs, i.e. on different SMs, which
// spreads the ~n/(3b) in-flight sweeps evenly (an atomic sweep ticket gives a data-dependent
// mapping that crowds some SMs: 1.54 s instead of 1.07 s at n = 49152).  The producer publishes
// its progress with st.release.gpu (after a CTA barrier, so the release covers both warps' band
// stores cumulatively; a fence.sc -- __threadfence, MEMBAR.SC -- is stronger than the pattern
// needs); the consumer polls the flag relaxed and then re-reads it once with ld.acquire before
// touching band data, which it reads through L2 (ld.cg).
//
// Per step the warp stages its region in shared memory (lane = row of the window):
//   left block  S[w0:w0+L, cg:w0]     (the column to annihilate + the bulge columns between)
//   window      S[w0:w0+L, w0:w0+L]   (symmetric, lower half stored)
//   coupling    S[w0+L:w0+L+b, w0:w0+L]
// and applies H = I - tau v v^T exactly as bulge.py:188-249: annihilate, left-apply, two-sided
// window update, right coupling.  Reflector (gi, j) is written to slot offset(j) + gi, the
// canonical chase-step-major order of bulge.py:51-60 (tau = 0 marks a step the reference
// skips because the column is already reduced).
#include "kernels.cuh"

namespace pevd {

namespace {

constexpr int BMAX = 32;
constexpr int LDS_ = BMAX + 1;
constexpr int DONE = 1 << 30;
#ifndef CHASE_LAG2_MINB
#define CHASE_LAG2_MINB 1  // no register cap: 240 registers, 4 CTAs per SM, measured fastest (5 or 6 per SM: 0.73 / 0.71 s vs 0.68 s at n = 49152)
#endif

// one sweep per CTA (two warps)
struct ChaseSmem {
  double SLC[3][BMAX * LDS_];  // left block / coupling block, a ring of three (see below)
  double SW[BMAX * LDS_];
  double vs[BMAX];
  double wv[BMAX];
  double tau;
};

__global__ void band_to_work(int64_t n, int b, const double* __restrict__ bands,
                             double* __restrict__ Bd, int64_t LDB, int* __restrict__ prog) {
  // b here is the INPUT band's semi-bandwidth (<= 2 b_chase for a relayed tail)
  const int64_t total = n * LDB;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / LDB, d = idx % LDB;
    Bd[idx] = (d <= b && c + d < n) ? bands[d * n + c] : 0.0;
    if (d == 0) prog[c] = 0;
  }
}

__global__ void work_to_band(int64_t n, int bw, const double* __restrict__ Bd, int64_t LDB,
                             double* __restrict__ out) {
  const int64_t total = (int64_t)(bw + 1) * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t dd = idx / n, c = idx % n;
    out[idx] = (c + dd < n) ? Bd[c * LDB + dd] : 0.0;
  }
}

__global__ void work_to_tridiag(int64_t n, const double* __restrict__ Bd, int64_t LDB,
                                double* __restrict__ d, double* __restrict__ e) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    d[i] = Bd[i * LDB];
    if (i + 1 < n) e[i] = Bd[i * LDB + 1];
  }
}

// Two warps per sweep.  Warp 0 owns the left block and the window (the Householder vector, the
// left application on the bulge columns, the two-sided window update), warp 1 the coupling block
// (its right application) and, on the sweep's last step, its store: the two halves of a step's
// work and of its loads / stores run side by side, which shortens the per-step critical path the
// whole wavefront waits on (~3n step slots).  Same arithmetic, in the same order, as one warp.
__global__ void __launch_bounds__(64)
    bc_chase_kernel(int64_t n, int b, double* __restrict__ Bd, int64_t LDB, int* prog,
                    double* __restrict__ tau_out, double* __restrict__ V_out, int vld,
                    int64_t sweep_end, int64_t slot_n, int64_t slot_col0, int poll_ns) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ChaseSmem& S = *reinterpret_cast<ChaseSmem*>(smraw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gend = sweep_end < n - 2 ? sweep_end : n - 2;
  const int64_t stp = LDB - 1;  // pointer step from one band column to the next, same row
  // step j's window (warp 0) / coupling rows (warp 1), loaded into registers: at the top of the
  // step, or -- when the predecessor's flag for step j is already up at the end of step j-1's
  // arithmetic -- before step j-1's write-back and publish, so the loads' L2 round trip hides
  // under them (the regions are disjoint from step j-1's stores)
  double rw[BMAX];
  auto wait_flag = [&](int64_t gi, int need, bool block) -> bool {
    bool ok = true;
    if (gi > 0) {
      if (lane == 0) {
        ok = ld_relaxed(prog + gi - 1) >= need;
        if (!ok && block) {
          const unsigned ns = (unsigned)poll_ns;
          while (ld_relaxed(prog + gi - 1) < need) {
            if (ns) __nanosleep(ns);
          }
          ok = true;
        }
        if (ok) (void)ld_acquire(prog + gi - 1);
      }
      ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
    }
    return ok;
  };
  auto load_step = [&](int64_t gi, int64_t j) {
    const int64_t w0 = gi + 1 + j * b;
    const int L = (int)((b < n - w0) ? b : n - w0);
    if (wid == 0) {
      const double* pw = Bd + w0 * LDB + lane;
#pragma unroll
      for (int q = 0; q < BMAX; ++q) {
        rw[q] = (q < L && lane >= q && lane < L) ? __ldcg(pw) : 0.0;
        pw += stp;
      }
    } else {
      const int64_t tend = (w0 + L + b < n) ? w0 + L + b : n;
      const int nT = (int)(tend - (w0 + L));
      const double* pc = Bd + w0 * LDB + lane + L;
#pragma unroll
      for (int q = 0; q < BMAX; ++q) {
        rw[q] = (q < L && lane < nT) ? __ldcg(pc) : 0.0;
        pc += stp;
      }
    }
  };
  for (int64_t gi = blockIdx.x; gi < gend; gi += gridDim.x) {
    // The coupling block of step j (rows [w0+L, w0+L+b) x columns [w0, w0+L)) IS the left block
    // of step j+1 of the same sweep, and nobody else touches it in between (the next sweep
    // reaches it only after this one completed step j+2): it stays in shared memory -- the two
    // buffers swap roles -- and is neither stored at step j nor reloaded at step j+1.
    // SLC[cur] = this step's left block, SLC[(cur + 1) % 3] its coupling block; the third buffer
    // keeps the previous step's left block readable while its deferred stores are issued
    int cur = 0;
    bool have = false;  // rw already holds this step's region (prefetched by the previous step)
    for (int64_t j = 0; gi + 1 + j * b <= n - 2; ++j) {
      // ---- wait for the predecessor sweep to complete step j+2 (both warps read band data).
      //      Polling is a relaxed L2 load; once the flag is seen one acquire load of it pairs
      //      with the producer's release store, and the shuffle extends the order to the other
      //      lanes, whose band reads then go through L2 (ld.cg).
      if (!have) {
        wait_flag(gi, (int)(j + 3), true);
        load_step(gi, j);
      }
      const int64_t cg = (j == 0) ? gi : gi + 1 + (j - 1) * b;
      const int64_t w0 = gi + 1 + j * b;
      const int L = (int)((b < n - w0) ? b : n - w0);
      const int nleft = (int)(w0 - cg);  // 1 (j = 0) or b
      const int64_t tend = (w0 + L + b < n) ? w0 + L + b : n;
      const int nT = (int)(tend - (w0 + L));
      const bool last = gi + 1 + (j + 1) * b > n - 2;  // no step j+1 in this sweep
      // reflector (slot_col0 + gi, j) of the slot_n problem (a relayed tail writes straight into
      // the whole matrix's fixed slots)
      const int64_t slot = (int64_t)j * (slot_n - 2) - (int64_t)b * j * (j - 1) / 2 + slot_col0 + gi;
      double* SL = S.SLC[cur];
      double* SC = S.SLC[cur == 2 ? 0 : cur + 1];
      // ---- stage the region into shared memory (the first step's left block loaded here)
      if (wid == 0) {
        if (j == 0) {
          double rl[BMAX];
          const double* pl = Bd + cg * LDB + (w0 - cg) + lane;
#pragma unroll
          for (int q = 0; q < BMAX; ++q) {
            rl[q] = (q < nleft && lane < L) ? __ldcg(pl) : 0.0;
            pl += stp;
          }
#pragma unroll
          for (int q = 0; q < BMAX; ++q) SL[lane * LDS_ + q] = rl[q];
        }
#pragma unroll
        for (int q = 0; q < BMAX; ++q) {
          if (lane >= q) {
            S.SW[lane * LDS_ + q] = rw[q];
            S.SW[q * LDS_ + lane] = rw[q];
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < BMAX; ++q) SC[lane * LDS_ + q] = rw[q];
      }
      // ---- the Householder vector (warp 0).  No CTA barrier before it: warp 0 reads only its own
      //      staging and (j >= 1) the left block warp 1 wrote before the previous step's last
      //      barrier, so warp 1's publish of the previous step (its release fence waits for the
      //      step's stores) runs in parallel with this
      __syncwarp();
      if (wid == 0) {
        const double x = (lane < L) ? SL[lane * LDS_] : 0.0;
        const double tail = warp_sum((lane >= 1 && lane < L) ? x * x : 0.0);
        if (tail == 0.0) {
          if (lane == 0) S.tau = 0.0;  // nothing to annihilate: the reference records no reflector
        } else {
          const double x0 = __shfl_sync(0xffffffffu, x, 0);
          const double nrm = sqrt(x0 * x0 + tail);
          const double alpha = (x0 >= 0.0) ? -nrm : nrm;
          const double denom = x0 - alpha;
          const double v = (lane == 0) ? 1.0 : ((lane < L) ? x / denom : 0.0);
          S.vs[lane] = v;
          // v^T v = 1 + tail / denom^2 in closed form (as the panel QR does): no second warp
          // reduction on the step-to-step path
          if (lane == 0) S.tau = 2.0 / (1.0 + tail / (denom * denom));
          if (lane < L) SL[lane * LDS_] = (lane == 0) ? alpha : 0.0;
        }
      }
      __syncthreads();  // v and tau visible to both warps
      const double tau = S.tau;
      // (all staged entries outside the live L x L / nT x L region are zero and v is zero beyond
      //  L, so every loop runs the full BMAX width without predicates; four partial sums break
      //  the dependent-FMA chains)
      if (wid == 0) {
        if (tau != 0.0) {
          const double v = S.vs[lane];
          // ---- H A H on the window (lane = row r)
          double u = 0.0;
          {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
            for (int c = 0; c < BMAX; c += 4) {
              a0 = fma(S.SW[lane * LDS_ + c], S.vs[c], a0);
              a1 = fma(S.SW[lane * LDS_ + c + 1], S.vs[c + 1], a1);
              a2 = fma(S.SW[lane * LDS_ + c + 2], S.vs[c + 2], a2);
              a3 = fma(S.SW[lane * LDS_ + c + 3], S.vs[c + 3], a3);
            }
            u = tau * ((a0 + a1) + (a2 + a3));
          }
          const double gam = 0.5 * tau * warp_sum(v * u);
          const double w = u - gam * v;
          S.wv[lane] = w;
          __syncwarp();
#pragma unroll
          for (int c = 0; c < BMAX; ++c) {
            if (c <= lane) S.SW[lane * LDS_ + c] -= v * S.wv[c] + w * S.vs[c];
          }
          __syncwarp();
        }
        // ---- next step's window now if its flag is already up (see rw above)
        have = !last && wait_flag(gi, (int)(j + 4), false);
        if (have) load_step(gi, j + 1);
        // ---- before the publish, only the one element of this step the successor sweep's newly
        //      unblocked step (j - 2) reads: (row w0, column cg), the corner of that step's
        //      coupling block.  The rest of the write-back follows the publish, so the release
        //      fence waits for one store (plus the previous step's, long since landed); the next
        //      publish covers them before any step that reads them is unblocked.
        if ((tau != 0.0 || j > 0) && lane == 0) Bd[cg * LDB + (w0 - cg)] = SL[0];
      } else {
        // ---- H from the left on the bulge columns strictly between (lane = column q; warp 1
        //      takes it so the two warps' shares of a step are about equal), then H from the
        //      right on the coupling rows (lane = row t)
        if (tau != 0.0) {
          // ---- H from the left on the bulge columns strictly between (lane = column q)
          if (lane >= 1 && lane < nleft) {
            const int q = lane;
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
            for (int r = 0; r < BMAX; r += 4) {
              d0 = fma(S.vs[r], SL[r * LDS_ + q], d0);
              d1 = fma(S.vs[r + 1], SL[(r + 1) * LDS_ + q], d1);
              d2 = fma(S.vs[r + 2], SL[(r + 2) * LDS_ + q], d2);
              d3 = fma(S.vs[r + 3], SL[(r + 3) * LDS_ + q], d3);
            }
            const double dot = tau * ((d0 + d1) + (d2 + d3));
#pragma unroll
            for (int r = 0; r < BMAX; ++r) SL[r * LDS_ + q] -= dot * S.vs[r];
          }
        }
        if (tau != 0.0) {
          double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int c = 0; c < BMAX; c += 4) {
            d0 = fma(SC[lane * LDS_ + c], S.vs[c], d0);
            d1 = fma(SC[lane * LDS_ + c + 1], S.vs[c + 1], d1);
            d2 = fma(SC[lane * LDS_ + c + 2], S.vs[c + 2], d2);
            d3 = fma(SC[lane * LDS_ + c + 3], S.vs[c + 3], d3);
          }
          const double dot = tau * ((d0 + d1) + (d2 + d3));
#pragma unroll
          for (int c = 0; c < BMAX; ++c) SC[lane * LDS_ + c] -= dot * S.vs[c];
        }
        // ---- next step's coupling rows now if its flag is already up
        have = !last && wait_flag(gi, (int)(j + 4), false);
        if (have) load_step(gi, j + 1);
      }
      // ---- publish progress (the barrier orders warp 0's store before warp 1's release, which
      //      covers it cumulatively); warp 1 publishes, so the fence's wait overlaps warp 0's
      //      deferred stores and next Householder vector
      __syncthreads();
      if (threadIdx.x == 32) st_release(prog + gi, (int)(j + 1));
      // ---- deferred write-back: the left block (it also carries the previous step's coupling
      //      update, never stored), the window when a reflector was applied, the reflector slot;
      //      the last step's coupling block (no next step carries it)
      if (wid == 0) {
        if (tau != 0.0 || j > 0) {
          // (not the corner stored above: the successor may already be updating it)
          double* pl = Bd + cg * LDB + (w0 - cg) + lane;
#pragma unroll 4
          for (int q = 0; q < nleft; ++q, pl += stp)
            if (lane < L && (lane | q) != 0) *pl = SL[lane * LDS_ + q];
        }
        if (tau != 0.0) {
          double* pw = Bd + w0 * LDB + lane;
#pragma unroll 4
          for (int c = 0; c < L; ++c, pw += stp)
            if (lane >= c && lane < L) *pw = S.SW[lane * LDS_ + c];
        }
        if (tau_out) {
          if (lane == 0) tau_out[slot] = tau;
          for (int r = lane; r < vld; r += 32)
            V_out[slot * vld + r] = (tau != 0.0) ? ((r < L) ? S.vs[r] : 0.0) : (r == 0 ? 1.0 : 0.0);
        }
        __syncwarp();  // these shared-memory reads precede the next step's staging (WAR)
      } else if (last) {
        double* pc = Bd + w0 * LDB + lane + L;
        for (int c = 0; c < L; ++c, pc += stp)
          if (lane < nT) *pc = SC[lane * LDS_ + c];
      }
      cur = (cur == 2) ? 0 : cur + 1;  // this step's coupling block is the next step's left block
    }
    __syncthreads();
    if (threadIdx.x == 32) st_release(prog + gi, DONE);
  }
}

__global__ void __launch_bounds__(64, CHASE_LAG2_MINB)
    bc_chase_lag2_kernel(int64_t n, int b, double* __restrict__ Bd, int64_t LDB, int* prog,
                    double* __restrict__ tau_out, double* __restrict__ V_out, int vld,
                    int64_t sweep_end, int64_t slot_n, int64_t slot_col0, int poll_ns) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ChaseSmem& S = *reinterpret_cast<ChaseSmem*>(smraw);
  __shared__ double defr[4];  // deferred coupling row b-1: its four partial-sum chains
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gend = sweep_end < n - 2 ? sweep_end : n - 2;
  const int64_t stp = LDB - 1;  // pointer step from one band column to the next, same row
  // step j's window (warp 0) / coupling rows (warp 1), loaded into registers: at the top of the
  // step, or -- when the predecessor's flag for step j is already up at the end of step j-1's
  // arithmetic -- before step j-1's write-back and publish, so the loads' L2 round trip hides
  // under them (the regions are disjoint from step j-1's stores)
  double rw[BMAX];
  auto wait_flag = [&](int64_t gi, int need, bool block) -> bool {
    bool ok = true;
    if (gi > 0) {
      if (lane == 0) {
        ok = ld_relaxed(prog + gi - 1) >= need;
        if (!ok && block) {
          const unsigned ns = (unsigned)poll_ns;
          while (ld_relaxed(prog + gi - 1) < need) {
            if (ns) __nanosleep(ns);
          }
          ok = true;
        }
        if (ok) (void)ld_acquire(prog + gi - 1);
      }
      ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
    }
    return ok;
  };
  auto load_step = [&](int64_t gi, int64_t j) {
    const int64_t w0 = gi + 1 + j * b;
    const int L = (int)((b < n - w0) ? b : n - w0);
    if (wid == 0) {
      const double* pw = Bd + w0 * LDB + lane;
#pragma unroll
      for (int q = 0; q < BMAX; ++q) {
        rw[q] = (q < L && lane >= q && lane < L) ? __ldcg(pw) : 0.0;
        pw += stp;
      }
    } else {
      const int64_t tend = (w0 + L + b < n) ? w0 + L + b : n;
      const int nT = (int)(tend - (w0 + L));
      const double* pc = Bd + w0 * LDB + lane + L;
#pragma unroll
      for (int q = 0; q < BMAX; ++q) {
        rw[q] = (q < L && lane < nT) ? __ldcg(pc) : 0.0;
        pc += stp;
      }
    }
  };
  for (int64_t gi = blockIdx.x; gi < gend; gi += gridDim.x) {
    // The coupling block of step j (rows [w0+L, w0+L+b) x columns [w0, w0+L)) IS the left block
    // of step j+1 of the same sweep, and nobody else touches it in between (the next sweep
    // reaches it only after this one completed step j+2): it stays in shared memory -- the two
    // buffers swap roles -- and is neither stored at step j nor reloaded at step j+1.
    // SLC[cur] = this step's left block, SLC[(cur + 1) % 3] its coupling block; the third buffer
    // keeps the previous step's left block readable while its deferred stores are issued
    int cur = 0;
    bool have = false;  // rw already holds this step's region (prefetched by the previous step)
    for (int64_t j = 0; gi + 1 + j * b <= n - 2; ++j) {
      // ---- wait for the predecessor sweep to complete step j+2 (both warps read band data).
      //      Polling is a relaxed L2 load; once the flag is seen one acquire load of it pairs
      //      with the producer's release store, and the shuffle extends the order to the other
      //      lanes, whose band reads then go through L2 (ld.cg).
      if (!have) {
        wait_flag(gi, (int)(j + 2), true);
        load_step(gi, j);
      }
      const int64_t cg = (j == 0) ? gi : gi + 1 + (j - 1) * b;
      const int64_t w0 = gi + 1 + j * b;
      const int L = (int)((b < n - w0) ? b : n - w0);
      const int nleft = (int)(w0 - cg);  // 1 (j = 0) or b
      const int64_t tend = (w0 + L + b < n) ? w0 + L + b : n;
      const int nT = (int)(tend - (w0 + L));
      const bool last = gi + 1 + (j + 1) * b > n - 2;  // no step j+1 in this sweep
      // Lag 2: step (gi, j) runs beside (gi-1, j+2), which shares ONE element with it: the
      // corner [b-1][b-1] of this step's coupling block is that step's pivot x0.  The coupling
      // row b-1 (whose dot product includes the corner) is therefore finished at the start of
      // step j+1, which waits for (gi-1, j+2) anyway; the corner's value is the one that step
      // stored before its publish.  (This step's own pivot row was deferred the same way by
      // step j-1.)
      const bool defer = gi > 0 && gi - 1 < gend && gi + (j + 2) * b <= n - 2;
      const bool fixup = j > 0 && gi > 0 && gi - 1 < gend && gi + (j + 1) * b <= n - 2;
      // reflector (slot_col0 + gi, j) of the slot_n problem (a relayed tail writes straight into
      // the whole matrix's fixed slots)
      const int64_t slot = (int64_t)j * (slot_n - 2) - (int64_t)b * j * (j - 1) / 2 + slot_col0 + gi;
      double* SL = S.SLC[cur];
      double* SC = S.SLC[cur == 2 ? 0 : cur + 1];
      // ---- stage the region into shared memory (the first step's left block loaded here)
      if (wid == 0) {
        if (j == 0) {
          double rl[BMAX];
          const double* pl = Bd + cg * LDB + (w0 - cg) + lane;
#pragma unroll
          for (int q = 0; q < BMAX; ++q) {
            rl[q] = (q < nleft && lane < L) ? __ldcg(pl) : 0.0;
            pl += stp;
          }
#pragma unroll
          for (int q = 0; q < BMAX; ++q) SL[lane * LDS_ + q] = rl[q];
        }
#pragma unroll
        for (int q = 0; q < BMAX; ++q) {
          if (lane >= q) {
            S.SW[lane * LDS_ + q] = rw[q];
            S.SW[q * LDS_ + lane] = rw[q];
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < BMAX; ++q) SC[lane * LDS_ + q] = rw[q];
      }
      // ---- the Householder vector (warp 0).  No CTA barrier before it: warp 0 reads only its own
      //      staging and (j >= 1) the left block warp 1 wrote before the previous step's last
      //      barrier, so warp 1's publish of the previous step (its release fence waits for the
      //      step's stores) runs in parallel with this
      __syncwarp();
      if (wid == 0 && fixup) {
        // finish the previous step's coupling row b-1 (now this step's left block row b-1) with
        // the corner (gi-1, j+1) stored: the same operations, in the same order, as unsplit
        // (the corner's term is the last nonzero one of its chain, (b-1) mod 4: the chains'
        //  later terms are exact zeros)
        const double Ec = __ldcg(Bd + (w0 - 1) * LDB + b);
        const int cb = b - 1;
        double c0 = defr[0], c1 = defr[1], c2 = defr[2], c3 = defr[3];
        const int rc = cb & 3;
        const double t = fma(Ec, S.vs[cb], rc == 0 ? c0 : rc == 1 ? c1 : rc == 2 ? c2 : c3);
        if (rc == 0) c0 = t; else if (rc == 1) c1 = t; else if (rc == 2) c2 = t; else c3 = t;
        const double dot = S.tau * ((c0 + c1) + (c2 + c3));
        const int row = cb * LDS_;
        const double cur = (lane == cb) ? Ec : SL[row + lane];
        SL[row + lane] = cur - dot * S.vs[lane];
        __syncwarp();
      }
      if (wid == 0) {
        const double x = (lane < L) ? SL[lane * LDS_] : 0.0;
        const double tail = warp_sum((lane >= 1 && lane < L) ? x * x : 0.0);
        if (tail == 0.0) {
          if (lane == 0) S.tau = 0.0;  // nothing to annihilate: the reference records no reflector
        } else {
          const double x0 = __shfl_sync(0xffffffffu, x, 0);
          const double nrm = sqrt(x0 * x0 + tail);
          const double alpha = (x0 >= 0.0) ? -nrm : nrm;
          const double denom = x0 - alpha;
          const double v = (lane == 0) ? 1.0 : ((lane < L) ? x / denom : 0.0);
          S.vs[lane] = v;
          // v^T v = 1 + tail / denom^2 in closed form (as the panel QR does): no second warp
          // reduction on the step-to-step path
          if (lane == 0) S.tau = 2.0 / (1.0 + tail / (denom * denom));
          if (lane < L) SL[lane * LDS_] = (lane == 0) ? alpha : 0.0;
        }
      }
      __syncthreads();  // v and tau visible to both warps
      const double tau = S.tau;
      // (all staged entries outside the live L x L / nT x L region are zero and v is zero beyond
      //  L, so every loop runs the full BMAX width without predicates; four partial sums break
      //  the dependent-FMA chains)
      if (wid == 0) {
        if (tau != 0.0) {
          const double v = S.vs[lane];
          // ---- H A H on the window (lane = row r)
          double u = 0.0;
          {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
            for (int c = 0; c < BMAX; c += 4) {
              a0 = fma(S.SW[lane * LDS_ + c], S.vs[c], a0);
              a1 = fma(S.SW[lane * LDS_ + c + 1], S.vs[c + 1], a1);
              a2 = fma(S.SW[lane * LDS_ + c + 2], S.vs[c + 2], a2);
              a3 = fma(S.SW[lane * LDS_ + c + 3], S.vs[c + 3], a3);
            }
            u = tau * ((a0 + a1) + (a2 + a3));
          }
          const double gam = 0.5 * tau * warp_sum(v * u);
          const double w = u - gam * v;
          S.wv[lane] = w;
          __syncwarp();
#pragma unroll
          for (int c = 0; c < BMAX; ++c) {
            if (c <= lane) S.SW[lane * LDS_ + c] -= v * S.wv[c] + w * S.vs[c];
          }
          __syncwarp();
        }
        // ---- next step's window now if its flag is already up (see rw above)
        have = !last && wait_flag(gi, (int)(j + 3), false);
        if (have) load_step(gi, j + 1);
        // ---- before the publish, only the one element of this step the successor sweep's newly
        //      unblocked step (j - 2) reads: (row w0, column cg), the corner of that step's
        //      coupling block.  The rest of the write-back follows the publish, so the release
        //      fence waits for one store (plus the previous step's, long since landed); the next
        //      publish covers them before any step that reads them is unblocked.
        if ((tau != 0.0 || j > 0) && lane == 0) Bd[cg * LDB + (w0 - cg)] = SL[0];
        // (lag 2: the window's column 0 is read by the successor's step j-1 too)
        if (tau != 0.0 && lane < L) Bd[w0 * LDB + lane] = S.SW[lane * LDS_];
      } else {
        // ---- H from the left on the bulge columns strictly between (lane = column q; warp 1
        //      takes it so the two warps' shares of a step are about equal), then H from the
        //      right on the coupling rows (lane = row t)
        if (tau != 0.0) {
          // ---- H from the left on the bulge columns strictly between (lane = column q)
          if (lane >= 1 && lane < nleft) {
            const int q = lane;
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
            for (int r = 0; r < BMAX; r += 4) {
              d0 = fma(S.vs[r], SL[r * LDS_ + q], d0);
              d1 = fma(S.vs[r + 1], SL[(r + 1) * LDS_ + q], d1);
              d2 = fma(S.vs[r + 2], SL[(r + 2) * LDS_ + q], d2);
              d3 = fma(S.vs[r + 3], SL[(r + 3) * LDS_ + q], d3);
            }
            const double dot = tau * ((d0 + d1) + (d2 + d3));
#pragma unroll
            for (int r = 0; r < BMAX; ++r) SL[r * LDS_ + q] -= dot * S.vs[r];
          }
        }
        // ---- lag 2: the successor's step j-1, unblocked by this step's publish, reads this
        //      left block, so it is stored before the publish (all but the corner, which warp 0
        //      stores; lane = row, coalesced)
        __syncwarp();
        if (tau != 0.0 || j > 0) {
          double* pl = Bd + cg * LDB + (w0 - cg) + lane;
#pragma unroll 4
          for (int q = 0; q < nleft; ++q, pl += stp)
            if (lane < L && (lane | q) != 0) *pl = SL[lane * LDS_ + q];
        }
        if (tau != 0.0) {
          // (row b-1 defers its corner term c = b-1: the chains skip it, the fixup adds it)
          const bool dl = defer && lane == b - 1;
          double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int c = 0; c < BMAX; c += 4) {
            d0 = fma((dl && c == b - 1) ? 0.0 : SC[lane * LDS_ + c], S.vs[c], d0);
            d1 = fma((dl && c + 1 == b - 1) ? 0.0 : SC[lane * LDS_ + c + 1], S.vs[c + 1], d1);
            d2 = fma((dl && c + 2 == b - 1) ? 0.0 : SC[lane * LDS_ + c + 2], S.vs[c + 2], d2);
            d3 = fma((dl && c + 3 == b - 1) ? 0.0 : SC[lane * LDS_ + c + 3], S.vs[c + 3], d3);
          }
          if (dl) {
            defr[0] = d0;
            defr[1] = d1;
            defr[2] = d2;
            defr[3] = d3;
          } else {
            const double dot = tau * ((d0 + d1) + (d2 + d3));
#pragma unroll
            for (int c = 0; c < BMAX; ++c) SC[lane * LDS_ + c] -= dot * S.vs[c];
          }
        } else if (defer && lane == b - 1) {
          // no reflector: the row stays as loaded except the corner, which the fixup sets to
          // (gi-1, j+2)'s stored value (tau = 0 there: dot = 0)
          defr[0] = defr[1] = defr[2] = defr[3] = 0.0;
        }
        // ---- next step's coupling rows now if its flag is already up
        have = !last && wait_flag(gi, (int)(j + 3), false);
        if (have) load_step(gi, j + 1);
        if (last) {  // lag 2: before the publish (the successor's step j-1 reads its corner)
          double* pc = Bd + w0 * LDB + lane + L;
          for (int c = 0; c < L; ++c, pc += stp)
            if (lane < nT) *pc = SC[lane * LDS_ + c];
        }
      }
      // ---- publish progress (the barrier orders warp 0's store before warp 1's release, which
      //      covers it cumulatively); warp 1 publishes, so the fence's wait overlaps warp 0's
      //      deferred stores and next Householder vector
      __syncthreads();
      if (threadIdx.x == 32) st_release(prog + gi, (int)(j + 1));
      // ---- deferred write-back: the left block (it also carries the previous step's coupling
      //      update, never stored), the window when a reflector was applied, the reflector slot;
      //      the last step's coupling block (no next step carries it)
      if (wid == 0) {
        if (tau != 0.0) {  // the window from column 1 (column 0 went before the publish)
          double* pw = Bd + w0 * LDB + lane + stp;
#pragma unroll 4
          for (int c = 1; c < L; ++c, pw += stp)
            if (lane >= c && lane < L) *pw = S.SW[lane * LDS_ + c];
        }
        if (tau_out) {
          if (lane == 0) tau_out[slot] = tau;
          for (int r = lane; r < vld; r += 32)
            V_out[slot * vld + r] = (tau != 0.0) ? ((r < L) ? S.vs[r] : 0.0) : (r == 0 ? 1.0 : 0.0);
        }
        __syncwarp();  // these shared-memory reads precede the next step's staging (WAR)
      }
      cur = (cur == 2) ? 0 : cur + 1;  // this step's coupling block is the next step's left block
    }
    __syncthreads();
    if (threadIdx.x == 32) st_release(prog + gi, DONE);
  }
}

// ------------------------------------------------------------ 32 < b <= 64
// The same wavefront, step and arithmetic for bandwidths past one warp's width, on four warps:
// warps 0-1 own the rows [32 w, 32 w + 32) of the left block and the window (and split the left
// application's columns the same way), warps 2-3 the coupling rows.  The region is staged
// straight into shared memory in 16-column batches of independent loads.
constexpr int WMAX = 64;
constexpr int LDW = WMAX + 1;
constexpr int WIDE_THREADS = 128;

struct ChaseWideSmem {
  double SLC[2][WMAX * LDW];
  double SW[WMAX * LDW];
  double vs[WMAX];
  double wv[WMAX];
  double red[2];
  double tau;
};

__global__ void __launch_bounds__(WIDE_THREADS)
    bc_chase_wide_kernel(int64_t n, int b, double* __restrict__ Bd, int64_t LDB, int* prog,
                         double* __restrict__ tau_out, double* __restrict__ V_out, int vld,
                         int64_t sweep_end, int64_t slot_n, int64_t slot_col0, int poll_ns) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ChaseWideSmem& S = *reinterpret_cast<ChaseWideSmem*>(smraw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool winw = wid < 2;                    // window warps 0-1, coupling warps 2-3
  const int r = 32 * (wid & 1) + lane;          // this thread's row (window or coupling)
  const int64_t gend = sweep_end < n - 2 ? sweep_end : n - 2;
  for (int64_t gi = blockIdx.x; gi < gend; gi += gridDim.x) {
    int cur = 0;
    for (int64_t j = 0; gi + 1 + j * b <= n - 2; ++j) {
      if (gi > 0) {
        if (lane == 0) {
          const int need = (int)(j + 3);
          if (ld_relaxed(prog + gi - 1) < need) {
            unsigned ns = (unsigned)poll_ns;
            while (ld_relaxed(prog + gi - 1) < need) {
              if (ns) __nanosleep(ns);
            }
          }
          (void)ld_acquire(prog + gi - 1);
        }
        __syncwarp();
      }
      const int64_t cg = (j == 0) ? gi : gi + 1 + (j - 1) * b;
      const int64_t w0 = gi + 1 + j * b;
      const int L = (int)((b < n - w0) ? b : n - w0);
      const int nleft = (int)(w0 - cg);
      const int64_t tend = (w0 + L + b < n) ? w0 + L + b : n;
      const int nT = (int)(tend - (w0 + L));
      const bool last = gi + 1 + (j + 1) * b > n - 2;
      const int64_t slot = (int64_t)j * (slot_n - 2) - (int64_t)b * j * (j - 1) / 2 + slot_col0 + gi;
      double* SL = S.SLC[cur];
      double* SC = S.SLC[cur ^ 1];
      // ---- stage this thread's row of its blocks (zero outside the live region)
      for (int q0 = 0; q0 < WMAX; q0 += 16) {
        double ra[16], rb[16];
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) {
          const int q = q0 + qq;
          if (winw) {
            ra[qq] = (j == 0 && q < nleft && r < L)
                         ? __ldcg(Bd + (cg + q) * LDB + (w0 + r - cg - q)) : 0.0;
            rb[qq] = (r >= q && r < L) ? __ldcg(Bd + (w0 + q) * LDB + (r - q)) : 0.0;
          } else {
            ra[qq] = (q < L && r < nT) ? __ldcg(Bd + (w0 + q) * LDB + (L + r - q)) : 0.0;
            rb[qq] = 0.0;
          }
        }
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) {
          const int q = q0 + qq;
          if (winw) {
            if (j == 0) SL[r * LDW + q] = ra[qq];
            if (r >= q) {
              S.SW[r * LDW + q] = rb[qq];
              S.SW[q * LDW + r] = rb[qq];
            }
          } else {
            SC[r * LDW + q] = ra[qq];
          }
        }
      }
      __syncthreads();
      // ---- the Householder vector (warp 0, two rows per lane)
      if (wid == 0) {
        double x[2], t2 = 0.0;
        for (int h = 0; h < 2; ++h) {
          const int rr = lane + 32 * h;
          x[h] = (rr < L) ? SL[rr * LDW] : 0.0;
          if (rr >= 1 && rr < L) t2 += x[h] * x[h];
        }
        const double tail = warp_sum(t2);
        if (tail == 0.0) {
          if (lane == 0) S.tau = 0.0;
        } else {
          const double x0 = __shfl_sync(0xffffffffu, x[0], 0);
          const double nrm = sqrt(x0 * x0 + tail);
          const double alpha = (x0 >= 0.0) ? -nrm : nrm;
          const double denom = x0 - alpha;
          double vv = 0.0;
          for (int h = 0; h < 2; ++h) {
            const int rr = lane + 32 * h;
            const double v = (rr == 0) ? 1.0 : ((rr < L) ? x[h] / denom : 0.0);
            S.vs[rr] = v;
            if (rr >= 1) vv += v * v;
            if (rr < L) SL[rr * LDW] = (rr == 0) ? alpha : 0.0;
          }
          const double vsq = 1.0 + warp_sum(vv);
          if (lane == 0) S.tau = 2.0 / vsq;
        }
      }
      __syncthreads();
      const double tau = S.tau;
      double u = 0.0;
      if (tau != 0.0) {
        if (winw) {
          // ---- H from the left on the bulge columns strictly between (column q = r)
          const int q = r;
          if (q >= 1 && q < nleft) {
            double d0 = 0.0, d1 = 0.0;
#pragma unroll 8
            for (int rr = 0; rr < WMAX; rr += 2) {
              d0 = fma(S.vs[rr], SL[rr * LDW + q], d0);
              d1 = fma(S.vs[rr + 1], SL[(rr + 1) * LDW + q], d1);
            }
            const double dot = tau * (d0 + d1);
#pragma unroll 8
            for (int rr = 0; rr < WMAX; ++rr) SL[rr * LDW + q] -= dot * S.vs[rr];
          }
          // ---- u = tau A v on this row of the window
          double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
          for (int c = 0; c < WMAX; c += 2) {
            a0 = fma(S.SW[r * LDW + c], S.vs[c], a0);
            a1 = fma(S.SW[r * LDW + c + 1], S.vs[c + 1], a1);
          }
          u = tau * (a0 + a1);
          const double part = warp_sum(S.vs[r] * u);
          if (lane == 0) S.red[wid] = part;
        } else {
          // ---- H from the right on this coupling row
          double d0 = 0.0, d1 = 0.0;
#pragma unroll 8
          for (int c = 0; c < WMAX; c += 2) {
            d0 = fma(SC[r * LDW + c], S.vs[c], d0);
            d1 = fma(SC[r * LDW + c + 1], S.vs[c + 1], d1);
          }
          const double dot = tau * (d0 + d1);
#pragma unroll 8
          for (int c = 0; c < WMAX; ++c) SC[r * LDW + c] -= dot * S.vs[c];
        }
      }
      __syncthreads();  // S.red complete; the left block's columns are final
      if (tau != 0.0 && winw) {
        const double gam = 0.5 * tau * (S.red[0] + S.red[1]);
        S.wv[r] = u - gam * S.vs[r];
      }
      __syncthreads();  // all of w visible
      if (winw) {
        if (tau != 0.0) {
          const double v = S.vs[r], w = S.wv[r];
          for (int c = 0; c <= r; ++c) S.SW[r * LDW + c] -= v * S.wv[c] + w * S.vs[c];
        }
        // ---- write back this row: left block, window (lower part), reflector slot
        if ((tau != 0.0 || j > 0) && r < L)
          for (int q = 0; q < nleft; ++q) Bd[(cg + q) * LDB + (w0 + r - cg - q)] = SL[r * LDW + q];
        if (tau != 0.0 && r < L)
          for (int c = 0; c <= r; ++c) Bd[(w0 + c) * LDB + (r - c)] = S.SW[r * LDW + c];
        if (tau_out) {
          if (threadIdx.x == 0) tau_out[slot] = tau;
          for (int rr = threadIdx.x; rr < vld; rr += 64)
            V_out[slot * vld + rr] =
                (tau != 0.0) ? ((rr < L) ? S.vs[rr] : 0.0) : (rr == 0 ? 1.0 : 0.0);
        }
      } else if (last && r < nT) {
        for (int c = 0; c < L; ++c) Bd[(w0 + c) * LDB + (L + r - c)] = SC[r * LDW + c];
      }
      __syncthreads();
      if (threadIdx.x == 0) st_release(prog + gi, (int)(j + 1));
      cur ^= 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) st_release(prog + gi, DONE);
  }
}

}  // namespace

int64_t bc_num_reflectors(int64_t n, int b) {
  int64_t tot = 0;
  for (int64_t j = 0; n - 2 - j * b > 0; ++j) tot += n - 2 - j * b;
  return tot;
}

int64_t bc_slot_offset(int64_t n, int b, int64_t j) {
  return j * (n - 2) - (int64_t)b * j * (j - 1) / 2;
}

static int64_t bc_ldb(int b) { return (2 * b + 2 + 1) / 2 * 2; }

int64_t bc_ws_bytes(int64_t n, int b) { return n * bc_ldb(b) * 8 + n * 4 + 256; }

// The chase of the sweeps [0, sweep_end) on a band of semi-bandwidth bw <= 2b (the relayed tail
// of a partition, bulge.py:348-385); band_out (optional, (2b+1) x n reference layout) receives the
// resulting band with its residual fill, d / e (optional) its tridiagonal part.
int bc_reduce_range(cudaStream_t st, int64_t n, int b, int bw, const double* bands_ref,
                    int64_t sweep_end, double* d, double* e, double* band_out, double* tau,
                    double* V, int vld, void* ws, int64_t slot_n, int64_t slot_col0) {
  if (slot_n <= 0) slot_n = n;
  if (b < 1 || b > WMAX) {
    set_error("bc_reduce: bandwidth %d outside [1, %d] (device kernel limit)", b, WMAX);
    return ERR_VALUE;
  }
  if (tau && vld < b) {
    set_error("bc_reduce: reflector stride %d < b=%d", vld, b);
    return ERR_VALUE;
  }
  const int64_t LDB = bc_ldb(b);
  double* Bd = (double*)ws;
  int* prog = (int*)(Bd + n * LDB);
  if (bw < 0 || bw > 2 * b) {
    set_error("bc_reduce: input bandwidth %d outside [0, 2b]", bw);
    return ERR_VALUE;
  }
  band_to_work<<<(unsigned)std::min<int64_t>(cdiv(n * LDB, 256), 8192), 256, 0, st>>>(
      n, bw, bands_ref, Bd, LDB, prog);
  PEVD_LAUNCH_CHECK();
  if (b >= 2 && n >= 3) {
    // per reflector about 7 b^2 multiply-adds (schedule.py:122): 14 b^2 flops
    {
      int64_t nref = 0;
      for (int64_t j = 0; n - 2 - j * b > 0; ++j)
        nref += std::max<int64_t>(0, std::min<int64_t>(sweep_end, n - 2 - j * b));
      flops_add(14.0 * b * b * (double)nref);
    }
    const bool wide = b > BMAX;
    static int lag = -1;  // PEVD_CHASE_LAG=3: the lag-3 schedule (b <= 32)
    if (lag < 0) {
      const char* e = getenv("PEVD_CHASE_LAG");
      lag = (e && atoi(e) == 3) ? 3 : 2;
    }
    const bool lag2 = !wide && lag == 2;
    const size_t smem = wide ? sizeof(ChaseWideSmem) : sizeof(ChaseSmem);
    auto kfn = wide ? bc_chase_wide_kernel : (lag2 ? bc_chase_lag2_kernel : bc_chase_kernel);
    static int attr_dev[3] = {-1, -1, -1};
    const int ki = wide ? 1 : (lag2 ? 2 : 0);
    int dev;
    PEVD_CUDA(cudaGetDevice(&dev));
    if (attr_dev[ki] != dev) {
      PEVD_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_dev[ki] = dev;
    }
    const int threads = wide ? WIDE_THREADS : 64;
    int per_sm = 0;
    PEVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, smem));
    if (per_sm < 1) {
      set_error("bc_reduce: chase kernel cannot be resident");
      return ERR_CUDA;
    }
    // (cooperative: one full wave at most)
    // about n/(3b) sweeps are in flight at once; 10% more CTAs keeps a CTA ready when a sweep's
    // turn comes, more only adds spinning CTAs; waiting CTAs poll with a 64 ns back-off (at
    // n = 49152: 1.068 s with twice the in-flight count and tight polling, 1.037 s like this)
    int poll = 64;
    if (const char* e = getenv("PEVD_CHASE_POLL_NS")) poll = std::max(0, atoi(e));  // probes
    // (lag 2: about n/(2b) sweeps in flight)
    const int64_t want_warps = std::min<int64_t>(
        n - 2, std::max<int64_t>(110 * n / ((lag2 ? 200 : 300) * b), 2 * num_sms()));
    const int64_t need = want_warps;  // one sweep (two warps) per CTA
    int grid = (int)std::min<int64_t>((int64_t)per_sm * num_sms(), need);
    if (const char* e = getenv("PEVD_CHASE_GRID"))  // probes: fewer CTAs (1 = sweeps in order)
      grid = std::max(1, std::min(grid, atoi(e)));
    int64_t n_ = n, sweep_end_ = sweep_end, LDB_ = LDB;
    int b_ = b, vld_ = vld;
    int poll_ns = poll;
    void* args[] = {&n_, &b_, &Bd, &LDB_, &prog, &tau, &V, &vld_, &sweep_end_, &slot_n, &slot_col0,
                    &poll_ns};
    PEVD_CUDA(cudaLaunchCooperativeKernel((const void*)kfn, dim3(grid), dim3(threads), args,
                                          smem, st));
    PEVD_LAUNCH_CHECK();
  } else if (tau && n >= 3 && slot_n == n && slot_col0 == 0) {
    PEVD_CUDA(cudaMemsetAsync(tau, 0, 8 * bc_num_reflectors(n, b), st));
  }
  if (d && e) {
    work_to_tridiag<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 4096), 256, 0, st>>>(n, Bd, LDB,
                                                                                    d, e);
    PEVD_LAUNCH_CHECK();
  }
  if (band_out) {
    work_to_band<<<(unsigned)std::min<int64_t>(cdiv(n * (2 * b + 1), 256), 8192), 256, 0, st>>>(
        n, 2 * b, Bd, LDB, band_out);
    PEVD_LAUNCH_CHECK();
  }
  return OK;
}

int bc_reduce(cudaStream_t st, int64_t n, int b, const double* bands_ref, double* d, double* e,
              double* tau, double* V, int vld, void* ws) {
  return bc_reduce_range(st, n, b, b, bands_ref, n, d, e, nullptr, tau, V, vld, ws);
}

}  // namespace pevd
