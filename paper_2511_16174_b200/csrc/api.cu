// C ABI of libpevd.so (include/pevd.h) and the single-GPU pipelined EVD orchestrator.
//
// Orchestration of pevd_syevd_device (pipeline.py:170-508 restated for one B200):
//   stream main : SBR -> BC -> D&C -> (wait back) -> final GEMM Q = (Q_s Q_b) Q_d
//   stream back : (wait SBR) SBR-Back forms Q_s -> (wait BC) BC-Back Q_s <- Q_s Q_b
// so the compute-bound Q_s formation overlaps the latency-bound bulge chase and BC-Back
// overlaps the divide and conquer ("pipelined").  "sequential" runs the same stages on one
// stream; "conventional" applies Q_b then Q_s to Q_d from the left (pipeline.py:367-387).
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <vector>
#include <memory>
#include "hostio.h"
#include "kernels.cuh"
#include "../../include/pevd.h"

namespace pevd {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct FlopState {
  int stage = 0;
  double host[ST_NSTAGE] = {};
  unsigned long long* dev = nullptr;
  int dev_id = -1;
  ~FlopState() {
    if (dev) cudaFree(dev);
  }
};
static thread_local FlopState g_flops;

void flops_set_stage(int stage) { g_flops.stage = stage; }
int flops_stage() { return g_flops.stage; }
void flops_add(double f) { g_flops.host[g_flops.stage] += f; }
unsigned long long* flops_dev() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  if (g_flops.dev && g_flops.dev_id == dev) return g_flops.dev;
  // one small buffer per (thread, device) for the life of the thread
  unsigned long long* p = nullptr;
  if (cudaMalloc(&p, ST_NSTAGE * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
  cudaMemset(p, 0, ST_NSTAGE * sizeof(unsigned long long));
  g_flops.dev = p;
  g_flops.dev_id = dev;
  return p;
}
void flops_reset() {
  for (double& h : g_flops.host) h = 0.0;
  if (unsigned long long* d = flops_dev()) cudaMemset(d, 0, ST_NSTAGE * sizeof(unsigned long long));
}
void flops_read(double out[ST_NSTAGE]) {
  unsigned long long d[ST_NSTAGE] = {};
  if (unsigned long long* p = flops_dev())
    cudaMemcpy(d, p, sizeof(d), cudaMemcpyDeviceToHost);
  for (int s = 0; s < ST_NSTAGE; ++s) out[s] = g_flops.host[s] + (double)d[s];
}

int num_sms() {
  static int cache[64];
  static bool init[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!init[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 1;
    init[dev] = true;
  }
  return cache[dev];
}

namespace {

struct Carve {
  char* base;
  int64_t off = 0, cap;
  Carve(void* b, int64_t c) : base((char*)b), cap(c) {}
  void* take(int64_t bytes) {
    void* p = base ? base + off : nullptr;
    off += (bytes + 255) / 256 * 256;
    return p;
  }
};

struct Layout {
  double *bands, *Tall, *d, *e, *tau, *V, *Qs, *Qd;
  void *ws_sbr, *ws_bc, *ws_dc, *ws_back, *ws_bcb;
  int vld;
  int64_t total;
};

// eigenvalues only by bisection (default; PEVD_VALUES_DC=1 keeps the divide and conquer)
bool values_by_bisection() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PEVD_VALUES_DC");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v != 0;
}

// The bulge chase treats the SBR's b-band as a band of width roundup8(b) (its entries beyond b
// are zero; the chase is valid for any band at most its width), so that its reflectors have the
// geometry of the DMMA BC-Back kernel, whose 8-wide blocks need b a multiple of 8.  Same
// eigenpairs to rounding; the per-stage entry points (pevd_bc, stages.bc_reduce) chase with b
// itself, exactly as bulge.py does.
int chase_bandwidth(int64_t n, int b) {
  const int r = (b + 7) / 8 * 8;
  return (r != b && r <= 64 && r <= n - 1) ? r : b;
}

Layout plan_layout(void* base, int64_t n, int b, int want_vectors, int order) {
  Carve c(base, 0);
  Layout L{};
  const int64_t R = sbr_num_rounds(n, b);
  const int bc_b = chase_bandwidth(n, b);
  L.vld = (int)pad8(bc_b);
  L.bands = (double*)c.take((int64_t)(b + 1) * n * 8);
  L.Tall = (double*)c.take(std::max<int64_t>(R, 1) * b * b * 8);
  L.d = (double*)c.take(n * 8);
  L.e = (double*)c.take(std::max<int64_t>(n, 1) * 8);
  const int64_t nref = (n >= 3) ? bc_num_reflectors(n, bc_b) : 0;
  if (want_vectors) {
    L.tau = (double*)c.take(std::max<int64_t>(nref, 1) * 8);
    L.V = (double*)c.take(std::max<int64_t>(nref, 1) * L.vld * 8);
    if (order != PEVD_ORDER_CONVENTIONAL) L.Qs = (double*)c.take(n * n * 8);
  }
  const bool bisect = !want_vectors && values_by_bisection();  // no Q_d, no merge buffers
  L.Qd = bisect ? nullptr : (double*)c.take(n * n * 8);
  L.ws_sbr = c.take(sbr_ws_bytes(n, b));
  L.ws_bc = c.take(bc_ws_bytes(n, bc_b));
  L.ws_dc = c.take(bisect ? stebz_ws_bytes(n) : stedc_ws_bytes(n));
  L.ws_back = c.take(sbr_back_ws_bytes(n, b));
  L.ws_bcb = c.take(bc_back_ws_bytes(n, n, bc_b));
  L.total = c.off;
  return L;
}

// max |A_ij - A_ji| and sum of squares over 32 x 32 tile pairs (one CTA per lower tile pair,
// read through shared memory so both tiles stream coalesced); per-CTA partials, reduced in a
// fixed order by asym_finish (deterministic)
__global__ void asym_partials(int64_t n, const double* __restrict__ A, int64_t lda, int64_t nt,
                              double* __restrict__ part) {
  __shared__ double t[32][33];
  __shared__ double rmax[8], rsum[8];
  const int64_t ntiles = nt * (nt + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int64_t id = blockIdx.x; id < ntiles; id += gridDim.x) {
    // tile (I, J), I >= J, row-major enumeration of the lower triangle of tiles
    int64_t I = (int64_t)((sqrt(8.0 * (double)id + 1.0) - 1.0) / 2.0);
    while (I * (I + 1) / 2 > id) --I;
    while ((I + 1) * (I + 2) / 2 <= id) ++I;
    const int64_t J = id - I * (I + 1) / 2;
    double mx = 0.0, sq = 0.0;
    // upper tile (J, I) transposed into shared memory: t[c][r] = A[J*32 + r, I*32 + c]
    for (int k = ty; k < 32; k += 8) {
      const int64_t r = J * 32 + tx, c = I * 32 + k;
      t[k][tx] = (r < n && c < n) ? A[r + c * lda] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int64_t r = I * 32 + tx, c = J * 32 + k;  // lower element A[r, c]
      if (r < n && c < n) {
        const double a = A[r + c * lda];
        const double m = t[tx][k];                   // A[c, r]
        mx = fmax(mx, fabs(a - m));
        sq += (I == J) ? a * a : a * a + m * m;
      }
    }
    __syncthreads();
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    for (int o = 16; o > 0; o >>= 1) {
      if (o < 16) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
    }
    if (tx == 0) {
      rmax[ty] = mx;
      rsum[ty] = sq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double m2 = 0.0, s2 = 0.0;
      for (int w = 0; w < 8; ++w) {
        m2 = fmax(m2, rmax[w]);
        s2 += rsum[w];
      }
      part[2 * blockIdx.x] = fmax(id == blockIdx.x ? 0.0 : part[2 * blockIdx.x], m2);
      part[2 * blockIdx.x + 1] = (id == blockIdx.x ? 0.0 : part[2 * blockIdx.x + 1]) + s2;
    }
    __syncthreads();
  }
}

__global__ void asym_finish(int nparts, const double* __restrict__ part, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double m = 0.0, s = 0.0;
    for (int i = 0; i < nparts; ++i) {
      m = fmax(m, part[2 * i]);
      s += part[2 * i + 1];
    }
    out[0] = m;
    out[1] = sqrt(s);
  }
}

struct Ev {
  cudaEvent_t a = nullptr, b = nullptr;
};


}  // namespace
}  // namespace pevd

using namespace pevd;

extern "C" {

const char* pevd_last_error(void) { return last_error(); }
const char* pevd_version(void) { return "pevd 0.1.0 (sm_100a, FP64 DMMA)"; }
int64_t pevd_kernel_launches(void) { return g_launches.load(); }

int64_t pevd_syevd_workspace_bytes(int64_t n, int b, int want_vectors, int order) {
  if (n < 1) return 0;
  if (b > n - 1) b = (int)std::max<int64_t>(n - 1, 1);
  return plan_layout(nullptr, n, b, want_vectors, order).total + 4096;
}

}  // extern "C"

namespace pevd {
namespace {

// The single-GPU orchestrator behind pevd_syevd_device / pevd_syevd_device_host_q / pevd_syevd.
// hq (optional): Q's host destination; its copies are queued as columns of Q become final.
int syevd_impl(int64_t n, int b, double* A, int64_t lda, double* lam, double* Q, int64_t ldq,
               int want_vectors, int order, void* workspace, int64_t workspace_bytes,
               cudaStream_t sm, pevd_stats* stats, HostQ* hq) {
  if (n < 1 || lda < n || (want_vectors && (!Q || ldq < n)) || b < 1) {
    set_error("pevd_syevd_device: bad arguments (n=%lld, b=%d)", (long long)n, b);
    return ERR_VALUE;
  }
  if (order < 0 || order > 2) {
    set_error("order must be 0 (pipelined), 1 (sequential) or 2 (conventional)");
    return ERR_VALUE;
  }
  if (stats) memset(stats, 0, sizeof(*stats));
  // trivial sizes (pipeline.py:90-93: b = min(b, n-1); n == 1 has nothing to reduce)
  if (n == 1) {
    PEVD_CUDA(cudaMemcpyAsync(lam, A, 8, cudaMemcpyDeviceToDevice, sm));
    if (want_vectors) {
      const double one = 1.0;
      PEVD_CUDA(cudaMemcpyAsync(Q, &one, 8, cudaMemcpyHostToDevice, sm));
      if (hq && hq->slab_ready(sm, Q, ldq, 1, 0, 1)) return ERR_CUDA;
    }
    PEVD_CUDA(cudaStreamSynchronize(sm));
    return OK;
  }
  b = (int)std::min<int64_t>(b, n - 1);
  if (b > 64) {
    set_error("bandwidth b=%d > 64 is not supported by the device kernels", b);
    return ERR_VALUE;
  }
  Layout L = plan_layout(workspace, n, b, want_vectors, order);
  const int bc_b = chase_bandwidth(n, b);
  if (workspace_bytes < L.total) {
    set_error("workspace too small: %lld < %lld bytes", (long long)workspace_bytes,
              (long long)L.total);
    return ERR_VALUE;
  }
  cudaStream_t sb = nullptr;
  const bool two_streams = want_vectors && order != PEVD_ORDER_SEQUENTIAL;
  if (two_streams) PEVD_CUDA(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  Ev ev[6];
  cudaEvent_t prep_done = nullptr;
  for (auto& e : ev) {
    PEVD_CUDA(cudaEventCreate(&e.a));
    PEVD_CUDA(cudaEventCreate(&e.b));
  }
  PEVD_CUDA(cudaEventCreateWithFlags(&prep_done, cudaEventDisableTiming));
  auto cleanup = [&]() {
    // the call is synchronous even on an error path: nothing may still write the caller's
    // workspace or Q once we return (errors of these waits are the error being reported)
    if (sb) cudaStreamSynchronize(sb);
    cudaStreamSynchronize(sm);
    if (prep_done) cudaEventDestroy(prep_done);
    for (auto& e : ev) {
      if (e.a) cudaEventDestroy(e.a);
      if (e.b) cudaEventDestroy(e.b);
    }
    if (sb) cudaStreamDestroy(sb);
  };
  int rc = OK;
  int info = 0;
  flops_reset();
  do {
    cudaStream_t sback = two_streams ? sb : sm;
    // ---- SBR
    flops_set_stage(ST_SBR);
    if ((rc = (cudaEventRecord(ev[0].a, sm) == cudaSuccess) ? OK : ERR_CUDA)) break;
    if ((rc = sbr_reduce(sm, n, b, A, lda, L.bands, want_vectors ? L.Tall : nullptr, L.ws_sbr)))
      break;
    cudaEventRecord(ev[0].b, sm);
    // ---- BC first: its persistent CTAs must become resident before the SBR-Back GEMMs
    //      (enqueued next, on the back stream) fill the SMs
    cudaEventRecord(ev[1].a, sm);
    flops_set_stage(ST_BC);
    if ((rc = bc_reduce_range(sm, n, bc_b, b, L.bands, n, L.d, L.e, nullptr,
                              want_vectors ? L.tau : nullptr, want_vectors ? L.V : nullptr, L.vld,
                              L.ws_bc)))
      break;
    cudaEventRecord(ev[1].b, sm);
    // ---- SBR-Back (forms Q_s) overlapping the chase
    if (want_vectors && order != PEVD_ORDER_CONVENTIONAL) {
      if (two_streams) cudaStreamWaitEvent(sback, ev[0].b, 0);
      flops_set_stage(ST_SBR_BACK);
      cudaEventRecord(ev[3].a, sback);
      if ((rc = sbr_back_form(sback, n, b, A, lda, L.Tall, L.Qs, n, L.ws_back))) break;
      cudaEventRecord(ev[3].b, sback);
    }
    // ---- BC-Back on Q_s (back stream) overlapping the divide and conquer
    if (want_vectors && order != PEVD_ORDER_CONVENTIONAL) {
      if (two_streams) cudaStreamWaitEvent(sback, ev[1].b, 0);
      flops_set_stage(ST_BC_BACK);
      cudaEventRecord(ev[4].a, sback);
      if ((rc = bc_back_right(sback, n, bc_b, L.tau, L.V, L.vld, L.Qs, n, n, L.ws_bcb))) break;
      cudaEventRecord(ev[4].b, sback);
    }
    // ---- conventional: the back-transform preparations on the side stream: the SBR-Back T
    //      aggregation needs only the SBR output, so it runs beside the latency-bound chase
    //      (enqueued after it, so the chase's cooperative grid is resident first); the Z factor
    //      of every BC-Back block needs the chase output and runs beside the divide and conquer
    // conventional order with b a multiple of 8 up to 64 runs BC-Back on the transpose (the DMMA
    // kernel's layout)
    const bool conv_t =
        want_vectors && order == PEVD_ORDER_CONVENTIONAL && bc_back_dmma_ok(bc_b, L.vld);
    if (want_vectors && order == PEVD_ORDER_CONVENTIONAL) {
      cudaStreamWaitEvent(sb, ev[0].b, 0);
      flops_set_stage(ST_SBR_BACK);
      if ((rc = sbr_back_prepare(sb, n, b, A, lda, L.Tall, L.ws_back))) break;
      cudaStreamWaitEvent(sb, ev[1].b, 0);
      flops_set_stage(ST_BC_BACK);
      if (conv_t &&
          (rc = bc_back_left_t(sb, n, bc_b, L.tau, L.V, L.vld, nullptr, n, n, L.ws_bcb, false)))
        break;
      cudaEventRecord(prep_done, sb);
    }
    // ---- D&C
    flops_set_stage(ST_SOLVER);
    cudaEventRecord(ev[2].a, sm);
    if (want_vectors || !values_by_bisection()) {
      if ((rc = stedc(sm, n, L.d, L.e, L.Qd, n, L.ws_dc, &info))) break;
      if ((rc = (cudaMemcpyAsync(lam, L.d, n * 8, cudaMemcpyDeviceToDevice, sm) == cudaSuccess)
                    ? OK
                    : ERR_CUDA))
        break;
    } else {  // eigenvalues only: no eigenvector merges at all
      if ((rc = stebz(sm, n, L.d, L.e, lam, L.ws_dc))) break;
    }
    cudaEventRecord(ev[2].b, sm);
    if (want_vectors) {
      if (order == PEVD_ORDER_CONVENTIONAL) cudaStreamWaitEvent(sm, prep_done, 0);
      if (conv_t) {
        // Q_b Q_d computed as its transpose Xt = Q_d^T Q_b^T, so the bulge reflectors meet X in
        // column-major order (the BC-Back kernel's coalesced pattern): Xt lives in the D&C's
        // (now free) ping-pong buffer; two n^2 transposes (~7 ms each)
        double* Xt = (double*)L.ws_dc;
        flops_set_stage(ST_BC_BACK);
        cudaEventRecord(ev[4].a, sm);
        if ((rc = transpose(sm, n, n, L.Qd, n, Xt, n))) break;
        if ((rc = bc_back_left_t(sm, n, bc_b, L.tau, L.V, L.vld, Xt, n, n, L.ws_bcb, true))) break;
        cudaEventRecord(ev[4].b, sm);
        // back to column-major in the output, where SBR-Back's left application (its faster
        // GEMM shapes) finishes Q = Q_s (Q_b Q_d) in place
        cudaEventRecord(ev[5].a, sm);
        if ((rc = transpose(sm, n, n, Xt, n, Q, ldq))) break;
        cudaEventRecord(ev[5].b, sm);
        flops_set_stage(ST_SBR_BACK);
        cudaEventRecord(ev[3].a, sm);
        if (hq) {
          // all but the last Q_SLAB_GROUPS aggregated blocks over every column, then those (the
          // largest, m ~ n) slab by slab: each slab's copy to the host overlaps the next
          // slab's GEMMs, and only the last slab's copy is exposed
          const std::vector<int64_t> sl = q_slab_bounds(n);
          const int64_t gsplit = sl.size() > 2 ? Q_SLAB_GROUPS : 0;
          if (gsplit > 0)
            rc = sbr_back_apply_left(sm, n, b, A, lda, L.Tall, Q, ldq, n, L.ws_back, true, gsplit);
          for (size_t s = 0; s + 1 < sl.size() && rc == OK; ++s) {
            rc = sbr_back_apply_left(sm, n, b, A, lda, L.Tall, Q + sl[s] * ldq, ldq,
                                     sl[s + 1] - sl[s], L.ws_back, true, 0, gsplit > 0 ? gsplit : -1);
            if (rc == OK && hq->slab_ready(sm, Q, ldq, n, sl[s], sl[s + 1] - sl[s])) rc = ERR_CUDA;
          }
          if (rc) break;
        } else if ((rc = sbr_back_apply_left(sm, n, b, A, lda, L.Tall, Q, ldq, n, L.ws_back,
                                             true))) {
          break;
        }
        cudaEventRecord(ev[3].b, sm);
      } else if (order == PEVD_ORDER_CONVENTIONAL) {
        flops_set_stage(ST_BC_BACK);
        cudaEventRecord(ev[4].a, sm);
        if ((rc = bc_back_left(sm, n, bc_b, L.tau, L.V, L.vld, L.Qd, n, n, L.ws_bcb))) break;
        cudaEventRecord(ev[4].b, sm);
        flops_set_stage(ST_SBR_BACK);
        cudaEventRecord(ev[3].a, sm);
        if ((rc = sbr_back_apply_left(sm, n, b, A, lda, L.Tall, L.Qd, n, n, L.ws_back, true))) break;
        cudaEventRecord(ev[3].b, sm);
        cudaEventRecord(ev[5].a, sm);
        if (cudaMemcpy2DAsync(Q, ldq * 8, L.Qd, n * 8, n * 8, n, cudaMemcpyDeviceToDevice, sm) !=
            cudaSuccess) {
          rc = ERR_CUDA;
          break;
        }
        cudaEventRecord(ev[5].b, sm);
      } else {
        if (two_streams) cudaStreamWaitEvent(sm, ev[4].b, 0);
        flops_set_stage(ST_FINAL);
        cudaEventRecord(ev[5].a, sm);
        if (hq && hq->row_major) {
          // Q^T = Q_d^T (Q_s Q_b)^T in column slabs (rows of Q), each slab's copy to the host
          // overlapping the next slab's GEMM
          const std::vector<int64_t> sl = q_slab_bounds(n);
          for (size_t s = 0; s + 1 < sl.size() && rc == OK; ++s) {
            const int64_t c0 = sl[s], nc = sl[s + 1] - sl[s];
            GemmArgs g{n, nc, n, 1.0, 0.0, L.Qd, n, L.Qs + c0, n, Q + c0 * ldq, ldq, 1, 1,
                       A_GENERAL, C_ALL};
            rc = gemm(sm, g, nullptr, 0);
            if (rc == OK && hq->slab_ready(sm, Q, ldq, n, c0, nc)) rc = ERR_CUDA;
          }
          if (rc) break;
        } else {
          GemmArgs g{n, n, n, 1.0, 0.0, L.Qs, n, L.Qd, n, Q, ldq, 0, 0, A_GENERAL, C_ALL};
          if ((rc = gemm(sm, g, nullptr, 0))) break;
        }
        cudaEventRecord(ev[5].b, sm);
      }
      if (hq && !conv_t && !(hq->row_major && order != PEVD_ORDER_CONVENTIONAL) &&
          hq->slab_ready(sm, Q, ldq, n, 0, n)) {
        rc = ERR_CUDA;
        break;
      }
    }
    if (cudaStreamSynchronize(sm) != cudaSuccess) {
      set_error("device failure: %s", cudaGetErrorString(cudaGetLastError()));
      rc = ERR_CUDA;
      break;
    }
    if (info != 0) {
      set_error(info > 0 ? "tridiagonal divide and conquer: leaf QL/QR did not converge near row %d"
                         : "tridiagonal divide and conquer: secular equation did not converge "
                           "(root %d)",
                info > 0 ? info - 1 : -info - 1);
      rc = ERR_CONVERGE;
      break;
    }
    if (stats) {
      auto el = [&](cudaEvent_t x) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[0].a, x);
        return (double)ms;
      };
      stats->sbr_ms[0] = 0.0; stats->sbr_ms[1] = el(ev[0].b);
      stats->bc_ms[0] = el(ev[1].a); stats->bc_ms[1] = el(ev[1].b);
      stats->solver_ms[0] = el(ev[2].a); stats->solver_ms[1] = el(ev[2].b);
      if (want_vectors) {
        stats->sbr_back_ms[0] = el(ev[3].a); stats->sbr_back_ms[1] = el(ev[3].b);
        stats->bc_back_ms[0] = el(ev[4].a); stats->bc_back_ms[1] = el(ev[4].b);
        stats->final_ms[0] = el(ev[5].a); stats->final_ms[1] = el(ev[5].b);
      }
      double tot = stats->solver_ms[1];
      tot = std::max(tot, std::max(stats->final_ms[1], stats->sbr_back_ms[1]));
      stats->total_ms = tot;
      stats->n_reflectors = bc_num_reflectors(n, bc_b);
      stats->n_rounds = sbr_num_rounds(n, b);
      flops_read(stats->flops);
    }
  } while (0);
  if (rc == ERR_CUDA && g_err[0] == '\0') set_error("CUDA failure");
  cleanup();
  return rc;
}

}  // namespace
}  // namespace pevd

extern "C" {

int pevd_syevd_device(int64_t n, int b, double* A, int64_t lda, double* lam, double* Q,
                      int64_t ldq, int want_vectors, int order, void* workspace,
                      int64_t workspace_bytes, void* stream, pevd_stats* stats) {
  return syevd_impl(n, b, A, lda, lam, Q, ldq, want_vectors, order, workspace, workspace_bytes,
                    (cudaStream_t)stream, stats, nullptr);
}

int pevd_syevd_device_host_q(int64_t n, int b, double* A, int64_t lda, double* lam, double* Q,
                             int64_t ldq, double* Qh, int64_t ldqh, int q_row_major,
                             int want_vectors, int order, void* workspace,
                             int64_t workspace_bytes, void* stream, pevd_stats* stats) {
  if (want_vectors && (!Qh || ldqh < n)) {
    set_error("pevd_syevd_device_host_q: bad host Q (ldqh=%lld, n=%lld)", (long long)ldqh,
              (long long)n);
    return ERR_VALUE;
  }
  if (!want_vectors)
    return syevd_impl(n, b, A, lda, lam, Q, ldq, 0, order, workspace, workspace_bytes,
                      (cudaStream_t)stream, stats, nullptr);
  int dev = 0;
  PEVD_CUDA(cudaGetDevice(&dev));
  HostQ hq;
  hq.Qh = Qh;
  hq.ldqh = ldqh;
  hq.pinned = host_is_pinned(Qh);
  hq.row_major = q_row_major != 0 && order != PEVD_ORDER_CONVENTIONAL;
  if (q_row_major && order == PEVD_ORDER_CONVENTIONAL) {
    set_error("pevd_syevd_device_host_q: row-major Q is produced by the pipelined and "
              "sequential orders only (conventional order returns it column-major)");
    return ERR_VALUE;
  }
  std::unique_ptr<Stager> stager;
  if (hq.pinned) {
    PEVD_CUDA(cudaStreamCreateWithFlags(&hq.cs, cudaStreamNonBlocking));
  } else {
    stager.reset(new Stager(dev));
    hq.stager = stager.get();
    stager->touch(Qh, ldqh, n, n);  // fault the pages in while the GPU reduces
  }
  int rc = syevd_impl(n, b, A, lda, lam, Q, ldq, 1, order, workspace, workspace_bytes,
                      (cudaStream_t)stream, stats, &hq);
  if (hq.finish() && rc == OK) {
    set_error("device -> host copy of Q failed");
    rc = ERR_CUDA;
  }
  if (hq.cs) cudaStreamDestroy(hq.cs);
  return rc;
}

int pevd_transpose(int64_t rows, int64_t cols, const double* in, int64_t ldi, double* out,
                   int64_t ldo, void* stream) {
  return transpose((cudaStream_t)stream, rows, cols, in, ldi, out, ldo);
}

int pevd_asymmetry(int64_t n, const double* A, int64_t lda, double* out2, void* stream) {
  if (n < 1 || lda < n || !A || !out2) {
    set_error("pevd_asymmetry: bad arguments");
    return ERR_VALUE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nt = cdiv(n, 32);
  const int64_t ntiles = nt * (nt + 1) / 2;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)num_sms() * 16);
  double* d = nullptr;
  if (cudaMallocAsync(&d, (2 * grid + 2) * 8, st) != cudaSuccess) {
    set_error("pevd_asymmetry: allocation failed");
    return ERR_NOMEM;
  }
  asym_partials<<<grid, 256, 0, st>>>(n, A, lda, nt, d + 2);
  count_launch();
  asym_finish<<<1, 32, 0, st>>>(grid, d + 2, d);
  count_launch();
  cudaError_t e = cudaMemcpyAsync(out2, d, 16, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (e != cudaSuccess) {
    set_error("pevd_asymmetry: %s", cudaGetErrorString(e));
    return ERR_CUDA;
  }
  return OK;
}

}  // extern "C"

namespace {

// pevd_syevd / pevd_syevd_checked.  sym_tol < 0: only the lower trapezoid of A goes up (the
// device never reads the strictly upper triangle); otherwise all of A goes up and the
// SymmetricMatrix test (core.py:75-84) runs on the device first.
int host_syevd(int64_t n, int b, const double* A, int64_t lda, double* lam, double* Q,
               int64_t ldq, int want_vectors, int order, double sym_tol, int q_row_major,
               pevd_stats* stats) {
  if (n < 1 || lda < n || !A || !lam || (want_vectors && (!Q || ldq < n))) {
    set_error("pevd_syevd: bad arguments");
    return ERR_VALUE;
  }
  const int bb = (int)std::min<int64_t>(std::max(b, 1), std::max<int64_t>(n - 1, 1));
  const int64_t wsb = pevd_syevd_workspace_bytes(n, bb, want_vectors, order);
  double *dA = nullptr, *dlam = nullptr, *dQ = nullptr;
  void* ws = nullptr;
  cudaStream_t st = nullptr;
  int dev = 0;
  int rc = OK;
  auto fail_alloc = [&](const char* what) {
    set_error("device allocation failed (%s)", what);
    rc = ERR_NOMEM;
  };
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    set_error("CUDA context unavailable: %s", cudaGetErrorString(cudaGetLastError()));
    return ERR_CUDA;
  }
  // PEVD_HOST_PHASES=1: wall time of each host-side phase on stderr (tools/hostio_probe.py)
  static const bool phases = getenv("PEVD_HOST_PHASES") && getenv("PEVD_HOST_PHASES")[0] == '1';
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!phases) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "pevd_syevd phase %-8s %8.1f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  if (cudaMalloc(&dA, n * n * 8) != cudaSuccess) fail_alloc("A");
  else if (cudaMalloc(&dlam, n * 8) != cudaSuccess) fail_alloc("lam");
  else if (want_vectors && cudaMalloc(&dQ, n * n * 8) != cudaSuccess) fail_alloc("Q");
  else if (cudaMalloc(&ws, wsb) != cudaSuccess) fail_alloc("workspace");
  phase("malloc");
  if (rc == OK) {
    // only the lower trapezoid of each column block goes up: the strictly upper triangle of A
    // is never referenced on the device (the SBR reads A through its lower triangle)
    const int64_t CB = 512;
    const bool full = sym_tol >= 0.0;
    cudaError_t e = cudaSuccess;
    if (host_is_pinned(A)) {
      for (int64_t j0 = 0; j0 < n && e == cudaSuccess; j0 += CB) {
        const int64_t r0 = full ? 0 : j0;
        e = cudaMemcpy2DAsync(dA + r0 + j0 * n, n * 8, A + r0 + j0 * lda, lda * 8, (n - r0) * 8,
                              std::min(CB, n - j0), cudaMemcpyHostToDevice, st);
      }
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    } else {
      Stager up(dev);
      for (int64_t j0 = 0; j0 < n; j0 += CB) {
        const int64_t r0 = full ? 0 : j0;
        up.h2d(A + r0 + j0 * lda, lda, dA + r0 + j0 * n, n, n - r0, std::min(CB, n - j0));
      }
      e = up.drain();
    }
    if (e != cudaSuccess) {
      set_error("H2D copy failed: %s", cudaGetErrorString(e));
      rc = ERR_CUDA;
    }
    if (rc == OK && full) {
      double out2[2] = {0.0, 0.0};
      rc = pevd_asymmetry(n, dA, n, out2, st);
      if (rc == OK && out2[0] > sym_tol * std::max(1.0, out2[1])) {
        set_error("asymmetry %.3e exceeds tolerance", out2[0]);
        rc = ERR_VALUE;
      }
    }
  }
  phase("upload");
  if (rc == OK)
    rc = want_vectors ? pevd_syevd_device_host_q(n, b, dA, n, dlam, dQ, n, Q, ldq, q_row_major,
                                                 1, order, ws, wsb, st, stats)
                      : pevd_syevd_device(n, b, dA, n, dlam, nullptr, n, 0, order, ws, wsb, st,
                                          stats);
  phase("evd");
  if (rc == OK && cudaMemcpy(lam, dlam, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    set_error("D2H copy failed");
    rc = ERR_CUDA;
  }
  cudaFree(dA);
  cudaFree(dlam);
  cudaFree(dQ);
  cudaFree(ws);
  cudaStreamDestroy(st);
  phase("free");
  return rc;
}

}  // namespace

extern "C" {

int pevd_syevd(int64_t n, int b, const double* A, int64_t lda, double* lam, double* Q, int64_t ldq,
               int want_vectors, int order, pevd_stats* stats) {
  return host_syevd(n, b, A, lda, lam, Q, ldq, want_vectors, order, -1.0, 0, stats);
}

int pevd_syevd_checked(int64_t n, int b, const double* A, int64_t lda, double* lam, double* Q,
                       int64_t ldq, int want_vectors, int order, double sym_tol, int q_row_major,
                       pevd_stats* stats) {
  if (sym_tol != sym_tol) {
    set_error("pevd_syevd_checked: sym_tol is NaN");
    return ERR_VALUE;
  }
  if (q_row_major && order == PEVD_ORDER_CONVENTIONAL) {
    set_error("pevd_syevd_checked: row-major Q is produced by the pipelined and sequential "
              "orders only (conventional order returns it column-major)");
    return ERR_VALUE;
  }
  return host_syevd(n, b, A, lda, lam, Q, ldq, want_vectors, order, sym_tol, q_row_major, stats);
}

int pevd_dgemm(int transA, int transB, int64_t m, int64_t n, int64_t k, double alpha,
               const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
               int64_t ldc, void* workspace, int64_t workspace_bytes, void* stream) {
  GemmArgs g{m, n, k, alpha, beta, A, lda, B, ldb, C, ldc, transA, transB, A_GENERAL, C_ALL};
  return gemm((cudaStream_t)stream, g, (double*)workspace, workspace_bytes / 8);
}

// Measurement helper (tools/kernel_probe.py gemm_grouped; not part of include/pevd.h): ONE
// problem through the grouped-GEMM path the divide and conquer's merges take, with an optional
// identity-free column map, so its rate can be set beside pevd_dgemm's on the same shape.
int pevd_probe_gemm_grouped(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double* C, int64_t ldc,
                            const int* d_cmap, void* d_args, void* stream) {
  GemmArgs g{m, n, k, 1.0, 0.0, A, lda, B, ldb, C, ldc, 0, 0, A_GENERAL, C_ALL};
  g.cmap = d_cmap;
  cudaStream_t st = (cudaStream_t)stream;
  PEVD_CUDA(cudaMemcpyAsync(d_args, &g, sizeof(GemmArgs), cudaMemcpyHostToDevice, st));
  return gemm_grouped(st, (const GemmArgs*)d_args, 1, m, n);
}

int pevd_dsymm_lower(int64_t m, int64_t n, double alpha, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                     void* workspace, int64_t workspace_bytes, void* stream) {
  GemmArgs g{m, n, m, alpha, beta, A, lda, B, ldb, C, ldc, 0, 0, A_SYM_LOWER, C_ALL};
  return gemm((cudaStream_t)stream, g, (double*)workspace, workspace_bytes / 8);
}

int64_t pevd_panel_qr_workspace_bytes(void) { return panel_qr_ws_bytes(); }

int pevd_panel_qr(int64_t m, int k, const double* P, int64_t ldp, double* R, double* Y,
                  int64_t ldy, double* W, int64_t ldw, double* T, void* workspace, void* stream) {
  return panel_qr((cudaStream_t)stream, m, k, P, ldp, R, Y, ldy, nullptr, 0, W, ldw, T, workspace);
}

int64_t pevd_sbr_workspace_bytes(int64_t n, int b) { return sbr_ws_bytes(n, b); }

int pevd_sbr(int64_t n, int b, double* A, int64_t lda, double* bands, double* Tall,
             void* workspace, void* stream) {
  return sbr_reduce((cudaStream_t)stream, n, b, A, lda, bands, Tall, workspace);
}

int64_t pevd_bc_num_reflectors(int64_t n, int b) { return n >= 3 ? bc_num_reflectors(n, b) : 0; }
int64_t pevd_bc_workspace_bytes(int64_t n, int b) { return bc_ws_bytes(n, b); }

int pevd_bc(int64_t n, int b, const double* bands, double* d, double* e, double* tau, double* V,
            int vld, void* workspace, void* stream) {
  return bc_reduce((cudaStream_t)stream, n, b, bands, d, e, tau, V, vld, workspace);
}

int pevd_bc_partition(int64_t n, int b, int bw, const double* bands, int64_t sweep_end,
                      double* band_out, double* tau, double* V, int vld, void* workspace,
                      void* stream) {
  return bc_reduce_range((cudaStream_t)stream, n, b, bw, bands, sweep_end, nullptr, nullptr,
                         band_out, tau, V, vld, workspace);
}

int64_t pevd_stedc_workspace_bytes(int64_t n) { return stedc_ws_bytes(n); }

int pevd_stedc(int64_t n, double* d, const double* e, double* Q, int64_t ldq, void* workspace,
               void* stream) {
  int info = 0;
  cudaStream_t st = (cudaStream_t)stream;
  PEVD_TRY(stedc(st, n, d, e, Q, ldq, workspace, &info));
  PEVD_CUDA(cudaStreamSynchronize(st));
  if (info != 0) {
    set_error("tridiagonal divide and conquer did not converge (info=%d)", info);
    return ERR_CONVERGE;
  }
  return OK;
}

int pevd_stedc_cols(int64_t n, double* d, const double* e, double* Q, int64_t ldq, int64_t col_lo,
                    int64_t col_hi, void* workspace, void* stream) {
  int info = 0;
  cudaStream_t st = (cudaStream_t)stream;
  PEVD_TRY(stedc(st, n, d, e, Q, ldq, workspace, &info, col_lo, col_hi));
  PEVD_CUDA(cudaStreamSynchronize(st));
  if (info != 0) {
    set_error("tridiagonal divide and conquer did not converge (info=%d)", info);
    return ERR_CONVERGE;
  }
  return OK;
}

int64_t pevd_sbr_back_workspace_bytes(int64_t n, int b) { return sbr_back_ws_bytes(n, b); }

int pevd_sbr_back_form(int64_t n, int b, const double* Ystair, int64_t ldy, const double* Tall,
                       double* Qs, int64_t ldq, void* workspace, void* stream) {
  if (ldy < n) {
    set_error("pevd_sbr_back_form: ldy=%lld < n=%lld", (long long)ldy, (long long)n);
    return ERR_VALUE;
  }
  return sbr_back_form((cudaStream_t)stream, n, b, Ystair, ldy, Tall, Qs, ldq, workspace);
}

int pevd_sbr_back_left(int64_t n, int b, const double* Ystair, int64_t ldy, const double* Tall,
                       double* X, int64_t ldx, int64_t ncols, void* workspace, void* stream) {
  if (ldy < n) {
    set_error("pevd_sbr_back_left: ldy=%lld < n=%lld", (long long)ldy, (long long)n);
    return ERR_VALUE;
  }
  return sbr_back_apply_left((cudaStream_t)stream, n, b, Ystair, ldy, Tall, X, ldx, ncols,
                             workspace);
}

static int64_t ws_round(int64_t x) { return (x + 255) / 256 * 256; }

// + room for the transpose of a left operand (the fast column-major BC-Back path, below)
int64_t pevd_bc_back_workspace_bytes(int64_t n, int64_t nrows, int b) {
  return ws_round(bc_back_ws_bytes(n, nrows, b)) + n * nrows * 8 + 256;
}

int pevd_bc_back_right(int64_t n, int b, const double* tau, const double* V, int vld, double* X,
                       int64_t ldx, int64_t nrows, void* workspace, void* stream) {
  return bc_back_right((cudaStream_t)stream, n, b, tau, V, vld, X, ldx, nrows, workspace);
}

int pevd_bc_back_left(int64_t n, int b, const double* tau, const double* V, int vld, double* X,
                      int64_t ldx, int64_t ncols, void* workspace, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (bc_back_dmma_ok(b, vld) && workspace && n >= 3 && ncols > 0) {
    // on the transpose: the DMMA kernel then reads X column-major (its coalesced pattern)
    double* Xt = (double*)((char*)workspace + ws_round(bc_back_ws_bytes(n, ncols, b)));
    PEVD_TRY(transpose(st, n, ncols, X, ldx, Xt, ncols));
    PEVD_TRY(bc_back_left_t(st, n, b, tau, V, vld, Xt, ncols, ncols, workspace));
    return transpose(st, ncols, n, Xt, ncols, X, ldx);
  }
  return bc_back_left(st, n, b, tau, V, vld, X, ldx, ncols, workspace);
}

}  // extern "C"
