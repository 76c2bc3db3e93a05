// Host <-> device staging for the host-buffer entry points (see hostio.h).
#include "hostio.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace pevd {

namespace {

constexpr int64_t kChunkBytes = 32ll << 20;

int stage_threads() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("PEVD_STAGE_THREADS");
    v = e ? std::max(1, atoi(e)) : 8;
  }
  return v;
}

// pinned staging chunks, allocated once per process and reused across calls
std::mutex g_pool_mu;
std::vector<void*> g_pool;

void* take_chunk() {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool.empty()) {
    void* p = g_pool.back();
    g_pool.pop_back();
    return p;
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, kChunkBytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void give_chunk(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool.push_back(p);
}

}  // namespace

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

Stager::Stager(int device) : device_(device) {
  const int T = stage_threads();
  for (int t = 0; t < T; ++t) threads_.emplace_back(&Stager::worker, this, t);
}

Stager::~Stager() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& th : threads_) th.join();
}

void Stager::enqueue(Task t) {
  // split into chunks of whole columns (or of rows when one column exceeds a chunk)
  const int64_t col_bytes = t.rows * 8;
  const int64_t rstep = std::min<int64_t>(t.rows, kChunkBytes / 8);
  const int64_t cstep = std::max<int64_t>(1, kChunkBytes / std::max<int64_t>(col_bytes, 8));
  std::lock_guard<std::mutex> lk(mu_);
  for (int64_t c = 0; c < t.cols; c += cstep)
    for (int64_t r = 0; r < t.rows; r += rstep) {
      Task s = t;
      s.rows = std::min(rstep, t.rows - r);
      s.cols = std::min(cstep, t.cols - c);
      s.src = t.src ? t.src + r + c * t.lds : nullptr;
      s.dst = t.dst + r + c * t.ldd;
      q_.push_back(s);
      ++pending_;
    }
  cv_.notify_all();
}

void Stager::d2h(const double* dsrc, int64_t ld, double* hdst, int64_t ldh, int64_t rows,
                 int64_t cols, cudaEvent_t after) {
  if (rows <= 0 || cols <= 0) return;
  enqueue(Task{DOWN, dsrc, hdst, ld, ldh, rows, cols, after});
}

void Stager::h2d(const double* hsrc, int64_t ldh, double* ddst, int64_t ld, int64_t rows,
                 int64_t cols) {
  if (rows <= 0 || cols <= 0) return;
  enqueue(Task{UP, hsrc, ddst, ldh, ld, rows, cols, nullptr});
}

void Stager::touch(double* hdst, int64_t ldh, int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return;
  enqueue(Task{TOUCH, nullptr, hdst, 0, ldh, rows, cols, nullptr});
}

cudaError_t Stager::drain() {
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return pending_ == 0; });
  const cudaError_t e = err_;
  err_ = cudaSuccess;
  return e;
}

void Stager::worker(int) {
  cudaSetDevice(device_);
  cudaStream_t st = nullptr;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  double* buf = (double*)take_chunk();
  for (;;) {
    Task t;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
      if (q_.empty()) break;
      t = q_.front();
      q_.pop_front();
    }
    cudaError_t e = (buf && st) ? cudaSuccess : cudaErrorMemoryAllocation;
    const size_t w = (size_t)t.rows * 8;
    if (t.kind == TOUCH) {
      for (int64_t c = 0; c < t.cols; ++c) memset(t.dst + c * t.ldd, 0, w);
    } else if (e == cudaSuccess && t.kind == DOWN) {
      if (t.after) e = cudaEventSynchronize(t.after);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(buf, w, t.src, t.lds * 8, w, t.cols, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e == cudaSuccess)
        for (int64_t c = 0; c < t.cols; ++c) memcpy(t.dst + c * t.ldd, buf + c * t.rows, w);
    } else if (e == cudaSuccess) {
      for (int64_t c = 0; c < t.cols; ++c) memcpy(buf + c * t.rows, t.src + c * t.lds, w);
      e = cudaMemcpy2DAsync(t.dst, t.ldd * 8, buf, w, w, t.cols, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    std::lock_guard<std::mutex> lk(mu_);
    if (e != cudaSuccess && err_ == cudaSuccess) err_ = e;
    if (--pending_ == 0) done_cv_.notify_all();
  }
  give_chunk(buf);
  if (st) cudaStreamDestroy(st);
}

int HostQ::slab_ready(cudaStream_t producer, const double* Q, int64_t ldq, int64_t n, int64_t c0,
                      int64_t nc) {
  if (!Qh || nc <= 0) return 0;
  cudaEvent_t e = nullptr;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return -1;
  evs.push_back(e);
  if (cudaEventRecord(e, producer) != cudaSuccess) return -1;
  if (pinned) {
    if (cudaStreamWaitEvent(cs, e, 0) != cudaSuccess) return -1;
    if (cudaMemcpy2DAsync(Qh + c0 * ldqh, ldqh * 8, Q + c0 * ldq, ldq * 8, n * 8, nc,
                          cudaMemcpyDeviceToHost, cs) != cudaSuccess)
      return -1;
  } else {
    stager->d2h(Q + c0 * ldq, ldq, Qh + c0 * ldqh, ldqh, n, nc, e);
  }
  return 0;
}

int HostQ::finish() {
  cudaError_t e = cudaSuccess;
  if (pinned && cs) e = cudaStreamSynchronize(cs);
  if (!pinned && stager) {
    const cudaError_t e2 = stager->drain();
    if (e == cudaSuccess) e = e2;
  }
  for (cudaEvent_t x : evs) cudaEventDestroy(x);
  evs.clear();
  return e == cudaSuccess ? 0 : -1;
}

std::vector<int64_t> q_slab_bounds(int64_t n) {
  std::vector<int64_t> b{0};
  if (n >= 4096) {
    for (int64_t num : {4, 6, 7}) {  // n/2, 3n/4, 7n/8
      const int64_t c = (n * num / 8) / 128 * 128;
      if (c > b.back() && c < n) b.push_back(c);
    }
  }
  b.push_back(n);
  return b;
}

}  // namespace pevd
