// Host <-> device movement of the EVD's n x n operands (the host-buffer entry points of
// include/pevd.h): A goes up as its lower trapezoid only (the strictly upper triangle is never
// referenced on the device), Q comes down slab by slab while the last back-transformation is
// still computing the next slab, so only the last slab's copy is exposed.
//
// Pinned host buffers are copied by the copy engines directly (cudaMemcpy2DAsync on a side
// stream).  Pageable buffers go through a pool of pinned staging chunks worked by several host
// threads (a single-threaded pageable copy of 19 GB runs at ~5 GB/s host -> device and ~2 GB/s
// device -> host on the pool's boxes; the threads overlap the DMA of one chunk with the host
// memcpy of another).
#pragma once
#include <cuda_runtime.h>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace pevd {

bool host_is_pinned(const void* p);

class Stager {
 public:
  // device: the CUDA device the chunks move to/from (the worker threads bind to it)
  explicit Stager(int device);
  ~Stager();
  // device (rows x cols, ld) -> host (ldh), after `after` (an event on the producing stream)
  void d2h(const double* dsrc, int64_t ld, double* hdst, int64_t ldh, int64_t rows, int64_t cols,
           cudaEvent_t after);
  // host -> device for a rectangle
  void h2d(const double* hsrc, int64_t ldh, double* ddst, int64_t ld, int64_t rows, int64_t cols);
  // first-touch a pageable host destination (zero fill) so the later d2h chunks copy into
  // resident pages instead of faulting them in on the critical path
  void touch(double* hdst, int64_t ldh, int64_t rows, int64_t cols);
  // wait for every queued chunk; returns the first CUDA error seen (cudaSuccess if none)
  cudaError_t drain();

 private:
  enum Kind { UP, DOWN, TOUCH };
  struct Task {
    Kind kind;
    const double* src;
    double* dst;
    int64_t lds, ldd, rows, cols;
    cudaEvent_t after;
  };
  void enqueue(Task t);
  void worker(int tid);
  int device_;
  std::vector<std::thread> threads_;
  std::deque<Task> q_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  int64_t pending_ = 0;
  bool stop_ = false;
  cudaError_t err_ = cudaSuccess;
};

// Where the EVD's Q goes on the host (nullptr Qh: Q stays on the device).
struct HostQ {
  double* Qh = nullptr;
  int64_t ldqh = 0;
  bool pinned = false;
  // pipelined / sequential orders: Qh receives Q ROW-major (Q^T column-major, the C-ordered Q of
  // pipeline.py:503); the final GEMM then forms Q^T slab by slab in the device buffer
  bool row_major = false;
  cudaStream_t cs = nullptr;      // copy stream (pinned destination)
  Stager* stager = nullptr;       // staging threads (pageable destination)
  std::vector<cudaEvent_t> evs;   // one per slab, destroyed by finish()
  // Q[:, c0:c0+nc] (device, column-major ldq, n rows) is final once `producer` reaches this
  // point: queue its copy to Qh[:, c0:c0+nc]
  int slab_ready(cudaStream_t producer, const double* Q, int64_t ldq, int64_t n, int64_t c0,
                 int64_t nc);
  int finish();
};

// Column slabs of the last back-transformation whose Q copies overlap the next slab's compute:
// geometric [n/2, n/4, n/8, n/8] (multiples of 128), one slab below n = 4096.
std::vector<int64_t> q_slab_bounds(int64_t n);
// aggregated SBR-Back blocks (the last ones applied, m ~ n) that run slab by slab: ~0.8 s of
// GEMMs at n = 49152 against 0.38 s to copy all of Q, and only 3 x 3 GEMMs split 4 ways
constexpr int64_t Q_SLAB_GROUPS = 3;

}  // namespace pevd
