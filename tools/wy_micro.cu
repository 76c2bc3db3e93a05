// Microbenchmark: the BC-Back DMMA block sequence (8 blocks x (10 + 10) DMMA per step, window of
// 12 accumulator tiles) with V/Z fragments from shared memory but no global traffic, no staging
// and (optionally) no per-step barrier.  Tells whether the kernel's 70% tensor-pipe activity is
// the dependency structure itself or the staging around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wy_micro tools/wy_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa8(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)), "l"(g));
}
__device__ __forceinline__ void cpa16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)), "l"(g));
}

// 0: as BC-Back (2 P chains + DADD), 1: + __syncthreads per step, 2: independent,
// 3: + cp.async staging of V (2048 x 8 B) and Z (1344 x 16 B) per step from a streamed buffer
template <int MODE>
__global__ void __launch_bounds__(256, 2) micro(double* out, int steps, const double* src) {
  __shared__ double va[2][64][20];
  __shared__ double zu[64][42];
  double* stage = &va[0][0][0];  // (va and zu are contiguous; contents do not matter here)
  const int tid = threadIdx.x, lane = tid & 31, qd = lane & 3, r8 = lane >> 2;
  for (int e = tid; e < 2 * 64 * 20; e += 256) (&va[0][0][0])[e] = 1e-3 * (e % 7);
  for (int e = tid; e < 64 * 42; e += 256) (&zu[0][0])[e] = 1e-3 * (e % 5);
  __syncthreads();
  double w[12][2];
#pragma unroll
  for (int c = 0; c < 12; ++c) w[c][0] = w[c][1] = 1e-3 * (c + lane);
  for (int s = 0; s < steps; ++s) {
#pragma unroll
    for (int bb = 0; bb < 8; ++bb) {
      const int blk = 7 - bb, tb = blk * 8;
      double p0 = 0, p1 = 0, e0 = 0, e1 = 0;
      const double* v0 = &va[0][tb + r8][qd];
      const double* v1 = &va[1][tb + r8][qd];
#pragma unroll
      for (int cc = 0; cc < 5; ++cc) {
        if (MODE == 2) {
          dmma(p0, p1, w[cc][0], v0[4 * cc]);
          dmma(e0, e1, w[cc][1], v1[4 * cc]);
        } else {
          dmma(p0, p1, w[blk + cc][0], v0[4 * cc]);
          dmma(e0, e1, w[blk + cc][1], v1[4 * cc]);
        }
      }
      p0 += e0;
      p1 += e1;
      const double* z0 = &zu[tb + 2 * qd][r8];
      const double* z1 = &zu[tb + 2 * qd + 1][r8];
#pragma unroll
      for (int cc = 0; cc < 5; ++cc) dmma(w[blk + cc][0], w[blk + cc][1], p0, z0[8 * cc]);
#pragma unroll
      for (int cc = 0; cc < 5; ++cc) dmma(w[blk + cc][0], w[blk + cc][1], p1, z1[8 * cc]);
    }
    if (MODE == 3) {
      const double* vs = src + ((size_t)(s % 4096) * 148 + blockIdx.x % 148) * 4736;
#pragma unroll
      for (int p = 0; p < 8; ++p) cpa8(&stage[(tid + 256 * p) % 2560], vs + tid + 256 * p);
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const int e = tid + 256 * p;
        if (e < 1344) cpa16(&zu[0][0] + 2 * e, vs + 2048 + 2 * e);
      }
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    if (MODE == 1 || MODE == 3) __syncthreads();
  }
  double acc = 0;
#pragma unroll
  for (int c = 0; c < 12; ++c) acc += w[c][0] + w[c][1];
  out[blockIdx.x * 256 + tid] = acc;
}

template <int MODE>
void run(double* out, int blocks, int steps, const double* src) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  micro<MODE><<<blocks, 256>>>(out, 10, src);
  cudaEventRecord(a);
  micro<MODE><<<blocks, 256>>>(out, steps, src);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 512.0 * 160.0 * 8.0 * blocks * (double)steps;  // DMMA = 512 flop
  printf("mode %d: %.3f ms, %.2f TF/s executed\n", MODE, ms, flops / ms / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * 256 * sms * 4);
  const int blocks = 2 * sms, steps = 20000;
  double* src;
  cudaMalloc(&src, sizeof(double) * (size_t)4096 * 148 * 4736 + 64);
  cudaMemset(src, 0, sizeof(double) * (size_t)4096 * 148 * 4736);
  run<0>(out, blocks, steps, src);
  run<1>(out, blocks, steps, src);
  run<2>(out, blocks, steps, src);
  run<3>(out, blocks, steps, src);
  return 0;
}
