// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Used once to establish the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    int iters = 20000;
    dmma_loop<<<sms, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * warps * sms * 2;
    printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", warps, flops / ms / 1e9);
  }
  for (int warps = 4; warps <= 32; warps *= 2) {
    int iters = 20000;
    dfma_loop<<<sms, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * (double)iters * warps * 32 * sms * 2;
    printf("{\"kind\":\"dfma\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", warps, flops / ms / 1e9);
  }
  return 0;
}
