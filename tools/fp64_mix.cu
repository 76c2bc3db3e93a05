// Can the DMMA (tensor) and DFMA (FP64) pipes of a B200 SM run at the same time?
// Runs DMMA-only, DFMA-only, interleaved (same warp) and warp-specialised (half the warps each)
// loops and prints the achieved FP64 TF/s of each.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NF>
__global__ void mix_loop(double* out, int iters, int split) {
  // split = 0: every warp runs ND DMMA and NF DFMA chains; split = 1: even warps DMMA only,
  // odd warps DFMA only (each with the same per-warp chain counts)
  const int w = threadIdx.x >> 5;
  const bool do_m = split ? (w % 2 == 0) : true;
  const bool do_f = split ? (w % 2 == 1) : true;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[ND > 0 ? ND : 1][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); i++) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); i++) f[i] = i;
  if (do_m && do_f) {
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int i = 0; i < ND; i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int i = 0; i < NF; i++) f[i] = fma(f[i], a, b);
    }
  } else if (do_m) {
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int i = 0; i < ND; i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  } else {
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int i = 0; i < NF; i++) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); i++) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); i++) s += f[i];
  if (s == 12345.678) out[0] = s;
}

template <int ND, int NF>
void run(const char* name, int sms, int warps, int split, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  mix_loop<ND, NF><<<sms, warps * 32>>>(out, 100, split);
  cudaEventRecord(e0);
  mix_loop<ND, NF><<<sms * 2, warps * 32>>>(out, iters, split);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double wm = split ? warps / 2.0 : warps, wf = split ? warps / 2.0 : warps;
  const double fm = 2.0 * 256 * ND * (double)iters * wm * sms * 2;
  const double ff = 2.0 * 32 * NF * (double)iters * wf * sms * 2;
  printf("{\"kind\":\"%s\",\"warps\":%d,\"split\":%d,\"ms\":%.3f,\"dmma_tflops\":%.2f,"
         "\"dfma_tflops\":%.2f,\"total_tflops\":%.2f}\n",
         name, warps, split, ms, fm / ms / 1e9, ff / ms / 1e9, (fm + ff) / ms / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int warps = 8; warps <= 16; warps *= 2) {
    run<8, 0>("dmma_only", sms, warps, 0, out);
    run<0, 16>("dfma_only", sms, warps, 0, out);
    run<8, 8>("mixed_8dmma_8dfma", sms, warps, 0, out);
    run<8, 16>("mixed_8dmma_16dfma", sms, warps, 0, out);
    run<8, 32>("mixed_8dmma_32dfma", sms, warps, 0, out);
    run<8, 16>("split_warps", sms, warps, 1, out);
  }
  return 0;
}
