// FP64 MMA shape microbenchmark (sm_100a): m8n8k4 vs the sm_90+ shapes m16n8k4 / m16n8k8 /
// m16n8k16.  Same peak flops would still matter: a larger shape needs fewer issue slots per flop,
// which is what the BC-Back kernel (DMMA + DADD on one warp) is short of.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void mma_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; i++) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
                     "{%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                     "{%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                     "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                       "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

template <int SHAPE>
void run(const char* name, double macs_per_mma, int sms, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    const int iters = SHAPE == 3 ? 2500 : SHAPE == 2 ? 5000 : 10000;
    mma_loop<SHAPE><<<sms, warps * 32>>>(out, 50);
    cudaEventRecord(e0);
    mma_loop<SHAPE><<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * macs_per_mma * 8 * (double)iters * warps * sms * 2;
    printf("{\"kind\":\"%s\",\"warps_per_cta\":%d,\"tflops\":%.2f,\"ns_per_mma_per_warp\":%.2f}\n", name,
           warps, flops / ms / 1e9, ms * 1e6 / (8.0 * iters) * (warps * sms * 2) / (4.0 * sms) / (warps * 2) * 4);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  run<0>("m8n8k4", 8 * 8 * 4, sms, out);
  run<1>("m16n8k4", 16 * 8 * 4, sms, out);
  run<2>("m16n8k8", 16 * 8 * 8, sms, out);
  run<3>("m16n8k16", 16 * 8 * 16, sms, out);
  return 0;
}
