// Microbenchmark: single-warp dependent-chain latencies (SM cycles) of the FP64 ops and
// SMEM loads that bound the tile sweep's serial per-strip step.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int n, double a, double b) {
  __shared__ int chase[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) chase[i] = (i + 33) % 1024;
  __syncwarp();
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x + a;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = x * a;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = b / x;
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = hypot(x, a);
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x);
  long long t6 = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < n; ++i) p = chase[p];
  long long t7 = clock64();
  out[threadIdx.x] = x + p;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    cyc[6] = t7 - t6;
  }
}
int main2();
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double)); cudaMallocManaged(&cyc, 8 * sizeof(long long));
  const int n = 4096;
  lat<<<1, 32>>>(out, cyc, n, 0.999999, 1e-3);
  lat<<<1, 32>>>(out, cyc, n, 0.999999, 1e-3);
  cudaDeviceSynchronize();
  const char* nm[7] = {"DFMA", "DADD", "DMUL", "div", "hypot", "sqrt", "LDS"};
  for (int k = 0; k < 7; ++k) printf("%s latency: %.1f cycles\n", nm[k], (double)cyc[k] / n);
  return main2();
}
// mbarrier try_wait / test_wait latency on an already-completed phase
__global__ void mbar_lat(long long* cyc, int n) {
  __shared__ __align__(8) unsigned long long bar[4];
  const unsigned a = (unsigned)__cvta_generic_to_shared(&bar[0]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a));  // phase 0 complete
  }
  __syncthreads();
  long long t0 = clock64();
  unsigned ok = 0;
  for (int i = 0; i < n; ++i) {
    unsigned p;
    asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n selp.u32 %0, 1, 0, q;\n}\n"
                 : "=r"(p) : "r"(a) : "memory");
    ok += p;
  }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) {
    unsigned p;
    asm volatile("{\n .reg .pred q;\n mbarrier.test_wait.parity.shared::cta.b64 q, [%1], 0;\n selp.u32 %0, 1, 0, q;\n}\n"
                 : "=r"(p) : "r"(a) : "memory");
    ok += p;
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = ok; }
}
int main2() {
  long long* cyc; cudaMallocManaged(&cyc, 4 * sizeof(long long));
  const int n = 4096;
  mbar_lat<<<1, 32>>>(cyc, n); mbar_lat<<<1, 32>>>(cyc, n); cudaDeviceSynchronize();
  printf("mbarrier try_wait (complete) latency: %.1f cycles\nmbarrier test_wait latency: %.1f cycles (ok=%lld)\n",
         (double)cyc[0] / n, (double)cyc[1] / n, cyc[2]);
  return 0;
}
