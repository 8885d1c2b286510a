// Microbenchmark: binary32 -> binary64 widening throughput (F2F.F64.F32 on the XU pipe vs
// an integer-pipe re-bias) next to DFMA, in lane-operations per clock per SM.  Decides how
// the complex64 kernels widen H.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double widen_int(uint32_t f) {
  const uint32_t s = f & 0x80000000u, a = f ^ s;
  const uint32_t hi = (a >> 3) + 0x38000000u + s, lo = a << 29;
  return __hiloint2double((int)hi, (int)lo);
}
// mode 0: F2F + DFMA (1:2, the ratio of a complex64 GEMV); 1: integer widening + DFMA; 2: DFMA only; 3: F2F only;
// 4: half the values by F2F, half by the integer re-bias, + DFMA (1:2); 5: as 0 with DFMA 1:4 (the packed-K apply's
// ratio: every element feeds the N part and the H part); 6: as 4 with DFMA 1:4
template <int MODE>
__global__ void loop(double* out, int iters, float seed) {
  float f0 = seed + threadIdx.x, f1 = f0 + 1.f, f2 = f0 + 2.f, f3 = f0 + 3.f;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
  double b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0, b5 = 0, b6 = 0, b7 = 0;
  const double q = 1.0000001, r = 0.999999;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double d0, d1, d2, d3;
      if (MODE == 0 || MODE == 3 || MODE == 5) { d0 = (double)f0; d1 = (double)f1; d2 = (double)f2; d3 = (double)f3; }
      else if (MODE == 4 || MODE == 6) { d0 = (double)f0; d1 = widen_int(__float_as_uint(f1)); d2 = (double)f2; d3 = widen_int(__float_as_uint(f3)); }
      else if (MODE == 1) { d0 = widen_int(__float_as_uint(f0)); d1 = widen_int(__float_as_uint(f1)); d2 = widen_int(__float_as_uint(f2)); d3 = widen_int(__float_as_uint(f3)); }
      else { d0 = a0; d1 = a1; d2 = a2; d3 = a3; }
      if (MODE != 3) {
        a0 = fma(d0, q, a0); a1 = fma(d1, q, a1); a2 = fma(d2, q, a2); a3 = fma(d3, q, a3);
        a4 = fma(d0, r, a4); a5 = fma(d1, r, a5); a6 = fma(d2, r, a6); a7 = fma(d3, r, a7);
        if (MODE == 5 || MODE == 6) {
          b0 = fma(d0, r, b0); b1 = fma(d1, r, b1); b2 = fma(d2, q, b2); b3 = fma(d3, q, b3);
          b4 = fma(d0, q, b4); b5 = fma(d1, q, b5); b6 = fma(d2, r, b6); b7 = fma(d3, r, b7);
        }
      } else { a0 += d0; a1 += d1; a2 += d2; a3 += d3; }
      // keep the floats changing with FP32-pipe work (not measured pipes)
      f0 += 1.0f; f1 += 2.0f; f2 += 3.0f; f3 += 5.0f;  // loop-carried: no two conversions share a value
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + b0 + b1 + b2 + b3 + b4 + b5 + b6 + b7;
}
template <int MODE>
void run(const char* name, double cvt_per_iter, double fma_per_iter) {
  int sms, khz; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  loop<MODE><<<blocks, threads>>>(out, 16, 1.5f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  loop<MODE><<<blocks, threads>>>(out, iters, 1.5f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double lanes = (double)iters * 8 * blocks * threads;
  const double clk = ms * 1e-3 * khz * 1e3 * sms;  // at the nominal max clock
  printf("%-28s %.3f ms  widen %.1f lanes/clk/SM  dfma %.1f lanes/clk/SM (max-clock basis)\n", name, ms,
         lanes * cvt_per_iter / clk, lanes * fma_per_iter / clk);
  cudaFree(out);
}
int main() {
  run<2>("DFMA only", 0, 8);
  run<3>("F2F.F64.F32 (+DADD)", 4, 4);
  run<0>("F2F + DFMA (1:2)", 4, 8);
  run<1>("integer widen + DFMA (1:2)", 4, 8);
  run<4>("half F2F half int + DFMA (1:2)", 4, 8);
  run<5>("F2F + DFMA (1:4)", 4, 16);
  run<6>("half F2F half int + DFMA (1:4)", 4, 16);
  // exactness of the integer widening on normal floats
  return 0;
}
