// Microbenchmark: FP64 complex multiply-accumulate throughput from registers, in DFMA
// lanes per clock per SM, for the operand patterns of the GEMV / sweep / K-apply kernels.
//   mode 0: cmac as written in admm_common.cuh (x: ax*bx, -ay*by; y: ax*by, ay*bx), 8 rows x 2 columns
//   mode 1: the same products ordered so consecutive DFMAs share an operand
//   mode 2: plain independent FMA chains with one shared multiplier (the fp_peak pattern)
#include <cstdio>
#include <cuda_runtime.h>
struct c2 { double x, y; };
template <int MODE>
__global__ void loop(double* out, int iters, double s) {
  c2 h[8][2], x[2], acc[8];
  for (int k = 0; k < 8; ++k) {
    acc[k] = {0.0, 0.0};
    for (int e = 0; e < 2; ++e) h[k][e] = {s + threadIdx.x * 1e-3 + k, s - e - k * 0.5};
  }
  x[0] = {s, -s}; x[1] = {0.5 * s, 2.0 * s};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const c2 a = h[k][e], b = x[e];
        if (MODE == 0) {
          acc[k].x = fma(a.x, b.x, acc[k].x); acc[k].x = fma(-a.y, b.y, acc[k].x);
          acc[k].y = fma(a.x, b.y, acc[k].y); acc[k].y = fma(a.y, b.x, acc[k].y);
        } else if (MODE == 1) {
          acc[k].x = fma(a.x, b.x, acc[k].x); acc[k].y = fma(a.x, b.y, acc[k].y);
          acc[k].x = fma(-a.y, b.y, acc[k].x); acc[k].y = fma(a.y, b.x, acc[k].y);
        } else {
          acc[k].x = fma(acc[k].x, s, b.x); acc[k].y = fma(acc[k].y, s, b.y);
          acc[k].x = fma(acc[k].x, s, b.y); acc[k].y = fma(acc[k].y, s, b.x);
        }
      }
    // rotate the operands so nothing is loop-invariant
    const c2 t = x[0]; x[0] = x[1]; x[1] = {t.y, t.x};
#pragma unroll
    for (int k = 0; k < 8; ++k) { const c2 t2 = h[k][0]; h[k][0] = h[(k + 1) & 7][1]; h[(k + 1) & 7][1] = t2; }
  }
  double r = 0;
  for (int k = 0; k < 8; ++k) r += acc[k].x + acc[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE>
void run(const char* name, int warps_per_sm) {
  int sms, khz; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const int threads = 256, blocks = sms * warps_per_sm / 8, iters = 20000;
  double* out; cudaMalloc(&out, sizeof(double) * blocks * threads);
  loop<MODE><<<blocks, threads>>>(out, 16, 1.0000001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  loop<MODE><<<blocks, threads>>>(out, iters, 1.0000001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = 64.0 * iters * blocks * threads;
  printf("%-44s %2d warps/SM: %.1f DFMA lanes/clk/SM (max-clock basis)\n", name, warps_per_sm,
         dfma / (ms * 1e-3 * khz * 1e3 * sms));
  cudaFree(out);
}
int main() {
  for (int w : {8, 16, 32}) {
    run<0>("cmac (admm_common order)", w);
    run<1>("cmac (operand-sharing order)", w);
    run<2>("independent chains, shared multiplier", w);
  }
  return 0;
}
