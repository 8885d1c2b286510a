// Microbenchmark: the arithmetic of one packed-K tile (64 x 64 complex64, hemv_bulk_kernel's lane
// mapping: warp = 8 rows, lane = 2 columns) from a tile resident in SMEM -- no global traffic, no
// CTA barrier.  Cycles per tile per SM against the FP64-pipe bound (4096 elements x 8 DFMA / 58
// lanes/clk = 565 cycles) and the HBM time of a tile (32 KiB at 6.45 TB/s / 148 SMs = 1,440 cycles).
//   mode 0: as in the kernel (H part: 4 chains of 16 dependent DFMAs)
//   mode 1: H part in 8 chains (even / odd rows)
//   mode 2: N part only;  mode 3: H part only
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ void cmac_conj(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
}
// binary32 -> binary64 on the integer pipes (normal, non-zero values; zero maps to 2^-127-ish garbage)
__device__ __forceinline__ double widen_int(float f) {
  const unsigned u = __float_as_uint(f);
  const unsigned a = u & 0x7fffffffu;
  const unsigned hi = ((a >> 3) + 0x38000000u) | (u & 0x80000000u), lo = u << 29;
  return __hiloint2double((int)hi, (int)lo);
}
// WM: 0 F2F for both components, 1 integer widening for both, 2 F2F for re / integer for im
template <int WM>
__device__ __forceinline__ double2 widen2(float x, float y) {
  if (WM == 0) return make_double2((double)x, (double)y);
  if (WM == 1) return make_double2(widen_int(x), widen_int(y));
  return make_double2((double)x, widen_int(y));
}
template <int MODE, int WARPS, int WM = 0>
__global__ void __launch_bounds__(WARPS * 32, 1) loop(double* out, long long* cyc, int tiles, float seed) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* tile = reinterpret_cast<float2*>(sm);           // 2 tiles of 64 x 64
  double2* tiled = reinterpret_cast<double2*>(sm);       // WM == 3: the tiles as complex128
  double2* xs = reinterpret_cast<double2*>(sm + 2 * 65536);  // 128 entries
  if (WM == 3)
    for (int e = threadIdx.x; e < 2 * 4096; e += blockDim.x) tiled[e] = make_double2(seed + e * 1e-4, seed - e * 2e-4);
  else
    for (int e = threadIdx.x; e < 2 * 4096; e += blockDim.x) tile[e] = make_float2(seed + e * 1e-4f, seed - e * 2e-4f);
  for (int e = threadIdx.x; e < 128; e += blockDim.x) xs[e] = make_double2(1.0 + e * 1e-3, 0.5 - e * 1e-3);
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int RW = 64 / WARPS;  // rows per warp
  double2 accN[RW], xI[RW];
  for (int k = 0; k < RW; ++k) accN[k] = make_double2(0, 0), xI[k] = xs[64 + warp * RW + k];
  double2 hsum = make_double2(0, 0);
  const long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    const double2 xj0 = xs[(lane * 2 + t) & 63], xj1 = xs[(lane * 2 + 1 + t) & 63];
    const float2* ts = tile + (t & 1) * 4096 + (warp * RW) * 64 + lane * 2;
    double2 h[RW][2];
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      if (WM == 3) {
        const double2* td = tiled + (t & 1) * 4096 + (warp * RW + k) * 64 + lane * 2;
        h[k][0] = td[0];
        h[k][1] = td[1];
      } else {
        const float4 f = *reinterpret_cast<const float4*>(ts + k * 64);
        h[k][0] = widen2<WM>(f.x, f.y);
        h[k][1] = widen2<WM>(f.z, f.w);
      }
    }
    if (MODE != 3) {
#pragma unroll
      for (int k = 0; k < RW; ++k) { cmac(accN[k], h[k][0], xj0); cmac(accN[k], h[k][1], xj1); }
    }
    if (MODE != 2) {
      double2 a0 = make_double2(0, 0), a1 = a0, b0 = a0, b1 = a0;
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        if (MODE == 1 && (k & 1)) { cmac_conj(b0, h[k][0], xI[k]); cmac_conj(b1, h[k][1], xI[k]); }
        else { cmac_conj(a0, h[k][0], xI[k]); cmac_conj(a1, h[k][1], xI[k]); }
      }
      hsum.x += a0.x + a1.x + b0.x + b1.x; hsum.y += a0.y + a1.y + b0.y + b1.y;
    }
  }
  const long long t1 = clock64();
  double r = hsum.x + hsum.y;
  for (int k = 0; k < RW; ++k) r += accN[k].x + accN[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE, int WARPS, int WM = 0>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc; cudaMalloc(&out, sizeof(double) * sms * WARPS * 32); cudaMalloc(&cyc, sizeof(long long) * sms);
  const size_t smem = 2 * 65536 + 128 * 16;
  cudaFuncSetAttribute(loop<MODE, WARPS, WM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = 4000;
  loop<MODE, WARPS, WM><<<sms, WARPS * 32, smem>>>(out, cyc, 16, 1.5f);
  loop<MODE, WARPS, WM><<<sms, WARPS * 32, smem>>>(out, cyc, tiles, 1.5f);
  long long c0 = 0; cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  printf("%-52s %2d warps: %7.0f cycles per tile\n", name, WARPS, (double)c0 / tiles);
  cudaFree(out); cudaFree(cyc);
}

// Software-pipelined variant: the raw rows of tile t + 1 are loaded (LDS.128) before the arithmetic of
// tile t, so the SMEM read latency / bandwidth phase of a warp overlaps its own FP64 phase.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) loop_pipe(double* out, long long* cyc, int tiles, float seed) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* tile = reinterpret_cast<float2*>(sm);
  double2* xs = reinterpret_cast<double2*>(sm + 2 * 65536);
  for (int e = threadIdx.x; e < 2 * 4096; e += blockDim.x) tile[e] = make_float2(seed + e * 1e-4f, seed - e * 2e-4f);
  for (int e = threadIdx.x; e < 128; e += blockDim.x) xs[e] = make_double2(1.0 + e * 1e-3, 0.5 - e * 1e-3);
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int RW = 64 / WARPS;
  double2 accN[RW], xI[RW];
  for (int k = 0; k < RW; ++k) accN[k] = make_double2(0, 0), xI[k] = xs[64 + warp * RW + k];
  double2 hsum = make_double2(0, 0);
  float4 raw[RW], nxt[RW];
  {
    const float2* ts = tile + (warp * RW) * 64 + lane * 2;
#pragma unroll
    for (int k = 0; k < RW; ++k) raw[k] = *reinterpret_cast<const float4*>(ts + k * 64);
  }
  const long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    const double2 xj0 = xs[(lane * 2 + t) & 63], xj1 = xs[(lane * 2 + 1 + t) & 63];
    const float2* tn = tile + ((t + 1) & 1) * 4096 + (warp * RW) * 64 + lane * 2;
#pragma unroll
    for (int k = 0; k < RW; ++k) nxt[k] = *reinterpret_cast<const float4*>(tn + k * 64);
    double2 a0 = make_double2(0, 0), a1 = a0;
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const double2 h0 = make_double2(raw[k].x, raw[k].y), h1 = make_double2(raw[k].z, raw[k].w);
      cmac(accN[k], h0, xj0);
      cmac(accN[k], h1, xj1);
      cmac_conj(a0, h0, xI[k]);
      cmac_conj(a1, h1, xI[k]);
    }
    hsum.x += a0.x + a1.x; hsum.y += a0.y + a1.y;
#pragma unroll
    for (int k = 0; k < RW; ++k) raw[k] = nxt[k];
  }
  const long long t1 = clock64();
  double r = hsum.x + hsum.y;
  for (int k = 0; k < RW; ++k) r += accN[k].x + accN[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int WARPS>
void run_pipe(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc; cudaMalloc(&out, sizeof(double) * sms * WARPS * 32); cudaMalloc(&cyc, sizeof(long long) * sms);
  const size_t smem = 2 * 65536 + 128 * 16;
  cudaFuncSetAttribute(loop_pipe<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = 4000;
  loop_pipe<WARPS><<<sms, WARPS * 32, smem>>>(out, cyc, 16, 1.5f);
  loop_pipe<WARPS><<<sms, WARPS * 32, smem>>>(out, cyc, tiles, 1.5f);
  long long c0 = 0; cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  printf("%-52s %2d warps: %7.0f cycles per tile\n", name, WARPS, (double)c0 / tiles);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run_pipe<8>("N + H parts, next tile's rows loaded ahead");
  run_pipe<16>("N + H parts, next tile's rows loaded ahead");
  run<0, 8>("N + H parts as in hemv_bulk_kernel");
  run<1, 8>("N + H parts, H in 8 chains");
  run<2, 8>("N part only");
  run<3, 8>("H part only");
  run<0, 16>("N + H parts as in the kernel, 4 rows per warp");
  run<1, 16>("N + H parts, H in 8 chains, 4 rows per warp");
  run<0, 8, 1>("N + H parts, integer widening");
  run<0, 8, 2>("N + H parts, re by F2F / im by integer widening");
  run<2, 8, 1>("N part only, integer widening");
  run<2, 8, 2>("N part only, half F2F / half integer");
  run<1, 8, 2>("N + H (8 chains), half F2F / half integer");
  run<2, 8, 3>("N part only, tile stored as complex128 (no widening)");
  run<0, 8, 3>("N + H parts, tile stored as complex128 (no widening)");
  run<0, 4>("N + H parts, 16 rows per warp");
  run<1, 4>("N + H parts, H in 8 chains, 16 rows per warp");
  return 0;
}
