// admm_common.cuh — shared device helpers for the B200 ADMM engine (sm_100a).
//
// Complex data are interleaved (re, im).  Storage of H and of the Woodbury
// inverse K is either complex128 (double2) or complex64 (float2); all arithmetic
// and every vector iterate is FP64 (double2) regardless of storage, so the c64
// path only rounds the two streamed matrices.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace admm {

constexpr int kWarp = 32;
constexpr int kCtaThreads = 256;  // 8 warps per CTA for every streaming kernel
constexpr int kCtaWarps = kCtaThreads / kWarp;

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += a * b
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cmac_conj(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }

// prox.hpp:15-19: |a| > kappa ? a (1 - kappa/|a|) : 0, with |a| = hypot.
// Same result as soft_threshold, with a short path for |a| clearly below kappa (most
// entries of a sparse iterate): |a|^2 < kappa^2 (1 - 2^-40) guarantees hypot(a) < kappa
// (both are within a few ulp), so hypot and the division are skipped.  kappa2_lo =
// kappa * kappa * (1 - 2^-40), precomputed.  NaN / overflow fall through to the full test.
__device__ __forceinline__ double2 soft_threshold_fast(double2 a, double kappa, double kappa2_lo) {
  const double r2 = a.x * a.x + a.y * a.y;
  if (r2 < kappa2_lo) return make_double2(0.0, 0.0);
  const double mag = hypot(a.x, a.y);
  if (mag > kappa) {
    const double f = 1.0 - kappa / mag;
    return make_double2(a.x * f, a.y * f);
  }
  return make_double2(0.0, 0.0);
}

// Latency-optimised variant for the slab sweep's D warps (4 active lanes, the result gates the
// next (A) pass): |a|^2 clearly above kappa^2 and inside the range where x^2 + y^2 neither
// overflows nor loses bits takes  a (1 - kappa rsqrt(|a|^2))  -- one rsqrt (MUFU.RSQ64H + Newton)
// instead of hypot and a division, equal to the reference expression to ~2 ulp (the soft
// threshold is continuous, so an ulp near |a| = kappa cannot flip anything that matters).
// Everything else (near the threshold, huge / tiny / non-finite) takes the exact path.
__device__ __forceinline__ double2 soft_threshold_lat(double2 a, double kappa, double kappa2_lo, double kappa2_hi) {
  const double r2 = a.x * a.x + a.y * a.y;
  if (r2 < kappa2_lo) return make_double2(0.0, 0.0);
  if (r2 > kappa2_hi && r2 > 1e-280 && r2 < 1e280) {
    const double f = fma(-kappa, rsqrt(r2), 1.0);
    return make_double2(a.x * f, a.y * f);
  }
  const double mag = hypot(a.x, a.y);
  if (mag > kappa) {
    const double f = 1.0 - kappa / mag;
    return make_double2(a.x * f, a.y * f);
  }
  return make_double2(0.0, 0.0);
}

__device__ __forceinline__ double2 soft_threshold(double2 a, double kappa) {
  const double mag = hypot(a.x, a.y);
  if (mag > kappa) {
    const double f = 1.0 - kappa / mag;
    return make_double2(a.x * f, a.y * f);
  }
  return make_double2(0.0, 0.0);
}

// ---- streaming loads of the matrix operand (read once per pass) -------------
// 256-bit LDG with L1 no-allocate and an L2 eviction priority:
//   kEvictNormal (default), kEvictFirst (stream through: the line is dead after this
//   read), kEvictLast (the line will be re-read soon — the fused sweep's second pass).
struct V256 {
  uint64_t w[4];
};
enum L2Hint { kEvictNormal = 0, kEvictFirst = 1, kEvictLast = 2 };
template <int Hint>
__device__ __forceinline__ V256 ld_stream256(const void* p) {
  V256 r;
  if constexpr (Hint == kEvictFirst) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r.w[0]), "=l"(r.w[1]), "=l"(r.w[2]), "=l"(r.w[3])
                 : "l"(p));
  } else if constexpr (Hint == kEvictLast) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r.w[0]), "=l"(r.w[1]), "=l"(r.w[2]), "=l"(r.w[3])
                 : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r.w[0]), "=l"(r.w[1]), "=l"(r.w[2]), "=l"(r.w[3])
                 : "l"(p));
  }
  return r;
}

// Storage traits: how many complex elements one 32-byte vector carries and how
// to widen them to FP64.
template <typename S>
struct Store;
template <>
struct Store<double2> {
  static constexpr int kPerVec = 2;  // 2 x 16 B
  __device__ __forceinline__ static double2 get(const V256& v, int e) {
    return make_double2(__longlong_as_double((long long)v.w[2 * e]),
                        __longlong_as_double((long long)v.w[2 * e + 1]));
  }
  __device__ __forceinline__ static double2 widen(double2 a) { return a; }
  __device__ __forceinline__ static double2 narrow(double2 a) { return a; }
};
template <>
struct Store<float2> {
  static constexpr int kPerVec = 4;  // 4 x 8 B
  __device__ __forceinline__ static double2 get(const V256& v, int e) {
    const uint64_t w = v.w[e];
    return make_double2((double)__uint_as_float((unsigned)(w & 0xffffffffu)),
                        (double)__uint_as_float((unsigned)(w >> 32)));
  }
  __device__ __forceinline__ static double2 widen(float2 a) { return make_double2(a.x, a.y); }
  __device__ __forceinline__ static float2 narrow(double2 a) {
    return make_float2((float)a.x, (float)a.y);
  }
};

// ---- stream-K work split ----------------------------------------------------
// Units [0, U) are split over P CTAs: CTA p owns [lo(p), lo(p+1)), lo(p) = p*U/P.
__host__ __device__ __forceinline__ uint64_t sk_lo(uint64_t p, uint64_t U, uint64_t P) {
  return (p * U) / P;
}
// The CTA that owns unit x.
__host__ __device__ __forceinline__ uint64_t sk_owner(uint64_t x, uint64_t U, uint64_t P) {
  return ((x + 1) * P - 1) / U;
}

// Warp index through a lane-0 broadcast.  ptxas cannot prove that threadIdx.x / 32 is the
// same in every lane, so a shuffle under a branch on it compiles to an out-of-line
// WARPSYNC.COLLECTIVE / ENDCOLLECTIVE sequence with fixed-register moves (about 7
// instructions per SHFL); the broadcast value is warp-uniform by construction, the role /
// tile branches move to the uniform datapath and the shuffles become bare SHFLs (slab sweep
// on config 3: 245 -> 169 us).  Call with all 32 lanes converged (kernel entry).
__device__ __forceinline__ int warp_index() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x / kWarp), 0); }

// ---- deterministic block reduction (fixed tree, no atomics) -----------------
template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double* smem) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = warp_index(), lane = threadIdx.x % kWarp;
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < kThreads / kWarp ? smem[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// cp.async helpers (size 8 or 16, zero-fill when src_bytes = 0)
__device__ __forceinline__ void cpa(void* smem, const void* src, bool ok) {
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cpa8(void* smem, const void* src, bool ok) {
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Index of the last descriptor with unit0 <= x (unit0 ascending, d[0].unit0 == 0) — the
// stream-K "which matrix does my first unit belong to" search.  The warp loads 32 unit0
// fields at once and takes the highest matching lane, instead of one dependent global load
// per step (7 serial L2 round trips for 8 blocks at every kernel start).  Warp-uniform:
// call with all 32 lanes.
template <typename D>
__device__ __forceinline__ int find_desc(const D* __restrict__ d, int n, uint64_t x) {
  const int lane = (int)(threadIdx.x % 32);
  int b = 0;
  for (int base = 0; base < n; base += 32) {
    const bool le = base + lane < n && d[base + lane].unit0 <= x;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    if (m) b = base + 31 - __clz(m);
    if (m != 0xffffffffu) break;
  }
  return b;
}

// Programmatic dependent launch: wait until the preceding grid in the stream has
// completed (its writes visible), then allow the next grid to be launched while this one
// runs.  A no-op when the launch carried no programmatic dependency.  Call first thing.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace admm
