// admm_setup.cuh — one-time per-plan setup kernels (not on the per-iteration path).
//
// Upload conversions, scaling (problem.hpp:59-66) and finiteness scans.  The Gram matrix
// and its inverse (gram.hpp:48-53,92-122; cholesky.hpp:48-74) are in admm_factor.cuh.
// The reference factors I + H H^H / rho = A_b / rho; K_b = (rho I + H_b H_b^H)^-1 therefore
// equals the reference's (rho * A_ref)^-1 and u = c + H^H K_b (g - H c).
#pragma once

#include "admm_common.cuh"
#include "admm_factor.cuh"

namespace admm {

// dst (storage S, row pitch ld) = scl * src (FP64 rows, pitch spitch), rows x cols.
template <typename S>
__global__ void narrow_rows_kernel(const double2* __restrict__ src, uint64_t spitch, S* __restrict__ dst,
                                   uint64_t ld, uint32_t rows, uint32_t cols, double scl) {
  const uint32_t r = blockIdx.y;
  if (r >= rows) return;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x)
    dst[(uint64_t)r * ld + c] = Store<S>::narrow(cscale(src[(uint64_t)r * spitch + c], scl));
}

// complex64 rows staged on the device -> storage S (scaled in FP64 first, as above).
template <typename S>
__global__ void widen_rows_kernel(const float2* __restrict__ src, uint64_t spitch, S* __restrict__ dst,
                                  uint64_t ld, uint32_t rows, uint32_t cols, double scl) {
  const uint32_t r = blockIdx.y;
  if (r >= rows) return;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x)
    dst[(uint64_t)r * ld + c] = Store<S>::narrow(cscale(Store<float2>::widen(src[(uint64_t)r * spitch + c]), scl));
}

// In-place scaling of a storage arena: p[i] *= scl (problem.hpp:59-66).
template <typename S>
__global__ void scale_kernel(S* __restrict__ p, uint64_t n, double scl) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    const double2 v = cscale(Store<S>::widen(p[t]), scl);
    p[t] = Store<S>::narrow(v);
  }
}

__global__ void scale_vec_kernel(double2* __restrict__ p, uint64_t n, double scl) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    p[t] = cscale(p[t], scl);
}

// flag |= 1 if any entry is non-finite.
template <typename S>
__global__ void finite_kernel(const S* __restrict__ p, uint64_t n, unsigned* flag) {
  bool bad = false;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    bad |= !cfinite(Store<S>::widen(p[t]));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

}  // namespace admm
