// admm_setup.cuh — one-time per-plan setup kernels (not on the per-iteration path).
//
// Replaces GramSolver construction (gram.hpp:48-53, inner_matrix 92-122) and
// CholeskyFactor::factor (cholesky.hpp:48-74):
//   A_b = rho I + H_b H_b^H               gram_kernel (FP64, lower tiles, mirrored)
//   K_b = A_b^-1                          Gauss-Jordan sweep without pivoting (A_b is
//                                         Hermitian positive definite); its pivots are
//                                         the Cholesky pivots d_j, so pivot <= 0 maps to
//                                         SingularityError exactly as cholesky.hpp:60-64.
// The reference factors I + H H^H / rho = A_b / rho; K_b therefore equals the
// reference's (rho * A_ref)^-1 and u = c + H^H K_b (g - H c).
#pragma once

#include "admm_common.cuh"

namespace admm {

struct GramDesc {
  uint64_t h_off;   // block in the H storage arena
  uint64_t a_off;   // dense FP64 m x m work matrix in the A arena
  uint64_t k_off;   // K_b in the K storage arena
  uint32_t m, n, ld, ldk;
};

constexpr int kGT = 64;  // Gram output tile
constexpr int kGK = 16;  // Gram k-chunk

// A_b = rho I + H_b H_b^H (lower tiles computed, upper mirrored).  flag[0] |= 1
// when a non-finite entry appears (NumericalError, cholesky.hpp:52-54).
template <typename S>
__global__ void __launch_bounds__(256)
gram_kernel(const S* __restrict__ H, const GramDesc* __restrict__ gd, double2* __restrict__ Aar,
            double rho, unsigned* flag) {
  __shared__ double2 As[kGK][kGT + 1];
  __shared__ double2 Bs[kGK][kGT + 1];
  const GramDesc d = gd[blockIdx.z];
  const uint32_t tr = blockIdx.y, tc = blockIdx.x;
  if (tc > tr || tr * kGT >= d.m) return;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = make_double2(0.0, 0.0);
  const S* hb = H + d.h_off;
  for (uint32_t k0 = 0; k0 < d.n; k0 += kGK) {
    for (int e = threadIdx.x; e < kGT * kGK; e += 256) {
      const int r = e / kGK, kk = e % kGK;
      const uint32_t col = k0 + kk;
      const uint32_t ra = tr * kGT + r, rb = tc * kGT + r;
      As[kk][r] = (ra < d.m && col < d.n) ? Store<S>::widen(hb[(uint64_t)ra * d.ld + col]) : make_double2(0.0, 0.0);
      Bs[kk][r] = (rb < d.m && col < d.n) ? Store<S>::widen(hb[(uint64_t)rb * d.ld + col]) : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kGK; ++kk) {
      double2 a[4], bb[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[kk][ty * 4 + q];
        bb[q] = Bs[kk][tx * 4 + q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w) {  // acc += a * conj(b)
          acc[q][w].x = fma(a[q].x, bb[w].x, acc[q][w].x);
          acc[q][w].x = fma(a[q].y, bb[w].y, acc[q][w].x);
          acc[q][w].y = fma(a[q].y, bb[w].x, acc[q][w].y);
          acc[q][w].y = fma(-a[q].x, bb[w].y, acc[q][w].y);
        }
    }
    __syncthreads();
  }
  bool bad = false;
  double2* A = Aar + d.a_off;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t r = tr * kGT + ty * 4 + q, c = tc * kGT + tx * 4 + w;
      if (r < d.m && c < d.m && c <= r) {
        double2 v = acc[q][w];
        if (r == c) v.x += rho;
        bad |= !cfinite(v);
        A[(uint64_t)r * d.m + c] = v;
        A[(uint64_t)c * d.m + r] = make_double2(v.x, -v.y);
      }
    }
  if (bad) atomicOr(flag, 1u);
}

// Gauss-Jordan step k, phase 1: save row k / column k of every block with m > k
// and test the pivot (flag bit 2 = SingularityError).
__global__ void gj_save_kernel(const double2* __restrict__ Aar, const GramDesc* __restrict__ gd,
                               double2* rowk, double2* colk, uint32_t maxm, uint32_t k,
                               unsigned* flag) {
  const GramDesc d = gd[blockIdx.y];
  if (k >= d.m) return;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const double2* A = Aar + d.a_off;
  if (t < d.m) {
    rowk[(uint64_t)blockIdx.y * maxm + t] = A[(uint64_t)k * d.m + t];
    colk[(uint64_t)blockIdx.y * maxm + t] = A[(uint64_t)t * d.m + k];
  }
  if (t == 0) {
    const double p = A[(uint64_t)k * d.m + k].x;
    if (!(p > 0.0) || !isfinite(p)) atomicOr(flag, 2u);
  }
}

// Gauss-Jordan step k, phase 2 (in place, no pivoting):
//   A_kk = 1/p, A_kj = a_kj / p, A_ik = -a_ik / p, A_ij -= a_ik a_kj / p.
__global__ void gj_update_kernel(double2* __restrict__ Aar, const GramDesc* __restrict__ gd,
                                 const double2* __restrict__ rowk, const double2* __restrict__ colk,
                                 uint32_t maxm, uint32_t k) {
  const GramDesc d = gd[blockIdx.z];
  if (k >= d.m) return;
  const uint32_t i = blockIdx.y;
  if (i >= d.m) return;
  const double2* rk = rowk + (uint64_t)blockIdx.z * maxm;
  const double pinv = 1.0 / rk[k].x;
  const double2 ci = colk[(uint64_t)blockIdx.z * maxm + i];
  double2* A = Aar + d.a_off + (uint64_t)i * d.m;
  for (uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x; jj < d.m; jj += gridDim.x * blockDim.x) {
    double2 v;
    if (i == k && jj == k) {
      v = make_double2(pinv, 0.0);
    } else if (i == k) {
      v = cscale(rk[jj], pinv);
    } else if (jj == k) {
      v = cscale(ci, -pinv);
    } else {
      const double2 f = cscale(rk[jj], pinv);
      v = A[jj];
      v.x -= ci.x * f.x - ci.y * f.y;
      v.y -= ci.x * f.y + ci.y * f.x;
    }
    A[jj] = v;
  }
}

// K_b (storage S, leading dimension ldk) = A_b (FP64).  flag bit 1 on non-finite.
template <typename S>
__global__ void k_store_kernel(const double2* __restrict__ Aar, const GramDesc* __restrict__ gd,
                               S* __restrict__ K, unsigned* flag) {
  const GramDesc d = gd[blockIdx.z];
  const uint32_t i = blockIdx.y;
  if (i >= d.m) return;
  bool bad = false;
  for (uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x; jj < d.m; jj += gridDim.x * blockDim.x) {
    const double2 v = Aar[d.a_off + (uint64_t)i * d.m + jj];
    bad |= !cfinite(v);
    K[d.k_off + (uint64_t)i * d.ldk + jj] = Store<S>::narrow(v);
  }
  if (bad) atomicOr(flag, 1u);
}

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
