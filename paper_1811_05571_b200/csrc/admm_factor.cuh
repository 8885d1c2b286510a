// admm_factor.cuh — the one dense contraction of the path, on the FP64 tensor cores.
//
// Replaces GramSolver::inner_matrix (gram.hpp:92-122) and CholeskyFactor::factor /
// solve (cholesky.hpp:24-74) for every block b:
//   A_b = rho I + H_b H_b^H        gram_dmma_kernel      (mma.sync m8n8k4 f64 = DMMA)
//   K_b = A_b^-1                   blocked Gauss-Jordan, panels of 64:
//        gj_diag_kernel    P = A_KK^-1 in shared memory (64 scalar pivots; they are the
//                          Cholesky pivots d_j of cholesky.hpp:56-64, so pivot <= 0 is the
//                          reference's SingularityError)
//        gj_panel_kernel   A_Kt <- P A_Kt (row panel, in place; its conjugate transpose to
//                          scratch), the old column panel A_tK copied to scratch
//        gj_update_kernel  A_ij <- A_ij - A_iK (P A_Kj)  and  A_iK <- -A_iK P: rank-64
//                          updates of every other tile, DMMA
// The work matrix of block b is padded to mp = 64 * ceil(m / 64) rows and columns with the
// identity, so no kernel masks: inv(blockdiag(A, I)) = blockdiag(A^-1, I).
//
// Complex products on a real tensor core: C = X Y^H with X = Xr + i Xi, Y = Yr + i Yi is
//   Cr = Xr Yr^T + Xi Yi^T,   Ci = Xi Yr^T - Xr Yi^T
// four real m8n8k4 products per 8 x 8 output tile and 4 complex k: one vector shared-memory
// load gives a lane both planes of its fragment element (re, im interleaved storage).
#pragma once

#include "admm_common.cuh"

namespace admm {

struct GramDesc {
  uint64_t h_off;   // block in the H storage arena
  uint64_t a_off;   // dense FP64 mp x mp work matrix in the A arena
  uint64_t k_off;   // K_b in the K storage arena
  uint32_t m, n, ld, ldk;
  uint32_t mp, pad_;  // padded dimension (multiple of 64) = leading dimension of the work matrix
};

constexpr int kFT = 64;            // output tile edge (complex)
constexpr int kFK = 16;            // k-chunk (complex columns) per pipeline stage
constexpr int kFLd = kFK + 4;      // shared row pitch: rows 64 B apart mod 128 -> conflict-free LDS.128
constexpr int kFThreads = 256;     // 8 warps: 4 (rows of 16) x 2 (columns of 32)
constexpr size_t kFStage = 2 * (size_t)kFT * kFLd * sizeof(double2);  // A and B tile of one stage

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Warp tile 16 x 32 of the 64 x 64 CTA tile: [mi][ni][e] = rows wr*16 + mi*8 + g,
// columns wc*32 + ni*8 + 2t + e (g = lane / 4, t = lane % 4).
struct FragAcc {
  double r[2][4][2];
  double i[2][4][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) r[a][b][0] = r[a][b][1] = i[a][b][0] = i[a][b][1] = 0.0;
  }
};

// acc += X Y^H over one staged chunk: Xs, Ys are [64][kFLd] double2 tiles (k contiguous).
__device__ __forceinline__ void dmma_chunk(const double2* __restrict__ Xs, const double2* __restrict__ Ys,
                                           FragAcc& c, int wr, int wc, int g, int t) {
#pragma unroll
  for (int kk = 0; kk < kFK; kk += 4) {
    double2 x[2], y[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) x[mi] = Xs[(wr * 16 + mi * 8 + g) * kFLd + kk + t];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) y[ni] = Ys[(wc * 32 + ni * 8 + g) * kFLd + kk + t];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        dmma(c.r[mi][ni], x[mi].x, y[ni].x);
        dmma(c.i[mi][ni], x[mi].y, y[ni].x);
      }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const double nyi = -y[ni].y;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        dmma(c.r[mi][ni], x[mi].y, y[ni].y);
        dmma(c.i[mi][ni], x[mi].x, nyi);
      }
    }
  }
}

// Stage one k-chunk of two 64-row operands (rows x0.., y0.. of a row-major matrix with k
// contiguous, leading dimension ld, kmax valid columns, rmax valid rows) as double2 tiles.
// complex128 storage: cp.async straight into the tile (zero-fill out of range).
// complex64 storage: 16-byte loads into registers (issue), widened once when stored (commit) —
// each element is converted once per CTA, not once per consuming warp.
template <typename S>
struct FStager;

template <>
struct FStager<double2> {
  __device__ __forceinline__ void issue(const double2* __restrict__ base, uint32_t ld, uint32_t x0, uint32_t y0,
                                        uint32_t rmax, uint32_t k0, uint32_t kmax, double2* Xs, double2* Ys) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + kFThreads * q, row = idx / kFK, col = idx % kFK;
      const bool kin = k0 + col < kmax;
      const bool okx = kin && x0 + row < rmax, oky = kin && y0 + row < rmax;
      cpa(Xs + row * kFLd + col, okx ? base + (uint64_t)(x0 + row) * ld + k0 + col : base, okx);
      cpa(Ys + row * kFLd + col, oky ? base + (uint64_t)(y0 + row) * ld + k0 + col : base, oky);
    }
    cpa_commit();
  }
  __device__ __forceinline__ void commit(double2*, double2*) { cpa_wait<0>(); }
};

template <>
struct FStager<float2> {
  float4 vx[2], vy[2];
  __device__ __forceinline__ void issue(const float2* __restrict__ base, uint32_t ld, uint32_t x0, uint32_t y0,
                                        uint32_t rmax, uint32_t k0, uint32_t kmax, double2*, double2*) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // 2 complex per 16-byte load; ld is a multiple of 8, pad zero
      const int idx = threadIdx.x + kFThreads * q, row = idx / (kFK / 2), col = (idx % (kFK / 2)) * 2;
      const bool kin = k0 + col < kmax;
      vx[q] = vy[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kin && x0 + row < rmax)
        vx[q] = __ldg(reinterpret_cast<const float4*>(base + (uint64_t)(x0 + row) * ld + k0 + col));
      if (kin && y0 + row < rmax)
        vy[q] = __ldg(reinterpret_cast<const float4*>(base + (uint64_t)(y0 + row) * ld + k0 + col));
    }
  }
  __device__ __forceinline__ void commit(double2* Xs, double2* Ys) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = threadIdx.x + kFThreads * q, row = idx / (kFK / 2), col = (idx % (kFK / 2)) * 2;
      Xs[row * kFLd + col] = make_double2(vx[q].x, vx[q].y);
      Xs[row * kFLd + col + 1] = make_double2(vx[q].z, vx[q].w);
      Ys[row * kFLd + col] = make_double2(vy[q].x, vy[q].y);
      Ys[row * kFLd + col + 1] = make_double2(vy[q].z, vy[q].w);
    }
  }
};

// acc = X Y^H over k in [0, kmax): X = rows x0.., Y = rows y0.. of `base`.  Double-buffered:
// chunk c + 1 is in flight (cp.async / registers) while chunk c is multiplied.
template <typename S>
__device__ __forceinline__ void dmma_tile(const S* __restrict__ base, uint32_t ld, uint32_t x0, uint32_t y0,
                                          uint32_t rmax, uint32_t kmax, double2* sm, FragAcc& acc) {
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int wr = warp >> 1, wc = warp & 1, g = lane >> 2, t = lane & 3;
  double2* Xs[2] = {sm, sm + 2 * kFT * kFLd};
  double2* Ys[2] = {sm + kFT * kFLd, sm + 3 * kFT * kFLd};
  FStager<S> st;
  st.issue(base, ld, x0, y0, rmax, 0, kmax, Xs[0], Ys[0]);
  st.commit(Xs[0], Ys[0]);
  __syncthreads();
  int s = 0;
  for (uint32_t k0 = 0; k0 < kmax; k0 += kFK, s ^= 1) {
    const bool more = k0 + kFK < kmax;
    if (more) st.issue(base, ld, x0, y0, rmax, k0 + kFK, kmax, Xs[s ^ 1], Ys[s ^ 1]);
    dmma_chunk(Xs[s], Ys[s], acc, wr, wc, g, t);
    if (more) st.commit(Xs[s ^ 1], Ys[s ^ 1]);
    __syncthreads();
  }
}

// Lower tile (I, J), I >= J, of unit u = I (I + 1) / 2 + J.
__device__ __forceinline__ void lower_tile(uint32_t u, uint32_t& I, uint32_t& J) {
  I = (uint32_t)((sqrt(8.0 * (double)u + 1.0) - 1.0) * 0.5);
  while ((uint64_t)(I + 1) * (I + 2) / 2 <= u) ++I;
  while ((uint64_t)I * (I + 1) / 2 > u) --I;
  J = u - I * (I + 1) / 2;
}

// A_b = rho I + H_b H_b^H for blocks b0 + blockIdx.y: one CTA per lower 64 x 64 tile, the
// upper triangle mirrored.  flag |= 1 on a non-finite entry (NumericalError, cholesky.hpp:52-54).
template <typename S>
__global__ void __launch_bounds__(kFThreads, 2)
gram_dmma_kernel(const S* __restrict__ H, const GramDesc* __restrict__ gd, uint32_t b0, double2* __restrict__ Aar,
                 double rho, unsigned* flag) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const GramDesc d = gd[b0 + blockIdx.y];
  uint32_t I, J;
  lower_tile(blockIdx.x, I, J);
  if (I * kFT >= d.mp) return;
  FragAcc acc;
  acc.zero();
  dmma_tile<S>(H + d.h_off, d.ld, I * kFT, J * kFT, d.m, d.n, reinterpret_cast<double2*>(fsm), acc);
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int wr = warp >> 1, wc = warp & 1, g = lane >> 2, t = lane & 3;
  double2* A = Aar + d.a_off;
  bool bad = false;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t r = I * kFT + wr * 16 + mi * 8 + g, c = J * kFT + wc * 32 + ni * 8 + 2 * t + e;
        if (c > r) continue;  // diagonal tiles: the lower half carries the values
        double2 v = make_double2(acc.r[mi][ni][e], acc.i[mi][ni][e]);
        if (r == c) v = make_double2(v.x + (r < d.m ? rho : 1.0), 0.0);
        bad |= !cfinite(v);
        A[(uint64_t)r * d.mp + c] = v;
        A[(uint64_t)c * d.mp + r] = make_double2(v.x, -v.y);
      }
  if (bad) atomicOr(flag, 1u);
}

// ---- blocked Gauss-Jordan inverse (in place, no pivoting: A is Hermitian positive definite)
// Scratch per block (mp_max = padded dimension of the largest block):
//   P  [64][64]   inverse of the current diagonal tile         PH [64][64] its conjugate transpose
//   WH [mp][64]   conjugate transpose of the new row panel P A_K,:
//   C  [mp][64]   the old column panel A_:,K
struct GjScratch {
  double2* P;
  double2* PH;
  double2* WH;
  double2* C;
  uint32_t mp_max;
  __device__ __forceinline__ double2* p(uint32_t b) const { return P + (uint64_t)b * kFT * kFT; }
  __device__ __forceinline__ double2* ph(uint32_t b) const { return PH + (uint64_t)b * kFT * kFT; }
  __device__ __forceinline__ double2* wh(uint32_t b) const { return WH + (uint64_t)b * mp_max * kFT; }
  __device__ __forceinline__ double2* c(uint32_t b) const { return C + (uint64_t)b * mp_max * kFT; }
};

// P = (A_KK)^-1 of panel kp, one CTA per block: 64 scalar Gauss-Jordan steps on the tile in
// shared memory (A_kk = 1/p, A_kj = a_kj / p, A_ik = -a_ik / p, A_ij -= a_ik a_kj / p).
// flag |= 2 when a pivot of a real (unpadded) row is not positive (SingularityError).
constexpr int kGjLd = kFT + 1;
constexpr size_t kGjDiagSmem = ((size_t)kFT * kGjLd + 2 * kFT) * sizeof(double2);
__global__ void __launch_bounds__(kFThreads)
gj_diag_kernel(double2* __restrict__ Aar, const GramDesc* __restrict__ gd, uint32_t kp, GjScratch sc, unsigned* flag) {
  extern __shared__ __align__(16) unsigned char fsm[];
  double2* D = reinterpret_cast<double2*>(fsm);
  double2* rowk = D + kFT * kGjLd;
  double2* colk = rowk + kFT;
  const GramDesc d = gd[blockIdx.x];
  if (kp * kFT >= d.mp) return;
  double2* A = Aar + d.a_off + (uint64_t)(kp * kFT) * d.mp + kp * kFT;
  for (int e = threadIdx.x; e < kFT * kFT; e += kFThreads) D[(e / kFT) * kGjLd + e % kFT] = A[(uint64_t)(e / kFT) * d.mp + e % kFT];
  __syncthreads();
  const int tj = threadIdx.x % kFT, ti0 = threadIdx.x / kFT;  // column tj, rows ti0 + 4 q
  for (int k = 0; k < kFT; ++k) {
    if (threadIdx.x < kFT) {
      rowk[threadIdx.x] = D[k * kGjLd + threadIdx.x];
      colk[threadIdx.x] = D[threadIdx.x * kGjLd + k];
    }
    __syncthreads();
    const double p = rowk[k].x;
    if (threadIdx.x == 0 && kp * kFT + k < d.m && (!(p > 0.0) || !isfinite(p))) atomicOr(flag, 2u);
    const double pinv = 1.0 / p;
    const double2 f = cscale(rowk[tj], pinv);
#pragma unroll 4
    for (int i = ti0; i < kFT; i += kFThreads / kFT) {
      double2 v;
      if (i == k) {
        v = tj == k ? make_double2(pinv, 0.0) : f;
      } else {
        const double2 ci = colk[i];
        if (tj == k) {
          v = cscale(ci, -pinv);
        } else {
          v = D[i * kGjLd + tj];
          v.x -= ci.x * f.x - ci.y * f.y;
          v.y -= ci.x * f.y + ci.y * f.x;
        }
      }
      D[i * kGjLd + tj] = v;
    }
    __syncthreads();
  }
  double2* P = sc.p(blockIdx.x);
  double2* PH = sc.ph(blockIdx.x);
  for (int e = threadIdx.x; e < kFT * kFT; e += kFThreads) {
    const int r = e / kFT, c = e % kFT;
    const double2 v = D[r * kGjLd + c];
    P[e] = v;
    A[(uint64_t)r * d.mp + c] = v;
    const double2 w = D[c * kGjLd + r];
    PH[e] = make_double2(w.x, -w.y);
  }
}

// Row panel of step kp, tile t != kp (grid: tiles x blocks): W = P A_Kt written in place and
// as W^H to scratch; the old column-panel tile A_tK copied to scratch.
constexpr size_t kGjPanelSmem = 2 * (size_t)kFT * kGjLd * sizeof(double2);
__global__ void __launch_bounds__(kFThreads)
gj_panel_kernel(double2* __restrict__ Aar, const GramDesc* __restrict__ gd, uint32_t kp, GjScratch sc) {
  extern __shared__ __align__(16) unsigned char fsm[];
  double2* Ps = reinterpret_cast<double2*>(fsm);
  double2* Ts = Ps + kFT * kGjLd;
  const GramDesc d = gd[blockIdx.y];
  const uint32_t t = blockIdx.x;
  if (kp * kFT >= d.mp || t * kFT >= d.mp || t == kp) return;
  double2* Arow = Aar + d.a_off + (uint64_t)(kp * kFT) * d.mp + t * kFT;  // A_Kt
  double2* Acol = Aar + d.a_off + (uint64_t)(t * kFT) * d.mp + kp * kFT;  // A_tK
  const double2* P = sc.p(blockIdx.y);
  double2* C = sc.c(blockIdx.y) + (uint64_t)t * kFT * kFT;
  double2* WH = sc.wh(blockIdx.y) + (uint64_t)t * kFT * kFT;
  for (int e = threadIdx.x; e < kFT * kFT; e += kFThreads) {
    const int r = e / kFT, c = e % kFT;
    Ps[r * kGjLd + c] = P[e];
    Ts[r * kGjLd + c] = Arow[(uint64_t)r * d.mp + c];
    C[e] = Acol[(uint64_t)r * d.mp + c];
  }
  __syncthreads();
  // thread: rows 4 ty .. +3, columns tx + 16 w (w = 0..3)
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
#pragma unroll 4
  for (int l = 0; l < kFT; ++l) {
    double2 pv[4], tv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) pv[a] = Ps[(ty * 4 + a) * kGjLd + l];
#pragma unroll
    for (int b = 0; b < 4; ++b) tv[b] = Ts[l * kGjLd + tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) cmac(acc[a][b], pv[a], tv[b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty * 4 + a, c = tx + 16 * b;
      Arow[(uint64_t)r * d.mp + c] = acc[a][b];
      WH[c * kFT + r] = make_double2(acc[a][b].x, -acc[a][b].y);
    }
}

// Step kp on every tile (i, j), i != kp (grid: tiles x tiles x blocks):
//   j != kp:  A_ij <- A_ij - C_i W_j          (C_i W_j = C_i (W_j^H)^H)
//   j == kp:  A_iK <- -C_i P                  (= -C_i (P^H)^H)
__global__ void __launch_bounds__(kFThreads, 2)
gj_update_kernel(double2* __restrict__ Aar, const GramDesc* __restrict__ gd, uint32_t kp, GjScratch sc) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const GramDesc d = gd[blockIdx.z];
  const uint32_t i = blockIdx.y, j = blockIdx.x;
  if (kp * kFT >= d.mp || i * kFT >= d.mp || j * kFT >= d.mp || i == kp) return;
  // one operand array: rows [0, mp) = C, rows [mp_max, mp_max + mp) = W^H live in separate
  // buffers, so the two 64-row operands are staged from their own bases
  const double2* X = sc.c(blockIdx.z) + (uint64_t)i * kFT * kFT;
  const double2* Y = j == kp ? sc.ph(blockIdx.z) : sc.wh(blockIdx.z) + (uint64_t)j * kFT * kFT;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int wr = warp >> 1, wc = warp & 1, g = lane >> 2, t = lane & 3;
  double2* sm = reinterpret_cast<double2*>(fsm);
  double2* Xs[2] = {sm, sm + 2 * kFT * kFLd};
  double2* Ys[2] = {sm + kFT * kFLd, sm + 3 * kFT * kFLd};
  auto issue = [&](int s, uint32_t k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + kFThreads * q, row = idx / kFK, col = idx % kFK;
      cpa(Xs[s] + row * kFLd + col, X + row * kFT + k0 + col, true);
      cpa(Ys[s] + row * kFLd + col, Y + row * kFT + k0 + col, true);
    }
    cpa_commit();
  };
  FragAcc acc;
  acc.zero();
  issue(0, 0);
  cpa_wait<0>();
  __syncthreads();
  int s = 0;
#pragma unroll
  for (uint32_t k0 = 0; k0 < kFT; k0 += kFK, s ^= 1) {
    const bool more = k0 + kFK < kFT;
    if (more) issue(s ^ 1, k0 + kFK);
    dmma_chunk(Xs[s], Ys[s], acc, wr, wc, g, t);
    if (more) cpa_wait<0>();
    __syncthreads();
  }
  double2* A = Aar + d.a_off + (uint64_t)(i * kFT) * d.mp + j * kFT;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const uint32_t r = wr * 16 + mi * 8 + g, c = wc * 32 + ni * 8 + 2 * t;
      double2* a = A + (uint64_t)r * d.mp + c;
      double2 v0, v1;
      if (j == kp) {
        v0 = make_double2(-acc.r[mi][ni][0], -acc.i[mi][ni][0]);
        v1 = make_double2(-acc.r[mi][ni][1], -acc.i[mi][ni][1]);
      } else {
        v0 = a[0];
        v1 = a[1];
        v0.x -= acc.r[mi][ni][0];
        v0.y -= acc.i[mi][ni][0];
        v1.x -= acc.r[mi][ni][1];
        v1.y -= acc.i[mi][ni][1];
      }
      a[0] = v0;
      a[1] = v1;
    }
}

// K_b (storage S, leading dimension ldk) = A_b (FP64, leading dimension mp).  flag bit 1 on
// a non-finite entry.
template <typename S>
__global__ void k_store_kernel(const double2* __restrict__ Aar, const GramDesc* __restrict__ gd,
                               S* __restrict__ K, unsigned* flag) {
  const GramDesc d = gd[blockIdx.z];
  const uint32_t i = blockIdx.y;
  if (i >= d.m) return;
  bool bad = false;
  for (uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x; jj < d.m; jj += gridDim.x * blockDim.x) {
    const double2 v = Aar[d.a_off + (uint64_t)i * d.mp + jj];
    bad |= !cfinite(v);
    K[d.k_off + (uint64_t)i * d.ldk + jj] = Store<S>::narrow(v);
  }
  if (bad) atomicOr(flag, 1u);
}

}  // namespace admm
