// admm_hemv.cuh — q_b = K_b r_b with K_b = (rho I + H_b H_b^H)^-1 Hermitian, streamed
// from a packed lower triangle: half the bytes of the dense K per iteration.
//
// Packed layout per block: 64 x 64 tiles (I, J), I >= J, in row-major tile order
// (unit u = I (I + 1) / 2 + J), each tile row-major; rows/columns past m are zero.  The
// diagonal tiles are stored full.  A tile (I, J), I > J, contributes
//     N part:  y_I += K_IJ r_J            (rows of the tile)
//     H part:  y_J += K_IJ^H r_I          (columns of the tile)
// and a diagonal tile only its N part.  Tiles are split stream-K over a persistent grid.
// Each warp owns 8 rows of a tile, each lane 2 columns (one 32-byte / 16-byte load per
// row): N partials stay in registers along a tile row and are reduced once per tile-row
// segment; H partials are reduced over the 8 warps through SMEM once per tile.  Both go
// to a partial buffer that hemv_finalize_kernel sums in a fixed order (no atomics).
// Numerics: K_IJ (lower) stands for both triangles — the inverse is Hermitian up to
// rounding (~1e-16 relative).
#pragma once

#include "admm_kernels.cuh"
#include "admm_slab.cuh"  // mbarrier / bulk-copy helpers

namespace admm {

constexpr int kHT = 64;                 // tile edge
constexpr int kHRows = kHT / kCtaWarps;  // rows per warp (8)

struct HemvDesc {       // one per local block
  uint64_t k_off;       // element offset of the block's packed tiles
  uint64_t unit0;       // first global unit (tile) of the block
  uint64_t part_off;    // double2 offset of the block's partials: N [n_units][64], H [n_units][64]
  uint32_t m;           // rows (= columns)
  uint32_t nT;          // tile rows
  uint32_t x_off;       // offset of r / q / ghat / gij (the block's mvec_off)
  uint32_t n_units;     // nT (nT + 1) / 2
  uint32_t cnt_off;     // first of the block's nT tile-row completion counters
  uint32_t pad_;
};

// (K r)[row] from the partials of row r of tile-row I: the N segments in CTA order, then
// the H parts of the tiles below the diagonal in ascending tile-row order.  Loads are
// issued 8 at a time (independent) and added in that fixed order; L1 bypassed (the
// partials come from other SMs).
__device__ __forceinline__ double2 hemv_sum_row(const double2* __restrict__ part, const HemvDesc& d, uint32_t I,
                                                uint32_t r, uint64_t U, uint64_t P) {
  const uint32_t urow = I * (I + 1) / 2;
  const uint32_t nseg = seg_count(d.unit0 + urow, I + 1, U, P);
  const uint32_t nh = d.nT - 1 - I;
  const double2* np = part + d.part_off + (uint64_t)urow * kHT + r;
  const double2* hp = part + d.part_off + (uint64_t)d.n_units * kHT + r;
  const uint32_t n = nseg + nh;
  double2 s = make_double2(0.0, 0.0);
  for (uint32_t k0 = 0; k0 < n; k0 += 8) {
    double2 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t k = k0 + e;
      if (k < nseg) {
        v[e] = __ldcg(np + (uint64_t)k * kHT);
      } else if (k < n) {
        const uint32_t I2 = I + 1 + (k - nseg);
        v[e] = __ldcg(hp + (uint64_t)(I2 * (I2 + 1) / 2 + I) * kHT);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (k0 + e < n) s = k0 + e == 0 ? v[e] : cadd(s, v[e]);
  }
  return s;
}

// Two complex elements of a tile row, widened to FP64 (c128: one 32-byte load; c64:
// one 16-byte load), L1 no-allocate, L2 policy `pol` (createpolicy).
template <typename S>
__device__ __forceinline__ void ld_pair(const S* p, double2 (&o)[2], uint64_t pol) {
  if constexpr (sizeof(S) == 16) {
    double a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p), "l"(pol));
    o[0] = make_double2(a, b);
    o[1] = make_double2(c, d);
  } else {
    float4 f;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w)
                 : "l"(p), "l"(pol));
    o[0] = make_double2(f.x, f.y);
    o[1] = make_double2(f.z, f.w);
  }
}

__device__ __forceinline__ double2 ld_masked(const double2* x, uint32_t i, uint32_t m) {
  return i < m ? x[i] : make_double2(0.0, 0.0);
}

// keep: K fits in L2 next to the sweep's open strips -> evict_last (re-read next
// iteration), else evict_first.
template <typename S, int OCC>
__global__ void __launch_bounds__(kCtaThreads, OCC)
hemv_kernel(const S* __restrict__ Kp, const double2* __restrict__ X, double2* __restrict__ part,
            const HemvDesc* __restrict__ hd, int nb, uint64_t U, int keep) {
  constexpr bool kPrefetch = OCC == 1;  // two tiles in registers only at one CTA per SM
  __shared__ double2 hbuf[2][kCtaWarps][kHT];
  uint64_t pol;
  if (keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint64_t P = gridDim.x, p = blockIdx.x;
  uint64_t x = sk_lo(p, U, P);
  const uint64_t xe = sk_lo(p + 1, U, P);
  if (x >= xe) {
    pdl_enter();
    return;
  }
  const int warp = warp_index(), lane = threadIdx.x % kWarp;
  // descriptors and K do not depend on the predecessor: located / requested before the
  // PDL wait, r (rows_finalize) only after it
  int b = find_desc(hd, nb, x);
  HemvDesc d = hd[b];
  uint32_t u = (uint32_t)(x - d.unit0);
  uint32_t I = 0;
  while ((I + 1) * (I + 2) / 2 <= u) ++I;
  uint32_t J = u - I * (I + 1) / 2;
  double2 accN[kHRows];
  double2 xI[kHRows];  // r_I on this warp's rows
  auto load_xI = [&]() {
#pragma unroll
    for (int k = 0; k < kHRows; ++k) xI[k] = ld_masked(X + d.x_off, I * kHT + warp * kHRows + k, d.m);
  };
#pragma unroll
  for (int k = 0; k < kHRows; ++k) accN[k] = make_double2(0.0, 0.0);
  uint32_t par = 0;
  // Tiles of all blocks are contiguous in unit order (k_off = unit0 * 64 * 64), so unit
  // x + 1 is the next 64 x 64 tile: its rows are loaded before tile x is reduced.
  const S* tp = Kp + x * (uint64_t)(kHT * kHT) + (uint64_t)(warp * kHRows) * kHT + lane * 2;
  double2 h[kHRows][2], hn[kHRows][2];
  if (kPrefetch) {
#pragma unroll
    for (int k = 0; k < kHRows; ++k) ld_pair<S>(tp + (uint64_t)k * kHT, h[k], pol);
  }
  pdl_enter();
  load_xI();
  for (;;) {
    if (kPrefetch) {
      if (x + 1 < xe) {
#pragma unroll
        for (int k = 0; k < kHRows; ++k) ld_pair<S>(tp + kHT * kHT + (uint64_t)k * kHT, hn[k], pol);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kHRows; ++k) ld_pair<S>(tp + (uint64_t)k * kHT, h[k], pol);
    }
    tp += kHT * kHT;
    const uint32_t c0 = J * kHT + lane * 2;
    const double2 xj0 = ld_masked(X + d.x_off, c0, d.m), xj1 = ld_masked(X + d.x_off, c0 + 1, d.m);
#pragma unroll
    for (int k = 0; k < kHRows; ++k) {
      cmac(accN[k], h[k][0], xj0);
      cmac(accN[k], h[k][1], xj1);
    }
    if (J < I) {  // H part of an off-diagonal tile: y_J += K_IJ^H r_I
      double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < kHRows; ++k) {
        cmac_conj(a0, h[k][0], xI[k]);
        cmac_conj(a1, h[k][1], xI[k]);
      }
      hbuf[par][warp][lane * 2] = a0;
      hbuf[par][warp][lane * 2 + 1] = a1;
      __syncthreads();
      if (warp == 0) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = lane * 2 + e;
          double2 s = hbuf[par][0][c];
#pragma unroll
          for (int w = 1; w < kCtaWarps; ++w) s = cadd(s, hbuf[par][w][c]);
          part[d.part_off + ((uint64_t)d.n_units + u) * kHT + c] = s;
        }
      }
      par ^= 1u;  // the next tile writes the other buffer; this one is reused after a barrier
    }
    ++x;
    const bool row_end = (J == I);
    if (row_end || x == xe) {  // flush the N partial of this tile-row segment
      const uint32_t urow = I * (I + 1) / 2;  // unit of (I, 0)
      const uint64_t seg = p - sk_owner(d.unit0 + urow, U, P);
      // reduce-scatter the 8 row partials over the 32 lanes: lane l ends with row (l >> 2)
#pragma unroll
      for (int o = 16, nv = kHRows / 2; o >= 4; o >>= 1, nv >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < nv; ++k) {
          double2 send = hi ? accN[k] : accN[k + nv];
          const double2 keep = hi ? accN[k + nv] : accN[k];
          send.x = __shfl_xor_sync(0xffffffffu, send.x, o);
          send.y = __shfl_xor_sync(0xffffffffu, send.y, o);
          accN[k] = cadd(keep, send);
        }
      }
      double2 a = accN[0];
#pragma unroll
      for (int o = 2; o >= 1; o >>= 1) {
        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
      }
      if ((lane & 3) == 0)
        part[d.part_off + (uint64_t)(urow + seg) * kHT + warp * kHRows + (lane >> 2)] = a;
#pragma unroll
      for (int k = 0; k < kHRows; ++k) accN[k] = make_double2(0.0, 0.0);
    }
    if (x == xe) break;
    if (kPrefetch) {
#pragma unroll
      for (int k = 0; k < kHRows; ++k) h[k][0] = hn[k][0], h[k][1] = hn[k][1];
    }
    ++u;
    if (row_end) {
      J = 0;
      if (++I == d.nT) {
        d = hd[++b];
        u = 0;
        I = 0;
      }
      load_xI();
    } else {
      ++J;
    }
  }
}

// Bulk-copy variant (default): the packed tiles are contiguous 64 x 64 blocks (32 KiB
// c64, 64 KiB c128), so each tile is ONE cp.async.bulk into an NS-deep SMEM ring
// (mbarrier complete_tx), issued by one thread as soon as all warps have read the stage
// it replaces.  NS tiles in flight per SM (192 KiB) instead of the register variant's one
// or two — that variant measured ~2 us per tile, latency-bound (2.2 TB/s on config 3).
// K does not depend on the previous kernel, so the first NS tiles are requested BEFORE
// the PDL wait and stream while rows_finalize is still finishing r.  Same tile/lane
// mapping, arithmetic order and partial layout as hemv_kernel (identical bits).
// OCC CTAs per SM: 1 -> NS = 5 (c64) / 2 (c128) stages; 2 -> NS = 2 per CTA.
template <typename S, int OCC>
struct HemvRing {
  static constexpr int NS = OCC == 2 ? 2 : sizeof(S) == 16 ? 2 : 5;
  static_assert(NS * sizeof(uint64_t) <= 128, "barrier area");
  static constexpr uint32_t TB = kHT * kHT * sizeof(S);
};
// ring + H-part buffers + barriers + the block's r (max_m complex)
template <typename S, int OCC>
constexpr size_t hemv_bulk_smem_fixed() {
  return (size_t)HemvRing<S, OCC>::NS * HemvRing<S, OCC>::TB + 2 * kCtaWarps * kHT * sizeof(double2) +
         128;  // NS barriers, padded so the r buffer behind them stays 16-byte aligned
}
template <typename S, int OCC>
size_t hemv_bulk_smem(uint32_t max_m) {
  return hemv_bulk_smem_fixed<S, OCC>() + (size_t)((max_m + kHT - 1) / kHT * kHT) * sizeof(double2);
}

template <typename S, int OCC>
__global__ void __launch_bounds__(kCtaThreads, OCC)
hemv_bulk_kernel(const S* __restrict__ Kp, const double2* __restrict__ X, double2* __restrict__ part,
                 const HemvDesc* __restrict__ hd, int nb, uint64_t U, int keep) {
  constexpr int NS = HemvRing<S, OCC>::NS;
  constexpr uint32_t TB = HemvRing<S, OCC>::TB;
  extern __shared__ __align__(128) unsigned char hsm[];
  const S* ring = reinterpret_cast<const S*>(hsm);
  double2(*hbuf)[kCtaWarps][kHT] = reinterpret_cast<double2(*)[kCtaWarps][kHT]>(hsm + NS * TB);
  uint64_t* full = reinterpret_cast<uint64_t*>(hsm + NS * TB + 2 * kCtaWarps * kHT * sizeof(double2));
  double2* xs = reinterpret_cast<double2*>(hsm + hemv_bulk_smem_fixed<S, OCC>());  // r of the current block
  uint64_t pol;
  if (keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint64_t P = gridDim.x, p = blockIdx.x;
  uint64_t x = sk_lo(p, U, P);
  const uint64_t x0 = x, xe = sk_lo(p + 1, U, P);
  if (x >= xe) {
    pdl_enter();
    return;
  }
  const uint32_t ring_s = smem_u32(hsm), full_s = smem_u32(full);
  if (threadIdx.x == 0) {
    for (int st = 0; st < NS; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint64_t t = 0; t < (uint64_t)NS && x0 + t < xe; ++t) {  // K is ready before the PDL wait
      mbar_expect_tx_s(full_s + 8 * (uint32_t)t, TB);
      bulk_g2s_s(ring_s + (uint32_t)t * TB, Kp + (x0 + t) * (uint64_t)(kHT * kHT), TB, full_s + 8 * (uint32_t)t, pol);
    }
  }
  const int warp = warp_index(), lane = threadIdx.x % kWarp;
  int b = find_desc(hd, nb, x);  // descriptors are constant: located before the PDL wait
  HemvDesc d = hd[b];
  __syncthreads();
  pdl_enter();  // r (rows_finalize) visible from here on
  uint32_t u = (uint32_t)(x - d.unit0);
  uint32_t I = 0;
  while ((I + 1) * (I + 2) / 2 <= u) ++I;
  uint32_t J = u - I * (I + 1) / 2;
  double2 accN[kHRows];
  double2 xI[kHRows];
  // the block's r, zero-padded to whole tiles, staged once per block: every X read of
  // the tile loop is an SMEM read (no L2 round trip on the per-tile critical path)
  auto stage_r = [&]() {
    const uint32_t mp = d.nT * kHT;
    for (uint32_t e = threadIdx.x; e < mp; e += kCtaThreads) xs[e] = ld_masked(X + d.x_off, e, d.m);
    __syncthreads();
  };
  auto load_xI = [&]() {
#pragma unroll
    for (int k = 0; k < kHRows; ++k) xI[k] = xs[I * kHT + warp * kHRows + k];
  };
#pragma unroll
  for (int k = 0; k < kHRows; ++k) accN[k] = make_double2(0.0, 0.0);
  stage_r();
  load_xI();
  uint32_t par = 0;
  for (uint64_t t = 0;; ++t) {
    const int st = (int)(t % NS);
    const uint32_t c0 = J * kHT + lane * 2;
    const double2 xj0 = xs[c0], xj1 = xs[c0 + 1];
    mbar_wait_s(full_s + 8 * st, (uint32_t)(t / NS) & 1u);
    double2 h[kHRows][2];
    const S* ts = ring + (size_t)st * (kHT * kHT) + (warp * kHRows) * kHT + lane * 2;
#pragma unroll
    for (int k = 0; k < kHRows; ++k) {
      if constexpr (sizeof(S) == 16) {
        h[k][0] = ts[k * kHT];
        h[k][1] = ts[k * kHT + 1];
      } else {
        const float4 f = *reinterpret_cast<const float4*>(ts + k * kHT);
        h[k][0] = make_double2(f.x, f.y);
        h[k][1] = make_double2(f.z, f.w);
      }
    }
#pragma unroll
    for (int k = 0; k < kHRows; ++k) {
      cmac(accN[k], h[k][0], xj0);
      cmac(accN[k], h[k][1], xj1);
    }
    const bool offdiag = J < I;
    if (offdiag) {  // H part of an off-diagonal tile: y_J += K_IJ^H r_I
      double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < kHRows; ++k) {
        cmac_conj(a0, h[k][0], xI[k]);
        cmac_conj(a1, h[k][1], xI[k]);
      }
      hbuf[par][warp][lane * 2] = a0;
      hbuf[par][warp][lane * 2 + 1] = a1;
    }
    __syncthreads();  // stage st read by every warp; hbuf[par] complete
    if (threadIdx.x == 0 && x + NS < xe) {
      mbar_expect_tx_s(full_s + 8 * st, TB);
      bulk_g2s_s(ring_s + (uint32_t)st * TB, Kp + (x + NS) * (uint64_t)(kHT * kHT), TB, full_s + 8 * st, pol);
    }
    if (offdiag) {
      if (warp == 0) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = lane * 2 + e;
          double2 sum = hbuf[par][0][c];
#pragma unroll
          for (int w = 1; w < kCtaWarps; ++w) sum = cadd(sum, hbuf[par][w][c]);
          part[d.part_off + ((uint64_t)d.n_units + u) * kHT + c] = sum;
        }
      }
      par ^= 1u;
    }
    ++x;
    const bool row_end = (J == I);
    if (row_end || x == xe) {  // flush the N partial of this tile-row segment (as hemv_kernel)
      const uint32_t urow = I * (I + 1) / 2;
      const uint64_t seg = p - sk_owner(d.unit0 + urow, U, P);
#pragma unroll
      for (int o = 16, nv = kHRows / 2; o >= 4; o >>= 1, nv >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < nv; ++k) {
          double2 send = hi ? accN[k] : accN[k + nv];
          const double2 kp = hi ? accN[k + nv] : accN[k];
          send.x = __shfl_xor_sync(0xffffffffu, send.x, o);
          send.y = __shfl_xor_sync(0xffffffffu, send.y, o);
          accN[k] = cadd(kp, send);
        }
      }
      double2 a = accN[0];
#pragma unroll
      for (int o = 2; o >= 1; o >>= 1) {
        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
      }
      if ((lane & 3) == 0)
        part[d.part_off + (uint64_t)(urow + seg) * kHT + warp * kHRows + (lane >> 2)] = a;
#pragma unroll
      for (int k = 0; k < kHRows; ++k) accN[k] = make_double2(0.0, 0.0);
    }
    if (x == xe) break;
    ++u;
    if (row_end) {
      J = 0;
      if (++I == d.nT) {
        d = hd[++b];
        u = 0;
        I = 0;
        __syncthreads();  // every warp is done with the previous block's r
        stage_r();
      }
      load_xI();
    } else {
      ++J;
    }
  }
}

// q = K r from the partials (tile-row N segments in CTA order, then the H parts of the
// tiles below the diagonal in ascending tile-row order), ghat = g_ij - rho q
// (the kQ stage of rows_finalize_kernel).
// Grid: (cdiv(max rows, kHFinRows), blocks).
constexpr int kHFinRows = 64;
__global__ void __launch_bounds__(kHFinRows)
hemv_finalize_kernel(RowVecs rv, const double2* __restrict__ part, const HemvDesc* __restrict__ hd, uint64_t U,
                     uint64_t P, const Params* __restrict__ prm) {
  const HemvDesc d = hd[blockIdx.y];  // constant: read before the PDL wait
  pdl_enter();
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= d.m) return;
  const double2 s = hemv_sum_row(part, d, row / kHT, row % kHT, U, P);
  const uint32_t o = d.x_off + row;
  rv.q[o] = s;
  rv.ghat[o] = csub(rv.gij[o], cscale(s, prm->rho));
}

// Packed tiles from the dense FP64 inverse (GramDesc a_off, leading dimension nT * 64 — the
// padded work matrix of admm_factor.cuh): tile (I, J), I >= J.
template <typename S>
__global__ void k_pack_kernel(const double2* __restrict__ Aar, uint64_t a_off, uint32_t m, uint32_t nT,
                              S* __restrict__ Kp, double diag = 0.0) {  // diag subtracted on the diagonal
  const uint64_t total = (uint64_t)nT * (nT + 1) / 2 * kHT * kHT;
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(idx / (kHT * kHT)), e = (uint32_t)(idx % (kHT * kHT));
    uint32_t I = 0;
    while ((I + 1) * (I + 2) / 2 <= u) ++I;
    const uint32_t J = u - I * (I + 1) / 2;
    const uint32_t row = I * kHT + e / kHT, col = J * kHT + e % kHT;
    double2 v = (row < m && col < m) ? Aar[a_off + (uint64_t)row * (nT * kHT) + col] : make_double2(0.0, 0.0);
    if (row == col && row < m) v.x -= diag;
    Kp[idx] = Store<S>::narrow(v);
  }
}

}  // namespace admm
