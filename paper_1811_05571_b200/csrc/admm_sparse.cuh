// admm_sparse.cuh — the "support" schedule: ONE dense pass over H per iteration plus a pass
// over only the columns in the support of the soft-thresholded variable v.
//
// Why it is the reference's iteration.  Per block b = (i, j) the column update of
// solvers.hpp (u = c + z, v' = S_kappa(mean_i(u + s)), s' = s + u - v', c' = v' - s';
// admm_core.hpp:80-89, prox.hpp:15) with c = v - s from the previous update gives
//     s' = v + z - v'      and      c' = 2 v' - v - z,        z = H_b^H q_b,
// so the next product the reference forms, w' = H_b c' (gram.hpp:71-77 inside the
// Woodbury solve), is exactly
//     w' = 2 a' - a - G_b q_b,      a = H_b v,  a' = H_b v',  G_b = H_b H_b^H.
// G_b q_b needs no product: q_b = K_b r_b with K_b = (rho I + G_b)^-1 (gram.hpp:63-78), so
//     G_b q_b = r_b - rho q_b
// from the r and q the iteration already holds (exact up to the rounding of the stored K,
// the same rounding the q-form's u = c + H^H q already carries).  a' = H_b v' touches
// only the columns where v' != 0: soft thresholding makes v sparse (config 4: ~1e3 of
// 262144 columns), and a skipped term is an exact zero (H is validated finite), so a'
// is bit-identical to the dense product in the same (ascending-column) order.  With v
// dense the same kernels read every column: the iteration then streams H twice, like
// the two-pass schedule.  Per iteration:
//
//   z = H^H q                 gemv_h_kernel (dense pass, row-major H)
//   u, v', s', c', residuals  zupdate_kernel (+ per-CTA support counts)
//   support list of v'        support_compact_kernel (ascending, deterministic)
//   a' = H v' on the support  support_a_kernel (column-major copy of H)
//   w' (Gq = r - rho q), r, objective rows     support_rows_kernel
//   trace[k]                  finalize_kernel
//   q = K r, ghat             hemv (packed K) + hemv_finalize
// Bit-reproducible: fixed-order sums, no atomics.
#pragma once

#include "admm_hemv.cuh"
#include "admm_kernels.cuh"
#include <type_traits>

namespace admm {

constexpr int kSupUnroll = 8;  // support columns in flight per thread

// Column-major copy of a block: Hc[x * ldc + r] = H[r * ld + x] (setup only).
template <typename S>
__global__ void colmajor_kernel(const S* __restrict__ H, uint64_t a_off, uint32_t ld, uint32_t rows, uint32_t cols,
                                S* __restrict__ Hc, uint64_t c_off, uint32_t ldc) {
  __shared__ S tile[32][33];
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (uint32_t k = threadIdx.y; k < 32; k += blockDim.y) {
    const uint32_t r = r0 + k, c = c0 + threadIdx.x;
    S v;
    v.x = 0;
    v.y = 0;
    if (r < rows && c < cols) v = H[a_off + (uint64_t)r * ld + c];
    tile[k][threadIdx.x] = v;
  }
  __syncthreads();
  for (uint32_t k = threadIdx.y; k < 32; k += blockDim.y) {
    const uint32_t c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < ldc) Hc[c_off + (uint64_t)c * ldc + r] = r < rows ? tile[threadIdx.x][k] : S{};
  }
}

// support list of segment j: CTA (x, j) covers columns [256x, 256x + 256); its offset is
// the sum of the counts of the CTAs before it (zupdate wrote them), so the list is in
// ascending column order.  The last CTA of a segment stores the segment's support size
// and adds it to the running total (diagnostics: mean support per iteration).
__global__ void __launch_bounds__(kCtaThreads)
support_compact_kernel(const double2* __restrict__ v, const BlockDesc* __restrict__ blocks,
                       const uint32_t* __restrict__ cnt, uint32_t gx, uint32_t* __restrict__ list,
                       uint32_t list_stride, uint32_t* __restrict__ nnz, unsigned long long* __restrict__ nnz_total) {
  __shared__ double sm[kCtaWarps];
  __shared__ uint32_t wsum[kCtaWarps];
  const uint32_t j = blockIdx.y, x = blockIdx.x;
  const BlockDesc b0 = blocks[j];
  double pre = 0.0;  // counts are < 2^32: exact in FP64 through block_sum
  for (uint32_t k = threadIdx.x; k < x; k += kCtaThreads) pre += (double)cnt[j * gx + k];
  pre = block_sum<kCtaThreads>(pre, sm);
  __shared__ uint32_t off;
  if (threadIdx.x == 0) off = (uint32_t)pre;
  const uint32_t t = x * kCtaThreads + threadIdx.x;
  bool nz = false;
  if (t < b0.cols) {
    const double2 a = v[b0.seg_off + t];
    nz = a.x != 0.0 || a.y != 0.0;
  }
  const int warp = warp_index(), lane = threadIdx.x % kWarp;
  const unsigned m = __ballot_sync(0xffffffffu, nz);
  if (lane == 0) wsum[warp] = __popc(m);
  __syncthreads();
  uint32_t base = off;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  if (nz) list[(uint64_t)j * list_stride + base + __popc(m & ((1u << lane) - 1u))] = t;
  if (x == gridDim.x - 1 && threadIdx.x == 0) {
    uint32_t tot = off;
    for (int w = 0; w < kCtaWarps; ++w) tot += wsum[w];
    nnz[j] = tot;
    atomicAdd(nnz_total, (unsigned long long)tot);  // integer: order-independent
  }
}

// a'_b = H_b v' over the support of segment j (ascending columns).  Grid (row tiles of
// kSupTile rows, local blocks, column chunks): thread t owns kSupRPT consecutive
// rows (one 32/64-byte load per support column), kSupUnroll columns in flight, so a CTA
// keeps ~kSupUnroll x 8 KiB of the column-major H in flight.  Column chunk c of the
// support list writes its partial; support_rows_kernel adds the chunks' partials of a
// row in chunk order (fixed order: bit-reproducible).
constexpr int kSupThreads = 256;
constexpr int kSupRPT = 4;                          // rows per thread
constexpr int kSupTile = kSupThreads * kSupRPT;     // rows per CTA
constexpr int kSupMaxChunks = 64;                   // column chunks of the support list: chosen per plan so that the
                                                    // grid is ~4 CTAs (32 warps) per SM -- with 16 chunks (1-2 CTAs per
                                                    // SM) the dense early iterations of config 4 ran at 3.5 TB/s
template <typename S>
__global__ void __launch_bounds__(kSupThreads)
support_a_kernel(const S* __restrict__ Hc, const uint64_t* __restrict__ coff, const uint32_t* __restrict__ ldc,
                 const BlockDesc* __restrict__ blocks, const double2* __restrict__ v, const uint32_t* __restrict__ list,
                 uint32_t list_stride, const uint32_t* __restrict__ nnz, double2* __restrict__ apart,
                 uint64_t chunk_stride) {
  const uint32_t b = blockIdx.y, chunk = blockIdx.z, chunks = gridDim.z;
  const BlockDesc bd = blocks[b];
  const uint32_t row0 = blockIdx.x * kSupTile + threadIdx.x * kSupRPT;
  if (blockIdx.x * kSupTile >= bd.rows) return;
  const uint32_t n = nnz[bd.jl];
  const uint32_t k0 = (uint32_t)((uint64_t)n * chunk / chunks), k1 = (uint32_t)((uint64_t)n * (chunk + 1) / chunks);
  const uint32_t* lj = list + (uint64_t)bd.jl * list_stride;
  const S* hb = Hc + coff[b] + row0;
  const uint32_t L = ldc[b];
  const double2* vj = v + bd.seg_off;
  const bool ok = row0 < bd.rows;  // ldc is a multiple of 8 >= rows: a thread's rows are all in the padded column
  double2 acc[kSupRPT];
#pragma unroll
  for (int e = 0; e < kSupRPT; ++e) acc[e] = make_double2(0.0, 0.0);
  uint32_t k = k0;
  for (; k + kSupUnroll <= k1; k += kSupUnroll) {
    uint32_t xs[kSupUnroll];
#pragma unroll
    for (int u = 0; u < kSupUnroll; ++u) xs[u] = __ldg(lj + k + u);
    S h[kSupUnroll][kSupRPT];
#pragma unroll
    for (int u = 0; u < kSupUnroll; ++u) {
      if (ok) {
        const S* p = hb + (uint64_t)xs[u] * L;
        if constexpr (sizeof(S) == 8) {
          const V256 w = ld_stream256<kEvictFirst>(p);  // the thread's 4 rows in one 32-byte load
#pragma unroll
          for (int e = 0; e < kSupRPT; ++e)
            h[u][e] = make_float2(__uint_as_float((unsigned)(w.w[e] & 0xffffffffu)), __uint_as_float((unsigned)(w.w[e] >> 32)));
        } else {
          const V256 w = ld_stream256<kEvictFirst>(p);
          const V256 w2 = ld_stream256<kEvictFirst>(p + 2);
          h[u][0] = Store<double2>::get(w, 0);
          h[u][1] = Store<double2>::get(w, 1);
          h[u][2] = Store<double2>::get(w2, 0);
          h[u][3] = Store<double2>::get(w2, 1);
        }
      } else {
#pragma unroll
        for (int e = 0; e < kSupRPT; ++e) h[u][e] = S{};
      }
    }
#pragma unroll
    for (int u = 0; u < kSupUnroll; ++u) {
      const double2 vx = __ldg(vj + xs[u]);
#pragma unroll
      for (int e = 0; e < kSupRPT; ++e) cmac(acc[e], Store<S>::widen(h[u][e]), vx);
    }
  }
  for (; k < k1; ++k) {
    const uint32_t x = __ldg(lj + k);
    const double2 vx = __ldg(vj + x);
    if (ok)
#pragma unroll
      for (int e = 0; e < kSupRPT; ++e) cmac(acc[e], Store<S>::widen(hb[(uint64_t)x * L + e]), vx);
  }
  double2* dst = apart + chunk * chunk_stride + bd.mvec_off;
#pragma unroll
  for (int e = 0; e < kSupRPT; ++e)
    if (row0 + e < bd.rows) dst[row0 + e] = acc[e];
}

// Per row r of row block i (NP = 2^np_log2 lanes per row, lane j = column block): for every
// local block b = (i, j): w' = 2 a' - a - (r - rho q)_b (first: w' = 0), a <- a', g_ij, r = g_ij - w';
// then |sum_j a'_ij - g_i|^2 (ascending j) into per-CTA objective partials.
__global__ void __launch_bounds__(kCtaThreads)
support_rows_kernel(RowVecs rv, const BlockDesc* __restrict__ blocks, const BlockDesc* __restrict__ gblocks,
                    uint32_t N, uint32_t np_log2, const double2* __restrict__ apart, uint64_t chunk_stride,
                    uint32_t chunks, double2* __restrict__ aold, const Params* __restrict__ prm, int first,
                    double* __restrict__ ored) {
  __shared__ double2 sa[kCtaThreads];
  __shared__ double sm[kCtaWarps];
  const uint32_t i = blockIdx.y;
  const BlockDesc b0 = blocks[i * N];
  const uint32_t NP = 1u << np_log2, j = threadIdx.x & (NP - 1), rl = threadIdx.x >> np_log2;
  const uint32_t row = blockIdx.x * (kCtaThreads >> np_log2) + rl;
  const bool on = row < b0.rows && j < N;
  double2 a = make_double2(0.0, 0.0);
  if (on) {
    const BlockDesc bd = blocks[i * N + j];
    const uint64_t o = (uint64_t)bd.mvec_off + row;
    double2 w = make_double2(0.0, 0.0);
    if (!first) {
      a = apart[o];  // a'_b = the column chunks' partials, in chunk order
#pragma unroll 4
      for (uint32_t c = 1; c < chunks; ++c) a = cadd(a, apart[(uint64_t)c * chunk_stride + o]);
      const double2 gq = csub(rv.r[o], cscale(rv.q[o], prm->rho));  // G q = (K^-1 - rho I) q = r - rho q
      w = csub(csub(cscale(a, 2.0), aold[o]), gq);
      aold[o] = a;
    }
    const double2 gij = gij_row(rv, gblocks, bd, N, row);
    rv.gij[o] = gij;
    rv.r[o] = csub(gij, w);
  }
  sa[threadIdx.x] = a;
  __syncthreads();
  double q = 0.0;
  if (!first && row < b0.rows && j == 0) {
    double2 hv = make_double2(0.0, 0.0);
    for (uint32_t jj = 0; jj < N; ++jj) hv = cadd(hv, sa[rl * NP + jj]);
    q = cabs2(csub(hv, rv.g[b0.row0 + row]));
  }
  const double r = block_sum<kCtaThreads>(q, sm);
  if (threadIdx.x == 0) ored[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

}  // namespace admm
