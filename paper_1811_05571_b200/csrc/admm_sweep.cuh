// admm_sweep.cuh — single-HBM-pass ADMM iteration ("column-strip sweep").
//
// The two H products of an iteration are separated only by elementwise-per-column
// work: z = H^H q feeds u = c + z, the replica mean, v = S_kappa(.), the dual update
// and the next iteration's c (solvers.hpp:116-139 / 236-242 / 377-414 are all
// per-column), and c feeds the next product w = H c.  So a CTA that owns a strip of
// W columns across ALL rows of a segment can
//   (C) stream the strip from HBM reducing z for its W columns   (evict_last),
//   (D) update u, v, s, c for those columns (all M replicas are in the strip),
//   (A) immediately re-stream the same strip — now an L2 hit — accumulating the
//       strip's contribution to the next iteration's w = H c   (evict_first).
// Per iteration H crosses HBM once instead of twice; the K apply stays a separate
// stream-K GEMV.  Strips are dealt to a persistent grid in contiguous runs (stream-K
// over strips); each CTA accumulates w for every row of its current segment in SMEM
// and flushes one partial per (segment, CTA), reduced in fixed CTA order by
// rows_finalize_sweep_kernel — bit-reproducible, no float atomics.
//
// Eligible when all replicas of a segment are on the device, the segment's rows fit
// the SMEM accumulator, and (#resident strips x strip bytes) fits in L2 (admm_plan.cu).
#pragma once

#include "admm_kernels.cuh"

namespace admm {

struct SweepDesc {    // one per segment j
  uint64_t unit0;     // first strip (work unit) of segment j
  uint64_t part_off;  // double2 offset of segment j's partial region: n_strips slots x n_meas rows
  uint32_t n_strips;
  uint32_t cols;      // segment width
};

constexpr int kSweepU = 8;   // producer: row-instructions in flight per lane

constexpr int kSweepUA = 8;  // consumer (L2 re-read): row-instructions in flight per lane

// Named barriers (id 0 is __syncthreads).
__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

constexpr int kSweepThreads = 512;           // 16 warps (8 producers with kSweepU = 16 and 4
                                             // consumers at 384 threads measured 191 vs 126 us)
constexpr int kProdWarps = 8;                // (C) HBM stream
constexpr int kConsWarps = 8;                // (D) column update + (A) L2 re-read
constexpr int kConsThreads = kConsWarps * kWarp;
enum SweepBar { kBarA = 2, kBarFull0 = 3, kBarEmpty0 = 5 };

// Warp-specialised sweep: 8 producer warps stream strip s+1 from HBM and reduce z
// while 8 consumer warps finish strip s (u/v/s/c update and the L2 re-read for w).
// Each producer warp hands its partial z over through a double-buffered SMEM slot
// guarded by named FULL/EMPTY barriers (the consumer adds the 8 partials in warp
// order), so the HBM stream never waits on a barrier of its own group.
// KeepL2: the whole local H (+ K) fits in L2 (multi-GPU shards): the re-read keeps the
// lines (evict_last) so the next iteration's stream is an L2 hit too.
template <typename S, int LPR, bool KeepL2>
__global__ void __launch_bounds__(kSweepThreads, 1)
sweep_kernel(const S* __restrict__ H, const MatDesc* __restrict__ hm, const BlockDesc* __restrict__ blocks,
             const SweepDesc* __restrict__ segs, uint32_t M, uint32_t N, uint32_t n_meas, uint64_t Utot,
             const double2* __restrict__ q, ColVecs cv, double2* __restrict__ wpart,
             const Params* __restrict__ prm, double* __restrict__ red, IterState* st) {
  pdl_enter();
  constexpr int PV = Store<S>::kPerVec;
  constexpr int W = LPR * PV;            // columns per strip
  constexpr int RPI = kWarp / LPR;       // rows per warp instruction
  constexpr int PSTEP = kProdWarps * RPI;
  constexpr int CSTEP = kConsWarps * RPI;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* wacc = reinterpret_cast<double2*>(smem_raw);            // n_meas               (consumer)
  double2* zbuf = wacc + n_meas;                                     // 2 x 12 x M x W       (hand-over)
  double2* us = zbuf + 2 * (size_t)kProdWarps * M * W;               // M x W                (consumer)
  double2* cs = us + (size_t)M * W;                                  // M x W                (consumer)
  double2* pre = cs + (size_t)M * W;                                 // 2 x M x W            (consumer)
  __shared__ double sm_red[kSweepThreads / kWarp];

  const uint64_t P = gridDim.x, p = blockIdx.x;
  const uint64_t x0 = sk_lo(p, Utot, P);
  const uint64_t xe = sk_lo(p + 1, Utot, P);
  const int gwarp = warp_index(), lane = threadIdx.x % kWarp;
  const bool producer = gwarp < kProdWarps;
  const int warp = producer ? gwarp : gwarp - kProdWarps;
  const int gt = threadIdx.x - (producer ? 0 : kProdWarps * kWarp);  // index within the group
  const int lr = lane / LPR, lc = lane % LPR;
  double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
  bool bad = false;

  if (x0 < xe) {
    uint32_t j = 0;
    while (j + 1 < N && segs[j + 1].unit0 <= x0) ++j;
    SweepDesc sd = segs[j];
    if (producer) {
      // ------------------------------------------------ (C) z = H^H q per strip
      uint32_t k = 0;
      for (uint64_t x = x0; x < xe; ++x, ++k) {
        if (x == sd.unit0 + sd.n_strips) sd = segs[++j];
        const int slot = k & 1;
        if (k >= 2) nb_sync(kBarEmpty0 + slot, kSweepThreads);  // consumer released the slot
        const uint32_t col = (uint32_t)(x - sd.unit0) * W + lc * PV;
        const bool cok = col < sd.cols;
        for (uint32_t i = 0; i < M; ++i) {
          const MatDesc md = hm[i * N + j];
          const S* hb = H + md.a_off + col;
          const double2* qb = q + blocks[i * N + j].mvec_off;
          double2 acc[PV];
#pragma unroll
          for (int e = 0; e < PV; ++e) acc[e] = make_double2(0.0, 0.0);
          for (uint32_t rb = warp * RPI; rb < md.rows; rb += PSTEP * kSweepU) {  // warp-uniform
            const uint32_t r0 = rb + lr;
            V256 hv[kSweepU];
#pragma unroll
            for (int u = 0; u < kSweepU; ++u) {
              const uint32_t row = r0 + u * PSTEP;
              if (row < md.rows && cok) {
                hv[u] = ld_stream256<kEvictLast>(hb + (uint64_t)row * md.ld);
              } else {
                hv[u].w[0] = hv[u].w[1] = hv[u].w[2] = hv[u].w[3] = 0;
              }
            }
#pragma unroll
            for (int u = 0; u < kSweepU; ++u) {
              const uint32_t row = r0 + u * PSTEP;
              const double2 qv = row < md.rows ? __ldg(qb + row) : make_double2(0.0, 0.0);
#pragma unroll
              for (int e = 0; e < PV; ++e) cmac_conj(acc[e], Store<S>::get(hv[u], e), qv);
            }
          }
#pragma unroll
          for (int e = 0; e < PV; ++e) {
#pragma unroll
            for (int o = LPR; o < kWarp; o <<= 1) {
              acc[e].x += __shfl_xor_sync(0xffffffffu, acc[e].x, o);
              acc[e].y += __shfl_xor_sync(0xffffffffu, acc[e].y, o);
            }
            if (lr == 0) zbuf[(((size_t)slot * kProdWarps + warp) * M + i) * W + lc * PV + e] = acc[e];
          }
        }
        nb_arrive(kBarFull0 + slot, kSweepThreads);  // z of this strip is ready
      }
      // drain: wait for the consumer's last releases so every barrier phase completes
      const uint32_t nk = k;
      for (uint32_t kk = (nk >= 2 ? nk - 2 : 0); kk < nk; ++kk) nb_sync(kBarEmpty0 + (kk & 1), kSweepThreads);
    } else {
      for (uint32_t r = gt; r < n_meas; r += kConsThreads) wacc[r] = make_double2(0.0, 0.0);
      uint32_t k = 0;
      for (uint64_t x = x0; x < xe; ++x, ++k) {
        const int slot = k & 1;
        const uint32_t col_lo = (uint32_t)(x - sd.unit0) * W;
        // prefetch this strip's iterates (independent of z) before waiting for z
        const uint32_t t = gt, cc = col_lo + t;
        const bool dcol = gt < W && cc < sd.cols;
        double2 vo = make_double2(0.0, 0.0);
        if (dcol) {  // pre[i] = c_i, pre[M + i] = s_i (SMEM: no dynamic register indexing)
          for (uint32_t i = 0; i < M; ++i) {
            const uint32_t o = blocks[i * N + j].vec_off + cc;
            pre[i * W + t] = cv.c[o];
            pre[(M + i) * W + t] = cv.s[o];
          }
          vo = cv.v[blocks[j].seg_off + cc];
        }
        nb_sync(kBarFull0 + slot, kSweepThreads);  // wait for z of strip x
        // ------------------------------------- (D) u, mean, v, residuals, s, next c
        if (gt < W) {
          if (dcol) {
            double2 mean = make_double2(0.0, 0.0);
            for (uint32_t i = 0; i < M; ++i) {
              const uint32_t o = blocks[i * N + j].vec_off + cc;
              double2 z = zbuf[((size_t)slot * kProdWarps * M + i) * W + t];
#pragma unroll
              for (int w = 1; w < kProdWarps; ++w) z = cadd(z, zbuf[(((size_t)slot * kProdWarps + w) * M + i) * W + t]);
              const double2 ci = pre[i * W + t];
              const double2 si = pre[(M + i) * W + t];
              const double2 u = cadd(ci, z);
              bad |= !cfinite(u);
              cv.u[o] = u;
              us[i * W + t] = u;
              mean = cadd(mean, cadd(u, si));
            }
            mean = make_double2(mean.x / prm->m_rep, mean.y / prm->m_rep);
            const double2 vn = soft_threshold(mean, prm->kappa);
            const uint32_t so = blocks[j].seg_off + cc;
            cv.vprev[so] = vo;
            cv.v[so] = vn;
            rd2 += cabs2(csub(vn, vo));
            l1 += hypot(vn.x, vn.y);
            for (uint32_t i = 0; i < M; ++i) {
              const uint32_t o = blocks[i * N + j].vec_off + cc;
              const double2 u = us[i * W + t];
              rp2 += cabs2(csub(u, vn));
              const double2 s = csub(cadd(pre[(M + i) * W + t], u), vn);
              cv.s[o] = s;
              const double2 c = csub(vn, s);
              cv.c[o] = c;
              cs[i * W + t] = c;
            }
          } else {
            for (uint32_t i = 0; i < M; ++i) cs[i * W + t] = make_double2(0.0, 0.0);
          }
        }
        nb_sync(kBarA, kConsThreads);               // cs visible to the consumer group
        nb_arrive(kBarEmpty0 + slot, kSweepThreads);  // zbuf[slot] may be refilled
        // ------------------------------------- (A) w_i += H_ij[:, strip] c_i  (L2 re-read)
        const uint32_t col = col_lo + lc * PV;
        const bool cok = col < sd.cols;
        for (uint32_t i = 0; i < M; ++i) {
          const MatDesc md = hm[i * N + j];
          const uint32_t row0 = blocks[i * N + j].row0;
          const S* hb = H + md.a_off + col;
          double2 cx[PV];
#pragma unroll
          for (int e = 0; e < PV; ++e) cx[e] = cs[i * W + lc * PV + e];
          for (uint32_t rb = warp * RPI; rb < md.rows; rb += CSTEP * kSweepUA) {  // warp-uniform
            const uint32_t r0 = rb + lr;
            V256 hv[kSweepUA];
#pragma unroll
            for (int u = 0; u < kSweepUA; ++u) {
              const uint32_t row = r0 + u * CSTEP;
              if (row < md.rows && cok) {
                hv[u] = ld_stream256<KeepL2 ? kEvictLast : kEvictFirst>(hb + (uint64_t)row * md.ld);
              } else {
                hv[u].w[0] = hv[u].w[1] = hv[u].w[2] = hv[u].w[3] = 0;
              }
            }
#pragma unroll
            for (int u = 0; u < kSweepUA; ++u) {
              double2 a = make_double2(0.0, 0.0);
#pragma unroll
              for (int e = 0; e < PV; ++e) cmac(a, Store<S>::get(hv[u], e), cx[e]);
#pragma unroll
              for (int o = 1; o < LPR; o <<= 1) {
                a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
                a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
              }
              const uint32_t row = r0 + u * CSTEP;
              if (lc == 0 && row < md.rows) {  // each row is owned by one lane group
                double2& dst = wacc[row0 + row];
                dst = cadd(dst, a);
              }
            }
          }
        }
        const bool seg_end = (x + 1 == sd.unit0 + sd.n_strips);
        if (seg_end || x + 1 == xe) {  // flush this segment's w partial
          nb_sync(kBarA, kConsThreads);
          const uint64_t slotp = p - sk_owner(sd.unit0, Utot, P);
          double2* dst = wpart + sd.part_off + slotp * n_meas;
          for (uint32_t r = gt; r < n_meas; r += kConsThreads) {
            dst[r] = wacc[r];
            wacc[r] = make_double2(0.0, 0.0);
          }
          nb_sync(kBarA, kConsThreads);
          if (seg_end && x + 1 < xe) sd = segs[++j];
        }
        // the next strip's (D) reads cs/us only after its FULL barrier, and this
        // group's (A) reads of cs finished before that (program order within the group
        // is enforced by the kBarA barrier at the next (D)).
        nb_sync(kBarA, kConsThreads);
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->nonfinite = 1u;
  double r = block_sum<kSweepThreads>(rp2, sm_red);
  if (threadIdx.x == 0) red[p] = r;
  r = block_sum<kSweepThreads>(rd2, sm_red);
  if (threadIdx.x == 0) red[P + p] = r;
  r = block_sum<kSweepThreads>(l1, sm_red);
  if (threadIdx.x == 0) red[2 * P + p] = r;
}

// ---- mbarrier / bulk-copy helpers (slab sweep, K apply) ---------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// r_b = g_ij - w_b with w_b summed from the sweep partials of segment j in fixed
// order (first = 1: w = 0, the prologue of a solve since c^0 = 0).  A CTA owns
// kRfRows rows; its kRfGroups warps-per-row-tile each sum every kRfGroups-th
// partial (a segment may have one partial per sweep CTA, ~148 when one block is
// resident), then group 0 adds the group sums in order: bit-reproducible.
// CTA (0,0) also closes the sweep's iteration: fin = 1 writes trace[k] (one
// device), fin = 2 writes this rank's 4 scalars into `slot` (sharded plans).
constexpr int kRfRows = 32;
constexpr int kRfGroups = kCtaThreads / kRfRows;

__global__ void __launch_bounds__(kCtaThreads)
rows_finalize_sweep_kernel(RowVecs rv, const double2* __restrict__ wpart, const SweepDesc* __restrict__ segs,
                           const BlockDesc* __restrict__ blocks, const BlockDesc* __restrict__ gblocks, uint32_t N,
                           uint32_t n_meas, uint64_t Utot, uint64_t Psweep, int first, int fin,
                           const double* __restrict__ red, const Params* __restrict__ prm,
                           double* __restrict__ trace, uint64_t trace_cap, IterState* st,
                           double* __restrict__ slot) {
  __shared__ double sm[kCtaWarps];
  __shared__ double2 gsum[kRfGroups][kRfRows];
  const uint32_t b = blockIdx.y;
  const BlockDesc bd = blocks[b];  // constant: read before the PDL wait
  const SweepDesc sd = segs[bd.jl];
  pdl_enter();
  const uint32_t tr = threadIdx.x % kRfRows, grp = threadIdx.x / kRfRows;
  const uint32_t row = blockIdx.x * kRfRows + tr;
  if (blockIdx.x * kRfRows < bd.rows) {  // CTA-uniform
    double2 w = make_double2(0.0, 0.0);
    if (!first && row < bd.rows) {
      const uint32_t ns = seg_count(sd.unit0, sd.n_strips, Utot, Psweep);
      const double2* src = wpart + sd.part_off + bd.row0 + row;
#pragma unroll 4
      for (uint32_t k = grp; k < ns; k += kRfGroups) w = cadd(w, src[(uint64_t)k * n_meas]);
    }
    gsum[grp][tr] = w;
    __syncthreads();
    if (grp == 0 && row < bd.rows) {
      for (int g2 = 1; g2 < kRfGroups; ++g2) w = cadd(w, gsum[g2][tr]);
      const double2 gij = gij_row(rv, gblocks, bd, N, row);
      const uint32_t o = bd.mvec_off + row;
      rv.gij[o] = gij;
      rv.r[o] = csub(gij, w);
    }
  }
  if (fin && blockIdx.x == 0 && blockIdx.y == 0) {
    double a = 0.0, d = 0.0, l = 0.0;
    for (uint32_t k = threadIdx.x; k < Psweep; k += kCtaThreads) {
      a += red[k];
      d += red[Psweep + k];
      if (fin == 2) l += red[2 * Psweep + k];
    }
    a = block_sum<kCtaThreads>(a, sm);
    d = block_sum<kCtaThreads>(d, sm);
    if (fin == 2) l = block_sum<kCtaThreads>(l, sm);
    if (threadIdx.x == 0) {
      if (fin == 2) {  // same values and order as local_scalars_kernel
        slot[0] = a;
        slot[1] = d;
        slot[2] = l;
        slot[3] = st->nonfinite ? 1.0 : 0.0;
        slot[4] = 0.0;
        st->nonfinite = 0u;
        return;
      }
      const uint64_t k = st->iter;
      if (k < trace_cap) {
        trace[3 * k] = sqrt(a);
        trace[3 * k + 1] = sqrt(prm->rho * prm->rho * prm->m_rep * d);
        trace[3 * k + 2] = __longlong_as_double(0x7ff8000000000000ll);
      }
      if (st->nonfinite && st->first_bad == ~0ull) st->first_bad = k;
      st->nonfinite = 0u;
      st->iter = k + 1;
    }
  }
}

}  // namespace admm
