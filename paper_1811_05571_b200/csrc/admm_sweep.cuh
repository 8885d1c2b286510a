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

constexpr int kSweepU = 8;  // row-instructions in flight per lane

template <typename S, int LPR>
__global__ void __launch_bounds__(kCtaThreads, 2)
sweep_kernel(const S* __restrict__ H, const MatDesc* __restrict__ hm, const BlockDesc* __restrict__ blocks,
             const SweepDesc* __restrict__ segs, uint32_t M, uint32_t N, uint32_t n_meas, uint64_t Utot,
             const double2* __restrict__ q, ColVecs cv, double2* __restrict__ wpart,
             const Params* __restrict__ prm, double* __restrict__ red, IterState* st) {
  constexpr int PV = Store<S>::kPerVec;
  constexpr int W = LPR * PV;            // columns per strip
  constexpr int RPI = kWarp / LPR;       // rows per warp instruction
  constexpr int ROWSTEP = kCtaWarps * RPI;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* wacc = reinterpret_cast<double2*>(smem_raw);            // n_meas
  double2* zred = wacc + n_meas;                                     // kCtaWarps x W
  double2* zs = zred + kCtaWarps * W;                                // M x W (z, then u)
  double2* cs = zs + (size_t)M * W;                                  // M x W (next c)
  __shared__ double sm_red[kCtaWarps];

  const uint64_t P = gridDim.x, p = blockIdx.x;
  uint64_t x = sk_lo(p, Utot, P);
  const uint64_t xe = sk_lo(p + 1, Utot, P);
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int lr = lane / LPR, lc = lane % LPR;
  double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
  bool bad = false;

  if (x < xe) {
    uint32_t j = 0;
    while (j + 1 < N && segs[j + 1].unit0 <= x) ++j;
    SweepDesc sd = segs[j];
    for (uint32_t r = threadIdx.x; r < n_meas; r += kCtaThreads) wacc[r] = make_double2(0.0, 0.0);
    __syncthreads();
    for (;;) {
#ifdef ADMM_DEBUG_SWEEP
      if (threadIdx.x == 0) printf("cta %llu x %llu xe %llu j %u\n", (unsigned long long)p, (unsigned long long)x, (unsigned long long)xe, j);
#endif
      const uint32_t col_lo = (uint32_t)(x - sd.unit0) * W;
      const uint32_t col = col_lo + lc * PV;
      const bool cok = col < sd.cols;
      // ---- (C) z_i = H_ij^H q_i over the strip, replica by replica
      for (uint32_t i = 0; i < M; ++i) {
        const MatDesc md = hm[i * N + j];
        const BlockDesc bd = blocks[i * N + j];
        const S* hb = H + md.a_off + col;
        const double2* qb = q + bd.mvec_off;
        double2 acc[PV];
#pragma unroll
        for (int e = 0; e < PV; ++e) acc[e] = make_double2(0.0, 0.0);
        for (uint32_t rb = warp * RPI; rb < md.rows; rb += ROWSTEP * kSweepU) {  // warp-uniform trip count
          const uint32_t r0 = rb + lr;
          V256 hv[kSweepU];
#pragma unroll
          for (int u = 0; u < kSweepU; ++u) {
            const uint32_t row = r0 + u * ROWSTEP;
            if (row < md.rows && cok) {
              hv[u] = ld_stream256<kEvictLast>(hb + (uint64_t)row * md.ld);
            } else {
              hv[u].w[0] = hv[u].w[1] = hv[u].w[2] = hv[u].w[3] = 0;
            }
          }
#pragma unroll
          for (int u = 0; u < kSweepU; ++u) {
            const uint32_t row = r0 + u * ROWSTEP;
            const double2 qv = row < md.rows ? __ldg(qb + row) : make_double2(0.0, 0.0);  // L1 hit
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
          if (lr == 0) zred[warp * W + lc * PV + e] = acc[e];
        }
        __syncthreads();
        if (threadIdx.x < W) {
          double2 z = zred[threadIdx.x];
#pragma unroll
          for (int w = 1; w < kCtaWarps; ++w) z = cadd(z, zred[w * W + threadIdx.x]);
          zs[i * W + threadIdx.x] = z;
        }
        __syncthreads();
      }
#ifdef ADMM_DEBUG_SWEEP
      if (threadIdx.x == 0) printf("cta %llu C done\n", (unsigned long long)p);
#endif
      // ---- (D) u, replica mean, v = S_kappa, residual partials, dual update, next c
      if (threadIdx.x < W) {
        const uint32_t t = threadIdx.x, cc = col_lo + t;
        if (cc < sd.cols) {
          double2 mean = make_double2(0.0, 0.0);
          for (uint32_t i = 0; i < M; ++i) {
            const uint32_t o = blocks[i * N + j].vec_off + cc;
            const double2 u = cadd(cv.c[o], zs[i * W + t]);
            bad |= !cfinite(u);
            cv.u[o] = u;
            zs[i * W + t] = u;
            mean = cadd(mean, cadd(u, cv.s[o]));
          }
          mean = make_double2(mean.x / prm->m_rep, mean.y / prm->m_rep);
          const double2 vn = soft_threshold(mean, prm->kappa);
          const uint32_t so = blocks[j].seg_off + cc;
          const double2 vo = cv.v[so];
          cv.vprev[so] = vo;
          cv.v[so] = vn;
          rd2 += cabs2(csub(vn, vo));
          l1 += hypot(vn.x, vn.y);
          for (uint32_t i = 0; i < M; ++i) {
            const uint32_t o = blocks[i * N + j].vec_off + cc;
            const double2 u = zs[i * W + t];
            rp2 += cabs2(csub(u, vn));
            const double2 s = csub(cadd(cv.s[o], u), vn);
            cv.s[o] = s;
            const double2 c = csub(vn, s);
            cv.c[o] = c;
            cs[i * W + t] = c;
          }
        } else {
          for (uint32_t i = 0; i < M; ++i) cs[i * W + t] = make_double2(0.0, 0.0);
        }
      }
      __syncthreads();
#ifdef ADMM_DEBUG_SWEEP
      if (threadIdx.x == 0) printf("cta %llu D done\n", (unsigned long long)p);
#endif
      // ---- (A) next iteration's w_i += H_ij[:, strip] c_i[strip]  (L2 re-read)
      for (uint32_t i = 0; i < M; ++i) {
        const MatDesc md = hm[i * N + j];
        const BlockDesc bd = blocks[i * N + j];
        const S* hb = H + md.a_off + col;
        double2 cx[PV];
#pragma unroll
        for (int e = 0; e < PV; ++e) cx[e] = cs[i * W + lc * PV + e];
        for (uint32_t rb = warp * RPI; rb < md.rows; rb += ROWSTEP * kSweepU) {  // warp-uniform trip count
          const uint32_t r0 = rb + lr;
          V256 hv[kSweepU];
#pragma unroll
          for (int u = 0; u < kSweepU; ++u) {
            const uint32_t row = r0 + u * ROWSTEP;
            if (row < md.rows && cok) {
              hv[u] = ld_stream256<kEvictFirst>(hb + (uint64_t)row * md.ld);
            } else {
              hv[u].w[0] = hv[u].w[1] = hv[u].w[2] = hv[u].w[3] = 0;
            }
          }
#pragma unroll
          for (int u = 0; u < kSweepU; ++u) {
            double2 a = make_double2(0.0, 0.0);
#pragma unroll
            for (int e = 0; e < PV; ++e) cmac(a, Store<S>::get(hv[u], e), cx[e]);
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) {
              a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
              a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
            }
            const uint32_t row = r0 + u * ROWSTEP;
            if (lc == 0 && row < md.rows) {
              double2& dst = wacc[bd.row0 + row];  // each row is owned by one lane group
              dst = cadd(dst, a);
            }
          }
        }
      }
#ifdef ADMM_DEBUG_SWEEP
      if (threadIdx.x == 0) printf("cta %llu A done\n", (unsigned long long)p);
#endif
      ++x;
      const bool seg_end = (x == sd.unit0 + sd.n_strips);
      if (seg_end || x == xe) {  // flush this segment's w partial
        __syncthreads();
        const uint64_t slot = p - sk_owner(sd.unit0, Utot, P);
        double2* dst = wpart + sd.part_off + slot * n_meas;
        for (uint32_t r = threadIdx.x; r < n_meas; r += kCtaThreads) {
          dst[r] = wacc[r];
          wacc[r] = make_double2(0.0, 0.0);
        }
        __syncthreads();
        if (x == xe) break;
        sd = segs[++j];
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->nonfinite = 1u;
  double r = block_sum<kCtaThreads>(rp2, sm_red);
  if (threadIdx.x == 0) red[p] = r;
  r = block_sum<kCtaThreads>(rd2, sm_red);
  if (threadIdx.x == 0) red[P + p] = r;
  r = block_sum<kCtaThreads>(l1, sm_red);
  if (threadIdx.x == 0) red[2 * P + p] = r;
}

// r_b = g_ij - w_b with w_b summed from the sweep partials of segment j in fixed
// CTA order (first = 1: w = 0, the prologue of a solve since c^0 = 0).  CTA (0,0)
// also closes the previous sweep's iteration (trace, non-finite bookkeeping).
__global__ void __launch_bounds__(kCtaThreads)
rows_finalize_sweep_kernel(RowVecs rv, const double2* __restrict__ wpart, const SweepDesc* __restrict__ segs,
                           const BlockDesc* __restrict__ blocks, uint32_t N, uint32_t n_meas, uint64_t Utot,
                           uint64_t Psweep, int first, int do_finalize, const double* __restrict__ red,
                           const Params* __restrict__ prm, double* __restrict__ trace, uint64_t trace_cap,
                           IterState* st) {
  __shared__ double sm[kCtaWarps];
  const uint32_t b = blockIdx.y;
  const BlockDesc bd = blocks[b];
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < bd.rows) {
    double2 w = make_double2(0.0, 0.0);
    if (!first) {
      const SweepDesc sd = segs[bd.j];
      const uint32_t ns = seg_count(sd.unit0, sd.n_strips, Utot, Psweep);
      const double2* src = wpart + sd.part_off + bd.row0 + row;
      w = src[0];
      for (uint32_t k = 1; k < ns; ++k) w = cadd(w, src[(uint64_t)k * n_meas]);
    }
    double2 gij = rv.g[bd.row0 + row];
    for (uint32_t qj = 0; qj < N; ++qj) {
      if (qj == bd.j) continue;
      gij = csub(gij, rv.ghat[blocks[bd.i * N + qj].mvec_off + row]);
    }
    const uint32_t o = bd.mvec_off + row;
    rv.gij[o] = gij;
    rv.r[o] = csub(gij, w);
  }
  if (do_finalize && blockIdx.x == 0 && blockIdx.y == 0) {
    double a = 0.0, d = 0.0;
    for (uint32_t k = threadIdx.x; k < Psweep; k += kCtaThreads) {
      a += red[k];
      d += red[Psweep + k];
    }
    a = block_sum<kCtaThreads>(a, sm);
    d = block_sum<kCtaThreads>(d, sm);
    if (threadIdx.x == 0) {
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
