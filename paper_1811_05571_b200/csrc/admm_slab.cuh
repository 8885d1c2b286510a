// admm_slab.cuh — single-HBM-pass ADMM iteration with per-warp row slabs ("slab sweep").
//
// Same iteration as sweep_kernel (admm_sweep.cuh): per column strip x of segment j,
//   (C) z_i = H_ij[:, x]^H q_ij for every replica i       (solvers.hpp:114-121 / 374-391 u-update, q-form)
//   (D) u, replica mean, v = S_kappa, s, next c            (solvers.hpp:116-139 / 236-242 / 377-414, prox.hpp:15)
//   (A) w_i += H_ij[:, x] c_i                               (the next iteration's H c)
// but organised so that no warp ever waits for another warp's data movement:
//
//  * H is re-laid out once at setup strip-major in row SLABS of RPW rows x 64 bytes
//    (Hs[x][slab][row][16-byte chunk], chunk order XOR-swizzled by (row >> 1) & 3), so a
//    slab of a strip is one contiguous 2-8 KiB block in HBM.
//  * Compute warp w of cluster rank r owns slab r*NW + w of EVERY strip.  Its lane 0
//    streams the slab into the warp's own stage of an NS-deep SMEM ring with one
//    cp.async.bulk (mbarrier complete_tx) — no producer warp, no cross-warp empty
//    barrier: the warp refills a stage the moment its own (A) pass has read it.
//  * Software pipeline per compute warp: (C) of strip k, then (A) of strip k-1 — the
//    latency of the strip-(k-1) column update hides behind the strip-k pass.
//  * (C) lanes own 16-byte column chunks and accumulate over the slab's rows in
//    registers (q of the slab's rows stays in registers for the whole segment); (A)
//    lanes own rows and form each row's dot in registers, accumulating w in registers
//    across every strip of the segment: no SMEM w, no per-row shuffles.  The swizzle
//    makes both access patterns bank-conflict-free.
//  * One D warp per CTA sums the warps' z partials (fixed order), exchanges CTA partials
//    with the other ranks of the thread-block cluster through DSMEM (rows of a strip are
//    split over the cluster; remote mbarrier arrive), does the column update redundantly
//    on every rank (identical bits) and publishes c through an mbarrier; rank 0 alone
//    stores the iterates and the residual partials.
//
// Outputs (w partials per (segment, cluster), residual partials per cluster) have the
// layout of sweep_kernel's with "cluster" in place of "CTA", so rows_finalize_sweep_kernel
// consumes them unchanged.  Bit-reproducible: every sum has a fixed order, no atomics.
#pragma once

#include "admm_sweep.cuh"

namespace admm {

constexpr int kSlabRB = 64;          // bytes per slab row (one strip row)
constexpr int kSlabNSL = kSlabRB / 16;  // 16-byte chunks per row
constexpr int kSlabMaxW = 16;        // compute warps per CTA (+1 D warp)
constexpr int kSlabThreads = (kSlabMaxW + 1) * kWarp;

struct SlabDesc {
  uint32_t rep;    // replica (row block) i
  uint32_t lrow0;  // first row of the slab inside block i
  uint32_t mrow0;  // ... in the plan's local measurement-row arena
  uint32_t nrows;  // valid rows (<= RPW; the rest of the slab is zero padding)
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_d2(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t a) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITC_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAITC_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ double2 lds_d2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// One 16-byte chunk of stored elements, widened to FP64 on use.
template <typename S>
struct Chunk;
template <>
struct Chunk<double2> {
  static constexpr int PV = 1;
  double2 v;
  __device__ __forceinline__ void load(uint32_t a) { v = lds_d2(a); }
  __device__ __forceinline__ double2 get(int) const { return v; }
};
template <>
struct Chunk<float2> {
  static constexpr int PV = 2;
  float4 v;
  __device__ __forceinline__ void load(uint32_t a) { v = lds_f4(a); }
  __device__ __forceinline__ double2 get(int e) const {
    return e == 0 ? make_double2((double)v.x, (double)v.y) : make_double2((double)v.z, (double)v.w);
  }
};

__host__ __device__ inline size_t slab_smem_bytes(uint32_t ns, uint32_t nw, uint32_t rpw, uint32_t C, uint32_t M,
                                                  uint32_t W) {
  return (size_t)ns * nw * rpw * kSlabRB            // ring
         + (size_t)nw * ns * sizeof(uint64_t)       // per-warp full barriers
         + 6 * sizeof(uint64_t)                     // zfull[2], cfull[2], xfull[2]
         + 2 * (size_t)nw * W * sizeof(double2)     // z partials per warp
         + 2 * (size_t)C * M * W * sizeof(double2)  // cluster exchange
         + 2 * (size_t)M * W * sizeof(double2);     // c of the strip
}

// RPL = rows per lane in (A) = RPW / 32.  Launched as NCl clusters of C CTAs, block
// (NW + 1) x 32 threads: warps 0..NW-1 compute, warp NW is the D warp.
template <typename S, int RPL>
__global__ void __launch_bounds__(kSlabThreads, 1)
sweep_slab_kernel(const S* __restrict__ Hs, const SlabDesc* __restrict__ slabs, const BlockDesc* __restrict__ blocks,
                  const SweepDesc* __restrict__ segs, uint32_t M, uint32_t N, uint32_t n_meas, uint64_t U, uint32_t NS,
                  uint32_t Ns, const double2* __restrict__ q, ColVecs cv, double2* __restrict__ wpart,
                  const Params* __restrict__ prm, double* __restrict__ red, IterState* st) {
  using CK = Chunk<S>;
  constexpr int PV = CK::PV;
  constexpr int W = kSlabNSL * PV;          // columns per strip
  constexpr int RPW = RPL * kWarp;          // rows per slab
  constexpr int SLAB_B = RPW * kSlabRB;     // bytes per slab
  constexpr int CRG = kWarp / kSlabNSL;     // (C) rows per warp instruction
  constexpr int CNU = RPW / CRG;            // (C) instructions per slab
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t NW = blockDim.x / kWarp - 1;
  const uint32_t C = cluster_size();
  unsigned char* ring = smem_raw;
  uint64_t* fullb = reinterpret_cast<uint64_t*>(ring + (size_t)NS * NW * SLAB_B);  // [NW][NS]
  uint64_t* zfull = fullb + (size_t)NW * NS;
  uint64_t* cfull = zfull + 2;
  uint64_t* xfull = cfull + 2;
  double2* zp = reinterpret_cast<double2*>(xfull + 2);  // [2][NW][W]
  double2* xb = zp + 2 * (size_t)NW * W;                // [2][C][M][W]
  double2* cb = xb + 2 * (size_t)C * M * W;             // [2][M][W]

  const uint32_t rank = cluster_rank();
  const uint64_t NCl = cluster_count(), cl = cluster_id();
  const uint64_t x0 = sk_lo(cl, U, NCl), xe = sk_lo(cl + 1, U, NCl);
  const uint32_t nstrip = (uint32_t)(xe - x0);
  const uint32_t warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;

  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < NW * NS; ++b) mbar_init(&fullb[b], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&zfull[b], NW);
      mbar_init(&cfull[b], 1);
      mbar_init(&xfull[b], C * kWarp);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (C > 1)
    cluster_sync_all();  // peers' barriers initialised before any remote arrive
  else
    __syncthreads();
  pdl_enter();  // q, c, s, v of the previous kernels are visible from here on

  if (warp < NW) {
    // ============================================================ compute warp
    const uint32_t sl = rank * NW + warp;
    const bool act = sl < Ns;
    SlabDesc sd{0, 0, 0, 0};
    if (act) sd = slabs[sl];
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint64_t* myfull = fullb + (size_t)warp * NS;
    const uint32_t ring_w = smem_u32(ring) + warp * SLAB_B;  // + stage * NW * SLAB_B
    const uint32_t stage_stride = NW * SLAB_B;
    const unsigned char* src0 = reinterpret_cast<const unsigned char*>(Hs) + ((x0 * Ns) + sl) * (uint64_t)SLAB_B;
    const uint64_t strip_stride = (uint64_t)Ns * SLAB_B;
    auto issue = [&](uint32_t k, uint32_t stg) {
      mbar_expect_tx(&myfull[stg], SLAB_B);
      bulk_g2s(ring_w + stg * stage_stride, src0 + k * strip_stride, SLAB_B, &myfull[stg], pol);
    };
    if (act && lane == 0)
      for (uint32_t k = 0; k < NS && k < nstrip; ++k) issue(k, k);

    // (C) lane geometry: rows crg + CRG u, logical chunk ccol at physical ccol ^ swz
    const uint32_t crg = lane / kSlabNSL, ccol = lane % kSlabNSL;
    const uint32_t c_off = crg * kSlabRB + ((ccol ^ ((crg >> 1) & 3)) * 16);
    // (A) lane geometry: rows lane + 32 m, logical chunk s at physical s ^ swz
    const uint32_t a_swz = (lane >> 1) & 3;
    uint32_t j = 0;
    if (nstrip > 0)
      while (j + 1 < N && segs[j + 1].unit0 <= x0) ++j;
    uint32_t jA = j;
    double2 qr[CNU];
    auto load_q = [&](uint32_t jj) {
      const double2* qb = q + blocks[sd.rep * N + jj].mvec_off + sd.lrow0;
#pragma unroll
      for (int u = 0; u < CNU; ++u) {
        const uint32_t r = crg + CRG * u;
        qr[u] = (act && r < sd.nrows) ? qb[r] : make_double2(0.0, 0.0);
      }
    };
    if (nstrip > 0) load_q(j);
    double2 wacc[RPL];
#pragma unroll
    for (int m = 0; m < RPL; ++m) wacc[m] = make_double2(0.0, 0.0);
    uint64_t seg_end = (nstrip > 0) ? segs[j].unit0 + segs[j].n_strips : 0;   // (C) side
    uint64_t seg_endA = seg_end;                                              // (A) side
    uint32_t stgC = 0, phC = 0, stgA = 0;

    for (uint32_t k = 0; k <= nstrip; ++k) {
      if (k < nstrip) {
        // ---------------------------------------------------------- (C) strip k
        if (x0 + k == seg_end) {
          ++j;
          seg_end = segs[j].unit0 + segs[j].n_strips;
          load_q(j);
        }
        if (act) {
          mbar_wait(&myfull[stgC], phC);
          const uint32_t base = ring_w + stgC * stage_stride + c_off;
          double2 acc[PV], acc2[PV];
#pragma unroll
          for (int e = 0; e < PV; ++e) acc[e] = acc2[e] = make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < CNU; u += 2) {
            CK h0, h1;
            h0.load(base + u * CRG * kSlabRB);
            h1.load(base + (u + 1) * CRG * kSlabRB);
#pragma unroll
            for (int e = 0; e < PV; ++e) {
              cmac_conj(acc[e], h0.get(e), qr[u]);
              cmac_conj(acc2[e], h1.get(e), qr[u + 1]);
            }
          }
#pragma unroll
          for (int e = 0; e < PV; ++e) {
            acc[e] = cadd(acc[e], acc2[e]);
#pragma unroll
            for (int o = kSlabNSL; o < kWarp; o <<= 1) {
              acc[e].x += __shfl_xor_sync(0xffffffffu, acc[e].x, o);
              acc[e].y += __shfl_xor_sync(0xffffffffu, acc[e].y, o);
            }
          }
          if (crg == 0) {
            double2* dst = zp + ((size_t)(k & 1) * NW + warp) * W + ccol * PV;
#pragma unroll
            for (int e = 0; e < PV; ++e) dst[e] = acc[e];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&zfull[k & 1]);
        if (++stgC == NS) stgC = 0, phC ^= 1u;
      }
      if (k >= 1) {
        // ---------------------------------------------------------- (A) strip k - 1
        const uint32_t kk = k - 1;
        mbar_wait(&cfull[kk & 1], (kk >> 1) & 1);
        if (act) {
          const double2* cbi = cb + ((size_t)(kk & 1) * M + sd.rep) * W;
          double2 cr[kSlabNSL][PV];
#pragma unroll
          for (int s2 = 0; s2 < kSlabNSL; ++s2)
#pragma unroll
            for (int e = 0; e < PV; ++e) cr[s2][e] = cbi[s2 * PV + e];
          const uint32_t base = ring_w + stgA * stage_stride + lane * kSlabRB;
#pragma unroll
          for (int m = 0; m < RPL; ++m) {
            CK h[kSlabNSL];
#pragma unroll
            for (int s2 = 0; s2 < kSlabNSL; ++s2) h[s2].load(base + m * kWarp * kSlabRB + ((s2 ^ a_swz) * 16));
            double2 ae = make_double2(0.0, 0.0), ao = make_double2(0.0, 0.0);
#pragma unroll
            for (int s2 = 0; s2 < kSlabNSL; ++s2)
#pragma unroll
              for (int e = 0; e < PV; ++e) {
                if ((s2 * PV + e) & 1)
                  cmac(ao, h[s2].get(e), cr[s2][e]);
                else
                  cmac(ae, h[s2].get(e), cr[s2][e]);
              }
            wacc[m] = cadd(wacc[m], cadd(ae, ao));
          }
          __syncwarp();  // every lane has consumed the stage
          if (lane == 0 && kk + NS < nstrip) issue(kk + NS, stgA);
        }
        if (++stgA == NS) stgA = 0;
        if (x0 + kk + 1 == seg_endA || kk + 1 == nstrip) {  // flush this segment's w partial
          if (act) {
            const SweepDesc sg = segs[jA];
            const uint64_t slotp = cl - sk_owner(sg.unit0, U, NCl);
            double2* dst = wpart + sg.part_off + slotp * n_meas + sd.mrow0;
#pragma unroll
            for (int m = 0; m < RPL; ++m) {
              const uint32_t r = lane + kWarp * m;
              if (r < sd.nrows) dst[r] = wacc[m];
              wacc[m] = make_double2(0.0, 0.0);
            }
          }
          if (kk + 1 < nstrip) {
            ++jA;
            seg_endA = segs[jA].unit0 + segs[jA].n_strips;
          }
        }
      }
    }
  } else {
    // ============================================================ D warp
    const uint32_t i = lane / W, t = lane % W;
    const bool dl = i < M;
    const bool store = rank == 0;
    // this CTA's warps of replica i: slabs are ordered by replica, so a contiguous range
    uint32_t wlo = 0, whi = 0;
    if (dl) {
      wlo = NW;
      for (uint32_t w = 0; w < NW; ++w) {
        const uint32_t s2 = rank * NW + w;
        if (s2 < Ns && slabs[s2].rep == i) {
          wlo = min(wlo, w);
          whi = w + 1;
        }
      }
      if (whi == 0) wlo = 0;
    }
    const double m_rep = prm->m_rep, kappa = prm->kappa;
    const double kappa2_lo = kappa * kappa * (1.0 - 0x1p-40);
    const double inv_m = 1.0 / m_rep;
    const bool pow2_m = inv_m * m_rep == 1.0 && (__double_as_longlong(m_rep) & 0xfffffffffffffull) == 0;
    double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
    bool bad = false;
    uint32_t j = 0;
    if (nstrip > 0)
      while (j + 1 < N && segs[j + 1].unit0 <= x0) ++j;
    SweepDesc sg = nstrip > 0 ? segs[j] : SweepDesc{0, 0, 0, 0};
    // iterates of strip k (prefetched one strip ahead)
    double2 cpre = make_double2(0.0, 0.0), spre = cpre, vpre = cpre;
    auto fetch = [&](uint64_t x, const SweepDesc& g, uint32_t jj, double2& c_, double2& s_, double2& v_) {
      const uint32_t col = (uint32_t)(x - g.unit0) * W + t;
      if (dl && col < g.cols) {
        const uint32_t o = blocks[i * N + jj].vec_off + col;
        c_ = cv.c[o];
        s_ = cv.s[o];
        v_ = cv.v[blocks[jj].seg_off + col];
      } else {
        c_ = s_ = v_ = make_double2(0.0, 0.0);
      }
    };
    if (nstrip > 0) fetch(x0, sg, j, cpre, spre, vpre);
    const uint32_t xb_me = smem_u32(xb);
    for (uint32_t k = 0; k < nstrip; ++k) {
      const uint64_t x = x0 + k;
      const uint32_t col = (uint32_t)(x - sg.unit0) * W + t;
      const bool dcol = dl && col < sg.cols;
      const uint32_t jc = j;
      // prefetch strip k + 1
      double2 cn = make_double2(0.0, 0.0), sn = cn, vn1 = cn;
      SweepDesc sgn = sg;
      uint32_t jn = j;
      if (k + 1 < nstrip) {
        if (x + 1 == sg.unit0 + sg.n_strips) sgn = segs[++jn];
        fetch(x + 1, sgn, jn, cn, sn, vn1);
      }
      const uint32_t kb = k & 1;
      mbar_wait(&zfull[kb], (k >> 1) & 1);
      double2 z = make_double2(0.0, 0.0);
      {
        const double2* zs = zp + (size_t)kb * NW * W + t;
        for (uint32_t w = wlo; w < whi; ++w) z = cadd(z, zs[(size_t)w * W]);
      }
      if (C > 1) {
        const uint32_t me = xb_me + (uint32_t)((((size_t)kb * C + rank) * M + (dl ? i : 0)) * W + t) * 16;
        if (dl)
          for (uint32_t r2 = 0; r2 < C; ++r2) st_cluster_d2(mapa(me, r2), z);
        const uint32_t xf = smem_u32(&xfull[kb]);
        for (uint32_t r2 = 0; r2 < C; ++r2) mbar_arrive_remote(mapa(xf, r2));
        mbar_wait_cluster(&xfull[kb], (k >> 1) & 1);
        z = make_double2(0.0, 0.0);
        if (dl) {
          const double2* xs = xb + ((size_t)kb * C * M + i) * W + t;
          for (uint32_t r2 = 0; r2 < C; ++r2) z = cadd(z, xs[(size_t)r2 * M * W]);
        }
      }
      // (D) u = c + z; mean over replicas of (u + s) in ascending i; v; s; next c
      const double2 u = cadd(cpre, z);
      const double2 a = cadd(u, spre);
      double2 mean = make_double2(0.0, 0.0);
      for (uint32_t i2 = 0; i2 < M; ++i2) {
        const double ax = __shfl_sync(0xffffffffu, a.x, i2 * W + t);
        const double ay = __shfl_sync(0xffffffffu, a.y, i2 * W + t);
        mean = cadd(mean, make_double2(ax, ay));
      }
      mean = pow2_m ? make_double2(mean.x * inv_m, mean.y * inv_m) : make_double2(mean.x / m_rep, mean.y / m_rep);
      const double2 vnew = soft_threshold_fast(mean, kappa, kappa2_lo);
      const double2 snew = csub(cadd(spre, u), vnew);
      const double2 cnew = csub(vnew, snew);
      if (dl) cb[((size_t)kb * M + i) * W + t] = dcol ? cnew : make_double2(0.0, 0.0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&cfull[kb]);
      if (store && dcol) {  // off the critical path
        const uint32_t o = blocks[i * N + jc].vec_off + col;
        bad |= !cfinite(u);
        cv.u[o] = u;
        cv.s[o] = snew;
        cv.c[o] = cnew;
        rp2 += cabs2(csub(u, vnew));
        if (i == 0) {
          const uint32_t so = blocks[jc].seg_off + col;
          cv.vprev[so] = vpre;
          cv.v[so] = vnew;
          rd2 += cabs2(csub(vnew, vpre));
          l1 += hypot(vnew.x, vnew.y);
        }
      }
      cpre = cn;
      spre = sn;
      vpre = vn1;
      sg = sgn;
      j = jn;
    }
    if (store) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rp2 += __shfl_xor_sync(0xffffffffu, rp2, o);
        rd2 += __shfl_xor_sync(0xffffffffu, rd2, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      const bool anybad = __any_sync(0xffffffffu, bad);
      if (lane == 0) {
        red[cl] = rp2;
        red[NCl + cl] = rd2;
        red[2 * NCl + cl] = l1;
        if (anybad) st->nonfinite = 1u;
      }
    }
  }
  if (C > 1) cluster_sync_all();  // no CTA leaves while a peer may still write its SMEM
}

// One-time re-layout into slabs: Hs[x][sl][rr][pc] (16-byte chunks) holds logical chunk
// pc ^ ((rr >> 1) & 3) of row lrow0(sl) + rr of block (rep(sl), j(x)), strip x; zero past
// the slab's valid rows or the segment's last column.  Setup only.
template <typename S>
__global__ void slab_h_kernel(const S* __restrict__ H, const MatDesc* __restrict__ hm, const SweepDesc* __restrict__ segs,
                              const SlabDesc* __restrict__ slabs, uint32_t N, uint32_t Ns, uint32_t RPW,
                              uint64_t total_chunks, S* __restrict__ Hs) {
  constexpr int PV = 16 / (int)sizeof(S);
  constexpr int W = kSlabNSL * PV;
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total_chunks;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t pc = (uint32_t)(idx % kSlabNSL);
    const uint64_t r1 = idx / kSlabNSL;
    const uint32_t rr = (uint32_t)(r1 % RPW);
    const uint64_t r2 = r1 / RPW;
    const uint32_t sl = (uint32_t)(r2 % Ns);
    const uint64_t x = r2 / Ns;
    const uint32_t lc = pc ^ ((rr >> 1) & 3);
    uint32_t j = 0;
    while (j + 1 < N && segs[j + 1].unit0 <= x) ++j;
    const SlabDesc sd = slabs[sl];
    const MatDesc md = hm[sd.rep * N + j];
#pragma unroll
    for (int e = 0; e < PV; ++e) {
      const uint32_t col = (uint32_t)(x - segs[j].unit0) * W + lc * PV + e;
      S val;
      val.x = 0;
      val.y = 0;
      if (rr < sd.nrows && col < segs[j].cols) val = H[md.a_off + (uint64_t)(sd.lrow0 + rr) * md.ld + col];
      Hs[idx * PV + e] = val;
    }
  }
}

}  // namespace admm
