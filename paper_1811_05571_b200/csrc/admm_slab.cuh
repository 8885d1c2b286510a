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

// Slab row width RB (bytes of one strip row): 64 (4 c128 / 8 c64 columns per strip), 32 or
// 16 (narrower strips for segments with many rows: the whole strip still fits one CTA's ring).  16-byte chunk c of row r is stored at
// position c ^ slab_swz<RB>(r): both SMEM access patterns below are then conflict-free.
template <int RB>
__host__ __device__ constexpr uint32_t slab_swz(uint32_t row) {
  return (row / (128 / RB)) % (RB / 16);
}
constexpr int kSlabMaxW = 16;        // compute warps per CTA (+ D warps)
constexpr int kSlabThreads = (kSlabMaxW + 4) * kWarp;  // + up to 4 D warps; 20 warps keep the 96-register cap

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
// Asynchronous 16-byte store into a peer CTA's shared memory that completes (tx bytes)
// on the peer's mbarrier: no release fence, so it never waits for this thread's
// outstanding global stores.
__device__ __forceinline__ void st_async_d2(uint32_t a, double2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(a), "d"(v.x),
               "d"(v.y), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITC_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAITC_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// mbarrier / bulk-copy helpers on 32-bit shared addresses (computed once per thread).
__device__ __forceinline__ void mbar_wait_s(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITU_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAITU_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// ... with a suspend-time hint: the warp sleeps in the barrier unit instead of re-polling (the
// compute warps' wait for c re-polled ~12 times per strip, issue slots the other warps want)
__device__ __forceinline__ void mbar_wait_hint_s(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITH_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra WAITH_%=;\n}\n" ::"r"(a),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

// mbarrier wait with a long suspend-time hint: the warp sleeps until the phase completes
// instead of re-polling.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITS_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra WAITS_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

// Bulk shared -> global copy (async proxy: no LSU store traffic from the issuing warp).
__device__ __forceinline__ void bulk_s2g(void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  __device__ __forceinline__ void ld(const unsigned char* p) { v = *reinterpret_cast<const double2*>(p); }
  __device__ __forceinline__ double2 get(int) const { return v; }
};
template <>
struct Chunk<float2> {
  static constexpr int PV = 2;
  float4 v;
  __device__ __forceinline__ void ld(const unsigned char* p) { v = *reinterpret_cast<const float4*>(p); }
  __device__ __forceinline__ double2 get(int e) const {
    return e == 0 ? make_double2((double)v.x, (double)v.y) : make_double2((double)v.z, (double)v.w);
  }
};

constexpr int kSlabZB = 4;   // z-partial / c / barrier slots (lag L <= kSlabZB - 1)
constexpr int kSlabXB = 8;   // cluster-exchange slots
constexpr int kSlabPF = 3;   // D warp: its strips of iterates prefetched ahead (cp.async)
constexpr int kSlabMaxD = 4; // D warps (config 2: 4 -> 94.8 us, 2 -> 97.1 us, 1 -> 103 us)

__host__ __device__ inline size_t slab_smem_bytes(uint32_t ns, uint32_t nw, uint32_t nd, uint32_t rpw, uint32_t rb,
                                                  uint32_t C, uint32_t M, uint32_t W, uint32_t N) {
  return (size_t)ns * nw * rpw * rb                             // ring
         + (size_t)nw * ns * sizeof(uint64_t)                   // per-warp full barriers
         + (2 * kSlabZB + kSlabXB) * sizeof(uint64_t)           // zfull, cfull, xfull
         + (size_t)kSlabZB * nw * W * sizeof(double2)           // z partials per warp
         + (size_t)kSlabXB * C * M * W * sizeof(double2)        // cluster exchange
         + (size_t)kSlabZB * M * W * sizeof(double2)            // c of the strip
         + (size_t)nd * (kSlabPF + 1) * 3 * kWarp * sizeof(double2)  // prefetched c, s, v
         + (size_t)(nw + nd) * 4 * sizeof(double)               // per-warp residual partials
         + (size_t)N * sizeof(SweepDesc) + (2 * (size_t)M * N + N) * sizeof(uint32_t);  // descriptor tables
}

// Valid (lag, D warps) pairs.  Slot reuse: a compute warp writes z partials of strip
// k + kSlabZB only after it has waited for c of every strip <= k + kSlabZB - 1 - L, so the
// D warp of strip k has read them (kSlabZB >= L + 1), and a D warp overwrites c of strip k
// only after every compute warp has passed (A) of strip k (same bound).  A peer's D warp
// writes exchange slot k % kSlabXB for strip k + kSlabXB only after this CTA sent its
// partials for some strip j in (k, k + kSlabXB - 1 - L] owned by the same D warp as k,
// i.e. after that D warp finished strip k: kSlabXB - 1 - L >= ND.
__host__ __device__ inline bool slab_lag_ok(uint32_t L, uint32_t ND) {
  return L >= 1 && L <= kSlabZB - 1 && kSlabXB - 1 - L >= ND;
}

// RPL = rows per lane in (A) = RPW / 32.  Launched as NCl clusters of C CTAs, block
// (NW + ND) x 32 threads: warps 0..NW-1 compute, warps NW.. are the D warps (strip k is
// updated by D warp k % ND).  L = lag of the (A) pass behind the (C) pass, in strips.
// 20 warps x 32 lanes: the register allocation granularity (4 warps) caps this at 96
// registers per thread (65536 / (20 x 32)).
// MAXW = compute warps the instantiation is launched with at most: (MAXW + 4) x 32 threads
// set the register cap (16 -> 96 registers, 12 -> 128, 8 -> 168).
template <typename S, int RPL, int RB, bool kTrace, int MAXW = kSlabMaxW>
__global__ void __launch_bounds__((MAXW + kSlabMaxD) * kWarp, 1)
sweep_slab_kernel(const S* __restrict__ Hs, const SlabDesc* __restrict__ slabs, const BlockDesc* __restrict__ blocks,
                  const SweepDesc* __restrict__ segs, uint32_t M, uint32_t N, uint32_t n_meas, uint64_t U, uint32_t NS,
                  uint32_t L, uint32_t Ns, uint32_t NW, const double2* __restrict__ q, ColVecs cv,
                  double2* __restrict__ wpart, const Params* __restrict__ prm, double* __restrict__ red, IterState* st,
                  unsigned long long* __restrict__ trace) {  // diagnostics (ADMM_B200_SLAB_TRACE), else null
  using CK = Chunk<S>;
  constexpr int PV = CK::PV;
  constexpr int NSL = RB / 16;              // 16-byte chunks per row
  constexpr int W = NSL * PV;               // columns per strip
  constexpr int RPW = RPL * kWarp;          // rows per slab
  constexpr int SLAB_B = RPW * RB;          // bytes per slab
  constexpr int CRG = kWarp / NSL;          // (C) rows per warp instruction
  constexpr int CNU = RPW / CRG;            // (C) instructions per slab
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t NWT = blockDim.x / kWarp, ND = NWT - NW;
  const uint32_t C = cluster_size();
  unsigned char* ring = smem_raw;
  uint64_t* fullb = reinterpret_cast<uint64_t*>(ring + (size_t)NS * NW * SLAB_B);  // [NW][NS]
  uint64_t* zfull = fullb + (size_t)NW * NS;              // [kSlabZB]
  uint64_t* cfull = zfull + kSlabZB;                      // [kSlabZB]
  uint64_t* xfull = cfull + kSlabZB;                      // [kSlabXB]
  double2* zp = reinterpret_cast<double2*>(xfull + kSlabXB);  // [kSlabZB][NW][W]
  double2* xb = zp + (size_t)kSlabZB * NW * W;            // [kSlabXB][C][M][W]
  double2* cb = xb + (size_t)kSlabXB * C * M * W;         // [kSlabZB][M][W]
  double2* pf = cb + (size_t)kSlabZB * M * W;             // [ND][kSlabPF + 1][3][32]
  double* wred = reinterpret_cast<double*>(pf + (size_t)ND * (kSlabPF + 1) * 3 * kWarp);  // [NWT][4]
  // descriptor tables in SMEM: nothing on the per-strip path reads global metadata
  SweepDesc* tseg = reinterpret_cast<SweepDesc*>(wred + (size_t)NWT * 4);  // [N]
  uint32_t* tvec = reinterpret_cast<uint32_t*>(tseg + N);                  // [M][N] vec_off
  uint32_t* tmvec = tvec + (size_t)M * N;                                  // [M][N] mvec_off
  uint32_t* tsego = tmvec + (size_t)M * N;                                 // [N] seg_off
  for (uint32_t b = threadIdx.x; b < M * N; b += blockDim.x) {
    tvec[b] = blocks[b].vec_off;
    tmvec[b] = blocks[b].mvec_off;
  }
  for (uint32_t b = threadIdx.x; b < N; b += blockDim.x) {
    tseg[b] = segs[b];
    tsego[b] = blocks[b].seg_off;
  }
  double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;  // residual partials (rank 0 D warps)
  bool bad = false;

  const uint32_t rank = cluster_rank();
  const uint64_t NCl = cluster_count(), cl = cluster_id();
  const uint64_t x0 = sk_lo(cl, U, NCl), xe = sk_lo(cl + 1, U, NCl);
  const uint32_t nstrip = (uint32_t)(xe - x0);
  // warp-uniform by construction (admm_common.cuh warp_index): bare SHFLs below
  const uint32_t warp = (uint32_t)warp_index(), lane = threadIdx.x % kWarp;
  // diagnostics: per-strip timestamps of compute warp 0 and the D warps (first 64 strips)
  auto mark = [&](uint32_t k, int ev) {
    if (kTrace && lane == 0 && k < 32 && (warp == 0 || warp >= NW))
      trace[((uint64_t)blockIdx.x * 64 + k) * 8 + ev] = clock64();
  };

  if (kTrace && threadIdx.x == 0) trace[((uint64_t)blockIdx.x * 64) * 8 + 6] = clock64();  // kernel entry
  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < NW * NS; ++b) mbar_init(&fullb[b], 1);
    for (int b = 0; b < kSlabZB; ++b) {
      mbar_init(&zfull[b], NW);
      mbar_init(&cfull[b], 1);
    }
    for (int b = 0; b < kSlabXB; ++b) mbar_init(&xfull[b], 1);  // + C x M x W x 16 tx bytes
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (C > 1)
    cluster_sync_all();  // peers' barriers initialised before any remote arrive
  else
    __syncthreads();

  if (warp < NW) {
    // ============================================================ compute warp
    // Static data first (H and the tables never change during a solve): the first NS
    // stages stream in while the previous kernel of the chain finishes (PDL).
    const uint32_t sl = rank * NW + warp;
    const bool act = sl < Ns;
    SlabDesc sd{0, 0, 0, 0};
    if (act) sd = slabs[sl];
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const uint32_t full_s = smem_u32(fullb) + warp * NS * 8;      // this warp's full barriers
    const uint32_t zfull_s = smem_u32(zfull), cfull_s = smem_u32(cfull);
    const uint32_t ring_off = warp * SLAB_B;                          // + stage * NW * SLAB_B
    const uint32_t ring_s = smem_u32(ring) + ring_off;
    const uint32_t stage_stride = NW * SLAB_B;
    const unsigned char* src0 = reinterpret_cast<const unsigned char*>(Hs) + ((x0 * Ns) + sl) * (uint64_t)SLAB_B;
    const uint64_t strip_stride = (uint64_t)Ns * SLAB_B;
    auto issue = [&](uint32_t k, uint32_t stg) {
      mbar_expect_tx_s(full_s + stg * 8, SLAB_B);
      bulk_g2s_s(ring_s + stg * stage_stride, src0 + k * strip_stride, SLAB_B, full_s + stg * 8, pol);
    };
    if (act && lane == 0)
      for (uint32_t k = 0; k < NS && k < nstrip; ++k) issue(k, k);
    uint32_t j = 0;
    if (nstrip > 0)
      while (j + 1 < N && tseg[j + 1].unit0 <= x0) ++j;
    uint32_t jA = j;
    // local strip index where the current segment ends, (C) side and (A) side (32-bit:
    // the strip loop runs at the 96-register cap)
    uint32_t kend = (nstrip > 0) ? (uint32_t)(tseg[j].unit0 + tseg[j].n_strips - x0) : 0;
    uint32_t kendA = kend;
    pdl_enter();  // q of the previous kernels is visible from here on
    if (kTrace && warp == 0 && lane == 0) trace[((uint64_t)blockIdx.x * 64 + 1) * 8 + 6] = clock64();

    // (C) lane geometry: rows crg + CRG u, logical chunk ccol at physical ccol ^ swz
    const uint32_t crg = lane / NSL, ccol = lane % NSL;
    const uint32_t c_off = crg * RB + ((ccol ^ slab_swz<RB>(crg)) * 16);  // swz(crg + CRG u) = swz(crg)
    // (A) lane geometry: rows lane + 32 m, logical chunk s at physical s ^ swz
    const uint32_t a_swz = slab_swz<RB>(lane);  // = swz(lane + 32 m)
    double2 qr[CNU];
    auto load_q = [&](uint32_t jj) {
      const double2* qb = q + tmvec[sd.rep * N + jj] + sd.lrow0;
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
    uint32_t stgC = 0, phC = 0, stgA = 0;
    const double2* cb_rep = cb + (size_t)sd.rep * W;
    double2* zp_w = zp + (size_t)warp * W + ccol * PV;

    // flush of a finished segment's w partial, then the next segment ((A) side)
    auto flush_w = [&](uint32_t kk) {
      if (kk + 1 == kendA || kk + 1 == nstrip) {
        if (act) {
          const SweepDesc sg = tseg[jA];
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
          kendA = (uint32_t)(tseg[jA].unit0 + tseg[jA].n_strips - x0);
        }
      }
    };

    long long t_full = 0, t_c = 0, t_n = 0, t_loop0 = 0;
    if (kTrace) t_loop0 = clock64();
    for (uint32_t k = 0; k < nstrip + L; ++k) {
      if (NSL == 1 && k < nstrip && k >= L) {
        // ------------------------------------------- (C) strip k and (A) strip k - L, fused
        // 16-byte strip rows: both passes map lane -> rows lane + 32 m, so one loop feeds the
        // z partial of strip k and the w accumulators from strip k - L; their loads, widenings
        // and FMAs interleave (the two passes alone are dependent chains: latency-bound with
        // five warps per scheduler).  The z partial is reduce-scattered over the lanes
        // (6 shuffle rounds of one double instead of 5 rounds of four).
        const uint32_t kk = k - L;
        if (k == kend) {
          ++j;
          kend = (uint32_t)(tseg[j].unit0 + tseg[j].n_strips - x0);
          load_q(j);
        }
        mark(k, 0);  // fused timeline: 0 loop top, 2 stage landed, 3 c landed, 1 end
        long long tw0 = 0;
        if (kTrace) tw0 = clock64();
        if (act) mbar_wait_s(full_s + stgC * 8, phC);
        mark(k, 2);
        long long tw1 = 0;
        if (kTrace) tw1 = clock64();
        mbar_wait_hint_s(cfull_s + (kk % kSlabZB) * 8, (kk / kSlabZB) & 1);
        mark(k, 3);
        if (kTrace) {  // per-warp totals (registers; written once at the end of the loop)
          const long long tw2 = clock64();
          t_full += tw1 - tw0;
          t_c += tw2 - tw1;
          ++t_n;
        }
        if (act) {
          const double2* cbi = cb_rep + (size_t)(kk % kSlabZB) * M * W;
          double2 cr[PV];
#pragma unroll
          for (int e = 0; e < PV; ++e) cr[e] = cbi[e];
          const unsigned char* baseC = ring + ring_off + stgC * stage_stride + lane * RB;
          const unsigned char* baseA = ring + ring_off + stgA * stage_stride + lane * RB;
          double2 acc[2][PV];
#pragma unroll
          for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
            for (int e = 0; e < PV; ++e) acc[a2][e] = make_double2(0.0, 0.0);
          // rows per batch (register cap)
          constexpr int FB = (MAXW <= 12 && RPL % 4 == 0) ? 4 : RPL % 3 == 0 ? 3 : RPL % 2 == 0 ? 2 : 1;
#pragma unroll
          for (int m0 = 0; m0 < RPL; m0 += FB) {
            CK hc[FB], ha[FB];
#pragma unroll
            for (int m = 0; m < FB; ++m) {
              hc[m].ld(baseC + (m0 + m) * kWarp * RB);
              ha[m].ld(baseA + (m0 + m) * kWarp * RB);
            }
#pragma unroll
            for (int m = 0; m < FB; ++m) {
#pragma unroll
              for (int e = 0; e < PV; ++e) cmac_conj(acc[(m0 + m) & 1][e], hc[m].get(e), qr[m0 + m]);
              double2 ae = make_double2(0.0, 0.0);
#pragma unroll
              for (int e = 0; e < PV; ++e) cmac(ae, ha[m].get(e), cr[e]);
              wacc[m0 + m] = cadd(wacc[m0 + m], ae);
            }
          }
          __syncwarp();  // every lane has consumed stage stgA
          if (lane == 0 && kk + NS < nstrip) issue(kk + NS, stgA);
          // reduce-scatter of the 2 PV doubles of z over the 32 lanes
          double v0, v1 = 0.0;
          if constexpr (PV == 2) {
            const double2 z0 = cadd(acc[0][0], acc[1][0]), z1 = cadd(acc[0][1], acc[1][1]);
            const bool hi = (lane & 16) != 0;
            const double sx = hi ? z0.x : z1.x, sy = hi ? z0.y : z1.y;
            v0 = (hi ? z1.x : z0.x) + __shfl_xor_sync(0xffffffffu, sx, 16);
            v1 = (hi ? z1.y : z0.y) + __shfl_xor_sync(0xffffffffu, sy, 16);
          } else {
            const double2 z0 = cadd(acc[0][0], acc[1][0]);
            v0 = z0.x;
            v1 = z0.y;
          }
          constexpr int O1 = PV == 2 ? 8 : 16;  // x / y split
          {
            const bool hi = (lane & O1) != 0;
            const double snd = hi ? v0 : v1;
            v0 = (hi ? v1 : v0) + __shfl_xor_sync(0xffffffffu, snd, O1);
          }
#pragma unroll
          for (int o = O1 / 2; o > 0; o >>= 1) v0 += __shfl_xor_sync(0xffffffffu, v0, o);
          if ((lane & (O1 - 1)) == 0)  // lane = (column e, component) * O1
            reinterpret_cast<double*>(zp + (size_t)(k % kSlabZB) * NW * W + (size_t)warp * W)[lane / O1] = v0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_s(zfull_s + (k % kSlabZB) * 8);
        mark(k, 1);
        if (++stgC == NS) stgC = 0, phC ^= 1u;
        if (++stgA == NS) stgA = 0;
        flush_w(kk);
        continue;
      }
      if (k < nstrip) {
        // ---------------------------------------------------------- (C) strip k
        if (k == kend) {
          ++j;
          kend = (uint32_t)(tseg[j].unit0 + tseg[j].n_strips - x0);
          load_q(j);
        }
        if (act) {
          mbar_wait_s(full_s + stgC * 8, phC);
          mark(k, 0);
          const unsigned char* base = ring + ring_off + stgC * stage_stride + c_off;
          double2 acc[4][PV];
#pragma unroll
          for (int a4 = 0; a4 < 4; ++a4)
#pragma unroll
            for (int e = 0; e < PV; ++e) acc[a4][e] = make_double2(0.0, 0.0);
          // loads in flight per batch (register cap); CB divides CNU
          constexpr int CB = CNU % 4 == 0 ? 4 : CNU % 3 == 0 ? 3 : CNU <= 4 ? CNU : 1;
#pragma unroll
          for (int u0 = 0; u0 < CNU; u0 += CB) {
            CK h[CB];
#pragma unroll
            for (int u = 0; u < CB; ++u) h[u].ld(base + (u0 + u) * CRG * RB);
#pragma unroll
            for (int u = 0; u < CB; ++u)
#pragma unroll
              for (int e = 0; e < PV; ++e) cmac_conj(acc[u & 3][e], h[u].get(e), qr[u0 + u]);
          }
#pragma unroll
          for (int e = 0; e < PV; ++e) {
            double2 z = cadd(cadd(acc[0][e], acc[1][e]), cadd(acc[2][e], acc[3][e]));
#pragma unroll
            for (int o = NSL; o < kWarp; o <<= 1) {
              z.x += __shfl_xor_sync(0xffffffffu, z.x, o);
              z.y += __shfl_xor_sync(0xffffffffu, z.y, o);
            }
            if (crg == 0) zp_w[(size_t)(k % kSlabZB) * NW * W + e] = z;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_s(zfull_s + (k % kSlabZB) * 8);
        mark(k, 1);
        if (++stgC == NS) stgC = 0, phC ^= 1u;
      }
      if (k >= L) {
        // ---------------------------------------------------------- (A) strip k - L
        const uint32_t kk = k - L;
        mbar_wait_hint_s(cfull_s + (kk % kSlabZB) * 8, (kk / kSlabZB) & 1);
        mark(kk, 2);
        if (act) {
          const double2* cbi = cb_rep + (size_t)(kk % kSlabZB) * M * W;
          double2 cr[NSL][PV];
#pragma unroll
          for (int s2 = 0; s2 < NSL; ++s2)
#pragma unroll
            for (int e = 0; e < PV; ++e) cr[s2][e] = cbi[s2 * PV + e];
          const unsigned char* base = ring + ring_off + stgA * stage_stride + lane * RB;
          CK h[RPL][NSL];
#pragma unroll
          for (int m = 0; m < RPL; ++m)
#pragma unroll
            for (int s2 = 0; s2 < NSL; ++s2) h[m][s2].ld(base + m * kWarp * RB + ((s2 ^ a_swz) * 16));
#pragma unroll
          for (int m = 0; m < RPL; ++m) {
            double2 ae = make_double2(0.0, 0.0), ao = make_double2(0.0, 0.0);
#pragma unroll
            for (int s2 = 0; s2 < NSL; ++s2)
#pragma unroll
              for (int e = 0; e < PV; ++e) {
                if ((s2 * PV + e) & 1)
                  cmac(ao, h[m][s2].get(e), cr[s2][e]);
                else
                  cmac(ae, h[m][s2].get(e), cr[s2][e]);
              }
            wacc[m] = cadd(wacc[m], cadd(ae, ao));
          }
          __syncwarp();  // every lane has consumed the stage
          if (lane == 0 && kk + NS < nstrip) issue(kk + NS, stgA);
          mark(kk, 3);
        }
        if (++stgA == NS) stgA = 0;
        flush_w(kk);
      }
    }
    if (kTrace && lane == 0) {  // slots 32..: per compute warp (loop cycles, stage wait, c wait, fused strips)
      unsigned long long* o = trace + ((uint64_t)blockIdx.x * 64 + 32 + warp) * 8;
      o[0] = (unsigned long long)(clock64() - t_loop0);
      o[1] = (unsigned long long)t_full;
      o[2] = (unsigned long long)t_c;
      o[3] = (unsigned long long)t_n;
    }
  } else {
    // ============================================================ D warps
    const uint32_t dw = warp - NW;
    const uint32_t i = lane / W, t = lane % W;
    const bool dl = i < M;
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
    pdl_enter();  // c, s, v, kappa of the previous kernels are visible from here on
    const double m_rep = prm->m_rep, kappa = prm->kappa;
    const double kappa2_lo = kappa * kappa * (1.0 - 0x1p-40), kappa2_hi = kappa * kappa * (1.0 + 0x1p-40);
    const double inv_m = 1.0 / m_rep;
    const bool pow2_m = inv_m * m_rep == 1.0 && (__double_as_longlong(m_rep) & 0xfffffffffffffull) == 0;
    // this D warp's strips dw, dw + ND, ...: the n-th is prefetched (cp.async, zero-filled
    // past the segment) into pfw[n % (kSlabPF + 1)] kSlabPF strips ahead
    double2* pfw = pf + (size_t)dw * (kSlabPF + 1) * 3 * kWarp + lane;
    auto seg_of = [&](uint64_t x, uint32_t& jj) {
      while (jj + 1 < N && tseg[jj + 1].unit0 <= x) ++jj;
    };
    uint32_t jf = 0;
    auto fetch = [&](uint32_t n) {
      const uint32_t kf = dw + n * ND;
      if (kf < nstrip) {
        const uint64_t x = x0 + kf;
        seg_of(x, jf);
        const SweepDesc g = tseg[jf];
        const uint32_t col = (uint32_t)(x - g.unit0) * W + t;
        const bool ok = dl && col < g.cols;
        const uint32_t o = tvec[(dl ? i : 0) * N + jf] + (ok ? col : 0);
        const uint32_t so = tsego[jf] + (ok ? col : 0);
        double2* dst = pfw + (size_t)(n % (kSlabPF + 1)) * 3 * kWarp;
        cpa(dst, cv.c + o, ok);
        cpa(dst + kWarp, cv.s + o, ok);
        cpa(dst + 2 * kWarp, cv.v + so, ok);
      }
      cpa_commit();
    };
    for (uint32_t n = 0; n < kSlabPF; ++n) fetch(n);
    uint32_t j = 0;
    const uint32_t xb_me = smem_u32(xb);
    uint32_t n = 0;
    for (uint32_t k = dw; k < nstrip; k += ND, ++n) {
      const uint64_t x = x0 + k;
      seg_of(x, j);
      const uint32_t col = (uint32_t)(x - tseg[j].unit0) * W + t;
      const bool dcol = dl && col < tseg[j].cols;
      const uint32_t kb = k % kSlabZB;
      cpa_wait<kSlabPF - 1>();  // this strip's iterates
      const double2* pk = pfw + (size_t)(n % (kSlabPF + 1)) * 3 * kWarp;
      const double2 cpre = pk[0], spre = pk[kWarp], vpre = pk[2 * kWarp];
      // tall strips (16-byte rows): a D warp is idle ~90% of a strip period and its spin loop (~220
      // polls per strip) takes issue slots from the compute warps, so it sleeps in the barrier unit;
      // short strips keep the spin (the hint costs config 1, where the wake-up latency shows, 5%)
      if constexpr (RB == 16)
        mbar_wait_sleep(&zfull[kb], (k / kSlabZB) & 1);
      else
        mbar_wait(&zfull[kb], (k / kSlabZB) & 1);
      mark(k, 4);
      double2 z = make_double2(0.0, 0.0);
      {
        // (a pairwise tree over 16 predicated loads measured slower than this loop: 5,729 vs
        // 5,823 it/s on config 3 -- the extra LDS / selects cost the compute warps issue slots)
        const double2* zs = zp + (size_t)kb * NW * W + t;
        for (uint32_t w = wlo; w < whi; ++w) z = cadd(z, zs[(size_t)w * W]);
      }
      if (C > 1) {
        // every rank sends its CTA partial to every rank (itself included) with st.async;
        // the local arrive.expect_tx arms this strip's phase for the C x M x W x 16 bytes
        const uint32_t xs_b = k % kSlabXB;
        const uint32_t xf = smem_u32(&xfull[xs_b]);
        if (lane == 0) mbar_expect_tx(&xfull[xs_b], C * M * W * 16);
        const uint32_t me = xb_me + (uint32_t)((((size_t)xs_b * C + rank) * M + (dl ? i : 0)) * W + t) * 16;
        if (dl)
          for (uint32_t r2 = 0; r2 < C; ++r2) st_async_d2(mapa(me, r2), z, mapa(xf, r2));
        mbar_wait_cluster(&xfull[xs_b], (k / kSlabXB) & 1);
        z = make_double2(0.0, 0.0);
        if (dl) {
          const double2* xs = xb + ((size_t)xs_b * C * M + i) * W + t;
          for (uint32_t r2 = 0; r2 < C; ++r2) z = cadd(z, xs[(size_t)r2 * M * W]);
        }
      }
      // (D) u = c + z; mean over replicas of (u + s) in ascending i; v; s; next c
      const double2 u = cadd(cpre, z);
      const double2 a = cadd(u, spre);
      double2 mean;
      if (M == 1) {
        mean = a;
      } else {
        mean = make_double2(0.0, 0.0);
        for (uint32_t i2 = 0; i2 < M; ++i2) {
          const double ax = __shfl_sync(0xffffffffu, a.x, i2 * W + t);
          const double ay = __shfl_sync(0xffffffffu, a.y, i2 * W + t);
          mean = cadd(mean, make_double2(ax, ay));
        }
      }
      mean = pow2_m ? make_double2(mean.x * inv_m, mean.y * inv_m) : make_double2(mean.x / m_rep, mean.y / m_rep);
      const double2 vnew = soft_threshold_lat(mean, kappa, kappa2_lo, kappa2_hi);
      const double2 snew = csub(cadd(spre, u), vnew);
      const double2 cnew = csub(vnew, snew);
      if (dl) cb[((size_t)kb * M + i) * W + t] = dcol ? cnew : make_double2(0.0, 0.0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&cfull[kb]);
      mark(k, 5);
      fetch(n + kSlabPF);  // into the slot of this warp's previous strip (consumed)
      if (rank == 0 && dcol) {  // off the critical path
        const uint32_t o = tvec[i * N + j] + col;
        bad |= !cfinite(u);
        cv.u[o] = u;
        cv.s[o] = snew;
        cv.c[o] = cnew;
        rp2 += cabs2(csub(u, vnew));
        if (i == 0) {
          const uint32_t so = tsego[j] + col;
          cv.vprev[so] = vpre;
          cv.v[so] = vnew;
          rd2 += cabs2(csub(vnew, vpre));
          l1 += hypot(vnew.x, vnew.y);
        }
      }
    }
    cpa_wait<0>();
  }
  if (kTrace && warp == 0 && lane == 0) trace[((uint64_t)blockIdx.x * 64 + 1) * 8 + 7] = clock64();
  // residual partials: warp sums, then the warps in order (rank 0 carries them)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rp2 += __shfl_xor_sync(0xffffffffu, rp2, o);
    rd2 += __shfl_xor_sync(0xffffffffu, rd2, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  const bool anybad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    wred[warp * 4 + 0] = rp2;
    wred[warp * 4 + 1] = rd2;
    wred[warp * 4 + 2] = l1;
    wred[warp * 4 + 3] = anybad ? 1.0 : 0.0;
  }
  __syncthreads();
  if (rank == 0 && threadIdx.x == 0) {
    double a = 0.0, d = 0.0, l = 0.0;
    bool nb = false;
    for (uint32_t w = NW; w < NWT; ++w) {
      a += wred[w * 4 + 0];
      d += wred[w * 4 + 1];
      l += wred[w * 4 + 2];
      nb |= wred[w * 4 + 3] != 0.0;
    }
    red[cl] = a;
    red[NCl + cl] = d;
    red[2 * NCl + cl] = l;
    if (nb) st->nonfinite = 1u;
  }
  if (C > 1) cluster_sync_all();  // no CTA leaves while a peer may still write its SMEM
  if (kTrace && threadIdx.x == 0) trace[((uint64_t)blockIdx.x * 64) * 8 + 7] = clock64();  // kernel exit
}

// One-time re-layout into slabs: Hs[x][sl][rr][pc] (16-byte chunks) holds logical chunk
// pc ^ slab_swz(rr) of row lrow0(sl) + rr of block (rep(sl), j(x)), strip x; zero past
// the slab's valid rows or the segment's last column.  Setup only.
template <typename S, int RB>
__global__ void slab_h_kernel(const S* __restrict__ H, const MatDesc* __restrict__ hm, const SweepDesc* __restrict__ segs,
                              const SlabDesc* __restrict__ slabs, uint32_t N, uint32_t Ns, uint32_t RPW,
                              uint64_t total_chunks, S* __restrict__ Hs) {
  constexpr int PV = 16 / (int)sizeof(S);
  constexpr int NSL = RB / 16;
  constexpr int W = NSL * PV;
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total_chunks;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t pc = (uint32_t)(idx % NSL);
    const uint64_t r1 = idx / NSL;
    const uint32_t rr = (uint32_t)(r1 % RPW);
    const uint64_t r2 = r1 / RPW;
    const uint32_t sl = (uint32_t)(r2 % Ns);
    const uint64_t x = r2 / Ns;
    const uint32_t lc = pc ^ slab_swz<RB>(rr);
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
