// admm_tile.cuh — SMEM-resident single-HBM-pass sweep over a strip-major copy of H.
//
// Same iteration as sweep_kernel (admm_sweep.cuh: (C) z = H^H q, (D) the column update
// of solvers.hpp:227-246 / 374-391, (A) the next w = H c), but H is re-laid out once at
// setup as column strips of W columns x all n_meas rows, each strip contiguous in HBM
// (Ht[x][row][0..W), zero-padded past a segment's last column).  A strip arrives as
// 32-row tasks (32 * RB bytes each), one cp.async.bulk per task into an SMEM ring slot,
// and stays there through (C), (D) and (A): H crosses HBM and L2 exactly once per
// iteration, and no register or scoreboard is held by loads in flight.  There is no
// producer warp: the warp that finishes a task in (A) refills its slot with the task NS
// positions later, so a slot is re-issued the moment it is free.
//
// Lane l of the warp that owns a task owns row 32 t + l: it reads the row's RB bytes as
// NSL 16-byte slots in a lane-permuted order (slot s ^ rot, rot = l / RPS mod NSL),
// which makes every quarter-warp LDS.128 bank-conflict-free, and does all the math of the
// row in registers: (C) accumulates NSL rotated z partials, (A) forms the row's full dot
// with the (rotated) new c — no per-row shuffles.  Per strip only z needs a cross-lane
// reduction (shuffles + one SMEM partial per warp).
//
// Strip bytes = n_meas * RB (RB = W * sizeof(S) = 128 or 64 bytes per row); the ring
// holds a strip plus >= 2 tasks of slack, so the next strip streams in while (A) of the
// current one drains it.  w partials, residual scalars and the segment partial layout are
// those of sweep_kernel (rows_finalize_sweep_kernel consumes them).
#pragma once

#include "admm_sweep.cuh"

namespace admm {

constexpr int kGroupWarps = 8;                           // (C) warps = (D)+(A) warps
constexpr int kTileWarps = 2 * kGroupWarps;
constexpr int kTileThreads = kTileWarps * kWarp;
constexpr int kTileRows = kWarp;                         // rows per task (one per lane)
// named barriers (0 is __syncthreads)
enum TileBar { kBarCG = 1, kBarAG = 2, kBarCDone0 = 3, kBarZFree0 = 5 };

template <typename S, int RB>
struct TileGeom {
  static constexpr int W = RB / (int)sizeof(S);     // columns per strip
  static constexpr int PV = 16 / (int)sizeof(S);    // elements per 16-byte slot
  static constexpr int NSL = RB / 16;               // 16-byte slots per row
  static constexpr int RPS = 128 / RB;              // rows per 128-byte bank line
  static constexpr int TB = kTileRows * RB;         // task bytes
};

__host__ __device__ inline size_t tile_smem_bytes(uint32_t ns, uint32_t task_bytes, uint32_t n_meas, uint32_t M,
                                                  uint32_t N, uint32_t W) {
  return (size_t)ns * task_bytes + 2 * (size_t)ns * sizeof(uint64_t) +
         ((size_t)2 * n_meas + ((size_t)2 * kGroupWarps + 6) * M * W + 2 * (size_t)W) * sizeof(double2) +
         (size_t)N * sizeof(SweepDesc) + ((size_t)M + 1 + 2 * (size_t)M * N + N) * sizeof(uint32_t);
}

// One 16-byte SMEM slot of stored elements, kept narrow in registers (c64: 2 elements
// as float4) and widened to FP64 at use.
template <typename S>
using Raw16 = typename std::conditional<sizeof(S) == 16, double2, float4>::type;

__device__ __forceinline__ double2 raw_get(const double2& r, int) { return r; }
__device__ __forceinline__ double2 raw_get(const float4& r, int e) {
  return e == 0 ? make_double2(r.x, r.y) : make_double2(r.z, r.w);
}

template <typename S, int RB, bool KeepL2, int CPS>
__global__ void __launch_bounds__(kTileThreads, CPS)
sweep_tile_kernel(const S* __restrict__ Ht, const BlockDesc* __restrict__ blocks, const SweepDesc* __restrict__ segs,
                  uint32_t M, uint32_t N, uint32_t n_meas, uint64_t Utot, uint32_t NS,
                  const double2* __restrict__ q, ColVecs cv, double2* __restrict__ wpart,
                  const Params* __restrict__ prm, double* __restrict__ red, IterState* st,
                  unsigned long long* __restrict__ trace) {  // diagnostics (ADMM_B200_TILE_TRACE), else null
  using TG = TileGeom<S, RB>;
  using R16 = Raw16<S>;
  constexpr int W = TG::W, PV = TG::PV, NSL = TG::NSL, RPS = TG::RPS, TB = TG::TB;
  constexpr int NG = kGroupWarps * kWarp;  // threads per group
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* ring = smem_raw;                                          // NS x TB
  uint64_t* fullb = reinterpret_cast<uint64_t*>(ring + (size_t)NS * TB);
  double2* q_s = reinterpret_cast<double2*>(fullb + 2 * NS);              // n_meas (16-B aligned)
  double2* wacc = q_s + n_meas;                                            // n_meas
  double2* zred = wacc + n_meas;                                           // 2 bufs x C warps x M x W
  double2* pre = zred + 2 * (size_t)kGroupWarps * M * W;                   // 2 bufs x (2M+1) x W (c, s, v)
  double2* us = pre + 2 * (2 * (size_t)M + 1) * W;                         // M x W
  double2* cs = us + (size_t)M * W;                                        // M x W
  SweepDesc* ssegs = reinterpret_cast<SweepDesc*>(cs + (size_t)M * W);     // N segment descriptors
  uint32_t* rbnd = reinterpret_cast<uint32_t*>(ssegs + N);                  // M + 1 row bounds
  uint32_t* tvec = rbnd + M + 1;                                            // M x N block vec_off
  uint32_t* tmvec = tvec + (size_t)M * N;                                   // M x N block mvec_off
  uint32_t* tseg = tmvec + (size_t)M * N;                                   // N segment seg_off
  __shared__ double sm_red[kTileThreads / kWarp];
  const double m_rep = prm->m_rep, kappa = prm->kappa;  // constant for the launch
  const double kappa2_lo = kappa * kappa * (1.0 - 0x1p-40);
  // mean = sum / m_rep: multiplying by 1/m_rep is exact when m_rep is a power of two
  const double inv_m = 1.0 / m_rep;
  const bool pow2_m = inv_m * m_rep == 1.0 && (__double_as_longlong(m_rep) & 0xfffffffffffffull) == 0;

  const uint64_t P = gridDim.x, p = blockIdx.x;
  const uint64_t x0 = sk_lo(p, Utot, P);
  const uint64_t xe = sk_lo(p + 1, Utot, P);
  const uint32_t nstrip = (uint32_t)(xe - x0);
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const bool cgroup = warp < kGroupWarps;               // (C) warps; the others do (D) + (A)
  const int gw = cgroup ? warp : warp - kGroupWarps;    // warp index within the group
  const int gt = threadIdx.x - (cgroup ? 0 : NG);       // thread index within the group
  const uint32_t nt = (n_meas + kTileRows - 1) / kTileRows;  // tasks per strip
  const uint64_t strip_bytes = (uint64_t)n_meas * RB;
  double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
  bool bad = false;

  uint64_t pol;
  if constexpr (KeepL2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const bool noload = trace && trace[7] == 1ull;  // diagnostics: consumer-only timing
  // Task t of strip k (the CTA's k-th strip) is the CTA's task g = k nt + t: it always
  // lives in ring slot g % NS, and its full barrier completes for the (g / NS)-th time
  // when it lands.  No divisions on the hot path: positions advance incrementally.
  auto issue = [&](uint32_t ks, uint32_t ts, uint32_t sl) {
    const uint32_t bytes = min((uint32_t)kTileRows, n_meas - ts * kTileRows) * RB;
    if (noload) {
      mbar_arrive(&fullb[sl]);
    } else {
      mbar_expect_tx(&fullb[sl], bytes);
      bulk_g2s(smem_u32(ring + (size_t)sl * TB),
               reinterpret_cast<const unsigned char*>(Ht) + (x0 + ks) * strip_bytes + (uint64_t)ts * TB, bytes,
               &fullb[sl], pol);
    }
  };
  const uint32_t ns_k = NS / nt, ns_t = NS % nt;  // NS = ns_k strips + ns_t tasks
  if (threadIdx.x == 0) {
    for (uint32_t k = 0; k < NS; ++k) mbar_init(&fullb[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t ks = 0, ts = 0;
    for (uint32_t sl = 0; sl < NS && ks < nstrip; ++sl) {
      issue(ks, ts, sl);
      if (++ts == nt) ts = 0, ++ks;
    }
  }
  // descriptor tables in SMEM: nothing on the per-strip path touches global metadata
  if (threadIdx.x <= M) {
    const uint32_t i = threadIdx.x;
    rbnd[i] = i < M ? blocks[i * N].row0 : blocks[(M - 1) * N].row0 + blocks[(M - 1) * N].rows;
  }
  for (uint32_t b = threadIdx.x; b < M * N; b += blockDim.x) {
    tvec[b] = blocks[b].vec_off;
    tmvec[b] = blocks[b].mvec_off;
  }
  for (uint32_t b = threadIdx.x; b < N; b += blockDim.x) {
    tseg[b] = blocks[b].seg_off;
    ssegs[b] = segs[b];
  }
  for (uint32_t r = threadIdx.x; r < n_meas; r += blockDim.x) wacc[r] = make_double2(0.0, 0.0);
  __syncthreads();

  auto mark = [&](uint32_t k, int ev) {
    if (trace && (threadIdx.x == 0 || threadIdx.x == NG) && k < 64) {
      trace[(p * 64 + k) * 8 + ev] = clock64();
    }
  };
  // per group: ring slot / parity of task 0 of the current strip (nt < NS: one wrap)
  uint32_t s0 = 0, ph0 = 0;
  auto ring_pos = [&](uint32_t t, uint32_t& ph) {
    uint32_t sl = s0 + t;
    ph = ph0;
    if (sl >= NS) sl -= NS, ph ^= 1u;
    return sl;
  };
  auto next_strip = [&]() {
    s0 += nt;
    if (s0 >= NS) s0 -= NS, ph0 ^= 1u;
  };

  if (nstrip > 0) {
    uint32_t j = 0;
    while (j + 1 < N && ssegs[j + 1].unit0 <= x0) ++j;
    SweepDesc sd = ssegs[j];
    if (cgroup) {
      // ===================================================== (C) group: z = H^H q per strip
      // Column-slot mapping: lane (lr, lc) reads slot lc of rows lr + RPI k of each task
      // (contiguous 512-byte warp accesses): its partial belongs to one column slot and the
      // end-of-strip reduction is an xor over the lanes sharing lc.
      constexpr int CRPI = kWarp / NSL;      // rows per warp instruction
      constexpr int CKI = kTileRows / CRPI;  // instructions per task
      const int clr = lane / NSL, clc = lane % NSL;
      auto load_q = [&](uint32_t jj) {
        for (uint32_t i = 0; i < M; ++i) {
          const double2* qb = q + tmvec[i * N + jj];
          const uint32_t r0 = rbnd[i], nr = rbnd[i + 1] - r0;
          for (uint32_t r = gt; r < nr; r += NG) q_s[r0 + r] = qb[r];
        }
      };
      load_q(j);
      nb_sync(kBarCG, NG);
      for (uint32_t k = 0; k < nstrip; ++k) {
        const uint64_t x = x0 + k;
        if (x == sd.unit0 + sd.n_strips) {  // next segment: its q
          sd = ssegs[++j];
          nb_sync(kBarCG, NG);
          load_q(j);
          nb_sync(kBarCG, NG);
        }
        const uint32_t zb = k & 1;
        if (k >= 2) nb_sync(kBarZFree0 + zb, kTileThreads);  // (D) of strip k-2 has read zred[zb]
        mark(k, 0);
        for (uint32_t i = 0; i < M; ++i) {
          const uint32_t ra = rbnd[i], rb = rbnd[i + 1];
          double2 acc[PV];
#pragma unroll
          for (int e = 0; e < PV; ++e) acc[e] = make_double2(0.0, 0.0);
          double2 acc2[PV];  // second accumulator set: two tasks in flight per pass
#pragma unroll
          for (int e = 0; e < PV; ++e) acc2[e] = make_double2(0.0, 0.0);
          const uint32_t t_lo = ra / kTileRows, t_hi = (rb + kTileRows - 1) / kTileRows;
          auto task_c = [&](uint32_t t, const R16 (&h)[CKI], double2 (&ac)[PV]) {
            const uint32_t row0 = t * kTileRows + clr;
            if (row0 >= ra && row0 + (CKI - 1) * CRPI < rb) {  // the whole task inside block i
#pragma unroll
              for (int u = 0; u < CKI; ++u) {
                const double2 qv = q_s[row0 + u * CRPI];
#pragma unroll
                for (int e = 0; e < PV; ++e) cmac_conj(ac[e], raw_get(h[u], e), qv);
              }
            } else {
#pragma unroll
              for (int u = 0; u < CKI; ++u) {
                const uint32_t row = row0 + u * CRPI;
                if (row >= ra && row < rb) {
                  const double2 qv = q_s[row];
#pragma unroll
                  for (int e = 0; e < PV; ++e) cmac_conj(ac[e], raw_get(h[u], e), qv);
                }
              }
            }
          };
          for (uint32_t t = t_lo + (gw - t_lo % kGroupWarps + kGroupWarps) % kGroupWarps; t < t_hi;
               t += 2 * kGroupWarps) {
            const uint32_t t2 = t + kGroupWarps;
            const bool two = t2 < t_hi;
            uint32_t ph, ph2;
            const uint32_t sl = ring_pos(t, ph);
            const uint32_t sl2 = two ? ring_pos(t2, ph2) : sl;
            mbar_wait(&fullb[sl], ph);
            if (two) mbar_wait(&fullb[sl2], ph2);
            const unsigned char* tb = ring + (size_t)sl * TB + (size_t)clr * RB + clc * 16;
            const unsigned char* tb2 = ring + (size_t)sl2 * TB + (size_t)clr * RB + clc * 16;
            R16 h[CKI], h2[CKI];
#pragma unroll
            for (int u = 0; u < CKI; ++u) h[u] = *reinterpret_cast<const R16*>(tb + (size_t)u * CRPI * RB);
#pragma unroll
            for (int u = 0; u < CKI; ++u) h2[u] = *reinterpret_cast<const R16*>(tb2 + (size_t)u * CRPI * RB);
            task_c(t, h, acc);
            if (two) task_c(t2, h2, acc2);
          }
#pragma unroll
          for (int e = 0; e < PV; ++e) acc[e] = cadd(acc[e], acc2[e]);
#pragma unroll
          for (int e = 0; e < PV; ++e) {
#pragma unroll
            for (int o = NSL; o < kWarp; o <<= 1) {
              acc[e].x += __shfl_xor_sync(0xffffffffu, acc[e].x, o);
              acc[e].y += __shfl_xor_sync(0xffffffffu, acc[e].y, o);
            }
            if (clr == 0) zred[(((size_t)zb * kGroupWarps + gw) * M + i) * W + clc * PV + e] = acc[e];
          }
        }
        mark(k, 1);
        nb_arrive(kBarCDone0 + zb, kTileThreads);  // z partials of strip k are in zred[zb]
        next_strip();
      }
    } else {
      // ===================================================== (D) + (A) group
      // Lane l of the warp that owns a task owns row 32 t + l and reads its NSL slots in
      // the lane-permuted order s ^ rot (bank-conflict-free), forming the row's full dot
      // with the permuted c in registers.
      const int rot = (lane / RPS) % NSL;
      const size_t pstride = (2 * (size_t)M + 1) * W;
      // the (D) threads (gt < W) stage the strip's iterates one strip ahead with cp.async
      auto stage = [&](uint64_t xs, uint32_t js, uint32_t buf) {
        const SweepDesc& sds = ssegs[js];
        const uint32_t cs_ = (uint32_t)(xs - sds.unit0) * W + gt;
        const bool ok = cs_ < sds.cols;
        double2* dst = pre + buf * pstride;
        for (uint32_t i = 0; i < M; ++i) {
          const uint32_t o = tvec[i * N + js] + (ok ? cs_ : 0);
          cpa(dst + i * W + gt, cv.c + o, ok);
          cpa(dst + (M + i) * W + gt, cv.s + o, ok);
        }
        cpa(dst + 2 * M * W + gt, cv.v + tseg[js] + (ok ? cs_ : 0), ok);
      };
      if (gt < W) stage(x0, j, 0);
      cpa_commit();
      for (uint32_t k = 0; k < nstrip; ++k) {
        const uint64_t x = x0 + k;
        const uint32_t zb = k & 1, pb = k & 1;
        const uint32_t col_lo = (uint32_t)(x - sd.unit0) * W;
        const uint32_t cc = col_lo + gt;
        const bool dcol = gt < W && cc < sd.cols;
        if (gt < W && k + 1 < nstrip) {
          const bool nseg = x + 1 == sd.unit0 + sd.n_strips;
          stage(x + 1, nseg ? j + 1 : j, pb ^ 1u);
        }
        cpa_commit();
        const double2* pc = pre + pb * pstride;
        cpa_wait<1>();                                // this strip's iterates
        nb_sync(kBarCDone0 + zb, kTileThreads);       // (C) of strip k done
        mark(k, 2);
        // ------------------------------------------- (D) u, mean, v, s, next c
        double2 vn = make_double2(0.0, 0.0);
        if (gt < W) {
          const int t = gt;
          if (dcol) {
            double2 mean = make_double2(0.0, 0.0);
            for (uint32_t i = 0; i < M; ++i) {
              double2 zw[kGroupWarps];  // all loads first, then the adds in warp order
#pragma unroll
              for (int w = 0; w < kGroupWarps; ++w) zw[w] = zred[(((size_t)zb * kGroupWarps + w) * M + i) * W + t];
              double2 z = zw[0];
#pragma unroll
              for (int w = 1; w < kGroupWarps; ++w) z = cadd(z, zw[w]);
              const double2 u = cadd(pc[i * W + t], z);
              us[i * W + t] = u;
              mean = cadd(mean, cadd(u, pc[(M + i) * W + t]));
            }
            mean = pow2_m ? make_double2(mean.x * inv_m, mean.y * inv_m)
                          : make_double2(mean.x / m_rep, mean.y / m_rep);
            vn = soft_threshold_fast(mean, kappa, kappa2_lo);
            for (uint32_t i = 0; i < M; ++i) {
              const double2 s = csub(cadd(pc[(M + i) * W + t], us[i * W + t]), vn);
              cs[i * W + t] = csub(vn, s);
            }
          } else {
            for (uint32_t i = 0; i < M; ++i) cs[i * W + t] = make_double2(0.0, 0.0);
          }
        }
        nb_sync(kBarAG, NG);  // cs visible to the group; zred[zb] consumed
        if (k + 2 < nstrip) nb_arrive(kBarZFree0 + zb, kTileThreads);
        mark(k, 3);
        if (dcol) {  // off the critical path: stores and residuals
          const int t = gt;
          const double2 vo = pc[2 * M * W + t];
          const uint32_t so = tseg[j] + cc;
          cv.vprev[so] = vo;
          cv.v[so] = vn;
          rd2 += cabs2(csub(vn, vo));
          l1 += hypot(vn.x, vn.y);
          for (uint32_t i = 0; i < M; ++i) {
            const uint32_t o = tvec[i * N + j] + cc;
            const double2 u = us[i * W + t];
            bad |= !cfinite(u);
            cv.u[o] = u;
            rp2 += cabs2(csub(u, vn));
            const double2 s = csub(cadd(pc[(M + i) * W + t], u), vn);
            cv.s[o] = s;
            cv.c[o] = cs[i * W + t];
          }
        }
        // ------------------------------------------- (A) w += H_ij[:, strip] c_i; refill
        // Two tasks per pass; the dot of a row is split in even/odd slot halves.
        {
          uint32_t bi = 0xffffffffu;
          double2 cr[NSL][PV];  // c of row block bi in this lane's permuted slot order
          auto use_block = [&](uint32_t row) {
            uint32_t b2 = 0;
            if (M > 1) {
              b2 = bi == 0xffffffffu ? 0 : bi;
              while (row >= rbnd[b2 + 1]) ++b2;  // rows ascend: row block of this row
            }
            if (b2 != bi) {
              bi = b2;
#pragma unroll
              for (int s2 = 0; s2 < NSL; ++s2)
#pragma unroll
                for (int e = 0; e < PV; ++e) cr[s2][e] = cs[bi * W + (s2 ^ rot) * PV + e];
            }
          };
          auto dot = [&](const R16 (&h)[NSL]) {
            double2 ae = make_double2(0.0, 0.0), ao = make_double2(0.0, 0.0);
#pragma unroll
            for (int s2 = 0; s2 < NSL; ++s2)
#pragma unroll
              for (int e = 0; e < PV; ++e) {
                if ((s2 * PV + e) & 1)
                  cmac(ao, raw_get(h[s2], e), cr[s2][e]);
                else
                  cmac(ae, raw_get(h[s2], e), cr[s2][e]);
              }
            return cadd(ae, ao);
          };
          auto refill = [&](uint32_t t, uint32_t sl) {  // the slot is free: task g + NS
            uint32_t kn = k + ns_k, tn = t + ns_t;
            if (tn >= nt) tn -= nt, ++kn;
            if (kn < nstrip) issue(kn, tn, sl);
          };
          for (uint32_t t = gw; t < nt; t += 2 * kGroupWarps) {
            const uint32_t t2 = t + kGroupWarps;
            const bool two = t2 < nt;
            uint32_t ph, ph2;
            const uint32_t sl = ring_pos(t, ph);
            const uint32_t sl2 = two ? ring_pos(t2, ph2) : sl;
            mbar_wait(&fullb[sl], ph);  // complete already ((C) saw it); orders this group's reads
            if (two) mbar_wait(&fullb[sl2], ph2);
            const unsigned char* b = ring + (size_t)sl * TB + (size_t)lane * RB;
            const unsigned char* b2 = ring + (size_t)sl2 * TB + (size_t)lane * RB;
            R16 h[NSL], h2[NSL];
#pragma unroll
            for (int s2 = 0; s2 < NSL; ++s2) h[s2] = *reinterpret_cast<const R16*>(b + (s2 ^ rot) * 16);
#pragma unroll
            for (int s2 = 0; s2 < NSL; ++s2) h2[s2] = *reinterpret_cast<const R16*>(b2 + (s2 ^ rot) * 16);
            const uint32_t row = t * kTileRows + lane, row2 = t2 * kTileRows + lane;
            double2 a1 = make_double2(0.0, 0.0), a2 = make_double2(0.0, 0.0);
            if (row < n_meas) {
              use_block(row);
              a1 = dot(h);
            }
            if (two && row2 < n_meas) {
              use_block(row2);
              a2 = dot(h2);
            }
            if (row < n_meas) wacc[row] = cadd(wacc[row], a1);  // one lane owns a row
            if (two && row2 < n_meas) wacc[row2] = cadd(wacc[row2], a2);
            __syncwarp();
            if (lane == 0) {  // the slot's reads have completed (their values are consumed)
              refill(t, sl);
              if (two) refill(t2, sl2);
            }
          }
        }
        mark(k, 4);
        next_strip();
        const bool seg_end = (x + 1 == sd.unit0 + sd.n_strips);
        if (seg_end || k + 1 == nstrip) {  // flush this segment's w partial
          nb_sync(kBarAG, NG);
          const uint64_t slotp = p - sk_owner(sd.unit0, Utot, P);
          double2* dst = wpart + sd.part_off + slotp * n_meas;
          for (uint32_t r = gt; r < n_meas; r += NG) {
            dst[r] = wacc[r];
            wacc[r] = make_double2(0.0, 0.0);
          }
          if (seg_end && k + 1 < nstrip) sd = ssegs[++j];
          nb_sync(kBarAG, NG);
        }
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->nonfinite = 1u;
  double r = block_sum<kTileThreads>(rp2, sm_red);
  if (threadIdx.x == 0) red[p] = r;
  r = block_sum<kTileThreads>(rd2, sm_red);
  if (threadIdx.x == 0) red[P + p] = r;
  r = block_sum<kTileThreads>(l1, sm_red);
  if (threadIdx.x == 0) red[2 * P + p] = r;
}

// One-time re-layout: Ht[x][row][e] = H_{i(row), j(x)}[row - row0_i][(x - unit0_j) * W + e]
// (zero past the segment's last column).  Setup only.
template <typename S>
__global__ void tile_h_kernel(const S* __restrict__ H, const MatDesc* __restrict__ hm,
                              const BlockDesc* __restrict__ blocks, const SweepDesc* __restrict__ segs, uint32_t M,
                              uint32_t N, uint32_t n_meas, uint32_t W, uint64_t total, S* __restrict__ Ht) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = idx / ((uint64_t)n_meas * W);
    const uint32_t rem = (uint32_t)(idx % ((uint64_t)n_meas * W));
    const uint32_t row = rem / W, e = rem % W;
    uint32_t j = 0;
    while (j + 1 < N && segs[j + 1].unit0 <= x) ++j;
    const uint32_t col = (uint32_t)(x - segs[j].unit0) * W + e;
    S val;
    val.x = 0;
    val.y = 0;
    if (col < segs[j].cols) {
      uint32_t i = 0;
      while (i + 1 < M && blocks[(i + 1) * N + j].row0 <= row) ++i;
      const MatDesc md = hm[i * N + j];
      val = H[md.a_off + (uint64_t)(row - blocks[i * N + j].row0) * md.ld + col];
    }
    Ht[idx] = val;
  }
}

}  // namespace admm
