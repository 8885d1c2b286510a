// admm_resident.cuh — the whole ADMM iteration of a SMALL problem in one persistent
// kernel, H resident in shared memory (schedule 4, "resident").
//
// BASELINE config 1 (256 x 2048 complex128, 8 MiB of H) is latency-bound on the launch
// chain of the other schedules: ~6 kernels of a few microseconds each per iteration,
// for 16 MiB of L2-resident H traffic.  Here each of the P = #SM CTAs loads ITS columns
// of H (all rows: every replica of its column segment) into SMEM once per launch
// (57 KiB per SM on config 1) and runs `iters` iterations with two grid-wide barriers
// each; no H byte moves after the first iteration.
//
//   phase A (every CTA, its columns t of segment j):
//     z_ij,t = sum_rows conj(H) q_ij              (adjoint_matvec, linalg.hpp:114)
//     u = c + z;  v = S_kappa(mean_i(u + s));  s = (s + u) - v;  c = v - s
//                                                  (solvers.hpp:116-136 / 242 / 377-415,
//                                                   prox.hpp:15, admm_core.hpp:73-89)
//     residual partials rp2, rd2, l1 (solvers.hpp:141-145), non-finite flag (solvers.hpp:47)
//     w partial: sum_{its columns} H c           (matvec, linalg.hpp:97)
//     [objective rows of the previous iteration: |sum_j a_ij - g|^2 over a row slice]
//   grid barrier
//   phase B (CTA b owns block b):
//     g_ij = g_i - sum_{q != j} ghat_iq (previous iteration's ghat, ascending q; Jacobi,
//     solvers.hpp:218-225 / 361-384);  w = sum of the segment's CTA partials (CTA order);
//     r = g_ij - w;  [a_b = (w + h_b + ghat_b)/2, h_b = a_b - w — objective recurrence,
//     DESIGN.md §2];  q = K r (dense K, warp per row);  ghat_new = g_ij - rho q
//     CTA 0: trace[k] = (r_p, r_d), trace[k-1].objective, non-finite bookkeeping, iter++
//   grid barrier
// ghat is double-buffered by iteration parity (phase B reads the previous iteration's
// values of all blocks while the owners write the new ones).  Deterministic: every sum
// has a fixed order, no float atomics.  Launched cooperatively (co-residency guaranteed).
#pragma once

#include "admm_kernels.cuh"

namespace admm {

constexpr int kResMaxM = 8;        // replicas (row blocks) per column segment
constexpr int kResMaxCols = 256;   // columns per CTA (thread per column in the update)
constexpr int kResMaxBlocks = 160; // blocks (one owner CTA each, <= #SMs)

struct ResCta {       // one per CTA
  uint32_t seg;       // column segment j
  uint32_t col_lo;    // first local column within the segment
  uint32_t ncols;     // columns owned
  uint32_t cta_lo;    // first CTA of this segment (its w partials are summed in CTA order)
  uint32_t cta_hi;    // one past the last CTA of this segment
  uint32_t pad_;
};

struct ResArgs {
  const void* H;               // storage arena (S)
  const void* K;               // dense inverses (S), kN descriptors
  const MatDesc* hN;           // per block: a_off, ld
  const MatDesc* kN;
  const BlockDesc* blocks;
  const ResCta* ctas;
  const uint32_t* seg_cta;     // [N][2]: first / one-past-last CTA of each segment
  const double2* g;
  double2* ghat[2];            // parity buffers
  double2* gij;
  double2* r;
  double2* q;
  ColVecs cv;
  double2* wpart;              // [P][n_meas]
  double* red;                 // [3][P]: rp2, rd2, l1
  double* opart;               // [P]
  double2* hs;                 // objective recurrence h_b (mvec) or nullptr
  double2* abuf;               // a_b (mvec)
  double* lprev;               // l1 of the previous iteration (objective of trace[k-1])
  const Params* prm;
  double* trace;
  uint64_t trace_cap;
  IterState* st;
  unsigned* bar;               // [2] grid barrier: count, generation
  uint32_t M, N, nb, n_meas;
  uint32_t max_cols;           // columns per CTA (SMEM tile width)
  uint32_t max_m;              // largest block row count (owner's K tile in SMEM: max_m^2)
  uint32_t iters;              // iterations in this launch
  uint32_t prologue;           // 1: run only the reset prologue (phase B with w = 0)
  uint32_t trace_obj;
  unsigned long long* dbg;     // optional clock64 trace [cta][iter][5] (ADMM_B200_RES_TRACE)
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free generation barrier over all CTAs (co-resident: cooperative launch).
__device__ __forceinline__ void res_grid_sync(unsigned* bar, unsigned nct) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire_gpu(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == nct - 1) {
      bar[0] = 0;
      __threadfence();
      atomicExch(bar + 1, g + 1);
    } else {
      while (ld_acquire_gpu(bar + 1) == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

template <typename S>
__device__ __forceinline__ double2 res_ld(const S* p) {
  return Store<S>::widen(*p);
}

template <typename S>
__global__ void __launch_bounds__(kCtaThreads, 1) resident_kernel(ResArgs a) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const uint32_t P = gridDim.x, cta = blockIdx.x;
  const ResCta rc = a.ctas[cta];
  const uint32_t nm = a.n_meas, M = a.M, N = a.N;
  // SMEM: H tile [max_cols][n_meas] (S), q [n_meas], z/u/s/c [M][max_cols], v, vp [max_cols],
  // owner scratch gij/r/w [n_meas], reduction scratch
  S* Hs = reinterpret_cast<S*>(rsm);
  size_t off = ((size_t)a.max_cols * nm * sizeof(S) + 15) & ~(size_t)15;
  const uint32_t nmx = nm > (uint32_t)kCtaThreads ? nm : (uint32_t)kCtaThreads;
  double2* qs = reinterpret_cast<double2*>(rsm + off);  // q of the segment; owner: K-apply run partials
  off += (size_t)nmx * 16;
  double2* zs = reinterpret_cast<double2*>(rsm + off);
  off += (size_t)M * a.max_cols * 16;
  double2* us = reinterpret_cast<double2*>(rsm + off);
  off += (size_t)M * a.max_cols * 16;
  double2* ss = reinterpret_cast<double2*>(rsm + off);
  off += (size_t)M * a.max_cols * 16;
  double2* csm = reinterpret_cast<double2*>(rsm + off);
  off += (size_t)M * a.max_cols * 16;
  double2* vs = reinterpret_cast<double2*>(rsm + off);
  off += (size_t)a.max_cols * 16;
  double2* vps = reinterpret_cast<double2*>(rsm + off);
  off += (size_t)a.max_cols * 16;
  double2* ob = reinterpret_cast<double2*>(rsm + off);  // owner: w partial runs, then r
  off += (size_t)nmx * 16;
  double2* wb = reinterpret_cast<double2*>(rsm + off);  // owner: w, then g_ij
  off += (size_t)nmx * 16;
  double* sm = reinterpret_cast<double*>(rsm + off);    // 5 x kCtaWarps doubles
  off += 5 * kCtaWarps * 8;
  S* Ks = reinterpret_cast<S*>(rsm + ((off + 15) & ~(size_t)15));  // owner: its block's K (row-major, m x m)
  // block table and segment CTA ranges, copied once per launch: every descriptor read of the
  // iteration loop is an SMEM read (no dependent global round trips on the critical path)
  __shared__ BlockDesc sblk[kResMaxBlocks];
  __shared__ uint32_t sseg[2 * kResMaxBlocks];
  for (uint32_t e = threadIdx.x; e < a.nb; e += kCtaThreads) sblk[e] = a.blocks[e];
  for (uint32_t e = threadIdx.x; e < 2 * N; e += kCtaThreads) sseg[e] = a.seg_cta[e];
  __syncthreads();

  const S* H = static_cast<const S*>(a.H);
  const uint32_t j = rc.seg;
  const uint32_t nc = rc.ncols;
  const double kappa = a.prm->kappa, rho = a.prm->rho, mrep = a.prm->m_rep;

  // ---- load this CTA's columns (all replicas) and iterates
  for (uint32_t i = 0; i < M && !a.prologue; ++i) {
    const BlockDesc bd = sblk[i * N + j];
    const MatDesc md = a.hN[i * N + j];
    for (uint32_t e = threadIdx.x; e < nc * bd.rows; e += kCtaThreads) {
      const uint32_t t = e % nc, row = e / nc;  // consecutive threads: consecutive columns of a row
      Hs[(size_t)t * nm + bd.row0 + row] = H[md.a_off + (uint64_t)row * md.ld + rc.col_lo + t];
    }
    for (uint32_t t = threadIdx.x; t < nc; t += kCtaThreads) {
      const uint32_t o = bd.vec_off + rc.col_lo + t;
      us[i * a.max_cols + t] = a.cv.u[o];
      ss[i * a.max_cols + t] = a.cv.s[o];
      csm[i * a.max_cols + t] = a.cv.c[o];
    }
  }
  if (cta < a.nb) {  // owner: K of its block, read once per launch
    const BlockDesc bd = sblk[cta];
    const MatDesc km = a.kN[cta];
    const S* K = static_cast<const S*>(a.K) + km.a_off;
    for (uint32_t e = threadIdx.x; e < bd.rows * bd.rows; e += kCtaThreads)  // transposed: Ks[col][row]
      Ks[(size_t)(e % bd.rows) * bd.rows + e / bd.rows] = K[(uint64_t)(e / bd.rows) * km.ld + e % bd.rows];
  }
  const BlockDesc s0 = sblk[j];  // replica 0: the segment's v offset
  for (uint32_t t = threadIdx.x; t < nc && !a.prologue; t += kCtaThreads) {
    vs[t] = a.cv.v[s0.seg_off + rc.col_lo + t];
    vps[t] = a.cv.vprev[s0.seg_off + rc.col_lo + t];
  }
  __syncthreads();

  const int warp = warp_index(), lane = threadIdx.x % kWarp;
  const uint32_t niter = a.prologue ? 1 : a.iters;
  for (uint32_t it = 0; it < niter; ++it) {
    const uint64_t k = ld_acquire_gpu64(&a.st->iter);  // iterations completed before this one
    if (!a.prologue) {
      // ---------------- phase A
      if (a.dbg && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 0] = clock64();
      // q of the segment's blocks, in global row order
      for (uint32_t row = threadIdx.x; row < nm; row += kCtaThreads) {  // one pass over all rows
        uint32_t i = 0;
        while (i + 1 < M && sblk[(i + 1) * N + j].row0 <= row) ++i;
        const BlockDesc bd = sblk[i * N + j];
        qs[row] = a.q[bd.mvec_off + row - bd.row0];
      }
      if (a.dbg && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 5] = clock64();
      // objective rows of the previous iteration (a_b written by the owners in its phase B)
      double oq = 0.0;
      if (a.trace_obj) {
        if (k >= 1) {
          const uint32_t r0 = (uint32_t)((uint64_t)nm * cta / P), r1 = (uint32_t)((uint64_t)nm * (cta + 1) / P);
          for (uint32_t row = r0 + threadIdx.x; row < r1; row += kCtaThreads) {
            uint32_t i = 0;
            while (i + 1 < M && sblk[(i + 1) * N].row0 <= row) ++i;
            const BlockDesc bi = sblk[i * N];
            double2 hv = make_double2(0.0, 0.0);
            for (uint32_t jj = 0; jj < N; ++jj) hv = cadd(hv, a.abuf[sblk[i * N + jj].mvec_off + row - bi.row0]);
            oq += cabs2(csub(hv, a.g[row]));
          }
        }
      }
      __syncthreads();
      if (a.dbg && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 6] = clock64();
      // z = H^H q per (replica, column): warp per column, lanes over the replica's rows
      // (all replicas' accumulators live together so their shuffle reductions interleave)
      for (uint32_t t = warp; t < nc; t += kCtaWarps) {
        const S* hc = Hs + (size_t)t * nm;
        double2 acc[kResMaxM];
#pragma unroll
        for (int i = 0; i < kResMaxM; ++i) {
          acc[i] = make_double2(0.0, 0.0);
          if (i < (int)M) {
            const BlockDesc bd = sblk[i * N + j];
            for (uint32_t row = lane; row < bd.rows; row += kWarp)
              cmac_conj(acc[i], res_ld(hc + bd.row0 + row), qs[bd.row0 + row]);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < kResMaxM; ++i)
            if (i < (int)M) {
              acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, o);
              acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, o);
            }
        if (lane < M) {
#pragma unroll
          for (int i = 0; i < kResMaxM; ++i)
            if (i == (int)lane) zs[i * a.max_cols + t] = acc[i];
        }
      }
      __syncthreads();
      if (a.dbg && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 7] = clock64();
      // column update (zupdate_kernel's arithmetic, same order)
      double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
      bool bad = false;
      for (uint32_t t = threadIdx.x; t < nc; t += kCtaThreads) {
        double2 mean = make_double2(0.0, 0.0);
        for (uint32_t i = 0; i < M; ++i) {
          const uint32_t x = i * a.max_cols + t;
          const double2 u = cadd(csm[x], zs[x]);
          bad |= !cfinite(u);
          us[x] = u;
          mean = cadd(mean, cadd(u, ss[x]));
        }
        mean = make_double2(mean.x / mrep, mean.y / mrep);
        const double2 vn = soft_threshold(mean, kappa);
        const double2 vo = vs[t];
        vps[t] = vo;
        vs[t] = vn;
        rd2 += cabs2(csub(vn, vo));
        l1 += hypot(vn.x, vn.y);
        for (uint32_t i = 0; i < M; ++i) {
          const uint32_t x = i * a.max_cols + t;
          const double2 u = us[x];
          rp2 += cabs2(csub(u, vn));
          const double2 s = csub(cadd(ss[x], u), vn);
          ss[x] = s;
          csm[x] = csub(vn, s);
        }
      }
      {  // rp2, rd2, l1, |Hv - g|^2 and the non-finite flag in one reduction (fixed order)
        double v4[4] = {rp2, rd2, l1, oq};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int f = 0; f < 4; ++f) v4[f] += __shfl_xor_sync(0xffffffffu, v4[f], o);
        const bool wbad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
#pragma unroll
          for (int f = 0; f < 4; ++f) sm[f * kCtaWarps + warp] = v4[f];
          sm[4 * kCtaWarps + warp] = wbad ? 1.0 : 0.0;
        }
        __syncthreads();
        if (threadIdx.x < 5) {
          double acc4 = 0.0;
          for (int w = 0; w < kCtaWarps; ++w) acc4 += sm[threadIdx.x * kCtaWarps + w];
          if (threadIdx.x < 3) a.red[threadIdx.x * P + cta] = acc4;
          else if (threadIdx.x == 3) a.opart[cta] = acc4;
          else if (acc4 != 0.0) a.st->nonfinite = 1u;
        }
      }
      if (a.dbg && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 8] = clock64();
      // w partial = H c over this CTA's columns, every row of the segment (row-parallel)
      for (uint32_t row = threadIdx.x; row < nm; row += kCtaThreads) {  // one pass over all rows
        uint32_t i = 0;
        while (i + 1 < M && sblk[(i + 1) * N + j].row0 <= row) ++i;
        const double2* ci = csm + i * a.max_cols;
        double2 acc = make_double2(0.0, 0.0);
        for (uint32_t t = 0; t < nc; ++t) cmac(acc, res_ld(Hs + (size_t)t * nm + row), ci[t]);
        a.wpart[(uint64_t)cta * nm + row] = acc;
      }
      if (a.dbg && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 1] = clock64();
      res_grid_sync(a.bar, P);
      if (a.dbg && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 2] = clock64();
    }
    // ---------------- phase B (owners)
    const uint32_t par = (uint32_t)(k & 1);  // ghat[par]: previous iteration's values
    const double2* gho = a.ghat[par];
    double2* ghn = a.ghat[par ^ 1];
    if (a.prologue) {  // reset: ghat^0 = 0 in buffer 0; the first iteration reads it
      gho = a.ghat[1];
      ghn = a.ghat[0];
    }
    for (uint32_t b = cta; b < a.nb; b += P) {  // (nb <= P: one block per owner)
      const BlockDesc bd = sblk[b];
      const uint32_t c_lo = sseg[2 * bd.j], c_hi = sseg[2 * bd.j + 1];  // segment j's CTAs
      // w = sum of the segment's CTA partials: G thread groups per row each sum a contiguous
      // run of CTAs (loads issued 8 at a time), then the runs are added in order — a fixed
      // association, so the result is deterministic
      const uint32_t G = bd.rows >= kCtaThreads ? 1u : kCtaThreads / bd.rows;
      if (!a.prologue) {
        const uint32_t ncta = c_hi - c_lo, per = (ncta + G - 1) / G;
        for (uint32_t e = threadIdx.x; e < G * bd.rows; e += kCtaThreads) {
          const uint32_t row = e % bd.rows, g = e / bd.rows;
          const uint32_t lo = c_lo + g * per, hi = min(c_hi, lo + per);
          double2 acc = make_double2(0.0, 0.0);
          for (uint32_t c0 = lo; c0 < hi; c0 += 16) {
            double2 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c0 + q < hi) v[q] = a.wpart[(uint64_t)(c0 + q) * nm + bd.row0 + row];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c0 + q < hi) acc = (c0 + q == lo) ? v[q] : cadd(acc, v[q]);
          }
          ob[(size_t)g * bd.rows + row] = acc;  // ob / wb are free until the rows below
        }
        __syncthreads();
        for (uint32_t row = threadIdx.x; row < bd.rows; row += kCtaThreads) {
          double2 w = ob[row];
          for (uint32_t g = 1; g < G; ++g) w = cadd(w, ob[(size_t)g * bd.rows + row]);
          wb[row] = w;
        }
        __syncthreads();
      }
      for (uint32_t row = threadIdx.x; row < bd.rows; row += kCtaThreads) {
        double2 gij = a.g[bd.row0 + row];
        for (uint32_t qj = 0; qj < N; ++qj)
          if (qj != bd.j) gij = csub(gij, a.prologue ? make_double2(0.0, 0.0) : gho[sblk[bd.i * N + qj].mvec_off + row]);
        const double2 w = a.prologue ? make_double2(0.0, 0.0) : wb[row];
        const double2 rr = csub(gij, w);
        const uint32_t o = bd.mvec_off + row;
        a.gij[o] = gij;
        a.r[o] = rr;
        ob[row] = rr;
        wb[row] = gij;
        if (a.trace_obj && !a.prologue) {
          const double2 ga = cscale(cadd(cadd(w, a.hs[o]), gho[o]), 0.5);
          a.hs[o] = csub(ga, w);
          a.abuf[o] = ga;
        }
      }
      __syncthreads();
      // q = K r: warp per row, lanes over columns (dense K, storage S)
      // G thread groups per row, each over a contiguous column run of the (transposed) K,
      // runs combined in order; conflict-free SMEM reads (consecutive rows)
      {
        double2* qp = qs;  // q scratch: phase A's q is dead until the next iteration reloads it
        const uint32_t per = (bd.rows + G - 1) / G;
        for (uint32_t e = threadIdx.x; e < G * bd.rows; e += kCtaThreads) {
          const uint32_t row = e % bd.rows, g = e / bd.rows;
          const uint32_t c0 = g * per, c1 = min(bd.rows, c0 + per);
          double2 acc = make_double2(0.0, 0.0);
          for (uint32_t col = c0; col < c1; ++col) cmac(acc, res_ld(Ks + (size_t)col * bd.rows + row), ob[col]);
          qp[(size_t)g * bd.rows + row] = acc;
        }
        __syncthreads();
        for (uint32_t row = threadIdx.x; row < bd.rows; row += kCtaThreads) {
          double2 acc = qp[row];
          for (uint32_t g = 1; g < G; ++g) acc = cadd(acc, qp[(size_t)g * bd.rows + row]);
          const uint32_t o2 = bd.mvec_off + row;
          a.q[o2] = acc;
          ghn[o2] = csub(wb[row], cscale(acc, rho));
        }
      }
      __syncthreads();
    }
    const uint32_t closer = P - 1 >= a.nb ? P - 1 : 0;  // a CTA without owner work, when there is one
    if (!a.prologue && cta == closer && threadIdx.x < kWarp) {  // close iteration k (finalize_kernel's sums)
      double rp = 0.0, rd = 0.0, l = 0.0, o = 0.0;
      for (uint32_t c = threadIdx.x; c < P; c += kWarp) {
        rp += a.red[c];
        rd += a.red[P + c];
        l += a.red[2 * P + c];
        if (a.trace_obj) o += a.opart[c];
      }
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        rp += __shfl_xor_sync(0xffffffffu, rp, s);
        rd += __shfl_xor_sync(0xffffffffu, rd, s);
        l += __shfl_xor_sync(0xffffffffu, l, s);
        o += __shfl_xor_sync(0xffffffffu, o, s);
      }
      if (threadIdx.x == 0) {
        if (k < a.trace_cap) {
          a.trace[3 * k] = sqrt(rp);
          a.trace[3 * k + 1] = sqrt(rho * rho * mrep * rd);
          a.trace[3 * k + 2] = __longlong_as_double(0x7ff8000000000000ll);
        }
        if (a.trace_obj && k >= 1 && k - 1 < a.trace_cap) a.trace[3 * (k - 1) + 2] = 0.5 * o + a.prm->lambda * *a.lprev;
        *a.lprev = l;
        if (*reinterpret_cast<volatile uint32_t*>(&a.st->nonfinite) && a.st->first_bad == ~0ull) a.st->first_bad = k;
        a.st->nonfinite = 0u;
        a.st->iter = k + 1;
      }
    }
    if (a.dbg && !a.prologue && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 3] = clock64();
    if (!a.prologue) res_grid_sync(a.bar, P);
    if (a.dbg && !a.prologue && threadIdx.x == 0 && it < 16) a.dbg[((uint64_t)cta * 16 + it) * 10 + 4] = clock64();
  }
  if (a.prologue) return;
  // ---- write back the column iterates
  for (uint32_t i = 0; i < M; ++i) {
    const BlockDesc bd = sblk[i * N + j];
    for (uint32_t t = threadIdx.x; t < nc; t += kCtaThreads) {
      const uint32_t o = bd.vec_off + rc.col_lo + t;
      a.cv.u[o] = us[i * a.max_cols + t];
      a.cv.s[o] = ss[i * a.max_cols + t];
      a.cv.c[o] = csm[i * a.max_cols + t];
    }
  }
  for (uint32_t t = threadIdx.x; t < nc; t += kCtaThreads) {
    a.cv.v[s0.seg_off + rc.col_lo + t] = vs[t];
    a.cv.vprev[s0.seg_off + rc.col_lo + t] = vps[t];
  }
}

template <typename S>
size_t resident_smem(uint32_t max_cols, uint32_t n_meas, uint32_t M, uint32_t max_m) {
  const size_t base = (((size_t)max_cols * n_meas * sizeof(S) + 15) & ~(size_t)15) +
                      (size_t)std::max<uint32_t>(n_meas, kCtaThreads) * 16 +
                      4 * (size_t)M * max_cols * 16 + 2 * (size_t)max_cols * 16 +
                      2 * (size_t)std::max<uint32_t>(n_meas, kCtaThreads) * 16 + 5 * kCtaWarps * 8;
  return ((base + 15) & ~(size_t)15) + (size_t)max_m * max_m * sizeof(S);
}

}  // namespace admm
