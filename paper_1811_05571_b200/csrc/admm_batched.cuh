// admm_batched.cuh — multi-scene (batched right-hand side) ADMM iteration.
//
// BASELINE config 5: B independent scenes g_b share H, the partition and the Woodbury
// factors; each scene is an independent hybrid_solve (solvers.hpp:306) with its own
// lambda_b.  With B right-hand sides the two H products of an iteration become skinny
// complex GEMMs, W = H C and Z = H^H Q (C: n x B, Q: m x B), compute-bound on SIMT
// (tensor cores are reserved for setup by the north star).  Register-tiled FP64 SIMT:
// a 256-thread CTA owns a 64 x 64 output tile (64 rows or columns x up to 64 scenes),
// each thread a 4 x 4 complex sub-tile (rows ty + 16q, scenes tx + 16w: both SMEM
// operand reads are conflict-free); A and X stream through SMEM in k-chunks of 16.
// Vectors are [row][scene] (scene fastest), FP64 like the single-scene engine.
#pragma once

#include "admm_kernels.cuh"

namespace admm {

constexpr int kBT = 64;   // output tile: rows (N) or columns (adjoint)
constexpr int kBB = 64;   // scenes per tile
constexpr int kBK = 16;   // k-chunk
// k-steps unrolled per chunk: 4 for W = H C (2.23 vs 2.29 ms on config 5), 2 for the
// adjoint (2.27 vs 2.31 ms; 4 spills there at the 128-register cap)
template <bool ADJ>
constexpr int kBUnroll = ADJ ? 2 : 4;

struct BTile {
  uint64_t a_off;   // matrix in the storage arena
  uint64_t x_off;   // X (k-major, [k][B]) in the vector arena
  uint64_t o_off;   // output (rows/cols x B) in the output arena
  uint32_t ld, rows, cols;
  uint32_t t0;      // first output row (N) / column (adjoint)
  uint32_t k0, k1;  // k range of this unit (split-K)
  uint32_t s0;      // first scene of this unit (scene tiles of SB)
  uint32_t pad_;
};

// out[t0 + i][b] = sum_{k in [k0,k1)} op(A)[t0 + i][k] X[k][b]
//   ADJ = false: op(A)[i][k] = A[i][k]          (W = H C, Q = K R)
//   ADJ = true:  op(A)[i][k] = conj(A[k][i])    (Z = H^H Q)
// A (storage precision) and X are staged by cp.async into double-buffered SMEM in the
// layout their global rows arrive in (no transposing stores); A is widened at read time.
// SB scenes per CTA tile: 64 (4 x 4 complex per thread, 2 CTAs/SM) or 32 (4 x 2, 3 CTAs/SM:
// more warps to keep the FP64 pipe fed, A staged twice as often).
template <typename S, bool ADJ, int SB>
__global__ void __launch_bounds__(256, SB == 64 ? 2 : 3)
bgemm_kernel(const S* __restrict__ A, const BTile* __restrict__ tiles, const double2* __restrict__ X,
             double2* __restrict__ out, uint32_t B) {
  constexpr int NW = SB / 16;  // scenes per thread
  constexpr int AR = ADJ ? kBK : kBT;      // As[2][AR][AC + 1]
  constexpr int AC = ADJ ? kBT : kBK;
  extern __shared__ __align__(16) unsigned char bsm[];
  S* As = reinterpret_cast<S*>(bsm);                                           // 2 x AR x (AC+1)
  constexpr size_t kAsBytes = (2 * AR * (AC + 1) * sizeof(S) + 15) & ~(size_t)15;
  double2* Xs = reinterpret_cast<double2*>(bsm + kAsBytes);  // 2 x kBK x (SB+1)
  double2* Ad = Xs + 2 * kBK * (SB + 1);                      // AR x (AC+1) FP64 (complex64 only)
  const BTile t = tiles[blockIdx.x];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const S* a = A + t.a_off;
  const uint32_t nout = ADJ ? t.cols : t.rows;
  auto stage = [&](int buf, uint32_t k0) {
    S* as = As + (size_t)buf * AR * (AC + 1);
    double2* xs = Xs + (size_t)buf * kBK * (SB + 1);
    // fixed trip counts, unrolled: the index math folds to per-thread constants
#pragma unroll
    for (int it = 0; it < kBT * kBK / 256; ++it) {
      const int e = (int)threadIdx.x + 256 * it;
      const int r = e / AC, c = e % AC;  // consecutive threads -> consecutive global and SMEM
      const uint32_t oi = t.t0 + (ADJ ? c : r), k = k0 + (ADJ ? r : c);
      const bool ok = oi < nout && k < t.k1;
      const S* src = ok ? (ADJ ? a + (uint64_t)k * t.ld + oi : a + (uint64_t)oi * t.ld + k) : a;
      if constexpr (sizeof(S) == 16)
        cpa(as + r * (AC + 1) + c, src, ok);
      else
        cpa8(as + r * (AC + 1) + c, src, ok);
    }
#pragma unroll
    for (int it = 0; it < kBK * SB / 256; ++it) {
      const int e = (int)threadIdx.x + 256 * it;
      const int kk = e / SB, b = e % SB;
      const uint32_t k = k0 + kk;
      const bool ok = k < t.k1 && t.s0 + b < B;
      cpa(xs + kk * (SB + 1) + b, ok ? X + t.x_off + (uint64_t)k * B + t.s0 + b : X, ok);
    }
    cpa_commit();
  };
  double2 acc[4][NW];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int w = 0; w < NW; ++w) acc[q][w] = make_double2(0.0, 0.0);
  int buf = 0;
  stage(0, t.k0);
  for (uint32_t k0 = t.k0; k0 < t.k1; k0 += kBK) {
    if (k0 + kBK < t.k1) {
      stage(buf ^ 1, k0 + kBK);
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    const S* as = As + (size_t)buf * AR * (AC + 1);
    const double2* xs = Xs + (size_t)buf * kBK * (SB + 1);
    const double2* ad = nullptr;  // complex64: the chunk widened once (not once per reader)
    if constexpr (sizeof(S) == 8) {
#pragma unroll
      for (int it = 0; it < AR * AC / 256; ++it) {  // the pad column is never read
        const int e = (int)threadIdx.x + 256 * it;
        const int o = e / AC * (AC + 1) + e % AC;
        Ad[o] = Store<S>::widen(as[o]);
      }
      __syncthreads();
      ad = Ad;
    }
#pragma unroll kBUnroll<ADJ>
    for (int kk = 0; kk < kBK; ++kk) {
      double2 av[4], xv[NW];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = ty + 16 * q;
        const int o = ADJ ? kk * (AC + 1) + i : i * (AC + 1) + kk;
        if constexpr (sizeof(S) == 8)
          av[q] = ad[o];
        else
          av[q] = Store<S>::widen(as[o]);
      }
#pragma unroll
      for (int w = 0; w < NW; ++w) xv[w] = xs[kk * (SB + 1) + tx + 16 * w];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          if (ADJ)
            cmac_conj(acc[q][w], av[q], xv[w]);
          else
            cmac(acc[q][w], av[q], xv[w]);
        }
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t oi = t.t0 + ty + 16 * q;
    if (oi >= nout) continue;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t b = t.s0 + tx + 16 * w;
      if (b < B) out[t.o_off + (uint64_t)oi * B + b] = acc[q][w];
    }
  }
}

template <typename S, bool ADJ, int SB>
constexpr size_t bgemm_smem() {
  constexpr int AR = ADJ ? kBK : kBT;
  constexpr int AC = ADJ ? kBT : kBK;
  return ((2 * AR * (AC + 1) * sizeof(S) + 15) & ~(size_t)15) + 2 * kBK * (SB + 1) * sizeof(double2) +
         (sizeof(S) == 8 ? AR * (AC + 1) * sizeof(double2) : 0);
}

struct BRowVecs {
  const double2* g;  // [n_meas][B]
  double2* ghat;     // [mvec][B]
  double2* gij;
  double2* r;
  double2* q;
};

// (b, row, scene) elementwise: kRhs: G_ij = G_i - sum_{q != j} Ghat_iq (ascending q),
// R = G_ij - sum_s Wpart_s.  kQ: Q = sum_s Qpart_s, Ghat = G_ij - rho Q.
template <int Stage>
__global__ void __launch_bounds__(kCtaThreads)
brows_kernel(BRowVecs rv, const double2* __restrict__ part, uint64_t part_stride, uint32_t nsplit,
             const BlockDesc* __restrict__ blocks, uint32_t N, uint32_t B, const Params* __restrict__ prm) {
  const uint32_t b = blockIdx.y;
  const BlockDesc bd = blocks[b];
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (uint64_t)bd.rows * B) return;
  const uint32_t row = (uint32_t)(e / B), sc = (uint32_t)(e % B);
  const uint64_t o = ((uint64_t)bd.mvec_off + row) * B + sc;
  double2 s = part[o];
  for (uint32_t k = 1; k < nsplit; ++k) s = cadd(s, part[(uint64_t)k * part_stride + o]);
  if constexpr (Stage == kRhs) {
    double2 gij = rv.g[((uint64_t)bd.row0 + row) * B + sc];
    for (uint32_t qj = 0; qj < N; ++qj) {
      if (qj == bd.j) continue;
      gij = csub(gij, rv.ghat[((uint64_t)blocks[bd.i * N + qj].mvec_off + row) * B + sc]);
    }
    rv.gij[o] = gij;
    rv.r[o] = csub(gij, s);
  } else {
    rv.q[o] = s;
    rv.ghat[o] = csub(rv.gij[o], cscale(s, prm->rho));
  }
}

// Per (segment column t, scene): u_i = c_i + z_i for all replicas i, the replica mean,
// v = S_{kappa_scene}(mean), residual partials per scene, dual update, next c.
// Threads: scene = tid % 64 group of 4 columns; grid-stride over the segment columns.
// z holds zsplit split-K slices (zstride apart), summed in slice order.
__global__ void __launch_bounds__(kCtaThreads)
bzupdate_kernel(ColVecs cv, const double2* __restrict__ z, uint32_t zsplit, uint64_t zstride,
                const BlockDesc* __restrict__ blocks, uint32_t M,
                uint32_t N, uint32_t B, const double* __restrict__ kappa, double* __restrict__ red,
                IterState* st) {
  __shared__ double sred[3][4][kBB];
  const uint32_t sc = threadIdx.x % kBB, grp = threadIdx.x / kBB;
  double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
  bool bad = false;
  if (sc < B) {
    const double kap = kappa[sc];
    const double mrep = (double)M;
    for (uint32_t j = 0; j < N; ++j) {
      const BlockDesc b0 = blocks[j];
      for (uint32_t t = blockIdx.x * 4 + grp; t < b0.cols; t += gridDim.x * 4) {
        double2 mean = make_double2(0.0, 0.0);
        for (uint32_t i = 0; i < M; ++i) {
          const uint64_t o = ((uint64_t)blocks[i * N + j].vec_off + t) * B + sc;
          double2 zo = z[o];  // split-K slices of Z = H^H Q, fixed order
          for (uint32_t k = 1; k < zsplit; ++k) zo = cadd(zo, z[(uint64_t)k * zstride + o]);
          const double2 u = cadd(cv.c[o], zo);
          bad |= !cfinite(u);
          cv.u[o] = u;
          mean = cadd(mean, cadd(u, cv.s[o]));
        }
        mean = make_double2(mean.x / mrep, mean.y / mrep);
        const double2 vn = soft_threshold(mean, kap);
        const uint64_t so = ((uint64_t)b0.seg_off + t) * B + sc;
        const double2 vo = cv.v[so];
        cv.vprev[so] = vo;
        cv.v[so] = vn;
        rd2 += cabs2(csub(vn, vo));
        l1 += hypot(vn.x, vn.y);
        for (uint32_t i = 0; i < M; ++i) {
          const uint64_t o = ((uint64_t)blocks[i * N + j].vec_off + t) * B + sc;
          const double2 u = cv.u[o];
          rp2 += cabs2(csub(u, vn));
          const double2 s = csub(cadd(cv.s[o], u), vn);
          cv.s[o] = s;
          cv.c[o] = csub(vn, s);
        }
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->nonfinite = 1u;
  sred[0][grp][sc] = rp2;
  sred[1][grp][sc] = rd2;
  sred[2][grp][sc] = l1;
  __syncthreads();
  if (threadIdx.x < kBB) {
    for (int f = 0; f < 3; ++f) {
      double a = sred[f][0][threadIdx.x];
      for (int g = 1; g < 4; ++g) a += sred[f][g][threadIdx.x];
      red[((uint64_t)f * gridDim.x + blockIdx.x) * kBB + threadIdx.x] = a;
    }
  }
}

// Per scene: fixed-order sums over the CTAs -> trace[k][scene] = (r_p, r_d, NaN).
// kBFinParts thread groups per scene each sum a strided subset of the CTA partials
// (loads independent, 4 in flight per thread), then the parts are added in order:
// a fixed association, so the trace is deterministic.  Launch: kBB * kBFinParts threads.
constexpr int kBFinParts = 16;
__device__ __forceinline__ double bfin_part_sum(const double* __restrict__ red, uint64_t base, uint32_t n,
                                                uint32_t part, uint32_t sc) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  uint32_t c = part;
  for (; c + 3 * kBFinParts < n; c += 4 * kBFinParts) {
    a0 += red[(base + c) * kBB + sc];
    a1 += red[(base + c + kBFinParts) * kBB + sc];
    a2 += red[(base + c + 2 * kBFinParts) * kBB + sc];
    a3 += red[(base + c + 3 * kBFinParts) * kBB + sc];
  }
  for (; c < n; c += kBFinParts) a0 += red[(base + c) * kBB + sc];
  return (a0 + a1) + (a2 + a3);
}

__global__ void __launch_bounds__(kBB * kBFinParts)
bfinalize_kernel(const double* __restrict__ red, uint32_t nct, uint32_t B, const Params* __restrict__ prm,
                 double* __restrict__ trace, uint64_t trace_cap, IterState* st) {
  __shared__ double sp[2][kBFinParts][kBB];
  const uint32_t sc = threadIdx.x % kBB, part = threadIdx.x / kBB;
  const uint64_t k = st->iter;
  sp[0][part][sc] = bfin_part_sum(red, 0, nct, part, sc);
  sp[1][part][sc] = bfin_part_sum(red, nct, nct, part, sc);
  __syncthreads();
  if (part == 0 && sc < B && k < trace_cap) {
    double a = sp[0][0][sc], d = sp[1][0][sc];
    for (int q = 1; q < kBFinParts; ++q) a += sp[0][q][sc], d += sp[1][q][sc];
    double* tr = trace + (k * B + sc) * 3;
    tr[0] = sqrt(a);
    tr[1] = sqrt(prm->rho * prm->rho * prm->m_rep * d);
    tr[2] = __longlong_as_double(0x7ff8000000000000ll);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (st->nonfinite && st->first_bad == ~0ull) st->first_bad = k;
    st->nonfinite = 0u;
    st->iter = k + 1;
  }
}

// Per-scene objective (admm_core.hpp:60-64) by the recurrence of objective_rec_kernel:
// a_b = (w' + h_b,prev + ghat_b) / 2, h_b = a_b - w', w' = G_ij - R after brows<kRhs>.
// Grid (gx, row blocks), 256 threads: scene = tid % 64, rows tid / 64 + 4 k.  Per-CTA,
// per-scene partials of |Hv - g|^2 (fixed order); skipped while st->iter < min_iter.
__global__ void __launch_bounds__(kCtaThreads)
bobjective_rec_kernel(BRowVecs rv, double2* __restrict__ hs, const BlockDesc* __restrict__ blocks, uint32_t N,
                      uint32_t B, double* __restrict__ ored, const IterState* st, uint64_t min_iter) {
  __shared__ double sm[kCtaThreads / kBB][kBB];
  const uint32_t i = blockIdx.y;
  const BlockDesc b0 = blocks[i * N];
  const uint32_t sc = threadIdx.x % kBB, grp = threadIdx.x / kBB;
  constexpr uint32_t G = kCtaThreads / kBB;
  double q = 0.0;
  if (sc < B && st->iter >= min_iter) {
    for (uint32_t row = blockIdx.x * G + grp; row < b0.rows; row += gridDim.x * G) {
      double2 hv = make_double2(0.0, 0.0);
      for (uint32_t j = 0; j < N; ++j) {
        const uint64_t o = ((uint64_t)blocks[i * N + j].mvec_off + row) * B + sc;
        const double2 w = csub(rv.gij[o], rv.r[o]);
        const double2 a = cscale(cadd(cadd(w, hs[o]), rv.ghat[o]), 0.5);
        hs[o] = csub(a, w);
        hv = cadd(hv, a);
      }
      q += cabs2(csub(hv, rv.g[((uint64_t)b0.row0 + row) * B + sc]));
    }
  }
  sm[grp][sc] = q;
  __syncthreads();
  if (threadIdx.x < kBB) {
    double a = sm[0][threadIdx.x];
    for (uint32_t g = 1; g < G; ++g) a += sm[g][threadIdx.x];
    ored[((uint64_t)blockIdx.y * gridDim.x + blockIdx.x) * kBB + threadIdx.x] = a;
  }
}

// trace[iter - 1][scene].objective = 0.5 sum |Hv - g|^2 + lambda_b ||v_b||_1 (the l1
// partials of bzupdate, red[2][pz][64]); one thread per scene, fixed order.
__global__ void __launch_bounds__(kBB * kBFinParts)
bobjective_trace_kernel(const double* __restrict__ red, uint32_t pz, const double* __restrict__ ored, uint32_t no,
                        const double* __restrict__ lam, uint32_t B, double* __restrict__ trace, uint64_t trace_cap,
                        const IterState* st) {
  __shared__ double sp[2][kBFinParts][kBB];
  const uint32_t sc = threadIdx.x % kBB, part = threadIdx.x / kBB;
  const uint64_t k = st->iter - 1;
  if (st->iter == 0 || k >= trace_cap) return;  // uniform over the CTA
  sp[0][part][sc] = bfin_part_sum(ored, 0, no, part, sc);
  sp[1][part][sc] = bfin_part_sum(red, 2 * (uint64_t)pz, pz, part, sc);
  __syncthreads();
  if (part == 0 && sc < B) {
    double o = sp[0][0][sc], l = sp[1][0][sc];
    for (int q = 1; q < kBFinParts; ++q) o += sp[0][q][sc], l += sp[1][q][sc];
    trace[(k * B + sc) * 3 + 2] = 0.5 * o + lam[sc] * l;
  }
}

// max_t |(H^H g_b)_t| per scene from Z = H^H G (segment sums over the row blocks).
__global__ void babsmax_kernel(const double2* __restrict__ z, const BlockDesc* __restrict__ blocks, uint32_t M,
                               uint32_t N, uint32_t B, double* __restrict__ out) {
  const uint32_t sc = threadIdx.x % kBB, grp = threadIdx.x / kBB;
  __shared__ double sm[4][kBB];
  double m = 0.0;
  if (sc < B)
    for (uint32_t j = 0; j < N; ++j)
      for (uint32_t t = blockIdx.x * 4 + grp; t < blocks[j].cols; t += gridDim.x * 4) {
        double2 a = make_double2(0.0, 0.0);
        for (uint32_t i = 0; i < M; ++i) a = cadd(a, z[((uint64_t)blocks[i * N + j].vec_off + t) * B + sc]);
        m = fmax(m, hypot(a.x, a.y));
      }
  sm[grp][sc] = m;
  __syncthreads();
  if (threadIdx.x < kBB) {
    double r = sm[0][threadIdx.x];
    for (int g = 1; g < 4; ++g) r = fmax(r, sm[g][threadIdx.x]);
    out[(uint64_t)blockIdx.x * kBB + threadIdx.x] = r;
  }
}

}  // namespace admm
