// admm_batched.cuh — multi-scene (batched right-hand side) ADMM iteration.
//
// BASELINE config 5: B independent scenes g_b share H, the partition and the Woodbury
// factors; each scene is an independent hybrid_solve (solvers.hpp:306) with its own
// lambda_b.  With B right-hand sides the two H products of an iteration become skinny
// complex GEMMs, W = H C and Z = H^H Q (C: n x B, Q: m x B), compute-bound on SIMT
// (tensor cores are reserved for setup by the north star).  Register-tiled FP64 SIMT:
// a 256-thread CTA owns a 64 x 64 output tile (64 rows or columns x up to 64 scenes),
// each thread a 4 x 4 complex sub-tile (rows ty + 16q, scenes tx + 16w: both SMEM
// operand reads are conflict-free); A and X stream through SMEM in k-chunks of 32.
// Vectors are [row][scene] (scene fastest), FP64 like the single-scene engine.
#pragma once

#include "admm_kernels.cuh"

namespace admm {

constexpr int kBT = 64;   // output tile: rows (N) or columns (adjoint)
constexpr int kBB = 64;   // scenes per tile
constexpr int kBK = 32;   // k-chunk

struct BTile {
  uint64_t a_off;   // matrix in the storage arena
  uint64_t x_off;   // X (k-major, [k][B]) in the vector arena
  uint64_t o_off;   // output (rows/cols x B) in the output arena
  uint32_t ld, rows, cols;
  uint32_t t0;      // first output row (N) / column (adjoint)
  uint32_t k0, k1;  // k range of this unit (split-K)
};

// out[t0 + i][b] = sum_{k in [k0,k1)} op(A)[t0 + i][k] X[k][b]
//   ADJ = false: op(A)[i][k] = A[i][k]          (W = H C, Q = K R)
//   ADJ = true:  op(A)[i][k] = conj(A[k][i])    (Z = H^H Q)
template <typename S, bool ADJ>
__global__ void __launch_bounds__(256, 2)
bgemm_kernel(const S* __restrict__ A, const BTile* __restrict__ tiles, const double2* __restrict__ X,
             double2* __restrict__ out, uint32_t B) {
  __shared__ double2 At[kBK][kBT + 1];
  __shared__ double2 Xs[kBK][kBB + 1];
  const BTile t = tiles[blockIdx.x];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const S* a = A + t.a_off;
  const uint32_t nout = ADJ ? t.cols : t.rows;
  double2 acc[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int w = 0; w < 4; ++w) acc[q][w] = make_double2(0.0, 0.0);
  for (uint32_t k0 = t.k0; k0 < t.k1; k0 += kBK) {
    for (int e = threadIdx.x; e < kBT * kBK; e += 256) {
      int i, kk;
      if (ADJ) {  // coalesced along the output columns
        kk = e / kBT;
        i = e % kBT;
      } else {    // coalesced along k
        i = e / kBK;
        kk = e % kBK;
      }
      const uint32_t oi = t.t0 + i, k = k0 + kk;
      double2 v = make_double2(0.0, 0.0);
      if (oi < nout && k < t.k1) {
        v = Store<S>::widen(ADJ ? a[(uint64_t)k * t.ld + oi] : a[(uint64_t)oi * t.ld + k]);
        if (ADJ) v.y = -v.y;
      }
      At[kk][i] = v;
    }
    for (int e = threadIdx.x; e < kBK * kBB; e += 256) {
      const int kk = e / kBB, b = e % kBB;
      const uint32_t k = k0 + kk;
      Xs[kk][b] = (k < t.k1 && (uint32_t)b < B) ? X[t.x_off + (uint64_t)k * B + b] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kBK; ++kk) {
      double2 av[4], xv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = At[kk][ty + 16 * q];
        xv[q] = Xs[kk][tx + 16 * q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w) cmac(acc[q][w], av[q], xv[w]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t oi = t.t0 + ty + 16 * q;
    if (oi >= nout) continue;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t b = tx + 16 * w;
      if (b < B) out[t.o_off + (uint64_t)oi * B + b] = acc[q][w];
    }
  }
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
__global__ void __launch_bounds__(kCtaThreads)
bzupdate_kernel(ColVecs cv, const double2* __restrict__ z, const BlockDesc* __restrict__ blocks, uint32_t M,
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
          const double2 u = cadd(cv.c[o], z[o]);
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
__global__ void bfinalize_kernel(const double* __restrict__ red, uint32_t nct, uint32_t B,
                                 const Params* __restrict__ prm, double* __restrict__ trace, uint64_t trace_cap,
                                 IterState* st) {
  const uint32_t sc = threadIdx.x;
  const uint64_t k = st->iter;
  if (sc < B && k < trace_cap) {
    double a = 0.0, d = 0.0;
    for (uint32_t c = 0; c < nct; ++c) {
      a += red[(uint64_t)c * kBB + sc];
      d += red[((uint64_t)nct + c) * kBB + sc];
    }
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
