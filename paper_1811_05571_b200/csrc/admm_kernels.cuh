// admm_kernels.cuh — per-iteration kernels of the B200 ADMM engine.
//
// One ADMM iteration for every block b = (i, j) of the M x N grid (SURVEY.md
// Appendix A, the two-pass "q-form" of the reference Woodbury u-update,
// gram.hpp:63-78 + solvers.hpp:114-121/227-246/374-391):
//
//   w_b   = H_b c_b                     gemv_n_kernel  (stream H_b once)
//   r_b   = g_ij - w_b                  rows_finalize_kernel(kRhs)
//           g_ij = g_i - sum_{q!=j} ghat_iq   (ascending q, solvers.hpp:378-384)
//   q_b   = K_b r_b                     gemv_n_kernel  (K_b = (rho I + H_b H_b^H)^-1)
//   ghat_b = g_ij - rho q_b             rows_finalize_kernel(kQ)   (= H_b u_b exactly)
//   z_b   = H_b^H q_b                   gemv_h_kernel  (stream H_b once)
//   u_b = c_b + z_b; v_j = S_kappa(mean_i(u_b + s_b)); s_b += u_b - v_j; c_b = v_j - s_b;
//   residual partials                   zupdate_kernel
//   trace[k] = (r_p, r_d, objective)     finalize_kernel
//
// Both GEMVs are "stream-K": the (matrix, row-group, column-chunk) work units
// of ALL blocks are linearised and split evenly over a persistent grid of
// P CTAs, so every SM streams the same number of bytes whatever the block
// shapes.  A CTA accumulates consecutive units of the same output in
// registers and writes one partial per (output, CTA); consumers reduce the
// partials in fixed CTA order, so results are bit-reproducible (no float
// atomics anywhere).
#pragma once

#include "admm_common.cuh"

namespace admm {

// One row-major matrix streamed by a GEMV launch.
struct MatDesc {
  uint64_t a_off;     // element offset of the matrix in the storage arena
  uint64_t x_off;     // element offset of its input vector in the FP64 vector arena
  uint64_t part_off;  // double2 offset of its partial-sum region
  uint64_t unit0;     // first global work unit of this matrix
  uint32_t rows, cols, ld;
  uint32_t n_chunks;  // gemv_n: column chunks per row group | gemv_h: column chunks
  uint32_t n_tiles;   // gemv_n: row groups                   | gemv_h: row tiles
  uint32_t lid;       // local block index (row of the plan's block table)
};

// Per-block indexing used by the elementwise kernels.
struct BlockDesc {
  uint32_t i, j;        // grid coordinates (worker id = i*N + j, solvers.hpp:305)
  uint32_t rows, cols;  // m_b, n_b
  uint32_t row0, col0;  // global row / column of the block's first entry
  uint32_t mvec_off;    // offset of the block's m-vectors (ghat, g_ij, r, q)
  uint32_t vec_off;     // offset of the block's n-vectors (u, s, c)
  uint32_t seg_off;     // offset of segment j in the segment arena (v, v_prev)
  uint32_t jl;          // local segment index of column block j (sharded plans)
  uint32_t box_off;     // offset of the block's u+s in the outbox exchange buffer
  uint32_t pad_;
};

// Scalars read by the kernels from device memory, so a captured CUDA graph
// stays valid when lambda / rho change between solves.
struct Params {
  double rho;
  double kappa;   // lambda/(M rho) (consensus, hybrid) or lambda/rho (sectioning, reference)
  double lambda;
  double m_rep;   // M as double (replica count in the mean and in r_d)
};

// Device-side iteration state (one per plan).
struct IterState {
  uint64_t iter;        // iterations completed since reset
  uint64_t first_bad;   // first iteration with a non-finite u (UINT64_MAX: none)
  uint32_t nonfinite;   // flag raised by zupdate in the current iteration
  uint32_t pad_;
};

constexpr int kRowsPerWarpN = 8;          // gemv_n: rows per warp per unit
constexpr int kRowsPerGroup = kCtaWarps * kRowsPerWarpN;  // gemv_n: rows per unit
constexpr int kRowsPerWarpH = 4;          // gemv_h: rows per warp per tile
constexpr int kRowTileH = kCtaWarps * kRowsPerWarpH;

// Number of partial segments written for a run of units [first, first+count).
__host__ __device__ __forceinline__ uint32_t seg_count(uint64_t first, uint64_t count, uint64_t U,
                                              uint64_t P) {
  return (uint32_t)(sk_owner(first + count - 1, U, P) - sk_owner(first, U, P) + 1);
}

// Load the FP64 x values matching one 32-byte storage vector (PV columns).
template <int PV>
__device__ __forceinline__ void load_x(const double2* __restrict__ x, double2 (&out)[PV]) {
  const V256 a = *reinterpret_cast<const V256*>(x);  // L1-cached: shared by the CTA's 8 rows
  out[0] = make_double2(__longlong_as_double((long long)a.w[0]), __longlong_as_double((long long)a.w[1]));
  out[1] = make_double2(__longlong_as_double((long long)a.w[2]), __longlong_as_double((long long)a.w[3]));
  if constexpr (PV == 4) {
    const V256 b = *reinterpret_cast<const V256*>(x + 2);
    out[2] = make_double2(__longlong_as_double((long long)b.w[0]), __longlong_as_double((long long)b.w[1]));
    out[3] = make_double2(__longlong_as_double((long long)b.w[2]), __longlong_as_double((long long)b.w[3]));
  }
}

// y_b = A_b x_b for a set of matrices; linalg.hpp:97-111 (matvec).
// Unit = (matrix, group of 32 rows, chunk of CN columns).  Lanes own columns, each
// warp owns 4 rows of the group, so one load of x (L1) serves 4 streamed rows of A.
template <typename S, int VN, int EF>
__global__ void __launch_bounds__(kCtaThreads, 2)
gemv_n_kernel(const S* __restrict__ A, const double2* __restrict__ X, double2* __restrict__ part,
              const MatDesc* __restrict__ mats, int nmats, uint64_t U) {
  constexpr int PV = Store<S>::kPerVec;
  constexpr int CN = kWarp * VN * PV;
  constexpr int RW = kRowsPerWarpN;
  const uint64_t P = gridDim.x, p = blockIdx.x;
  uint64_t x = sk_lo(p, U, P);
  const uint64_t xe = sk_lo(p + 1, U, P);
  if (x >= xe) return;
  const int warp = warp_index(), lane = threadIdx.x % kWarp;
  int b = find_desc(mats, nmats, x);
  MatDesc md = mats[b];
  uint64_t local = x - md.unit0;
  uint32_t rg = (uint32_t)(local / md.n_chunks), cc = (uint32_t)(local % md.n_chunks);
  double2 acc[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) acc[r] = make_double2(0.0, 0.0);
  for (;;) {
    const uint32_t row0 = rg * kRowsPerGroup + warp * RW;
    const uint32_t c0 = cc * CN + lane * PV;
    V256 hv[RW][VN];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const S* arow = A + md.a_off + (uint64_t)(row0 + r) * md.ld;
#pragma unroll
      for (int v = 0; v < VN; ++v) {
        const uint32_t col = c0 + v * kWarp * PV;
        if (row0 + r < md.rows && col < md.cols) {
          hv[r][v] = ld_stream256<EF>(arow + col);
        } else {
          hv[r][v].w[0] = hv[r][v].w[1] = hv[r][v].w[2] = hv[r][v].w[3] = 0;
        }
      }
    }
    const double2* xv = X + md.x_off;
#pragma unroll
    for (int v = 0; v < VN; ++v) {
      const uint32_t col = c0 + v * kWarp * PV;
      if (col < md.cols) {
        double2 xs[PV];
        load_x<PV>(xv + col, xs);
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
          for (int e = 0; e < PV; ++e) cmac(acc[r], Store<S>::get(hv[r][v], e), xs[e]);
      }
    }
    ++x;
    ++cc;
    if (cc == md.n_chunks || x == xe) {  // flush this row group's partial
      const uint64_t first = md.unit0 + (uint64_t)rg * md.n_chunks;
      const uint64_t seg = p - sk_owner(first, U, P);
      double2* dst = part + md.part_off + ((uint64_t)rg * md.n_chunks + seg) * kRowsPerGroup + warp * RW;
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        double2 a = acc[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
          a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
        }
        if (lane == 0 && row0 + r < md.rows) dst[r] = a;
        acc[r] = make_double2(0.0, 0.0);
      }
      if (x == xe) break;
      if (cc == md.n_chunks) {
        cc = 0;
        if (++rg == md.n_tiles) {
          md = mats[++b];
          rg = 0;
        }
      }
    }
  }
}

// z_b = A_b^H q_b for a set of matrices; linalg.hpp:114-127 (adjoint_matvec).
// Unit = (matrix, chunk of CH columns, tile of 32 rows); lanes own columns,
// warps split the rows; partials are combined across warps through SMEM.
template <typename S, int VH, int EF>
__global__ void __launch_bounds__(kCtaThreads, 3)
gemv_h_kernel(const S* __restrict__ A, const double2* __restrict__ Q, double2* __restrict__ part,
              const MatDesc* __restrict__ mats, int nmats, uint64_t U) {
  constexpr int PV = Store<S>::kPerVec;
  constexpr int CH = kWarp * VH * PV;
  constexpr int NACC = VH * PV;
  __shared__ double2 red[kCtaWarps][CH];
  const uint64_t P = gridDim.x, p = blockIdx.x;
  uint64_t x = sk_lo(p, U, P);
  const uint64_t xe = sk_lo(p + 1, U, P);
  if (x >= xe) return;
  const int warp = warp_index(), lane = threadIdx.x % kWarp;
  int b = find_desc(mats, nmats, x);
  MatDesc md = mats[b];
  uint64_t local = x - md.unit0;
  uint32_t cc = (uint32_t)(local / md.n_tiles), rt = (uint32_t)(local % md.n_tiles);
  double2 acc[NACC];
#pragma unroll
  for (int a = 0; a < NACC; ++a) acc[a] = make_double2(0.0, 0.0);
  for (;;) {
    const uint32_t c0 = cc * CH + lane * PV;
    V256 hv[kRowsPerWarpH][VH];
    double2 qv[kRowsPerWarpH];
#pragma unroll
    for (int r = 0; r < kRowsPerWarpH; ++r) {
      const uint32_t row = rt * kRowTileH + r * kCtaWarps + warp;
      const bool rok = row < md.rows;
      qv[r] = rok ? Q[md.x_off + row] : make_double2(0.0, 0.0);
      // Unconditional loads from clamped addresses (no zero-fill, no predicated LDG): a row past
      // the block reads the last row against q = 0 (H is validated finite), a column past the
      // padded row reads the row's last vector into accumulators of columns >= cols, which no
      // consumer reads (columns in [cols, ld) are the arena's zero padding).
      const S* arow = A + md.a_off + (uint64_t)(rok ? row : md.rows - 1) * md.ld;
#pragma unroll
      for (int v = 0; v < VH; ++v) {
        const uint32_t col = c0 + v * kWarp * PV;
        hv[r][v] = ld_stream256<EF>(arow + min(col, md.ld - PV));
      }
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarpH; ++r)
#pragma unroll
      for (int v = 0; v < VH; ++v)
#pragma unroll
        for (int e = 0; e < PV; ++e) cmac_conj(acc[v * PV + e], Store<S>::get(hv[r][v], e), qv[r]);
    ++x;
    ++rt;
    if (rt == md.n_tiles || x == xe) {  // flush this column chunk's partial
#pragma unroll
      for (int v = 0; v < VH; ++v)
#pragma unroll
        for (int e = 0; e < PV; ++e) {
          red[warp][lane * PV + v * kWarp * PV + e] = acc[v * PV + e];
          acc[v * PV + e] = make_double2(0.0, 0.0);
        }
      __syncthreads();
      const uint64_t first = md.unit0 + (uint64_t)cc * md.n_tiles;
      const uint64_t seg = p - sk_owner(first, U, P);
      double2* dst = part + md.part_off + ((uint64_t)cc * md.n_tiles + seg) * CH;
      for (int c = threadIdx.x; c < CH; c += kCtaThreads) {
        double2 s = red[0][c];
#pragma unroll
        for (int w = 1; w < kCtaWarps; ++w) s = cadd(s, red[w][c]);
        dst[c] = s;
      }
      __syncthreads();
      if (x == xe) break;
      if (rt == md.n_tiles) {
        rt = 0;
        if (++cc == md.n_chunks) {
          md = mats[++b];
          cc = 0;
        }
      }
    }
  }
}

// Sum of the gemv_n partials of row `row` of matrix md (fixed CTA order).
__device__ __forceinline__ double2 sum_rows_part(const double2* __restrict__ part, const MatDesc& md,
                                                 uint32_t row, uint64_t U, uint64_t P) {
  const uint32_t rg = row / kRowsPerGroup, w = row % kRowsPerGroup;
  const uint64_t first = md.unit0 + (uint64_t)rg * md.n_chunks;
  const uint32_t nseg = seg_count(first, md.n_chunks, U, P);
  const double2* src = part + md.part_off + (uint64_t)rg * md.n_chunks * kRowsPerGroup + w;
  double2 s = src[0];
#pragma unroll 8
  for (uint32_t k = 1; k < nseg; ++k) s = cadd(s, src[(uint64_t)k * kRowsPerGroup]);  // loads hoisted, adds in order
  return s;
}

// Sum of the gemv_h partials of column `col` of matrix md (fixed CTA order).
template <int CH>
__device__ __forceinline__ double2 sum_cols_part(const double2* __restrict__ part, const MatDesc& md,
                                                 uint32_t col, uint64_t U, uint64_t P) {
  const uint32_t cc = col / CH, cl = col % CH;
  const uint64_t first = md.unit0 + (uint64_t)cc * md.n_tiles;
  const uint32_t nseg = seg_count(first, md.n_tiles, U, P);
  const double2* src = part + md.part_off + (uint64_t)cc * md.n_tiles * CH + cl;
  double2 s = src[0];
#pragma unroll 8
  for (uint32_t k = 1; k < nseg; ++k) s = cadd(s, src[(uint64_t)k * CH]);
  return s;
}

struct RowVecs {
  const double2* g;      // full g (scaled), n_meas
  double2* ghat;         // per-block m-vectors
  double2* gij;
  double2* r;
  double2* q;
};

// kRhs: g_ij = g_i - sum_{q != j} ghat_iq (ascending q), r_b = g_ij - H_b c_b.
// kQ:   q_b = sum(partials of K_b r_b), ghat_b = g_ij - rho q_b.
enum RowStage { kRhs = 0, kQ = 1 };

// g_ij[row] = g_i - sum_{q != j} ghat_iq in ascending q (solvers.hpp:378-384); the ghat
// loads are issued 8 at a time (independent), the subtractions stay in order.
// gblocks: the global block table (a sharded plan's peers too).
__device__ __forceinline__ double2 gij_row(const RowVecs& rv, const BlockDesc* __restrict__ gblocks,
                                           const BlockDesc& bd, uint32_t N, uint32_t row) {
  double2 gij = rv.g[bd.row0 + row];
  for (uint32_t q0 = 0; q0 < N; q0 += 8) {
    double2 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t qj = q0 + e;
      if (qj < N && qj != bd.j) v[e] = rv.ghat[gblocks[bd.i * N + qj].mvec_off + row];
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t qj = q0 + e;
      if (qj < N && qj != bd.j) gij = csub(gij, v[e]);
    }
  }
  return gij;
}

template <int Stage>
__global__ void __launch_bounds__(kCtaThreads)
rows_finalize_kernel(RowVecs rv, const double2* __restrict__ part, const MatDesc* __restrict__ mats,
                     const BlockDesc* __restrict__ blocks, const BlockDesc* __restrict__ gblocks, uint32_t N,
                     uint64_t U, uint64_t P, const Params* __restrict__ prm) {
  const uint32_t b = blockIdx.y;
  const BlockDesc bd = blocks[b];
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= bd.rows) return;
  const MatDesc md = mats[b];
  const double2 s = sum_rows_part(part, md, row, U, P);
  const uint32_t o = bd.mvec_off + row;
  if constexpr (Stage == kRhs) {
    const double2 gij = gij_row(rv, gblocks, bd, N, row);
    rv.gij[o] = gij;
    rv.r[o] = csub(gij, s);
  } else {
    rv.q[o] = s;
    rv.ghat[o] = csub(rv.gij[o], cscale(s, prm->rho));
  }
}

struct ColVecs {
  double2* u;      // per-block n-vectors
  double2* s;
  double2* c;
  double2* v;      // segment arena
  double2* vprev;
};

// Per column t of segment j: u_ij = c_ij + z_ij for every replica i; the
// replica mean of (u + s) in ascending i (solvers.hpp:130-136 / 404-415);
// v = S_kappa(mean) (prox.hpp); residual partials (solvers.hpp:141-145,
// 417-424); and the dual update for the next iteration (admm_core.hpp:87-89,
// applied here instead of at the start of the next iteration — same values).
template <int CH>
__global__ void __launch_bounds__(kCtaThreads)
zupdate_kernel(ColVecs cv, const double2* __restrict__ part, const MatDesc* __restrict__ mats,
               const BlockDesc* __restrict__ blocks, uint32_t M, uint32_t N, uint64_t U, uint64_t P,
               const Params* __restrict__ prm, double* __restrict__ red, IterState* st,
               uint32_t* __restrict__ nzcnt = nullptr) {  // support counts per CTA (admm_sparse.cuh)
  __shared__ double sm[kCtaWarps];
  const uint32_t j = blockIdx.y;
  const BlockDesc b0 = blocks[j];  // replica 0 of segment j
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
  bool bad = false, nz = false;
  if (t < b0.cols) {
    const double kappa = prm->kappa;
    double2 mean = make_double2(0.0, 0.0);
    for (uint32_t i = 0; i < M; ++i) {
      const BlockDesc bd = blocks[i * N + j];
      const double2 z = sum_cols_part<CH>(part, mats[i * N + j], t, U, P);
      const uint32_t o = bd.vec_off + t;
      const double2 u = cadd(cv.c[o], z);
      bad |= !cfinite(u);
      cv.u[o] = u;
      mean = cadd(mean, cadd(u, cv.s[o]));
    }
    mean = make_double2(mean.x / prm->m_rep, mean.y / prm->m_rep);
    const double2 vn = soft_threshold(mean, kappa);
    nz = vn.x != 0.0 || vn.y != 0.0;
    const uint32_t so = b0.seg_off + t;
    const double2 vo = cv.v[so];
    cv.vprev[so] = vo;
    cv.v[so] = vn;
    rd2 = cabs2(csub(vn, vo));
    l1 = hypot(vn.x, vn.y);
    for (uint32_t i = 0; i < M; ++i) {
      const uint32_t o = blocks[i * N + j].vec_off + t;
      const double2 u = cv.u[o];
      rp2 += cabs2(csub(u, vn));
      const double2 s = csub(cadd(cv.s[o], u), vn);  // (s + u) - v
      cv.s[o] = s;
      cv.c[o] = csub(vn, s);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->nonfinite = 1u;
  if (nzcnt) {
    const int c = __syncthreads_count(nz);
    if (threadIdx.x == 0) nzcnt[blockIdx.y * gridDim.x + blockIdx.x] = (uint32_t)c;
  }
  const uint32_t cta = blockIdx.y * gridDim.x + blockIdx.x;
  const uint32_t nct = gridDim.x * gridDim.y;
  double r = block_sum<kCtaThreads>(rp2, sm);
  if (threadIdx.x == 0) red[cta] = r;
  r = block_sum<kCtaThreads>(rd2, sm);
  if (threadIdx.x == 0) red[nct + cta] = r;
  r = block_sum<kCtaThreads>(l1, sm);
  if (threadIdx.x == 0) red[2 * nct + cta] = r;
}

// Objective rows: res = (sum_j H_ij v_j) - g_i per global row (ascending j),
// partial sums of |res|^2 (admm_core.hpp:60-64).
__global__ void __launch_bounds__(kCtaThreads)
objective_rows_kernel(const double2* __restrict__ g, const double2* __restrict__ part,
                      const MatDesc* __restrict__ mats, const BlockDesc* __restrict__ blocks,
                      uint32_t N, uint64_t U, uint64_t P, double* __restrict__ red) {
  __shared__ double sm[kCtaWarps];
  const uint32_t i = blockIdx.y;
  const BlockDesc b0 = blocks[i * N];
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  double q = 0.0;
  if (row < b0.rows) {
    double2 hv = make_double2(0.0, 0.0);
    for (uint32_t jj = 0; jj < N; ++jj) hv = cadd(hv, sum_rows_part(part, mats[i * N + jj], row, U, P));
    q = cabs2(csub(hv, g[b0.row0 + row]));
  }
  const double r = block_sum<kCtaThreads>(q, sm);
  if (threadIdx.x == 0) red[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

// Per-iteration objective (admm_core.hpp:60-64) WITHOUT a pass over H.  For block b
// let a_b = H_b v and h_b = H_b s_b (this iteration's v and s).  Two products the
// iteration already has pin them: w' = H_b c' with c' = v - s_b (the next w, read back as
// g_ij - r after rows_finalize), and ghat_b = H_b u_b (still in the ghat buffer).  The
// dual update s_b = s_b,prev + u_b - v (admm_core.hpp:87-89) gives
//     h_b = h_b,prev + ghat_b - a_b,   a_b - h_b = w'   =>   a_b = (w' + h_b,prev + ghat_b) / 2,
// with h_b = 0 before the first iteration (s = 0).  Row r of row block i:
// (H v)_r = sum_j a_ij,r (ascending j).  Writes per-CTA partials of |Hv - g|^2; skipped
// (zero partials, h untouched) while st->iter < min_iter.
// Parallel over (row, column block): 256 threads = RT rows x NP lanes (NP = 2^np_log2 >=
// N), so a sectioning row block of 1024 rows and N = 8 spreads over 32 CTAs instead of 4.
// Each lane updates one a_ij / h_ij; lane 0 of each row sums the row's a_ij in ascending j.
__global__ void __launch_bounds__(kCtaThreads)
objective_rec_kernel(RowVecs rv, double2* __restrict__ hs, const BlockDesc* __restrict__ blocks, uint32_t N,
                     uint32_t np_log2, double* __restrict__ red, const IterState* st, uint64_t min_iter) {
  __shared__ double2 sa[kCtaThreads];
  __shared__ double sm[kCtaWarps];
  const uint32_t i = blockIdx.y;
  const BlockDesc b0 = blocks[i * N];  // descriptors are constant: read before the PDL wait
  const uint32_t NP = 1u << np_log2, j = threadIdx.x & (NP - 1), rl = threadIdx.x >> np_log2;
  const uint32_t mv = j < N ? blocks[i * N + j].mvec_off : 0u;
  pdl_enter();
  const uint32_t row = blockIdx.x * (kCtaThreads >> np_log2) + rl;
  const bool on = st->iter >= min_iter && row < b0.rows;
  double2 a = make_double2(0.0, 0.0);
  if (on && j < N) {
    const uint64_t o = (uint64_t)mv + row;
    const double2 w = csub(rv.gij[o], rv.r[o]);
    a = cscale(cadd(cadd(w, hs[o]), rv.ghat[o]), 0.5);
    hs[o] = csub(a, w);
  }
  sa[threadIdx.x] = a;
  __syncthreads();
  double q = 0.0;
  if (on && j == 0) {
    double2 hv = make_double2(0.0, 0.0);
    for (uint32_t jj = 0; jj < N; ++jj) hv = cadd(hv, sa[rl * NP + jj]);
    q = cabs2(csub(hv, rv.g[b0.row0 + row]));
  }
  const double r = block_sum<kCtaThreads>(q, sm);
  if (threadIdx.x == 0) red[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

// Single-CTA epilogue of an iteration: fixed-order sums of the per-CTA
// partials, trace[k] = (sqrt(rp2), sqrt(rho*rho*M*rd2), objective), and the
// non-finite bookkeeping behind NumericalError(last_good_iteration).
__global__ void __launch_bounds__(kCtaThreads)
finalize_kernel(const double* __restrict__ red, uint32_t nz, const double* __restrict__ ored,
                uint32_t no, const Params* __restrict__ prm, double* __restrict__ trace,
                uint64_t trace_cap, IterState* st) {
  __shared__ double sm[kCtaWarps];
  double a = 0.0, d = 0.0, l = 0.0, o = 0.0;
  for (uint32_t k = threadIdx.x; k < nz; k += kCtaThreads) {
    a += red[k];
    d += red[nz + k];
    l += red[2 * nz + k];
  }
  for (uint32_t k = threadIdx.x; k < no; k += kCtaThreads) o += ored[k];
  a = block_sum<kCtaThreads>(a, sm);
  d = block_sum<kCtaThreads>(d, sm);
  l = block_sum<kCtaThreads>(l, sm);
  o = block_sum<kCtaThreads>(o, sm);
  if (threadIdx.x == 0) {
    const uint64_t k = st->iter;
    if (k < trace_cap) {
      trace[3 * k] = sqrt(a);
      trace[3 * k + 1] = sqrt(prm->rho * prm->rho * prm->m_rep * d);
      trace[3 * k + 2] = no ? 0.5 * o + prm->lambda * l : __longlong_as_double(0x7ff8000000000000ll);
    }
    if (st->nonfinite && st->first_bad == ~0ull) st->first_bad = k;
    st->nonfinite = 0u;
    st->iter = k + 1;
  }
}

// ---- sharded two-pass iteration (replicas of a segment on different GPUs) -------
// (after gemv_h) u_b = c_b + z_b for the local blocks; u_b + s_b goes to this rank's
// slot of the outbox exchange buffer (all-gathered over the column communicator).
template <int CH>
__global__ void __launch_bounds__(kCtaThreads)
uupdate_kernel(ColVecs cv, double2* __restrict__ outbox, const double2* __restrict__ part,
               const MatDesc* __restrict__ mats, const BlockDesc* __restrict__ blocks, uint64_t U, uint64_t P,
               IterState* st) {
  const uint32_t b = blockIdx.y;
  const BlockDesc bd = blocks[b];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (t < bd.cols) {
    const double2 z = sum_cols_part<CH>(part, mats[b], t, U, P);
    const uint32_t o = bd.vec_off + t;
    const double2 u = cadd(cv.c[o], z);
    bad = !cfinite(u);
    cv.u[o] = u;
    outbox[bd.box_off + t] = cadd(u, cv.s[o]);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->nonfinite = 1u;
}

// (after the outbox all-gather) per local segment jl: the replica mean over ALL M row
// blocks in ascending i (solvers.hpp:404-415), v = S_kappa(mean), and the dual / next-c
// update of the local blocks.  r_d and |v|_1 are counted by the pr == 0 rank only (the
// other ranks of the column communicator hold the same segment).
__global__ void __launch_bounds__(kCtaThreads)
zfinal_kernel(ColVecs cv, const double2* __restrict__ outbox, const BlockDesc* __restrict__ blocks,
              uint32_t M, uint32_t Mr, uint32_t Nc, uint32_t npad, int count_v, const Params* __restrict__ prm,
              double* __restrict__ red,
              uint32_t* __restrict__ nzcnt = nullptr) {  // support counts per CTA (sharded support schedule)
  __shared__ double sm[kCtaWarps];
  const uint32_t jl = blockIdx.y;
  const BlockDesc b0 = blocks[jl];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  double rp2 = 0.0, rd2 = 0.0, l1 = 0.0;
  bool nz = false;
  if (t < b0.cols) {
    double2 mean = make_double2(0.0, 0.0);
    for (uint32_t i = 0; i < M; ++i) mean = cadd(mean, outbox[((uint64_t)i * Nc + jl) * npad + t]);
    mean = make_double2(mean.x / prm->m_rep, mean.y / prm->m_rep);
    const double2 vn = soft_threshold(mean, prm->kappa);
    nz = vn.x != 0.0 || vn.y != 0.0;
    const uint32_t so = b0.seg_off + t;
    const double2 vo = cv.v[so];
    cv.vprev[so] = vo;
    cv.v[so] = vn;
    if (count_v) {
      rd2 = cabs2(csub(vn, vo));
      l1 = hypot(vn.x, vn.y);
    }
    for (uint32_t il = 0; il < Mr; ++il) {
      const uint32_t o = blocks[il * Nc + jl].vec_off + t;
      const double2 u = cv.u[o];
      rp2 += cabs2(csub(u, vn));
      const double2 s = csub(cadd(cv.s[o], u), vn);
      cv.s[o] = s;
      cv.c[o] = csub(vn, s);
    }
  }
  const uint32_t cta = blockIdx.y * gridDim.x + blockIdx.x, nct = gridDim.x * gridDim.y;
  if (nzcnt) {
    const int c = __syncthreads_count(nz);
    if (threadIdx.x == 0) nzcnt[cta] = (uint32_t)c;
  }
  double r = block_sum<kCtaThreads>(rp2, sm);
  if (threadIdx.x == 0) red[cta] = r;
  r = block_sum<kCtaThreads>(rd2, sm);
  if (threadIdx.x == 0) red[nct + cta] = r;
  r = block_sum<kCtaThreads>(l1, sm);
  if (threadIdx.x == 0) red[2 * nct + cta] = r;
}

// Scalar slot of one rank in the exchange (doubles): rp2, rd2, |v|_1, non-finite flag,
// objective rows |Hv - g|^2 partial, spare.
constexpr int kScalDoubles = 8;

// This rank's iteration scalars (rp2, rd2, l1, non-finite; objective-rows partials when
// objp != null) into its slot of the scalar exchange buffer (all-gathered over all ranks).
__global__ void local_scalars_kernel(const double* __restrict__ red, uint32_t n, const double* __restrict__ objp,
                                     uint32_t nobj, double* __restrict__ slot, IterState* st) {
  __shared__ double sm[kCtaWarps];
  double a = 0.0, d = 0.0, l = 0.0, o = 0.0;
  for (uint32_t k = threadIdx.x; k < n; k += kCtaThreads) {
    a += red[k];
    d += red[n + k];
    l += red[2 * n + k];
  }
  if (objp)
    for (uint32_t k = threadIdx.x; k < nobj; k += kCtaThreads) o += objp[k];
  a = block_sum<kCtaThreads>(a, sm);
  d = block_sum<kCtaThreads>(d, sm);
  l = block_sum<kCtaThreads>(l, sm);
  o = block_sum<kCtaThreads>(o, sm);
  if (threadIdx.x == 0) {
    slot[0] = a;
    slot[1] = d;
    slot[2] = l;
    slot[3] = st->nonfinite ? 1.0 : 0.0;
    slot[4] = o;
    st->nonfinite = 0u;
  }
}

// Objective of a sharded plan (admm_core.hpp:60-64 without an H pass; the recurrence of
// objective_rec_kernel): a_b of every LOCAL block into the A region of its ghat exchange
// slot (gathered over the row communicator with ghat), h_b updated.  Skipped while
// st->iter < min_iter (the two-pass schedule computes the previous iteration's a_b).
__global__ void __launch_bounds__(kCtaThreads)
objective_arec_kernel(RowVecs rv, double2* __restrict__ hs, const BlockDesc* __restrict__ blocks, uint64_t aoff,
                      const IterState* st, uint64_t min_iter) {
  const BlockDesc bd = blocks[blockIdx.y];
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= bd.rows || st->iter < min_iter) return;
  const uint64_t o = (uint64_t)bd.mvec_off + row;
  const double2 w = csub(rv.gij[o], rv.r[o]);
  const double2 a = cscale(cadd(cadd(w, hs[o]), rv.ghat[o]), 0.5);
  hs[o] = csub(a, w);
  rv.ghat[o + aoff] = a;
}

// After the gather: |sum_q a_iq - g_i|^2 per row of the local row blocks (ascending q over
// ALL N column blocks, every a_iq from the gathered A regions), per-CTA partials (zero when
// count == 0 or st->iter < min_iter: that rank's rows are counted by another rank).
__global__ void __launch_bounds__(kCtaThreads)
objective_grows_kernel(const double2* __restrict__ g, const double2* __restrict__ xg, uint64_t aoff,
                       const BlockDesc* __restrict__ gblocks, uint32_t N, uint32_t i0, int count,
                       const IterState* st, uint64_t min_iter, double* __restrict__ objp) {
  __shared__ double sm[kCtaWarps];
  const uint32_t i = i0 + blockIdx.y;
  const BlockDesc b0 = gblocks[i * N];
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  double q = 0.0;
  if (count && row < b0.rows && st->iter >= min_iter) {
    double2 hv = make_double2(0.0, 0.0);
    for (uint32_t jj = 0; jj < N; ++jj) hv = cadd(hv, xg[gblocks[i * N + jj].mvec_off + aoff + row]);
    q = cabs2(csub(hv, g[b0.row0 + row]));
  }
  const double r = block_sum<kCtaThreads>(q, sm);
  if (threadIdx.x == 0) objp[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

// Final objective pass of a sharded plan: a_b = H_b v_j (row sums of gemv_n partials) into
// the A region of the ghat slot.
__global__ void __launch_bounds__(kCtaThreads)
arows_kernel(double2* __restrict__ xg, uint64_t aoff, const double2* __restrict__ part,
             const MatDesc* __restrict__ mats, const BlockDesc* __restrict__ blocks, uint64_t U, uint64_t P) {
  const uint32_t b = blockIdx.y;
  const BlockDesc bd = blocks[b];
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < bd.rows) xg[(uint64_t)bd.mvec_off + aoff + row] = sum_rows_part(part, mats[b], row, U, P);
}

// Final objective pass: slot[4] = sum of the rows partials, slot[2] = |v|_1 of the local
// segments (when count_v: one rank per column block counts them).
__global__ void obj_scalars_kernel(const double* __restrict__ objp, uint32_t nobj, const double2* __restrict__ v,
                                   const BlockDesc* __restrict__ blocks, uint32_t Nc, int count_v,
                                   double* __restrict__ slot) {
  __shared__ double sm[kCtaWarps];
  double o = 0.0, l = 0.0;
  for (uint32_t k = threadIdx.x; k < nobj; k += kCtaThreads) o += objp[k];
  if (count_v)
    for (uint32_t jl = 0; jl < Nc; ++jl) {
      const BlockDesc bd = blocks[jl];
      for (uint32_t t = threadIdx.x; t < bd.cols; t += kCtaThreads) {
        const double2 x = v[bd.seg_off + t];
        l += hypot(x.x, x.y);
      }
    }
  o = block_sum<kCtaThreads>(o, sm);
  l = block_sum<kCtaThreads>(l, sm);
  if (threadIdx.x == 0) {
    slot[2] = l;
    slot[4] = o;
  }
}

// Close an iteration from the all-gathered scalars (rank order): trace[k] and the
// non-finite bookkeeping, identically on every rank.  Objective (obj_mode):
//   0  none (NaN);
//   1  two-pass, lagged: trace[k-1] from the gathered rows partials of this iteration and
//      the |v|_1 of iteration k-1 (kept in *l1prev); trace[k] is filled next iteration or
//      by the final exact pass;
//   2  sweep (Pr == 1): trace[k] from this rank's complete rows sum (objp, every rank holds
//      all rows after the gather) and the gathered |v|_1.
__global__ void close_kernel(const double* __restrict__ all, uint32_t nranks, uint64_t stride,
                             const Params* __restrict__ prm, double* __restrict__ trace, uint64_t trace_cap,
                             IterState* st, int obj_mode, const double* __restrict__ objp, uint32_t nobj,
                             double* __restrict__ l1prev) {
  __shared__ double sm[kCtaWarps];
  double o = 0.0;
  if (obj_mode == 2)
    for (uint32_t k = threadIdx.x; k < nobj; k += kCtaThreads) o += objp[k];
  o = block_sum<kCtaThreads>(o, sm);
  if (threadIdx.x != 0) return;
  double a = 0.0, d = 0.0, l = 0.0, og = 0.0;
  bool bad = false;
  for (uint32_t r = 0; r < nranks; ++r) {  // rank order; `stride` doubles between rank slots
    a += all[stride * r];
    d += all[stride * r + 1];
    l += all[stride * r + 2];
    bad |= all[stride * r + 3] != 0.0;
    og += all[stride * r + 4];
  }
  const uint64_t k = st->iter;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  if (k < trace_cap) {
    trace[3 * k] = sqrt(a);
    trace[3 * k + 1] = sqrt(prm->rho * prm->rho * prm->m_rep * d);
    trace[3 * k + 2] = obj_mode == 2 ? 0.5 * o + prm->lambda * l : nan;
  }
  if (obj_mode == 1) {
    if (k >= 1 && k - 1 < trace_cap) trace[3 * (k - 1) + 2] = 0.5 * og + prm->lambda * *l1prev;
    *l1prev = l;
  }
  if (bad && st->first_bad == ~0ull) st->first_bad = k;
  st->iter = k + 1;
}

}  // namespace admm
