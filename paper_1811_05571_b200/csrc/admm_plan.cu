// admm_plan.cu — host runtime of the B200 ADMM engine and its C ABI (admm_b200.h).
//
// One plan = one solve configuration on one device: the partition (partition.hpp),
// the uploaded blocks, the per-block Woodbury inverses (gram.hpp), the iterate
// vectors, and a captured CUDA graph of one ADMM iteration.  The reference's
// simulated node runtime (parallel_for + coordinator copies, parallel.hpp /
// solvers.hpp:109-136) becomes a single stream: all M*N blocks are processed by
// each kernel launch, and the coordinator reductions are fixed-order device sums.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <thread>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "admm_b200.h"
#include "admm_kernels.cuh"
#include "admm_setup.cuh"
#include "admm_sweep.cuh"
#include "admm_slab.cuh"
#include "admm_hemv.cuh"
#include "admm_batched.cuh"
#include "admm_sparse.cuh"
#include "admm_resident.cuh"
#include "admm_host.h"

using namespace admm;

namespace {

thread_local std::string g_last_error;
thread_local uint64_t g_last_good = 0;
thread_local uint64_t g_last_offset = 0;

struct Fail {
  admm_status st;
  std::string msg;
  uint64_t last_good = 0;
};

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw Fail{ADMM_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};       \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t b) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = b;
    CK(cudaMalloc(&p, std::max<size_t>(b, 256)));
    CK(cudaMemset(p, 0, std::max<size_t>(b, 256)));
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
uint64_t cdiv(uint64_t x, uint64_t a) { return (x + a - 1) / a; }

// partition.hpp:34-52 (split_bounds) with the reference's PartitionError texts.
std::vector<uint64_t> split_bounds(uint64_t total, uint64_t parts, bool ragged, const char* axis) {
  if (parts < 1 || parts > total)
    throw Fail{ADMM_E_PARTITION, std::string("make_partition: ") + axis + " division count " +
                                     std::to_string(parts) + " not in [1, " + std::to_string(total) + "]"};
  if (!ragged && total % parts != 0)
    throw Fail{ADMM_E_PARTITION, "make_partition: " + std::to_string(parts) + " does not divide " +
                                     std::to_string(total) + " " + axis +
                                     "s (pass ragged=true to allow uneven blocks)"};
  const uint64_t base = total / parts, rem = total % parts;
  std::vector<uint64_t> b(parts + 1, 0);
  for (uint64_t k = 0; k < parts; ++k) b[k + 1] = b[k] + base + (k < rem ? 1 : 0);
  return b;
}

template <typename T>
bool host_all_finite(const T* p, uint64_t n) {  // multi-threaded problem.validate() scan
  unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < (1u << 20)) nt = 1;
  std::vector<char> ok(nt, 1);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
      for (uint64_t i = lo; i < hi; ++i)
        if (!std::isfinite(p[i])) {
          ok[t] = 0;
          return;
        }
    });
  for (auto& x : th) x.join();
  for (char c : ok)
    if (!c) return false;
  return true;
}

// Streaming geometry (see admm_kernels.cuh).
constexpr int kVN = 1;  // 32-byte vectors per lane per row in gemv_n
constexpr int kVH = 2;  // 32-byte vectors per lane per row in gemv_h
template <typename S>
constexpr int chunk_n() { return kWarp * kVN * Store<S>::kPerVec; }
template <typename S>
constexpr int chunk_h() { return kWarp * kVH * Store<S>::kPerVec; }

struct Geom {
  uint64_t U = 0, P = 0;
};

}  // namespace

void admm_host_set_error(const char* msg, uint64_t byte_offset) {
  g_last_error = msg ? msg : "";
  g_last_offset = byte_offset;
}

struct admm_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;  // the plan's stream; `stream` may be a caller's (graph capture)
  admm_dtype dtype = ADMM_C128;
  admm_method method = ADMM_HYBRID;
  uint64_t n_meas = 0, n_pix = 0, M = 1, N = 1;
  // sharding over a Pr x Pc process grid; 1 x 1 for a single GPU
  uint64_t Pr = 1, Pc = 1, pr = 0, pc = 0, Mr = 1, Nc = 1, i0 = 0, j0 = 0;
  uint64_t mpad = 0, npad = 0, outbox_total = 0;
  std::vector<BlockDesc> gblocks;  // global M x N table (ghost entries for exchange layouts)
  DevBuf dgblocks, doutbox, dscal;
  double2* ghat_ptr = nullptr;     // ghat exchange buffer (internal or attached)
  double2* outbox_ptr = nullptr;
  double* scal_ptr = nullptr;
  bool fused_scal = false;   // Pr == 1, Pc > 1: scalars ride in the ghat all-gather slot
  uint64_t gslot = 0;        // ghat slot per rank (complex elements)
  bool keep_l2 = false;      // local H + K fit in L2: keep H resident across iterations
  bool ragged = false, trace_obj = false, obj_pass = false;  // obj_pass: objective by an extra H pass
  admm_solver_config cfg{};
  std::vector<uint64_t> rb, cb;
  std::vector<BlockDesc> blocks;
  std::vector<MatDesc> hN, hNv, kN, hH, hHg;
  std::vector<GramDesc> gram;
  uint64_t mvec_total = 0, vec_total = 0, seg_total = 0, h_elems = 0, k_elems = 0, a_elems = 0;
  uint32_t max_rows = 0, max_seg = 0, max_rowblock = 0, max_m = 0;
  DevBuf dH, dK, dg, dghat, dgij, dr, dq, du, ds, dc, dv, dvprev;
  DevBuf dwpart, dqpart, dzpart, dopart, dgpart, dhs;  // dhs: H_b s_b per block (objective recurrence)
  DevBuf dred, dored, dtrace, dstate, dparams, dblocks, dhN, dhNv, dkN, dhH, dhHg, dgram, dobj;
  Geom gN, gK, gH, gO, gG;
  // batched scenes (admm_batched.cuh): B right-hand sides sharing H and the factors
  uint64_t batch = 1;
  std::vector<BTile> tN, tK, tH, tG;
  DevBuf dtN, dtK, dtH, dtG, dz, dkappa, dbred, dblam, dbored;  // dblam: lambda_b; dbored: objective partials
  uint32_t bogx = 1;  // bobjective_rec_kernel grid x
  uint32_t splitN = 1, splitK = 1, splitH = 1, pz = 1;
  uint32_t bsb = 64;  // scenes per bgemm CTA tile (64 or 32)
  std::vector<double> lambdas;
  // sweep schedule (admm_sweep.cuh)
  int schedule = 1;             // 1 two-pass, 2 single-HBM-pass sweep
  int sweep_lpr = 8;
  int slab_rpl = 0;         // > 0: per-warp slab sweep (sweep_slab_kernel), rows per lane
  uint32_t slab_C = 1, slab_nw = 0, slab_ns = 0, slab_Ns = 0, slab_lag = 1, slab_nd = 1, slab_rb = 64;  // cluster size, compute warps, stages, slabs, (A) lag
  std::vector<SlabDesc> slabs;
  DevBuf dHs, dslabs;       // slab-major copy of H, slab table
  bool kpacked = false;     // K applied from the packed Hermitian tiles (hemv_kernel)
  bool h_evict_first = false;  // two-pass GEMVs stream H with L2 evict_first
  bool kkeep = false;       // ... with an L2 evict_last policy (ADMM_B200_KKEEP)
  int hemv_bulk = 0;        // hemv_bulk_kernel CTAs per SM (0: register variant hemv_kernel)
  DevBuf dkcnt;
  std::vector<HemvDesc> hv;
  DevBuf dKp, dhv, dkppart;
  Geom gP;
  DevBuf dtrace_tile;       // ADMM_B200_SLAB_TRACE: per-strip phase timestamps
  std::vector<SweepDesc> segs;
  DevBuf dsegs, dwpart_s;
  Geom gS;
  size_t sweep_smem = 0;
  uint32_t zgx = 0, rgx = 0, rgx_s = 0, ogx = 0, nz = 0, no = 0;
  uint32_t orgx = 1, onp = 0, nor = 1;  // objective_rec_kernel: grid x, log2 lanes per row, partials
  DevBuf drored;
  // resident schedule (4): per-CTA column ranges, w / residual / objective partials
  DevBuf dres_dbg;
  DevBuf dres_cta, dres_seg, dres_w, dres_red, dres_opart, dres_abuf, dres_lprev, dres_bar, dghat2;
  uint32_t res_P = 0, res_cols = 0;
  bool is_shard = false;  // created by admm_plan_create_sharded (driven phase by phase)
  // sharded objective (admm_kernels.cuh objective_arec/grows): offset of the A region in a
  // ghat slot (0: no per-iteration objective), rows partials, |v|_1 of the previous iteration
  uint64_t aoff = 0;
  bool shard_obj = false;   // sharded plan with the per-iteration objective
  uint32_t objgx = 1;
  DevBuf dobjp, dl1prev;
  // multi-GPU with plan-owned NCCL communicators (admm_dist.inc): a rank of a distributed
  // plan (dist != null), or a single-process container of one sub-plan per device (subs)
  struct Dist* dist = nullptr;
  std::vector<admm_plan*> subs;
  // support schedule (5, admm_sparse.cuh): column-major H, packed G = H H^H, a = H v
  DevBuf dHc, dhcoff, dhcld, danew, daold, dnzcnt, dnzlist, dnnz, dnnz_tot;
  uint32_t nzstride = 0, supgx = 1, sup_np = 0, sup_rgx = 1, sup_chunks = 16;
  size_t res_smem = 0;
  uint64_t trace_cap = 0;
  cudaGraphExec_t exec = nullptr;
  uint64_t graph_iters = 0;
  double setup_s = 0.0;
  double setup_phase[4] = {0, 0, 0, 0};  // validate (host scans), upload (+ layouts), Gram, inverse + packing
  double gram_device_s = 0.0, gram_flops = 0.0, inverse_device_s = 0.0, inverse_flops = 0.0;
  size_t elem = 16;
  int num_sms = 148;
  Params params{};
  // host scratch for snapshots
  std::vector<double> h_v, h_vprev, h_u, h_seg;

  ~admm_plan();
};

namespace {

template <typename S, typename K>
uint64_t grid_for(K kernel, uint64_t U, int sms, size_t smem = 0) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kCtaThreads, smem));
  occ = std::max(occ, 1);
  return std::max<uint64_t>(1, std::min<uint64_t>(U, (uint64_t)sms * occ));
}

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled
// while its predecessor runs; it must call pdl_enter() before touching the
// predecessor's output (sweep_kernel, rows_finalize_sweep_kernel, hemv_kernel,
// hemv_finalize_kernel do).  ADMM_B200_PDL=0 launches plainly.
bool pdl_enabled() { return true; }
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

template <typename S>
void build_geometry(admm_plan* p) {
  const uint64_t CN = chunk_n<S>(), CH = chunk_h<S>();
  const uint64_t nb = p->blocks.size();
  p->hN.assign(nb, {});
  p->hNv.assign(nb, {});
  p->kN.assign(nb, {});
  p->hH.assign(nb, {});
  p->hHg.assign(nb, {});
  p->gram.assign(nb, {});
  uint64_t uN = 0, uK = 0, uH = 0, pN = 0, pK = 0, pH = 0, hoff = 0, koff = 0, aoff = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    const BlockDesc& bd = p->blocks[b];
    const uint32_t ld = (uint32_t)round_up(bd.cols, 8), ldk = (uint32_t)round_up(bd.rows, 8);
    MatDesc n{};
    n.a_off = hoff;
    n.x_off = bd.vec_off;
    n.rows = bd.rows;
    n.cols = bd.cols;
    n.ld = ld;
    n.n_chunks = (uint32_t)cdiv(bd.cols, CN);
    n.n_tiles = (uint32_t)cdiv(bd.rows, kRowsPerGroup);
    n.unit0 = uN;
    n.part_off = pN;
    uN += (uint64_t)n.n_chunks * n.n_tiles;
    pN += (uint64_t)n.n_chunks * n.n_tiles * kRowsPerGroup;
    p->hN[b] = n;
    MatDesc nv = n;
    nv.x_off = bd.seg_off;
    p->hNv[b] = nv;
    MatDesc k{};
    k.a_off = koff;
    k.x_off = bd.mvec_off;
    k.rows = bd.rows;
    k.cols = bd.rows;
    k.ld = ldk;
    k.n_chunks = (uint32_t)cdiv(bd.rows, CN);
    k.n_tiles = (uint32_t)cdiv(bd.rows, kRowsPerGroup);
    k.unit0 = uK;
    k.part_off = pK;
    uK += (uint64_t)k.n_chunks * k.n_tiles;
    pK += (uint64_t)k.n_chunks * k.n_tiles * kRowsPerGroup;
    p->kN[b] = k;
    MatDesc h{};
    h.a_off = hoff;
    h.x_off = bd.mvec_off;
    h.rows = bd.rows;
    h.cols = bd.cols;
    h.ld = ld;
    h.n_chunks = (uint32_t)cdiv(bd.cols, CH);
    h.n_tiles = (uint32_t)cdiv(bd.rows, kRowTileH);
    h.unit0 = uH;
    h.part_off = pH;
    uH += (uint64_t)h.n_chunks * h.n_tiles;
    pH += (uint64_t)h.n_chunks * h.n_tiles * CH;
    p->hH[b] = h;
    MatDesc hg = h;
    hg.x_off = bd.row0;  // gemv_h over g itself: Q = g (global rows)
    p->hHg[b] = hg;
    GramDesc gd{};
    gd.h_off = hoff;
    gd.a_off = aoff;
    gd.k_off = koff;
    gd.m = bd.rows;
    gd.n = bd.cols;
    gd.ld = ld;
    gd.ldk = ldk;
    gd.mp = (uint32_t)round_up(bd.rows, kFT);
    p->gram[b] = gd;
    hoff += (uint64_t)bd.rows * ld;
    koff += (uint64_t)bd.rows * ldk;
    aoff += (uint64_t)gd.mp * gd.mp;
  }
  p->h_elems = hoff;
  p->k_elems = koff;
  p->a_elems = aoff;
  p->gN.U = uN;
  p->gK.U = uK;
  p->gH.U = uH;
  p->gO.U = uN;
  p->gG.U = uH;
  p->gN.P = grid_for<S>(gemv_n_kernel<S, kVN, kEvictNormal>, uN, p->num_sms);
  p->gK.P = grid_for<S>(gemv_n_kernel<S, kVN, kEvictNormal>, uK, p->num_sms);
  p->gH.P = grid_for<S>(gemv_h_kernel<S, kVH, kEvictNormal>, uH, p->num_sms);
  p->gO.P = p->gN.P;
  p->gG.P = p->gH.P;
  p->dwpart.alloc(pN * sizeof(double2));
  p->dopart.alloc(pN * sizeof(double2));
  p->dqpart.alloc(pK * sizeof(double2));
  p->dzpart.alloc(pH * sizeof(double2));
  p->dgpart.alloc(pH * sizeof(double2));
  p->dH.alloc(p->h_elems * sizeof(S));
}

void upload_desc(DevBuf& d, const void* src, size_t bytes);

template <typename S, int LPR>
size_t sweep_smem_bytes(const admm_plan* p) {
  constexpr int W = LPR * Store<S>::kPerVec;
  return ((size_t)p->n_meas + (2 * (size_t)kProdWarps + 4) * p->Mr * W) * sizeof(double2);
}

// The L2-re-read sweep with LPR lanes per row (the fallback single-pass kernel when the slab
// geometry does not fit).  False when the segment rows do not fit the SMEM accumulator or
// the open strips would not fit in L2 (then the two-pass schedule is used).
template <typename S, int LPR>
bool try_sweep(admm_plan* p, size_t l2_budget) {
  constexpr int W = LPR * Store<S>::kPerVec;
  const size_t smem = sweep_smem_bytes<S, LPR>(p);
  if (smem > 225 * 1024) return false;
  for (auto fn : {sweep_kernel<S, LPR, false>, sweep_kernel<S, LPR, true>})
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::min<size_t>(smem, 225 * 1024)));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_kernel<S, LPR, false>, kSweepThreads, smem));
  if (occ < 1) return false;
  occ = 1;  // one warp-specialised CTA per SM (exactly num_sms CTAs: no wave imbalance)
  if (p->Pr != 1) return false;  // the replica mean needs every row block of a strip
  std::vector<SweepDesc> segs(p->Nc);
  uint64_t u = 0, po = 0;
  for (uint64_t j = 0; j < p->Nc; ++j) {
    const uint32_t cols = p->blocks[j].cols;
    segs[j] = SweepDesc{u, po, (uint32_t)cdiv(cols, W), cols};
    u += segs[j].n_strips;
    po += (uint64_t)segs[j].n_strips * p->n_meas;
  }
  uint64_t P = std::min<uint64_t>(u, (uint64_t)p->num_sms * occ);
  const uint64_t strip = 2 * (uint64_t)p->n_meas * W * sizeof(S);  // two strips open per CTA
  if (P * strip > l2_budget) {
    const uint64_t cap = l2_budget / strip;
    if (cap < (uint64_t)p->num_sms) return false;
    P = std::min<uint64_t>(P, cap);
  }
  p->segs = segs;
  p->gS.U = u;
  p->gS.P = P;
  p->sweep_lpr = LPR;
  p->sweep_smem = smem;
  p->keep_l2 = (p->h_elems + p->k_elems) * sizeof(S) <= (96ull << 20);
  p->dwpart_s.alloc(po * sizeof(double2));
  upload_desc(p->dsegs, segs.data(), segs.size() * sizeof(SweepDesc));
  return true;
}

template <typename S>
using SlabFn = void (*)(const S*, const SlabDesc*, const BlockDesc*, const SweepDesc*, uint32_t, uint32_t, uint32_t,
                        uint64_t, uint32_t, uint32_t, uint32_t, uint32_t, const double2*, ColVecs, double2*,
                        const Params*, double*, IterState*, unsigned long long*);
template <typename S, int RB>
SlabFn<S> slab_fn_rb(int rpl, bool tr) {
  if (rpl == 1) return tr ? sweep_slab_kernel<S, 1, RB, true> : sweep_slab_kernel<S, 1, RB, false>;
  if (rpl == 2) return tr ? sweep_slab_kernel<S, 2, RB, true> : sweep_slab_kernel<S, 2, RB, false>;
  return tr ? sweep_slab_kernel<S, 4, RB, true> : sweep_slab_kernel<S, 4, RB, false>;
}
// 16-byte strip rows: tall strips (many rows per segment) in one CTA, 16 slabs of 192 rows
template <typename S>
SlabFn<S> slab_fn_rb16(int rpl, bool tr) {
  // fewer, fatter warps on request (ADMM_B200_SLAB_RPW=256 / 384): 12 x 256 rows at 128 registers, 8 x 384 at 168
  if (rpl == 8) return tr ? sweep_slab_kernel<S, 8, 16, true, 12> : sweep_slab_kernel<S, 8, 16, false, 12>;
  if (rpl == 12) return tr ? sweep_slab_kernel<S, 12, 16, true, 8> : sweep_slab_kernel<S, 12, 16, false, 8>;
  return tr ? sweep_slab_kernel<S, 6, 16, true> : sweep_slab_kernel<S, 6, 16, false>;
}
template <typename S>
SlabFn<S> slab_fn(int rpl, uint32_t rb, bool tr) {
  if (rb == 16) return slab_fn_rb16<S>(rpl, tr);
  return rb == 32 ? slab_fn_rb<S, 32>(rpl, tr) : slab_fn_rb<S, 64>(rpl, tr);
}

// Per-warp slab sweep (admm_slab.cuh): rows of every strip cut into RPW-row slabs (each
// inside one replica), C x NW slabs per cluster; NS ring stages of NW slabs per CTA.
// Chosen to avoid padding rows (padding is streamed from HBM), then the smallest
// cluster with >= 3 stages.  ADMM_B200_SLAB_C / ADMM_B200_SLAB_RPW force a geometry.
template <typename S>
bool try_slab(admm_plan* p) {
  if (p->Pr != 1) return false;  // the replica mean needs every row block of a strip
  const uint32_t M = (uint32_t)p->Mr, N = (uint32_t)p->Nc;
  int fC = 0, fR = 0, fB = 0;
  if (const char* e = std::getenv("ADMM_B200_SLAB_C")) fC = std::atoi(e);
  if (const char* e = std::getenv("ADMM_B200_SLAB_RPW")) fR = std::atoi(e);
  if (const char* e = std::getenv("ADMM_B200_SLAB_RB")) fB = std::atoi(e);
  const size_t cap = 227 * 1024;
  struct Cand { uint32_t rb, rpl, C, nw, ns, Ns; uint64_t pad; };
  bool have = false;
  Cand best{};
  for (uint32_t rb : {64u, 32u, 16u}) {
    if (fB && (uint32_t)fB != rb) continue;
    const uint32_t W = rb / 16 * (16 / sizeof(S));
    if (M * W > kWarp) continue;  // the D warp maps (replica, column) onto lanes
    for (uint32_t rpl : {2u, 1u, 4u, 6u, 8u, 12u}) {
      if ((rpl >= 6) != (rb == 16)) continue;  // 16-byte rows come with 192-row slabs (16 warps x 192 = 3072 rows)
      if (rpl > 8 && !fR) continue;            // 384-row slabs (8 warps at 168 registers) only on request: measured slower
      const uint32_t maxw = rpl == 8 ? 12u : rpl == 12 ? 8u : (uint32_t)kSlabMaxW;
      const uint32_t rpw = rpl * kWarp;
      if (fR && (uint32_t)fR != rpw) continue;
      uint32_t Ns = 0;
      uint64_t pad = 0;
      for (uint32_t i = 0; i < M; ++i) {
        const uint32_t R = p->blocks[(size_t)i * N].rows;
        Ns += (uint32_t)cdiv(R, rpw);
        pad += cdiv(R, rpw) * rpw - R;
      }
      for (uint32_t C : {1u, 2u, 4u, 8u}) {
        if (fC && (uint32_t)fC != C) continue;
        // clusters only on request: every cluster geometry measured so far loses to the
        // single-CTA slab (config 2: 120 vs 96 us) or to two-pass (config 3: 276-362 us vs
        // 265 us) -- the per-strip DSMEM exchange sits on the D warps' critical path
        if (!fC && C > 1) continue;
        const uint32_t nw = (uint32_t)cdiv(Ns, C);
        if (nw > maxw || (C > 1 && nw * (C - 1) >= Ns)) continue;  // no empty rank
        const size_t fixed = slab_smem_bytes(0, nw, kSlabMaxD, rpw, rb, C, M, W, N);
        const size_t per = (size_t)nw * rpw * rb + nw * sizeof(uint64_t);
        const uint32_t ns = (uint32_t)std::min<size_t>((cap - fixed) / per, 8);
        if (ns < 3) continue;
        Cand c{rb, rpl, C, nw, ns, Ns, pad};
        // fewest padding rows (they are streamed), then the smallest cluster, then the
        // widest rows (fewer strips, fewer per-strip overheads)
        // ... and at 16-byte rows 12 warps x 256 rows (128 registers, 4-row batches) over 16 x 192
        // (config 3: 5,823 vs 5,625 it/s)
        const bool better = !have || c.pad < best.pad || (c.pad == best.pad && c.C < best.C) ||
                            (c.pad == best.pad && c.C == best.C && c.rb > best.rb) ||
                            (c.pad == best.pad && c.C == best.C && c.rb == best.rb && c.rpl == 8 && best.rpl == 6);
        if (better) best = c, have = true;
      }
    }
  }
  if (!have) return false;
  const uint32_t W = best.rb / 16 * (16 / sizeof(S));
  // lag of (A) behind (C) and D warps: the deepest lag the ring allows, two D warps when
  // the slot-reuse rules permit (slab_lag_ok)
  uint32_t lag = std::max<uint32_t>(1, std::min<uint32_t>(best.ns - 2, kSlabZB - 1));
  if (const char* e = std::getenv("ADMM_B200_SLAB_LAG"))
    lag = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)std::atoi(e), std::min<uint32_t>(best.ns - 2, kSlabZB - 1)));
  uint32_t nd = kSlabMaxD;
  if (const char* e = std::getenv("ADMM_B200_SLAB_ND")) nd = std::max(1, std::min(kSlabMaxD, std::atoi(e)));
  while (lag > 1 && !slab_lag_ok(lag, nd) && !slab_lag_ok(lag, 1)) --lag;
  if (!slab_lag_ok(lag, nd)) nd = 1;
  if (!slab_lag_ok(lag, nd)) return false;
  const size_t smem = slab_smem_bytes(best.ns, best.nw, nd, best.rpl * kWarp, best.rb, best.C, M, W, N);
  const auto fn = slab_fn<S>(best.rpl, best.rb, std::getenv("ADMM_B200_SLAB_TRACE") != nullptr);
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  std::vector<SweepDesc> segs(N);
  uint64_t u = 0;
  for (uint32_t j = 0; j < N; ++j) {
    const uint32_t cols = p->blocks[j].cols;
    segs[j] = SweepDesc{u, 0, (uint32_t)cdiv(cols, W), cols};
    u += segs[j].n_strips;
  }
  // co-resident clusters (one CTA per SM)
  uint64_t ncl = (uint64_t)p->num_sms / best.C;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ncl * best.C));
    cfg.blockDim = dim3((best.nw + nd) * kWarp);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = best.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, fn, &cfg);
    if (std::getenv("ADMM_B200_DEBUG")) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, fn);
      int ob = -1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob, fn, (best.nw + nd) * kWarp, smem);
      std::fprintf(stderr, "slab attrs: regs=%d maxthr=%d static_smem=%zu maxdyn=%d occ_blocks=%d\n", fa.numRegs,
                   fa.maxThreadsPerBlock, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, ob);
    }
    if (std::getenv("ADMM_B200_DEBUG"))
      std::fprintf(stderr, "slab: rb=%u C=%u rpw=%u nw=%u nd=%u lag=%u ns=%u smem=%zu clusters=%d (%s)\n", best.rb, best.C,
                   best.rpl * kWarp, best.nw, nd, lag, best.ns, smem, nc, cudaGetErrorString(e));
    if (e != cudaSuccess || nc < 1) {
      cudaGetLastError();
      return false;
    }
    ncl = std::min<uint64_t>(ncl, (uint64_t)nc);
  }
  const uint64_t P = std::min<uint64_t>(u, ncl);
  uint64_t po = 0;
  for (auto& sd : segs) {  // one partial slot per cluster overlapping the segment
    sd.part_off = po;
    po += (uint64_t)seg_count(sd.unit0, sd.n_strips, u, P) * p->n_meas;
  }
  std::vector<SlabDesc> slabs;
  const uint32_t rpw = best.rpl * kWarp;
  for (uint32_t i = 0; i < M; ++i) {
    const BlockDesc& b = p->blocks[(size_t)i * N];
    for (uint32_t r = 0; r < b.rows; r += rpw) slabs.push_back(SlabDesc{i, r, b.row0 + r, std::min(rpw, b.rows - r)});
  }
  p->segs = segs;
  p->slabs = slabs;
  p->gS.U = u;
  p->gS.P = P;
  p->slab_rpl = (int)best.rpl;
  p->slab_C = best.C;
  p->slab_nw = best.nw;
  p->slab_ns = best.ns;
  p->slab_Ns = best.Ns;
  p->slab_lag = lag;
  p->slab_nd = nd;
  p->sweep_smem = smem;
  p->dwpart_s.alloc(po * sizeof(double2));
  upload_desc(p->dsegs, segs.data(), segs.size() * sizeof(SweepDesc));
  upload_desc(p->dslabs, slabs.data(), slabs.size() * sizeof(SlabDesc));
  p->dHs.alloc(u * best.Ns * (uint64_t)rpw * best.rb);
  p->slab_rb = best.rb;
  if (std::getenv("ADMM_B200_SLAB_TRACE")) {
    const uint64_t n = P * best.C * 64 * 8;
    p->dtrace_tile.alloc(n * sizeof(unsigned long long));
    CK(cudaMemset(p->dtrace_tile.p, 0, n * sizeof(unsigned long long)));
  }
  return true;
}

// Resident schedule (admm_resident.cuh): H of each CTA's columns kept in SMEM, one
// persistent cooperative kernel per launch.  On request (schedule 4 / ADMM_B200_SCHEDULE=
// resident) for small problems: single GPU, one scene, <= 8 replicas per segment, one
// owner CTA per block, and the SMEM tile (H columns + the owner's K) must fit.
template <typename S>
bool try_resident(admm_plan* p, int requested) {
  // opt-in: on config 1 it measured 45.5k it/s vs 46k for the sweep launch chain (two
  // grid barriers + dependent L2 round trips per iteration)
  if (requested != 4) return false;
  if (p->batch > 1 || p->is_shard || p->Mr > (uint64_t)kResMaxM || p->Mr * p->Nc > (uint64_t)p->num_sms) return false;
  const char* oe = std::getenv("ADMM_B200_OBJ");
  if (oe && !std::strcmp(oe, "pass")) return false;
  int coop = 0;
  CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, p->device));
  if (!coop) return false;
  // CTAs per segment in proportion to its columns (at least one each).  Fewer, wider CTAs
  // shorten phase B (the owners sum one w partial per CTA) and the grid barriers:
  // at least kResMinCols columns per CTA.
  uint64_t min_cols = 32;
  const uint64_t Pmax = std::max<uint64_t>(std::min<uint64_t>(p->num_sms, cdiv(p->n_pix, min_cols)),
                                           p->blocks.size()),
                 ncol = p->n_pix;
  std::vector<uint32_t> pj(p->Nc);
  uint64_t tot = 0;
  for (uint64_t j = 0; j < p->Nc; ++j) {
    pj[j] = (uint32_t)std::max<uint64_t>(1, (Pmax * p->blocks[j].cols) / std::max<uint64_t>(ncol, 1));
    pj[j] = std::min<uint32_t>(pj[j], p->blocks[j].cols);
    tot += pj[j];
  }
  while (tot > Pmax) {
    auto it = std::max_element(pj.begin(), pj.end());
    if (*it <= 1) return false;
    --*it;
    --tot;
  }
  std::vector<ResCta> ctas;
  std::vector<uint32_t> seg(2 * p->Nc);
  uint32_t maxc = 0;
  for (uint64_t j = 0; j < p->Nc; ++j) {
    const uint32_t lo = (uint32_t)ctas.size(), n = p->blocks[j].cols;
    for (uint32_t c = 0; c < pj[j]; ++c) {
      const uint32_t c0 = (uint32_t)((uint64_t)n * c / pj[j]), c1 = (uint32_t)((uint64_t)n * (c + 1) / pj[j]);
      ctas.push_back(ResCta{(uint32_t)j, c0, c1 - c0, lo, lo + pj[j], 0});
      maxc = std::max(maxc, c1 - c0);
    }
    seg[2 * j] = lo;
    seg[2 * j + 1] = lo + pj[j];
  }
  if (maxc > (uint32_t)kResMaxCols || p->blocks.size() > ctas.size() || p->blocks.size() > (size_t)kResMaxBlocks)
    return false;  // one owner CTA per block
  const size_t smem = resident_smem<S>(maxc, (uint32_t)p->n_meas, (uint32_t)p->Mr, p->max_rows);
  if (smem > 225 * 1024) return false;
  CK(cudaFuncSetAttribute(resident_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, resident_kernel<S>, kCtaThreads, smem));
  if (occ < 1) return false;
  p->res_P = (uint32_t)ctas.size();
  p->res_cols = maxc;
  p->res_smem = smem;
  upload_desc(p->dres_cta, ctas.data(), ctas.size() * sizeof(ResCta));
  upload_desc(p->dres_seg, seg.data(), seg.size() * sizeof(uint32_t));
  p->dres_w.alloc((size_t)p->res_P * p->n_meas * sizeof(double2));
  p->dres_red.alloc((size_t)3 * p->res_P * sizeof(double));
  p->dres_opart.alloc((size_t)p->res_P * sizeof(double));
  p->dres_abuf.alloc(p->mvec_total * sizeof(double2));
  p->dres_lprev.alloc(sizeof(double));
  p->dres_bar.alloc(2 * sizeof(unsigned));
  CK(cudaMemset(p->dres_bar.p, 0, 2 * sizeof(unsigned)));
  p->dghat2.alloc(p->mvec_total * sizeof(double2));
  return true;
}

template <typename S>
void launch_resident(admm_plan* p, cudaStream_t s, uint32_t iters, bool prologue, bool obj) {
  ResArgs a{};
  a.H = p->dH.p;
  a.K = p->dK.p;
  a.hN = p->dhN.as<MatDesc>();
  a.kN = p->dkN.as<MatDesc>();
  a.blocks = p->dblocks.as<BlockDesc>();
  a.ctas = p->dres_cta.as<ResCta>();
  a.seg_cta = p->dres_seg.as<uint32_t>();
  a.g = p->dg.as<double2>();
  a.ghat[0] = p->ghat_ptr;
  a.ghat[1] = p->dghat2.as<double2>();
  a.gij = p->dgij.as<double2>();
  a.r = p->dr.as<double2>();
  a.q = p->dq.as<double2>();
  a.cv = ColVecs{p->du.as<double2>(), p->ds.as<double2>(), p->dc.as<double2>(), p->dv.as<double2>(),
                 p->dvprev.as<double2>()};
  a.wpart = p->dres_w.as<double2>();
  a.red = p->dres_red.as<double>();
  a.opart = p->dres_opart.as<double>();
  a.hs = p->dhs.as<double2>();
  a.abuf = p->dres_abuf.as<double2>();
  a.lprev = p->dres_lprev.as<double>();
  a.prm = p->dparams.as<Params>();
  a.trace = p->dtrace.as<double>();
  a.trace_cap = p->trace_cap;
  a.st = p->dstate.as<IterState>();
  a.bar = p->dres_bar.as<unsigned>();
  a.M = (uint32_t)p->Mr;
  a.N = (uint32_t)p->Nc;
  a.nb = (uint32_t)p->blocks.size();
  a.n_meas = (uint32_t)p->n_meas;
  a.max_cols = p->res_cols;
  a.max_m = p->max_rows;
  a.dbg = nullptr;
  if (const char* tf = std::getenv("ADMM_B200_RES_TRACE")) {
    if (!p->dres_dbg.p) {
      p->dres_dbg.alloc((size_t)p->res_P * 16 * 10 * 8);
      CK(cudaMemset(p->dres_dbg.p, 0, p->dres_dbg.bytes));
    }
    a.dbg = p->dres_dbg.as<unsigned long long>();
    (void)tf;
  }
  a.iters = iters;
  a.prologue = prologue ? 1u : 0u;
  a.trace_obj = (obj && p->dhs.p) ? 1u : 0u;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->res_P);
  cfg.blockDim = dim3(kCtaThreads);
  cfg.dynamicSmemBytes = p->res_smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the grid barriers cannot deadlock
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, resident_kernel<S>, a));
}

void launch_resident_any(admm_plan* p, cudaStream_t s, uint64_t iters, bool prologue, bool obj) {
  do {
    const uint32_t n = (uint32_t)std::min<uint64_t>(iters, 1u << 30);
    if (p->dtype == ADMM_C128)
      launch_resident<double2>(p, s, n, prologue, obj);
    else
      launch_resident<float2>(p, s, n, prologue, obj);
    iters -= n;
  } while (iters > 0 && !prologue);
}

// Support schedule (admm_sparse.cuh): one dense H pass + a pass over the columns in the
// support of v.  Automatic for a single-GPU, single-scene plan whose H exceeds L2 and whose
// column update is a consensus one (M > 1, N = 1: every replica sees the whole v, whose
// soft threshold makes it sparse); on request (schedule 5) for any shape.
template <typename S>
bool try_support(admm_plan* p, int requested) {
  if (p->batch > 1) return false;
  // a shard of a multi-GPU plan: consensus over row-block ranks (Pc = 1, every rank holds the whole
  // v after the replica-mean exchange); driven by the two-pass phase program with phase 1 replaced
  if (p->is_shard && (p->method != ADMM_CONSENSUS || p->Pc != 1 || p->Nc != 1)) return false;
  if (!p->is_shard && p->Pr * p->Pc > 1) return false;
  if (requested != 5) {
    if (requested != 0 || p->method != ADMM_CONSENSUS || p->M < 2) return false;
    if (p->h_elems * sizeof(S) <= (256ull << 20)) return false;
  }
  if (p->Nc > kCtaThreads) return false;  // support_rows_kernel spreads <= 256 column blocks per row
  return true;
}

template <typename S>
void choose_schedule(admm_plan* p, int requested) {
  p->schedule = 1;
  if (requested == 1) return;
  if (try_support<S>(p, requested)) {
    p->schedule = 5;
    return;
  }
  if (requested == 5) throw Fail{ADMM_E_PARAMETER, "support schedule not possible for this plan"};
  if (try_resident<S>(p, requested)) {
    p->schedule = 4;
    return;
  }
  if (requested == 4) throw Fail{ADMM_E_PARAMETER, "resident schedule not possible for this shape"};
  if (try_slab<S>(p)) {
    p->schedule = 2;
    return;
  }
  const size_t budget = 80ull << 20;  // open strips must stay well inside the 126 MB L2
  // 64-byte strips (LPR = 2) only on request: measured slower than two-pass on config 3
  if (try_sweep<S, 8>(p, budget) || try_sweep<S, 4>(p, budget) || (requested == 2 && try_sweep<S, 2>(p, budget))) {
    p->schedule = 2;
    return;
  }
  if (requested == 2) throw Fail{ADMM_E_PARAMETER, "sweep schedule not possible for this shape"};
}

void upload_desc(DevBuf& d, const void* src, size_t bytes) {
  d.alloc(bytes);
  CK(cudaMemcpy(d.p, src, bytes, cudaMemcpyHostToDevice));
}

// Upload the blocks of the host matrix into the storage arena (partition.hpp:79-125
// materialises the same blocks as host copies).
// Host rows -> pinned staging (pitch n_pix -> the block's ld, zero pad), on every host
// core (OpenMP), checking finiteness of what it copies when asked (problem.hpp:44-46 for
// the large matrices whose separate scan would cost a pass).  Returns false on a
// non-finite entry.
bool pack_rows(void* dst, const char* src, uint64_t nr, uint64_t cols, uint64_t src_pitch, uint64_t ld,
               size_t esz, bool check) {
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t r = 0; r < (int64_t)nr; ++r) {
    char* d = static_cast<char*>(dst) + (uint64_t)r * ld * esz;
    const char* s = src + (uint64_t)r * src_pitch * esz;
    std::memcpy(d, s, cols * esz);
    if (ld > cols) std::memset(d + cols * esz, 0, (ld - cols) * esz);
    if (check) {
      if (esz == 16) {
        const double* v = reinterpret_cast<const double*>(d);
        for (uint64_t e = 0; e < 2 * cols; ++e) bad |= !std::isfinite(v[e]);
      } else {
        const float* v = reinterpret_cast<const float*>(d);
        for (uint64_t e = 0; e < 2 * cols; ++e) bad |= !std::isfinite(v[e]);
      }
    }
  }
  return !bad;
}

// Upload the blocks of the host matrix into the storage arena (partition.hpp:79-125
// materialises the same blocks as host copies).  Large matrices go through two pinned
// staging buffers: host cores pack chunk k + 1 while the copy engine moves chunk k, so H
// crosses PCIe at DMA speed with one host pass that also checks finiteness
// (check_finite).  c128 <-> c64 conversions run on the device (scl applied in FP64).
// on_block(b) runs once block b's rows (final values) are enqueued on p->stream.
template <typename S, typename OnBlock>
void upload_h(admm_plan* p, const void* h, admm_dtype h_dtype, bool check_finite, OnBlock on_block) {
  const size_t hsz = h_dtype == ADMM_C128 ? 16 : 8;
  const bool direct = (h_dtype == ADMM_C128) == std::is_same<S, double2>::value;
  uint64_t total = 0, maxld = 0;
  for (size_t b = 0; b < p->blocks.size(); ++b) {
    total += (uint64_t)p->blocks[b].rows * p->hN[b].ld * hsz;
    maxld = std::max<uint64_t>(maxld, p->hN[b].ld);
  }
  const bool staged = check_finite || total >= (256ull << 20);
  DevBuf tmp;
  const size_t chunk = staged ? std::min<uint64_t>(total, 128ull << 20) : (size_t)std::min<uint64_t>(total, 1ull << 30);
  if (!direct) tmp.alloc(std::max<size_t>(chunk, maxld * hsz));
  void* pin[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  struct Cleanup {
    void** pin;
    cudaEvent_t* ev;
    ~Cleanup() {
      for (int k = 0; k < 2; ++k) {
        if (ev[k]) cudaEventDestroy(ev[k]);
        if (pin[k]) cudaFreeHost(pin[k]);
      }
    }
  } cleanup{pin, done};
  if (staged)
    for (int k = 0; k < 2; ++k) {
      CK(cudaHostAlloc(&pin[k], std::max<size_t>(chunk, maxld * hsz), cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
    }
  int slot = 0;
  bool finite = true;
  for (size_t b = 0; b < p->blocks.size(); ++b) {
    const BlockDesc& bd = p->blocks[b];
    const MatDesc& md = p->hN[b];
    const char* src = static_cast<const char*>(h) + ((uint64_t)bd.row0 * p->n_pix + bd.col0) * hsz;
    if (!staged && direct) {
      CK(cudaMemcpy2DAsync(p->dH.as<S>() + md.a_off, (size_t)md.ld * sizeof(S), src, p->n_pix * hsz,
                           (size_t)bd.cols * sizeof(S), bd.rows, cudaMemcpyHostToDevice, p->stream));
      on_block(b);
      continue;
    }
    const uint64_t rows_per = std::max<uint64_t>(1, chunk / ((uint64_t)md.ld * hsz));
    for (uint64_t r0 = 0; r0 < bd.rows; r0 += rows_per) {
      const uint32_t nr = (uint32_t)std::min<uint64_t>(rows_per, bd.rows - r0);
      const void* dev_src = nullptr;  // where the chunk's rows are on the device (pitch ld)
      if (staged) {
        CK(cudaEventSynchronize(done[slot]));  // the copy out of this buffer has finished
        finite &= pack_rows(pin[slot], src + r0 * p->n_pix * hsz, nr, bd.cols, p->n_pix, md.ld, hsz, check_finite);
        void* dst = direct ? (void*)(p->dH.as<S>() + md.a_off + r0 * md.ld) : tmp.p;
        CK(cudaMemcpyAsync(dst, pin[slot], (size_t)nr * md.ld * hsz, cudaMemcpyHostToDevice, p->stream));
        dev_src = tmp.p;
      } else {
        CK(cudaMemcpy2DAsync(tmp.p, (size_t)md.ld * hsz, src + r0 * p->n_pix * hsz, p->n_pix * hsz,
                             (size_t)bd.cols * hsz, nr, cudaMemcpyHostToDevice, p->stream));
        dev_src = tmp.p;
      }
      if (!direct) {
        dim3 grid((unsigned)std::min<uint64_t>(cdiv(bd.cols, 256), 64), nr);
        if (h_dtype == ADMM_C64)
          widen_rows_kernel<S><<<grid, 256, 0, p->stream>>>(static_cast<const float2*>(dev_src), md.ld,
                                                             p->dH.as<S>() + md.a_off + r0 * md.ld, md.ld, nr,
                                                             bd.cols, p->cfg.scl);
        else
          narrow_rows_kernel<S><<<grid, 256, 0, p->stream>>>(static_cast<const double2*>(dev_src), md.ld,
                                                              p->dH.as<S>() + md.a_off + r0 * md.ld, md.ld, nr,
                                                              bd.cols, p->cfg.scl);
        CK(cudaGetLastError());
      }
      if (staged) {
        CK(cudaEventRecord(done[slot], p->stream));
        if (!direct) CK(cudaStreamSynchronize(p->stream));  // tmp is reused by the next chunk
        slot ^= 1;
      } else {
        CK(cudaStreamSynchronize(p->stream));
      }
    }
    on_block(b);
  }
  CK(cudaStreamSynchronize(p->stream));
  if (!finite) throw Fail{ADMM_E_NUMERICAL, "SensingProblem: non-finite entries"};
  if (direct && p->cfg.scl != 1.0) {  // apply_scaling, problem.hpp:59-66 (converted
                                      // uploads scale in FP64 before rounding)
    scale_kernel<S><<<p->num_sms * 8, 256, 0, p->stream>>>(p->dH.as<S>(), p->h_elems, p->cfg.scl);
    CK(cudaGetLastError());
  }
  DevBuf flag;
  flag.alloc(4);
  finite_kernel<S><<<p->num_sms * 8, 256, 0, p->stream>>>(p->dH.as<S>(), p->h_elems, flag.as<unsigned>());
  CK(cudaGetLastError());
  unsigned hf = 0;
  CK(cudaMemcpyAsync(&hf, flag.p, 4, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  if (hf) throw Fail{ADMM_E_NUMERICAL, "SensingProblem: non-finite entries"};
}

// Slab-major copy of the (scaled) H for sweep_slab_kernel.
template <typename S>
void build_slab(admm_plan* p) {
  const uint64_t chunks = p->gS.U * p->slab_Ns * (uint64_t)p->slab_rpl * kWarp * (p->slab_rb / 16);
  auto kern = p->slab_rb == 16 ? slab_h_kernel<S, 16> : p->slab_rb == 32 ? slab_h_kernel<S, 32> : slab_h_kernel<S, 64>;
  kern<<<p->num_sms * 8, 256, 0, p->stream>>>(p->dH.as<S>(), p->dhN.as<MatDesc>(),
                                                          p->dsegs.as<SweepDesc>(), p->dslabs.as<SlabDesc>(),
                                                          (uint32_t)p->Nc, p->slab_Ns, (uint32_t)p->slab_rpl * kWarp,
                                                          chunks, p->dHs.as<S>());
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(p->stream));
}

// Gram phase (gram.hpp:92-122): A_b = rho I + H_b H_b^H on the FP64 tensor cores, one launch
// per block on a second stream as soon as the block's rows are on the device, so the Gram of
// block b runs under the PCIe upload of block b + 1.
struct GramWork {
  DevBuf A, flag;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev = nullptr;
  std::vector<cudaEvent_t> marks;  // start / stop of every Gram launch (device time of the phase)
  ~GramWork() {
    for (cudaEvent_t e : marks) cudaEventDestroy(e);
    if (ev) cudaEventDestroy(ev);
    if (stream) cudaStreamDestroy(stream);
  }
};

template <typename S>
void gram_begin(admm_plan* p, GramWork& w) {
  upload_desc(p->dgram, p->gram.data(), p->blocks.size() * sizeof(GramDesc));
  w.A.alloc(p->a_elems * sizeof(double2));
  w.flag.alloc(4);
  CK(cudaMemsetAsync(w.flag.p, 0, 4, p->stream));
  CK(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&w.ev, cudaEventDisableTiming));
  CK(cudaFuncSetAttribute(gram_dmma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * kFStage)));
  CK(cudaStreamSynchronize(p->stream));
}

// Blocks [b0, b1): their rows are complete on p->stream.
template <typename S>
void gram_blocks(admm_plan* p, GramWork& w, size_t b0, size_t b1) {
  uint32_t mp = 0;
  for (size_t b = b0; b < b1; ++b) mp = std::max(mp, p->gram[b].mp);
  const uint32_t nT = mp / kFT;
  CK(cudaEventRecord(w.ev, p->stream));
  CK(cudaStreamWaitEvent(w.stream, w.ev, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  w.marks.push_back(e0);
  CK(cudaEventCreate(&e1));
  w.marks.push_back(e1);
  CK(cudaEventRecord(e0, w.stream));
  gram_dmma_kernel<S><<<dim3(nT * (nT + 1) / 2, (unsigned)(b1 - b0)), kFThreads, 2 * kFStage, w.stream>>>(
      p->dH.as<S>(), p->dgram.as<GramDesc>(), (uint32_t)b0, w.A.as<double2>(), p->cfg.rho, w.flag.as<unsigned>());
  CK(cudaGetLastError());
  CK(cudaEventRecord(e1, w.stream));
  for (size_t b = b0; b < b1; ++b) {  // lower tiles (diagonal ones whole) x n complex MACs x 8 flops
    const double nt = p->gram[b].mp / kFT;
    p->gram_flops += nt * (nt + 1) / 2 * kFT * kFT * (double)p->gram[b].n * 8.0;
  }
}

// Gram done -> blocked Gauss-Jordan inverse, store K (cholesky.hpp:48-74; admm_factor.cuh).
template <typename S>
void factor_blocks(admm_plan* p, GramWork& w) {
  const uint64_t nb = p->blocks.size();
  DevBuf& A = w.A;
  DevBuf& flag = w.flag;
  unsigned hf = 0;
  const auto tf0 = std::chrono::steady_clock::now();
  CK(cudaStreamSynchronize(w.stream));
  CK(cudaMemcpyAsync(&hf, flag.p, 4, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  if (hf & 1u) throw Fail{ADMM_E_NUMERICAL, "CholeskyFactor: non-finite entries in input matrix"};
  for (size_t k = 0; k + 1 < w.marks.size(); k += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, w.marks[k], w.marks[k + 1]));
    p->gram_device_s += ms * 1e-3;
  }
  const auto tf1 = std::chrono::steady_clock::now();
  p->setup_phase[2] = std::chrono::duration<double>(tf1 - tf0).count();  // Gram time not hidden under the upload
  uint64_t kpacked_elems = 0;
  if (p->kpacked) {  // packed Hermitian tile layout (shared by K and, for the support schedule, G)
    uint64_t koff = 0, u0 = 0, po = 0, co = 0;
    p->hv.assign(nb, HemvDesc{});
    for (uint64_t b = 0; b < nb; ++b) {
      HemvDesc& h = p->hv[b];
      h.m = p->blocks[b].rows;
      h.nT = (uint32_t)cdiv(h.m, kHT);
      h.n_units = h.nT * (h.nT + 1) / 2;
      h.k_off = koff;
      h.unit0 = u0;
      h.part_off = po;
      h.x_off = p->blocks[b].mvec_off;
      h.cnt_off = (uint32_t)co;
      co += h.nT;
      koff += (uint64_t)h.n_units * kHT * kHT;
      u0 += h.n_units;
      po += 2ull * h.n_units * kHT;
    }
    kpacked_elems = koff;
    p->gP.U = u0;
    p->dkppart.alloc(po * sizeof(double2));
    p->dkcnt.alloc(std::max<uint64_t>(co, 1) * sizeof(unsigned));
    CK(cudaMemset(p->dkcnt.p, 0, std::max<uint64_t>(co, 1) * sizeof(unsigned)));
  }
  if (p->schedule == 5 && !p->kpacked) throw Fail{ADMM_E_PARAMETER, "support schedule needs the packed Hermitian apply"};
  const unsigned gx = (unsigned)std::min<uint64_t>(cdiv(p->max_m, 256), 8);
  {  // blocked Gauss-Jordan: per 64-wide panel the diagonal inverse, the row panel, the rank-64 update
    const uint32_t mpmax = (uint32_t)round_up(p->max_m, kFT), np = mpmax / kFT;
    DevBuf P, PH, WH, C;
    P.alloc(nb * kFT * kFT * sizeof(double2));
    PH.alloc(nb * kFT * kFT * sizeof(double2));
    WH.alloc(nb * (uint64_t)mpmax * kFT * sizeof(double2));
    C.alloc(nb * (uint64_t)mpmax * kFT * sizeof(double2));
    const GjScratch sc{P.as<double2>(), PH.as<double2>(), WH.as<double2>(), C.as<double2>(), mpmax};
    CK(cudaFuncSetAttribute(gj_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGjDiagSmem));
    CK(cudaFuncSetAttribute(gj_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGjPanelSmem));
    CK(cudaFuncSetAttribute(gj_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * kFStage)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, p->stream));
    for (uint32_t kp = 0; kp < np; ++kp) {
      gj_diag_kernel<<<(unsigned)nb, kFThreads, kGjDiagSmem, p->stream>>>(A.as<double2>(), p->dgram.as<GramDesc>(), kp,
                                                                         sc, flag.as<unsigned>());
      if (np > 1) {
        gj_panel_kernel<<<dim3(np, (unsigned)nb), kFThreads, kGjPanelSmem, p->stream>>>(
            A.as<double2>(), p->dgram.as<GramDesc>(), kp, sc);
        gj_update_kernel<<<dim3(np, np, (unsigned)nb), kFThreads, 2 * kFStage, p->stream>>>(
            A.as<double2>(), p->dgram.as<GramDesc>(), kp, sc);
      }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, p->stream));
    CK(cudaStreamSynchronize(p->stream));  // the scratch buffers are released here
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    p->inverse_device_s = ms * 1e-3;
    for (uint64_t b = 0; b < nb; ++b) p->inverse_flops += 8.0 * std::pow((double)p->gram[b].mp, 3.0);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&hf, flag.p, 4, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  if (hf & 2u)
    throw Fail{ADMM_E_SINGULARITY,
               "CholeskyFactor: pivot is not positive (matrix not positive definite or "
               "contaminated by non-finite values)"};
  p->dK.alloc(p->k_elems * sizeof(S));
  k_store_kernel<S><<<dim3(gx, p->max_m, (unsigned)nb), 256, 0, p->stream>>>(
      A.as<double2>(), p->dgram.as<GramDesc>(), p->dK.as<S>(), flag.as<unsigned>());
  if (p->kpacked) {  // packed Hermitian tiles of the same inverse
    p->dKp.alloc(kpacked_elems * sizeof(S));
    for (uint64_t b = 0; b < nb; ++b)
      k_pack_kernel<S><<<p->num_sms * 4, 256, 0, p->stream>>>(A.as<double2>(), p->gram[b].a_off, p->hv[b].m,
                                                             p->hv[b].nT, p->dKp.as<S>() + p->hv[b].k_off);
    upload_desc(p->dhv, p->hv.data(), nb * sizeof(HemvDesc));
    const uint64_t u0 = p->gP.U;
    p->gP.P = grid_for<S>(hemv_kernel<S, 1>, u0, p->num_sms);
    // complex64 K (streamed from HBM: configs 3/4): the bulk-copy ring variant, one CTA per
    // SM (35 -> 25 us on config 3); complex128 K (config 2, L2-resident between iterations):
    // the register variant (15.0 vs 18.4 us)
    const size_t bsm = hemv_bulk_smem<S, 1>(p->max_rows);
    p->hemv_bulk = sizeof(S) == 8 && bsm <= 227 * 1024 ? 1 : 0;
    if (p->hemv_bulk) {
      CK(cudaFuncSetAttribute(hemv_bulk_kernel<S, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      p->gP.P = std::max<uint64_t>(1, std::min<uint64_t>(u0, (uint64_t)p->num_sms));
    }
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&hf, flag.p, 4, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  if (hf & 1u) throw Fail{ADMM_E_NUMERICAL, "GramSolver: non-finite inverse"};
  p->setup_phase[3] = std::chrono::duration<double>(std::chrono::steady_clock::now() - tf1).count();
}

// Sweep schedule with a per-iteration objective: trace[k-1].objective after the
// finalize of iteration k-1 (l1 partials of the sweep + |Hv - g|^2 partials).
__global__ void objective_trace_kernel(const double* __restrict__ red, uint32_t P, const double* __restrict__ ored,
                                       uint32_t no, const Params* __restrict__ prm, double* __restrict__ trace,
                                       uint64_t trace_cap, const IterState* st) {
  pdl_enter();
  __shared__ double sm[kCtaWarps];
  double l = 0.0, o = 0.0;
  for (uint32_t k = threadIdx.x; k < P; k += kCtaThreads) l += red[2 * P + k];
  for (uint32_t k = threadIdx.x; k < no; k += kCtaThreads) o += ored[k];
  l = block_sum<kCtaThreads>(l, sm);
  o = block_sum<kCtaThreads>(o, sm);
  if (threadIdx.x == 0) {
    const uint64_t k = st->iter - 1;
    if (k < trace_cap) trace[3 * k + 2] = 0.5 * o + prm->lambda * l;
  }
}

RowVecs row_vecs(admm_plan* p) {
  return RowVecs{p->dg.as<double2>(), p->ghat_ptr, p->dgij.as<double2>(), p->dr.as<double2>(),
                 p->dq.as<double2>()};
}
ColVecs col_vecs(admm_plan* p) {
  return ColVecs{p->du.as<double2>(), p->ds.as<double2>(), p->dc.as<double2>(), p->dv.as<double2>(),
                 p->dvprev.as<double2>()};
}

// q = K r and ghat = g_ij - rho q for every local block: packed Hermitian K (half the
// bytes) unless disabled, else the dense K through gemv_n.
// `mid` runs between the two launches (profiling events).
template <typename S, typename Mid>
void enqueue_kapply(admm_plan* p, cudaStream_t s, Mid mid) {
  const int nb = (int)p->blocks.size();
  if (p->kpacked) {
    if (p->hemv_bulk) {
      auto fb = hemv_bulk_kernel<S, 1>;
      const size_t sm = hemv_bulk_smem<S, 1>(p->max_rows);
      launch_pdl(fb, dim3((unsigned)p->gP.P), dim3(kCtaThreads), sm, s,
                 p->dKp.as<S>(), p->dr.as<double2>(), p->dkppart.as<double2>(), p->dhv.as<HemvDesc>(), nb, p->gP.U,
                 p->kkeep ? 1 : 0);
      mid();
      launch_pdl(hemv_finalize_kernel, dim3((unsigned)cdiv(p->max_rows, kHFinRows), nb), dim3(kHFinRows), 0, s,
                 row_vecs(p), p->dkppart.as<double2>(), p->dhv.as<HemvDesc>(), p->gP.U, p->gP.P,
                 p->dparams.as<Params>());
      return;
    }
    auto fn = hemv_kernel<S, 1>;
    launch_pdl(fn, dim3((unsigned)p->gP.P), dim3(kCtaThreads), 0, s, p->dKp.as<S>(), p->dr.as<double2>(),
               p->dkppart.as<double2>(), p->dhv.as<HemvDesc>(), nb, p->gP.U, p->kkeep ? 1 : 0);
    mid();
    launch_pdl(hemv_finalize_kernel, dim3((unsigned)cdiv(p->max_rows, kHFinRows), nb), dim3(kHFinRows), 0, s,
                 row_vecs(p), p->dkppart.as<double2>(), p->dhv.as<HemvDesc>(), p->gP.U, p->gP.P,
                 p->dparams.as<Params>());
    return;
  }
  gemv_n_kernel<S, kVN, kEvictNormal><<<(unsigned)p->gK.P, kCtaThreads, 0, s>>>(
      p->dK.as<S>(), p->dr.as<double2>(), p->dqpart.as<double2>(), p->dkN.as<MatDesc>(), nb, p->gK.U);
  mid();
  rows_finalize_kernel<kQ><<<dim3(p->rgx, nb), kCtaThreads, 0, s>>>(
      row_vecs(p), p->dqpart.as<double2>(), p->dkN.as<MatDesc>(), p->dblocks.as<BlockDesc>(),
      p->dgblocks.as<BlockDesc>(), (uint32_t)p->N, p->gK.U, p->gK.P, p->dparams.as<Params>());
}
template <typename S>
void enqueue_kapply(admm_plan* p, cudaStream_t s) {
  enqueue_kapply<S>(p, s, [] {});
}

// Support schedule rows step: w' = 2a' - a - (r - rho q), g_ij, r; objective rows (first: r = g_ij).
void enqueue_support_rows(admm_plan* p, cudaStream_t s, bool first) {
  support_rows_kernel<<<dim3(p->sup_rgx, (unsigned)p->Mr), kCtaThreads, 0, s>>>(
      row_vecs(p), p->dblocks.as<BlockDesc>(), p->dgblocks.as<BlockDesc>(), (uint32_t)p->Nc, p->sup_np,
      p->danew.as<double2>(), p->mvec_total, p->sup_chunks, p->daold.as<double2>(), p->dparams.as<Params>(), first ? 1 : 0,
      p->dored.as<double>());
}

// One iteration of the support schedule (admm_sparse.cuh).
template <typename S>
void enqueue_iteration_support(admm_plan* p, cudaStream_t s, bool with_objective, std::vector<cudaEvent_t>* ev) {
  constexpr int CH = chunk_h<S>();
  const int nb = (int)p->blocks.size();
  const uint32_t N = (uint32_t)p->Nc, M = (uint32_t)p->Mr;
  auto mark = [&](size_t k) {
    if (ev) CK(cudaEventRecord((*ev)[k], s));
  };
  mark(0);
  gemv_h_kernel<S, kVH, kEvictFirst><<<(unsigned)p->gH.P, kCtaThreads, 0, s>>>(
      p->dH.as<S>(), p->dq.as<double2>(), p->dzpart.as<double2>(), p->dhH.as<MatDesc>(), nb, p->gH.U);
  mark(1);
  zupdate_kernel<CH><<<dim3(p->zgx, N), kCtaThreads, 0, s>>>(
      col_vecs(p), p->dzpart.as<double2>(), p->dhH.as<MatDesc>(), p->dblocks.as<BlockDesc>(), M, N, p->gH.U,
      p->gH.P, p->dparams.as<Params>(), p->dred.as<double>(), p->dstate.as<IterState>(), p->dnzcnt.as<uint32_t>());
  support_compact_kernel<<<dim3(p->zgx, N), kCtaThreads, 0, s>>>(
      p->dv.as<double2>(), p->dblocks.as<BlockDesc>(), p->dnzcnt.as<uint32_t>(), p->zgx, p->dnzlist.as<uint32_t>(),
      p->nzstride, p->dnnz.as<uint32_t>(), p->dnnz_tot.as<unsigned long long>());
  mark(2);
  support_a_kernel<S><<<dim3(p->supgx, (unsigned)nb, p->sup_chunks), kSupThreads, 0, s>>>(
      p->dHc.as<S>(), p->dhcoff.as<uint64_t>(), p->dhcld.as<uint32_t>(), p->dblocks.as<BlockDesc>(),
      p->dv.as<double2>(), p->dnzlist.as<uint32_t>(), p->nzstride, p->dnnz.as<uint32_t>(), p->danew.as<double2>(),
      p->mvec_total);
  mark(3);
  enqueue_support_rows(p, s, false);
  finalize_kernel<<<1, kCtaThreads, 0, s>>>(p->dred.as<double>(), p->nz, p->dored.as<double>(),
                                            with_objective ? p->sup_rgx * M : 0, p->dparams.as<Params>(),
                                            p->dtrace.as<double>(), p->trace_cap, p->dstate.as<IterState>());
  mark(4);
  enqueue_kapply<S>(p, s, [&] { mark(5); });
  mark(6);
  CK(cudaGetLastError());
}

// Setup of the support schedule: column-major copy of every block and the vectors.
template <typename S>
void build_support(admm_plan* p) {
  const uint64_t nb = p->blocks.size();
  std::vector<uint64_t> coff(nb);
  std::vector<uint32_t> ld(nb);
  uint64_t tot = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    ld[b] = (uint32_t)round_up(p->blocks[b].rows, 8);
    coff[b] = tot;
    tot += (uint64_t)ld[b] * p->blocks[b].cols;
  }
  p->dHc.alloc(tot * sizeof(S));
  upload_desc(p->dhcoff, coff.data(), nb * sizeof(uint64_t));
  upload_desc(p->dhcld, ld.data(), nb * sizeof(uint32_t));
  for (uint64_t b = 0; b < nb; ++b) {
    const MatDesc& md = p->hN[b];
    dim3 grid((unsigned)cdiv(md.cols, 32), (unsigned)cdiv(ld[b], 32));
    colmajor_kernel<S><<<grid, dim3(32, 8), 0, p->stream>>>(p->dH.as<S>(), md.a_off, md.ld, md.rows, md.cols,
                                                            p->dHc.as<S>(), coff[b], ld[b]);
  }
  CK(cudaGetLastError());
  p->nzstride = (uint32_t)round_up(p->max_seg, 4);
  p->dnzcnt.alloc((uint64_t)p->zgx * p->Nc * sizeof(uint32_t));
  p->dnzlist.alloc((uint64_t)p->nzstride * p->Nc * sizeof(uint32_t));
  p->dnnz.alloc(p->Nc * sizeof(uint32_t));
  p->dnnz_tot.alloc(sizeof(unsigned long long));
  p->supgx = (uint32_t)cdiv(p->max_rows, kSupTile);
  // column chunks: ~4 CTAs of support_a per SM (a whole number of waves when it divides)
  p->sup_chunks = (uint32_t)std::min<uint64_t>(kSupMaxChunks, std::max<uint64_t>(1, cdiv((uint64_t)4 * p->num_sms, p->supgx * nb)));
  p->danew.alloc(p->mvec_total * 16 * p->sup_chunks);  // column-chunk partials of a'
  p->daold.alloc(p->mvec_total * 16);
  while ((1u << p->sup_np) < p->Nc) ++p->sup_np;
  p->sup_rgx = (uint32_t)std::max<uint64_t>(1, cdiv(p->max_rowblock, kCtaThreads >> p->sup_np));
  p->dored.alloc((size_t)std::max<uint64_t>(p->dored.bytes / sizeof(double), (uint64_t)p->sup_rgx * p->Mr) *
                 sizeof(double));
  CK(cudaStreamSynchronize(p->stream));
}

// Launch list of one iteration (the order of solvers.hpp's phases).
template <typename S>
void enqueue_iteration_twopass(admm_plan* p, cudaStream_t s, bool with_objective, std::vector<cudaEvent_t>* ev) {
  constexpr int CH = chunk_h<S>();
  const int nb = (int)p->blocks.size();
  const uint32_t N = (uint32_t)p->Nc, M = (uint32_t)p->Mr;  // local table
  auto mark = [&](size_t k) {
    if (ev) CK(cudaEventRecord((*ev)[k], s));
  };
  mark(0);
  // H streams through L2 (evict_first) so the packed K, re-read every iteration, can stay
  auto gn = p->h_evict_first ? gemv_n_kernel<S, kVN, kEvictFirst> : gemv_n_kernel<S, kVN, kEvictNormal>;
  auto gh = p->h_evict_first ? gemv_h_kernel<S, kVH, kEvictFirst> : gemv_h_kernel<S, kVH, kEvictNormal>;
  gn<<<(unsigned)p->gN.P, kCtaThreads, 0, s>>>(p->dH.as<S>(), p->dc.as<double2>(), p->dwpart.as<double2>(),
                                               p->dhN.as<MatDesc>(), nb, p->gN.U);
  mark(1);
  rows_finalize_kernel<kRhs><<<dim3(p->rgx, nb), kCtaThreads, 0, s>>>(
      row_vecs(p), p->dwpart.as<double2>(), p->dhN.as<MatDesc>(), p->dblocks.as<BlockDesc>(),
      p->dgblocks.as<BlockDesc>(), (uint32_t)p->N, p->gN.U,
      p->gN.P, p->dparams.as<Params>());
  if (with_objective && !p->obj_pass) {  // trace[k-1].objective from this iteration's w = H c
    launch_pdl(objective_rec_kernel, dim3(p->orgx, M), dim3(kCtaThreads), 0, s, row_vecs(p), p->dhs.as<double2>(),
               p->dblocks.as<BlockDesc>(), N, p->onp, p->drored.as<double>(), (const IterState*)p->dstate.as<IterState>(),
               (uint64_t)1);
    launch_pdl(objective_trace_kernel, dim3(1), dim3(kCtaThreads), 0, s, (const double*)p->dred.as<double>(), p->nz,
               (const double*)p->drored.as<double>(), p->nor, (const Params*)p->dparams.as<Params>(),
               p->dtrace.as<double>(), p->trace_cap, (const IterState*)p->dstate.as<IterState>());
  }
  mark(2);
  enqueue_kapply<S>(p, s, [&] { mark(3); });
  mark(4);
  gh<<<(unsigned)p->gH.P, kCtaThreads, 0, s>>>(p->dH.as<S>(), p->dq.as<double2>(), p->dzpart.as<double2>(),
                                               p->dhH.as<MatDesc>(), nb, p->gH.U);
  mark(5);
  zupdate_kernel<CH><<<dim3(p->zgx, N), kCtaThreads, 0, s>>>(
      col_vecs(p), p->dzpart.as<double2>(), p->dhH.as<MatDesc>(), p->dblocks.as<BlockDesc>(), M, N, p->gH.U,
      p->gH.P, p->dparams.as<Params>(), p->dred.as<double>(), p->dstate.as<IterState>());
  mark(6);
  const bool pass = with_objective && p->obj_pass;
  if (pass) {
    gemv_n_kernel<S, kVN, kEvictNormal><<<(unsigned)p->gO.P, kCtaThreads, 0, s>>>(
        p->dH.as<S>(), p->dv.as<double2>(), p->dopart.as<double2>(), p->dhNv.as<MatDesc>(), nb, p->gO.U);
    objective_rows_kernel<<<dim3(p->ogx, M), kCtaThreads, 0, s>>>(
        p->dg.as<double2>(), p->dopart.as<double2>(), p->dhNv.as<MatDesc>(), p->dblocks.as<BlockDesc>(), N,
        p->gO.U, p->gO.P, p->dored.as<double>());
  }
  finalize_kernel<<<1, kCtaThreads, 0, s>>>(p->dred.as<double>(), p->nz, p->dored.as<double>(),
                                            pass ? p->no : 0, p->dparams.as<Params>(),
                                            p->dtrace.as<double>(), p->trace_cap, p->dstate.as<IterState>());
  mark(7);
  CK(cudaGetLastError());
}

// Sweep schedule.  Prologue (after reset): r = g_ij (w = H c^0 = 0), q = K r, ghat.
template <typename S>
void enqueue_sweep_prologue(admm_plan* p, cudaStream_t s) {
  const int nb = (int)p->blocks.size();
  rows_finalize_sweep_kernel<<<dim3(p->rgx_s, nb), kCtaThreads, 0, s>>>(
      row_vecs(p), p->dwpart_s.as<double2>(), p->dsegs.as<SweepDesc>(), p->dblocks.as<BlockDesc>(),
      p->dgblocks.as<BlockDesc>(), (uint32_t)p->N, (uint32_t)p->n_meas, p->gS.U, p->gS.P, 1, 0, p->dred.as<double>(),
      p->dparams.as<Params>(), p->dtrace.as<double>(), p->trace_cap, p->dstate.as<IterState>(), nullptr);
  enqueue_kapply<S>(p, s);
  CK(cudaGetLastError());
}

template <typename S, int LPR>
void launch_sweep_lpr(admm_plan* p, cudaStream_t s) {
  auto fn = p->keep_l2 ? sweep_kernel<S, LPR, true> : sweep_kernel<S, LPR, false>;
  launch_pdl(fn, dim3((unsigned)p->gS.P), dim3(kSweepThreads), p->sweep_smem, s, p->dH.as<S>(),
             p->dhN.as<MatDesc>(), p->dblocks.as<BlockDesc>(), p->dsegs.as<SweepDesc>(), (uint32_t)p->Mr,
             (uint32_t)p->Nc, (uint32_t)p->n_meas, p->gS.U, p->dq.as<double2>(), col_vecs(p),
             p->dwpart_s.as<double2>(), p->dparams.as<Params>(), p->dred.as<double>(), p->dstate.as<IterState>());
}

template <typename S>
void launch_slab(admm_plan* p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p->gS.P * p->slab_C));
  cfg.blockDim = dim3((p->slab_nw + p->slab_nd) * kWarp);
  cfg.dynamicSmemBytes = p->sweep_smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p->slab_C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const auto fn = slab_fn<S>(p->slab_rpl, p->slab_rb, p->dtrace_tile.p != nullptr);
  CK(cudaLaunchKernelEx(&cfg, fn, (const S*)p->dHs.as<S>(), (const SlabDesc*)p->dslabs.as<SlabDesc>(),
                        (const BlockDesc*)p->dblocks.as<BlockDesc>(), (const SweepDesc*)p->dsegs.as<SweepDesc>(),
                        (uint32_t)p->Mr, (uint32_t)p->Nc, (uint32_t)p->n_meas, p->gS.U, p->slab_ns, p->slab_lag,
                        p->slab_Ns, p->slab_nw, (const double2*)p->dq.as<double2>(), col_vecs(p),
                        p->dwpart_s.as<double2>(), (const Params*)p->dparams.as<Params>(), p->dred.as<double>(),
                        p->dstate.as<IterState>(),
                        p->dtrace_tile.p ? p->dtrace_tile.as<unsigned long long>() : nullptr));
}

template <typename S>
void launch_sweep(admm_plan* p, cudaStream_t s) {
  if (p->slab_rpl) return launch_slab<S>(p, s);
  if (p->sweep_lpr == 8)
    launch_sweep_lpr<S, 8>(p, s);
  else if (p->sweep_lpr == 4)
    launch_sweep_lpr<S, 4>(p, s);
  else
    launch_sweep_lpr<S, 2>(p, s);
}

// One iteration: sweep (z, u/v/s/c, next w) -> [objective] -> r (+ close iteration) ->
// q = K r -> ghat.
template <typename S>
void enqueue_iteration_sweep(admm_plan* p, cudaStream_t s, bool with_objective, std::vector<cudaEvent_t>* ev) {
  const int nb = (int)p->blocks.size();
  auto mark = [&](size_t k) {
    if (ev) CK(cudaEventRecord((*ev)[k], s));
  };
  mark(0);
  launch_sweep<S>(p, s);
  mark(1);
  if (with_objective && p->obj_pass) {
    gemv_n_kernel<S, kVN, kEvictNormal><<<(unsigned)p->gO.P, kCtaThreads, 0, s>>>(
        p->dH.as<S>(), p->dv.as<double2>(), p->dopart.as<double2>(), p->dhNv.as<MatDesc>(), nb, p->gO.U);
    objective_rows_kernel<<<dim3(p->ogx, (uint32_t)p->Mr), kCtaThreads, 0, s>>>(
        p->dg.as<double2>(), p->dopart.as<double2>(), p->dhNv.as<MatDesc>(), p->dblocks.as<BlockDesc>(),
        (uint32_t)p->Nc, p->gO.U, p->gO.P, p->dored.as<double>());
  }
  launch_pdl(rows_finalize_sweep_kernel, dim3(p->rgx_s, nb), dim3(kCtaThreads), 0, s, row_vecs(p),
             p->dwpart_s.as<double2>(), p->dsegs.as<SweepDesc>(), p->dblocks.as<BlockDesc>(),
             p->dgblocks.as<BlockDesc>(), (uint32_t)p->N, (uint32_t)p->n_meas, p->gS.U, p->gS.P, 0, 1,
             p->dred.as<double>(), p->dparams.as<Params>(), p->dtrace.as<double>(), p->trace_cap,
             p->dstate.as<IterState>(), (double*)nullptr);
  mark(2);
  if (with_objective && !p->obj_pass)  // this iteration's a_b from the sweep's next w (no H pass)
    launch_pdl(objective_rec_kernel, dim3(p->orgx, (uint32_t)p->Mr), dim3(kCtaThreads), 0, s, row_vecs(p),
               p->dhs.as<double2>(), p->dblocks.as<BlockDesc>(), (uint32_t)p->Nc, p->onp, p->drored.as<double>(),
               (const IterState*)p->dstate.as<IterState>(), (uint64_t)0);
  if (with_objective) {  // the sweep's finalize wrote NaN: fill the objective of this iteration
    const bool rec = !p->obj_pass;
    launch_pdl(objective_trace_kernel, dim3(1), dim3(kCtaThreads), 0, s, (const double*)p->dred.as<double>(),
               (uint32_t)p->gS.P, (const double*)(rec ? p->drored.as<double>() : p->dored.as<double>()),
               rec ? p->nor : p->no, (const Params*)p->dparams.as<Params>(), p->dtrace.as<double>(), p->trace_cap,
               (const IterState*)p->dstate.as<IterState>());
  }
  enqueue_kapply<S>(p, s, [&] { mark(3); });
  mark(4);
  CK(cudaGetLastError());
}

// ---- batched scenes (config 5) ----------------------------------------------------
template <typename S>
void bgemm_attrs() {
  CK(cudaFuncSetAttribute(bgemm_kernel<S, false, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)bgemm_smem<S, false, 64>()));
  CK(cudaFuncSetAttribute(bgemm_kernel<S, true, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)bgemm_smem<S, true, 64>()));
  CK(cudaFuncSetAttribute(bgemm_kernel<S, false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)bgemm_smem<S, false, 32>()));
  CK(cudaFuncSetAttribute(bgemm_kernel<S, true, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)bgemm_smem<S, true, 32>()));
}

// One skinny GEMM launch over a tile list, in the plan's scene-tile width.
template <typename S, bool ADJ>
void launch_bgemm(const admm_plan* p, cudaStream_t s, size_t ntiles, const S* A, const BTile* tiles,
                  const double2* X, double2* out, uint32_t B) {
  if (p->bsb == 32)
    bgemm_kernel<S, ADJ, 32><<<(unsigned)ntiles, 256, bgemm_smem<S, ADJ, 32>(), s>>>(A, tiles, X, out, B);
  else
    bgemm_kernel<S, ADJ, 64><<<(unsigned)ntiles, 256, bgemm_smem<S, ADJ, 64>(), s>>>(A, tiles, X, out, B);
}

// Split-K count s in [1, smax] (and at most kmax) whose tiles*s work units fill the
// `slots` resident CTAs in the most nearly whole waves; each extra split costs a
// partial slice, so ties go to the smaller s.
uint32_t wave_split(uint64_t tiles, uint64_t slots, uint32_t smax, uint64_t kmax) {
  smax = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(smax, kmax));
  double best = -1.0;
  uint32_t bs = 1;
  for (uint32_t sp = 1; sp <= smax; ++sp) {
    const double waves = (double)(tiles * sp) / (double)slots;
    const double score = waves / std::ceil(waves) - 0.01 * (sp - 1);
    if (score > best + 1e-12) best = score, bs = sp;
  }
  return bs;
}

void build_batched(admm_plan* p) {
  const uint64_t B = p->batch;
  if (p->dtype == ADMM_C128)
    bgemm_attrs<double2>();
  else
    bgemm_attrs<float2>();
  const uint64_t nb = p->blocks.size();
  uint64_t rtiles = 0, ctiles = 0;
  for (auto& b : p->blocks) rtiles += cdiv(b.rows, kBT), ctiles += cdiv(b.cols, kBT);
  // split-K counts chosen for whole waves over the resident CTA slots (bgemm runs 2 CTAs
  // per SM): config 5 has 192 row tiles (x3 -> 1.95 waves) and 1024 column tiles
  // (x2 -> 6.9 waves) instead of 2.6 / 3.5 waves
  int occ = 0;
  p->bsb = 64;
  if (p->dtype == ADMM_C128)
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->bsb == 32 ? bgemm_kernel<double2, false, 32> : bgemm_kernel<double2, false, 64>, 256,
                                                     p->bsb == 32 ? bgemm_smem<double2, false, 32>() : bgemm_smem<double2, false, 64>()));
  else
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->bsb == 32 ? bgemm_kernel<float2, false, 32> : bgemm_kernel<float2, false, 64>, 256,
                                                     p->bsb == 32 ? bgemm_smem<float2, false, 32>() : bgemm_smem<float2, false, 64>()));
  const uint64_t nsc = cdiv(B, (uint64_t)p->bsb);  // scene tiles
  rtiles *= nsc;
  ctiles *= nsc;
  const uint64_t slots = (uint64_t)std::max(1, occ) * p->num_sms;
  p->splitN = wave_split(rtiles, slots, 16, p->max_seg / (4 * kBK));
  p->splitK = wave_split(rtiles, slots, 16, p->max_rows / (4 * kBK));
  p->splitH = wave_split(ctiles, slots, 4, p->max_rows / (4 * kBK));
  if (const char* e = std::getenv("ADMM_B200_BSPLIT")) {  // diagnostics: "N,K,H"
    unsigned a = 0, b = 0, c = 0;
    if (std::sscanf(e, "%u,%u,%u", &a, &b, &c) == 3 && a && b && c) p->splitN = a, p->splitK = b, p->splitH = c;
  }
  const uint64_t stride = p->mvec_total * B;
  const uint64_t zstride = p->vec_total * B;
  p->tN.clear();
  p->tK.clear();
  p->tH.clear();
  p->tG.clear();
  for (uint32_t s0 = 0; s0 < B; s0 += p->bsb)  // scene tiles outermost: a wave streams each A tile once per scene tile
    for (uint64_t b = 0; b < nb; ++b) {
      const BlockDesc& bd = p->blocks[b];
      const MatDesc& hn = p->hN[b];
      const MatDesc& kn = p->kN[b];
      const uint32_t kcN = (uint32_t)round_up(cdiv(bd.cols, p->splitN), kBK);
      const uint32_t kcK = (uint32_t)round_up(cdiv(bd.rows, p->splitK), kBK);
      for (uint32_t t0 = 0; t0 < bd.rows; t0 += kBT)
        for (uint32_t sp = 0; sp < p->splitN; ++sp)
          p->tN.push_back(BTile{hn.a_off, (uint64_t)bd.vec_off * B, sp * stride + (uint64_t)bd.mvec_off * B, hn.ld,
                                bd.rows, bd.cols, t0, std::min(bd.cols, sp * kcN), std::min(bd.cols, (sp + 1) * kcN),
                                s0, 0});
      for (uint32_t t0 = 0; t0 < bd.rows; t0 += kBT)
        for (uint32_t sp = 0; sp < p->splitK; ++sp)
          p->tK.push_back(BTile{kn.a_off, (uint64_t)bd.mvec_off * B, sp * stride + (uint64_t)bd.mvec_off * B, kn.ld,
                                bd.rows, bd.rows, t0, std::min(bd.rows, sp * kcK), std::min(bd.rows, (sp + 1) * kcK),
                                s0, 0});
      const uint32_t kcH = (uint32_t)round_up(cdiv(bd.rows, p->splitH), kBK);
      for (uint32_t t0 = 0; t0 < bd.cols; t0 += kBT)
        for (uint32_t sp = 0; sp < p->splitH; ++sp)
          p->tH.push_back(BTile{hn.a_off, (uint64_t)bd.mvec_off * B, sp * zstride + (uint64_t)bd.vec_off * B, hn.ld,
                                bd.rows, bd.cols, t0, std::min(bd.rows, sp * kcH), std::min(bd.rows, (sp + 1) * kcH),
                                s0, 0});
      for (uint32_t t0 = 0; t0 < bd.cols; t0 += kBT)
        p->tG.push_back(BTile{hn.a_off, (uint64_t)bd.row0 * B, (uint64_t)bd.vec_off * B, hn.ld, bd.rows, bd.cols, t0,
                              0, bd.rows, s0, 0});
    }
  upload_desc(p->dtN, p->tN.data(), p->tN.size() * sizeof(BTile));
  upload_desc(p->dtK, p->tK.data(), p->tK.size() * sizeof(BTile));
  upload_desc(p->dtH, p->tH.data(), p->tH.size() * sizeof(BTile));
  upload_desc(p->dtG, p->tG.data(), p->tG.size() * sizeof(BTile));
  p->dwpart.alloc((size_t)p->splitN * stride * 16);
  p->dqpart.alloc((size_t)p->splitK * stride * 16);
  p->dz.alloc((size_t)p->splitH * p->vec_total * B * 16);
  p->dkappa.alloc(B * sizeof(double));
  uint64_t pzm = 5;  // bzupdate CTAs per SM (48 registers: 5 x 256 threads fit; 127 -> 113 us on config 5)
  p->pz = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(pzm * p->num_sms, cdiv(p->max_seg, 4)));
  p->dbred.alloc((size_t)3 * p->pz * kBB * sizeof(double));
  p->dblam.alloc(B * sizeof(double));
  p->bogx = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(2ull * p->num_sms / std::max<uint64_t>(1, p->Mr),
                                                                cdiv(p->max_rows, kCtaThreads / kBB)));
  p->dbored.alloc((size_t)p->bogx * p->Mr * kBB * sizeof(double));
}

BRowVecs brow_vecs(admm_plan* p) {
  return BRowVecs{p->dg.as<double2>(), p->ghat_ptr, p->dgij.as<double2>(), p->dr.as<double2>(), p->dq.as<double2>()};
}

void enqueue_bobjective(admm_plan* p, cudaStream_t s) {
  const uint32_t B = (uint32_t)p->batch;
  bobjective_rec_kernel<<<dim3(p->bogx, (unsigned)p->Mr), kCtaThreads, 0, s>>>(
      brow_vecs(p), p->dhs.as<double2>(), p->dblocks.as<BlockDesc>(), (uint32_t)p->Nc, B, p->dbored.as<double>(),
      p->dstate.as<IterState>(), 1);
  bobjective_trace_kernel<<<1, kBB * kBFinParts, 0, s>>>(p->dbred.as<double>(), p->pz, p->dbored.as<double>(),
                                            p->bogx * (uint32_t)p->Mr, p->dblam.as<double>(), B,
                                            p->dtrace.as<double>(), p->trace_cap, p->dstate.as<IterState>());
}

// After the last iteration: w = H c of the would-be next iteration (bgemm + brows<kRhs>),
// then the recurrence fills the last trace entry.  Leaves the iterates untouched.
template <typename S>
void enqueue_bobjective_last(admm_plan* p, cudaStream_t s) {
  const uint32_t B = (uint32_t)p->batch, nb = (uint32_t)p->blocks.size();
  const uint64_t stride = p->mvec_total * B;
  const unsigned rgx = (unsigned)cdiv((uint64_t)p->max_rows * B, kCtaThreads);
  launch_bgemm<S, false>(p, s, p->tN.size(), p->dH.as<S>(), p->dtN.as<BTile>(),
                                                                  p->dc.as<double2>(), p->dwpart.as<double2>(), B);
  brows_kernel<kRhs><<<dim3(rgx, nb), kCtaThreads, 0, s>>>(brow_vecs(p), p->dwpart.as<double2>(), stride, p->splitN,
                                                          p->dblocks.as<BlockDesc>(), (uint32_t)p->Nc, B,
                                                          p->dparams.as<Params>());
  enqueue_bobjective(p, s);
  CK(cudaGetLastError());
}

template <typename S>
void enqueue_iteration_batched(admm_plan* p, cudaStream_t s, bool with_objective, std::vector<cudaEvent_t>* ev) {
  const uint32_t B = (uint32_t)p->batch, nb = (uint32_t)p->blocks.size();
  const uint64_t stride = p->mvec_total * B;
  const unsigned rgx = (unsigned)cdiv((uint64_t)p->max_rows * B, kCtaThreads);
  auto mark = [&](size_t k) {
    if (ev) CK(cudaEventRecord((*ev)[k], s));
  };
  mark(0);
  launch_bgemm<S, false>(p, s, p->tN.size(), p->dH.as<S>(), p->dtN.as<BTile>(),
                                                                  p->dc.as<double2>(), p->dwpart.as<double2>(), B);
  mark(1);
  brows_kernel<kRhs><<<dim3(rgx, nb), kCtaThreads, 0, s>>>(brow_vecs(p), p->dwpart.as<double2>(), stride, p->splitN,
                                                          p->dblocks.as<BlockDesc>(), (uint32_t)p->Nc, B,
                                                          p->dparams.as<Params>());
  if (with_objective) enqueue_bobjective(p, s);  // trace[k-1].objective per scene (w = H c of this iteration)
  mark(2);
  launch_bgemm<S, false>(p, s, p->tK.size(), p->dK.as<S>(), p->dtK.as<BTile>(),
                                                                  p->dr.as<double2>(), p->dqpart.as<double2>(), B);
  mark(3);
  brows_kernel<kQ><<<dim3(rgx, nb), kCtaThreads, 0, s>>>(brow_vecs(p), p->dqpart.as<double2>(), stride, p->splitK,
                                                        p->dblocks.as<BlockDesc>(), (uint32_t)p->Nc, B,
                                                        p->dparams.as<Params>());
  mark(4);
  launch_bgemm<S, true>(p, s, p->tH.size(), p->dH.as<S>(), p->dtH.as<BTile>(), p->dq.as<double2>(),
                                                                 p->dz.as<double2>(), B);
  mark(5);
  bzupdate_kernel<<<p->pz, kCtaThreads, 0, s>>>(col_vecs(p), p->dz.as<double2>(), p->splitH, p->vec_total * B,
                                                p->dblocks.as<BlockDesc>(),
                                                (uint32_t)p->Mr, (uint32_t)p->Nc, B, p->dkappa.as<double>(),
                                                p->dbred.as<double>(), p->dstate.as<IterState>());
  mark(6);
  bfinalize_kernel<<<1, kBB * kBFinParts, 0, s>>>(p->dbred.as<double>(), p->pz, B, p->dparams.as<Params>(), p->dtrace.as<double>(),
                                     p->trace_cap, p->dstate.as<IterState>());
  mark(7);
  CK(cudaGetLastError());
}

void enqueue_iteration_any(admm_plan* p, cudaStream_t s, bool obj, std::vector<cudaEvent_t>* ev) {
  if (p->schedule == 4) {
    if (ev) CK(cudaEventRecord((*ev)[0], s));
    launch_resident_any(p, s, 1, false, obj);
    if (ev) CK(cudaEventRecord((*ev)[1], s));
    return;
  }
  if (p->batch > 1) {
    if (p->dtype == ADMM_C128)
      enqueue_iteration_batched<double2>(p, s, obj, ev);
    else
      enqueue_iteration_batched<float2>(p, s, obj, ev);
    return;
  }
  if (p->schedule == 5) {
    if (p->dtype == ADMM_C128)
      enqueue_iteration_support<double2>(p, s, obj, ev);
    else
      enqueue_iteration_support<float2>(p, s, obj, ev);
  } else if (p->schedule == 2) {
    if (p->dtype == ADMM_C128)
      enqueue_iteration_sweep<double2>(p, s, obj, ev);
    else
      enqueue_iteration_sweep<float2>(p, s, obj, ev);
  } else {
    if (p->dtype == ADMM_C128)
      enqueue_iteration_twopass<double2>(p, s, obj, ev);
    else
      enqueue_iteration_twopass<float2>(p, s, obj, ev);
  }
}

// Objective of the current v (admm_core.hpp:60-64) into *d_obj, without touching
// the iteration state.
__global__ void objective_final_kernel(const double* __restrict__ red, uint32_t nz,
                                       const double* __restrict__ ored, uint32_t no,
                                       const Params* __restrict__ prm, double* out) {
  __shared__ double sm[kCtaWarps];
  double l = 0.0, o = 0.0;
  for (uint32_t k = threadIdx.x; k < nz; k += kCtaThreads) l += red[2 * nz + k];
  for (uint32_t k = threadIdx.x; k < no; k += kCtaThreads) o += ored[k];
  l = block_sum<kCtaThreads>(l, sm);
  o = block_sum<kCtaThreads>(o, sm);
  if (threadIdx.x == 0) *out = 0.5 * o + prm->lambda * l;
}

template <typename S>
void enqueue_objective(admm_plan* p, cudaStream_t s) {
  const int nb = (int)p->blocks.size();
  gemv_n_kernel<S, kVN, kEvictNormal><<<(unsigned)p->gO.P, kCtaThreads, 0, s>>>(
      p->dH.as<S>(), p->dv.as<double2>(), p->dopart.as<double2>(), p->dhNv.as<MatDesc>(), nb, p->gO.U);
  objective_rows_kernel<<<dim3(p->ogx, (unsigned)p->Mr), kCtaThreads, 0, s>>>(
      p->dg.as<double2>(), p->dopart.as<double2>(), p->dhNv.as<MatDesc>(), p->dblocks.as<BlockDesc>(),
      (uint32_t)p->Nc, p->gO.U, p->gO.P, p->dored.as<double>());
  // l1 partials of the last column update ([3][n] layout: rp2, rd2, l1)
  const uint32_t nred = p->schedule == 4 ? p->res_P : p->schedule == 2 ? (uint32_t)p->gS.P : p->nz;
  const double* red = p->schedule == 4 ? p->dres_red.as<double>() : p->dred.as<double>();
  objective_final_kernel<<<1, kCtaThreads, 0, s>>>(red, nred, p->dored.as<double>(), p->no, p->dparams.as<Params>(),
                                                   p->dobj.as<double>());
  CK(cudaGetLastError());
}

// max |(H^H g)_t| over all columns: gemv_h with q = g, then the row-block sum.
template <int CH>
__global__ void adjoint_absmax_kernel(const double2* __restrict__ part, const MatDesc* __restrict__ mats,
                                      const BlockDesc* __restrict__ blocks, uint32_t M, uint32_t N, uint64_t U,
                                      uint64_t P, double* __restrict__ out) {
  __shared__ double sm[kCtaThreads];
  const uint32_t j = blockIdx.y;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  double m = 0.0;
  if (t < blocks[j].cols) {
    double2 z = make_double2(0.0, 0.0);
    for (uint32_t i = 0; i < M; ++i) z = cadd(z, sum_cols_part<CH>(part, mats[i * N + j], t, U, P));
    m = hypot(z.x, z.y);
  }
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int o = kCtaThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.y * gridDim.x + blockIdx.x] = sm[0];
}

void set_params(admm_plan* p) {
  const double m = (double)p->M;
  p->params.rho = p->cfg.rho;
  p->params.lambda = p->cfg.lambda;
  p->params.m_rep = m;
  // kappa: solvers.hpp:104 / 344 (lambda/(M rho)); solvers.hpp:212 and
  // reference.hpp:43 (lambda/rho).
  p->params.kappa = (p->method == ADMM_CONSENSUS || p->method == ADMM_HYBRID)
                        ? p->cfg.lambda / (m * p->cfg.rho)
                        : p->cfg.lambda / p->cfg.rho;
  CK(cudaMemcpyAsync(p->dparams.p, &p->params, sizeof(Params), cudaMemcpyHostToDevice, p->stream));
  if (p->batch > 1) {  // per-scene kappa_b (same rule, lambda_b per scene)
    if (p->lambdas.size() != p->batch) p->lambdas.assign(p->batch, p->cfg.lambda);
    std::vector<double> k(p->batch);
    for (uint64_t b = 0; b < p->batch; ++b) k[b] = p->params.kappa * (p->lambdas[b] / p->cfg.lambda);
    CK(cudaMemcpyAsync(p->dkappa.p, k.data(), k.size() * 8, cudaMemcpyHostToDevice, p->stream));
    if (p->dblam.p)
      CK(cudaMemcpyAsync(p->dblam.p, p->lambdas.data(), p->batch * 8, cudaMemcpyHostToDevice, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  }
}

void upload_g(admm_plan* p, const double* g) {
  CK(cudaMemcpyAsync(p->dg.p, g, p->n_meas * p->batch * 16, cudaMemcpyHostToDevice, p->stream));
  if (p->cfg.scl != 1.0) {
    scale_vec_kernel<<<64, 256, 0, p->stream>>>(p->dg.as<double2>(), p->n_meas * p->batch, p->cfg.scl);
    CK(cudaGetLastError());
  }
}

void reset_state(admm_plan* p) {
  cudaStream_t s = p->stream;
  for (DevBuf* d : {&p->du, &p->ds, &p->dc, &p->dv, &p->dvprev, &p->dgij, &p->dr, &p->dq, &p->dhs, &p->danew,
                    &p->daold})
    if (d->p) CK(cudaMemsetAsync(d->p, 0, d->bytes, s));
  CK(cudaMemsetAsync(p->ghat_ptr, 0, p->mvec_total * 16 * p->batch, s));
  CK(cudaMemsetAsync(p->outbox_ptr, 0, p->outbox_total * 16, s));
  if (p->dl1prev.p) CK(cudaMemsetAsync(p->dl1prev.p, 0, sizeof(double), s));
  IterState st{0, ~0ull, 0u, 0u};
  CK(cudaMemcpyAsync(p->dstate.p, &st, sizeof(st), cudaMemcpyHostToDevice, s));
  if (p->schedule == 2) {
    if (p->dtype == ADMM_C128)
      enqueue_sweep_prologue<double2>(p, s);
    else
      enqueue_sweep_prologue<float2>(p, s);
  }
  if (p->schedule == 4) launch_resident_any(p, s, 0, true, false);
  if (p->schedule == 5 && p->is_shard) {  // phase 1 of the first iteration is the prologue (v = 0: empty support)
    CK(cudaMemsetAsync(p->dnzcnt.p, 0, p->dnzcnt.bytes, s));
  } else if (p->schedule == 5) {  // prologue: r = g_ij (w = H c^0 = 0), q = K r, ghat
    enqueue_support_rows(p, s, true);
    if (p->dtype == ADMM_C128)
      enqueue_kapply<double2>(p, s);
    else
      enqueue_kapply<float2>(p, s);
    CK(cudaGetLastError());
  }
}

void ensure_trace(admm_plan* p, uint64_t iters) {
  if (iters <= p->trace_cap) return;
  p->trace_cap = std::max<uint64_t>(iters, 64);
  p->dtrace.alloc(p->trace_cap * 3 * p->batch * sizeof(double));
  if (p->exec) {  // the graph captured the old trace pointer
    cudaGraphExecDestroy(p->exec);
    p->exec = nullptr;
  }
}

constexpr uint64_t kGraphIters = 8;  // iterations per captured graph

void ensure_graph(admm_plan* p) {
  if (p->exec) return;
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
  try {
    for (uint64_t k = 0; k < kGraphIters; ++k) enqueue_iteration_any(p, p->stream, p->trace_obj, nullptr);
  } catch (...) {
    cudaStreamEndCapture(p->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CK(cudaStreamEndCapture(p->stream, &g));
  cudaError_t e = cudaGraphInstantiate(&p->exec, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  // single-iteration graph for the tail / stepping path
  p->graph_iters = kGraphIters;
}

void enqueue_iters(admm_plan* p, uint64_t iters) {
  if (p->schedule == 4) {  // one persistent launch for all of them
    if (iters) launch_resident_any(p, p->stream, iters, false, p->trace_obj);
    return;
  }
  ensure_graph(p);
  uint64_t k = 0;
  for (; k + kGraphIters <= iters; k += kGraphIters) CK(cudaGraphLaunch(p->exec, p->stream));
  for (; k < iters; ++k) enqueue_iteration_any(p, p->stream, p->trace_obj, nullptr);
}

IterState read_state(admm_plan* p) {
  IterState st{};
  CK(cudaMemcpyAsync(&st, p->dstate.p, sizeof(st), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return st;
}

void read_segments(admm_plan* p, const DevBuf& src, double* dst) {
  const uint64_t B = p->batch;  // rows of B scenes
  p->h_seg.resize(p->seg_total * 2 * B);
  CK(cudaMemcpyAsync(p->h_seg.data(), src.p, p->seg_total * 16 * B, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  for (uint64_t j = 0; j < p->Nc; ++j) {  // local segments (all of them on a single GPU)
    const BlockDesc& b = p->blocks[j];
    std::memcpy(dst + 2 * (uint64_t)b.col0 * B, p->h_seg.data() + 2 * (uint64_t)b.seg_off * B, (size_t)b.cols * 16 * B);
  }
}

admm_status run_guarded(const std::function<void()>& fn) {
  try {
    fn();
    return ADMM_OK;
  } catch (const Fail& f) {
    g_last_error = f.msg;
    g_last_good = f.last_good;
    return f.st;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ADMM_E_CUDA;
  }
}

void validate_cfg(const admm_solver_config& c) {  // SolverConfig::validate, admm_core.hpp:26-34
  if (!(c.rho > 0.0)) throw Fail{ADMM_E_PARAMETER, "SolverConfig: rho must be positive"};
  if (!(c.lambda > 0.0)) throw Fail{ADMM_E_PARAMETER, "SolverConfig: lambda must be positive"};
  if (!(c.scl > 0.0)) throw Fail{ADMM_E_PARAMETER, "SolverConfig: scl must be positive"};
  if (c.max_iters < 1) throw Fail{ADMM_E_PARAMETER, "SolverConfig: max_iters must be >= 1"};
  if (c.eps_pri < 0.0 || c.eps_dual < 0.0)
    throw Fail{ADMM_E_PARAMETER, "SolverConfig: residual thresholds must be non-negative"};
}

// Build a plan.  skip_cfg_validation is used by the GramSolver op (no lambda).
admm_plan* create_plan(const admm_plan_options& o, const admm_solver_config& cfg, uint64_t n_meas,
                       uint64_t n_pix, const void* h, admm_dtype h_dtype, const double* g,
                       bool skip_cfg_validation, const admm_shard* shard = nullptr) {
  const auto t0 = std::chrono::steady_clock::now();
  auto since = [](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  };
  if (!skip_cfg_validation) validate_cfg(cfg);
  // SensingProblem::validate (problem.hpp:35-49)
  if (n_meas == 0 || n_pix == 0 || !h || !g)
    throw Fail{ADMM_E_DIMENSION, "SensingProblem: empty sensing matrix"};
  // Finiteness of H: a separate host pass for small matrices; large ones are checked by the
  // staged upload's packing pass (upload_h).  Any error raised before that point is then
  // preceded by the scan, so NumericalError keeps its place in the reference's order
  // (problem.hpp:35-49 before the partition, partition.hpp:56-65).
  auto h_finite = [&] {
    return h_dtype == ADMM_C128 ? host_all_finite(static_cast<const double*>(h), 2 * n_meas * n_pix)
                                : host_all_finite(static_cast<const float*>(h), 2 * n_meas * n_pix);
  };
  const bool defer_h = n_meas * n_pix * (h_dtype == ADMM_C128 ? 16 : 8) >= (256ull << 20);
  if ((!defer_h && !h_finite()) || !host_all_finite(g, 2 * n_meas * std::max<uint64_t>(1, o.batch)))
    throw Fail{ADMM_E_NUMERICAL, "SensingProblem: non-finite entries"};
  std::unique_ptr<admm_plan> p;
  bool h_checked = false;  // the staged upload has scanned H
  try {
  if (o.noise_sigma < 0.0) throw Fail{ADMM_E_PARAMETER, "SensingProblem: negative noise_sigma"};
  if (o.method < ADMM_REFERENCE || o.method > ADMM_HYBRID) throw Fail{ADMM_E_PARAMETER, "unknown method"};
  if (o.dtype != ADMM_C128 && o.dtype != ADMM_C64) throw Fail{ADMM_E_PARAMETER, "unknown dtype"};

  p = std::make_unique<admm_plan>();
  p->device = o.device;
  p->dtype = o.dtype;
  p->method = o.method;
  p->n_meas = n_meas;
  p->n_pix = n_pix;
  p->cfg = cfg;
  p->ragged = o.ragged != 0;
  p->trace_obj = o.trace_objective != 0;
  p->M = (o.method == ADMM_CONSENSUS || o.method == ADMM_HYBRID) ? o.M : 1;
  p->N = (o.method == ADMM_SECTIONING || o.method == ADMM_HYBRID) ? o.N : 1;
  p->elem = o.dtype == ADMM_C128 ? 16 : 8;
  p->batch = std::max<uint64_t>(1, o.batch);
  if (p->batch > kBB) throw Fail{ADMM_E_PARAMETER, "batch larger than 64 scenes"};
  if (p->batch > 1 && shard && shard->Pr * shard->Pc > 1)
    throw Fail{ADMM_E_PARAMETER, "batched scenes run on a single GPU"};
  if (p->batch > 1 && (cfg.eps_pri != 0.0 || cfg.eps_dual != 0.0))
    throw Fail{ADMM_E_PARAMETER, "batched scenes run a fixed iteration count (eps = 0)"};
  // make_partition (partition.hpp:56-65): rows then columns
  p->rb = split_bounds(n_meas, p->M, p->ragged, "row");
  p->cb = split_bounds(n_pix, p->N, p->ragged, "column");
  if (p->M * p->N > 65535) throw Fail{ADMM_E_PARAMETER, "too many blocks"};

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Fail{ADMM_E_CUDA, "no CUDA device: libadmm_b200 has no CPU fallback"};
  CK(cudaSetDevice(o.device));
  CK(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, o.device));
  CK(cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking));
  p->stream = p->own_stream;

  // sharding: this plan owns row blocks [i0, i0+Mr) x column blocks [j0, j0+Nc)
  p->is_shard = shard != nullptr;
  if (shard) {
    p->Pr = shard->Pr;
    p->Pc = shard->Pc;
    p->pr = shard->pr;
    p->pc = shard->pc;
    if (p->Pr < 1 || p->Pc < 1 || p->pr >= p->Pr || p->pc >= p->Pc)
      throw Fail{ADMM_E_INDEX, "shard coordinates out of range"};
    if (p->M % p->Pr || p->N % p->Pc)
      throw Fail{ADMM_E_PARTITION, "process grid " + std::to_string(p->Pr) + "x" + std::to_string(p->Pc) +
                                       " does not divide the " + std::to_string(p->M) + "x" +
                                       std::to_string(p->N) + " block grid"};
    if (p->Pr * p->Pc > 1 && p->ragged) throw Fail{ADMM_E_PARTITION, "sharded plans need uniform blocks"};
  }
  p->Mr = p->M / p->Pr;
  p->Nc = p->N / p->Pc;
  p->i0 = p->pr * p->Mr;
  p->j0 = p->pc * p->Nc;
  uint64_t mmax = 0, nmax = 0;
  for (uint64_t i = 0; i < p->M; ++i) mmax = std::max<uint64_t>(mmax, p->rb[i + 1] - p->rb[i]);
  for (uint64_t j = 0; j < p->N; ++j) nmax = std::max<uint64_t>(nmax, p->cb[j + 1] - p->cb[j]);
  p->mpad = round_up(mmax, 4);
  p->npad = round_up(nmax, 4);
  // Global table (worker id = i*N + j, solvers.hpp:305).  Offsets follow the exchange
  // layouts so that all-gathers land every peer vector where the kernels look for it:
  //   ghat:   [pc'][il][jl][mpad]  for blocks in this plan's row blocks (row comm order)
  //   outbox: [i][jl][npad]        for blocks in this plan's column blocks (column comm order)
  // A sharded plan with the per-iteration objective carries a_b = H_b v next to ghat_b (the
  // A region, gathered with it).  Column-sharded grids reserve kScalDoubles after each
  // rank's ghat slot; the sweep schedule (scalars ready before the ghat exchange) uses them
  // instead of a separate all-gather.
  if (p->is_shard && p->trace_obj && (p->Nc > kCtaThreads || o.batch > 1)) p->trace_obj = false;
  p->aoff = p->is_shard ? p->Mr * p->Nc * p->mpad : 0;  // (the final objective pass uses it too)
  p->shard_obj = p->is_shard && p->trace_obj;
  p->gslot = p->Mr * p->Nc * p->mpad + p->aoff + (p->Pr == 1 && p->Pc > 1 ? kScalDoubles / 2 : 0);
  p->gblocks.assign(p->M * p->N, BlockDesc{});
  for (uint64_t i = 0; i < p->M; ++i)
    for (uint64_t q = 0; q < p->N; ++q) {
      BlockDesc& b = p->gblocks[i * p->N + q];
      b.i = (uint32_t)i;
      b.j = (uint32_t)q;
      b.rows = (uint32_t)(p->rb[i + 1] - p->rb[i]);
      b.cols = (uint32_t)(p->cb[q + 1] - p->cb[q]);
      b.row0 = (uint32_t)p->rb[i];
      b.col0 = (uint32_t)p->cb[q];
      const bool own_row = i >= p->i0 && i < p->i0 + p->Mr;
      const bool own_col = q >= p->j0 && q < p->j0 + p->Nc;
      const uint64_t il = i - p->i0, jl = q - p->j0;
      if (own_row) b.mvec_off = (uint32_t)((q / p->Nc) * p->gslot + (il * p->Nc + q % p->Nc) * p->mpad);
      if (own_col) {
        b.jl = (uint32_t)jl;
        b.seg_off = (uint32_t)(jl * p->npad);
        b.box_off = (uint32_t)((i * p->Nc + jl) * p->npad);
      }
      if (own_row && own_col) b.vec_off = (uint32_t)((il * p->Nc + jl) * p->npad);
    }
  for (uint64_t il = 0; il < p->Mr; ++il)
    for (uint64_t jl = 0; jl < p->Nc; ++jl) {
      const BlockDesc& b = p->gblocks[(p->i0 + il) * p->N + p->j0 + jl];
      p->blocks.push_back(b);
      p->max_rows = std::max(p->max_rows, b.rows);
      p->max_m = std::max(p->max_m, b.rows);
      p->max_seg = std::max(p->max_seg, b.cols);
      p->max_rowblock = std::max(p->max_rowblock, b.rows);
    }
  p->mvec_total = p->Pc * p->gslot;
  p->vec_total = p->Mr * p->Nc * p->npad;
  p->seg_total = p->Nc * p->npad;
  p->outbox_total = p->M * p->Nc * p->npad;

  int requested = o.schedule;
  if (const char* env = std::getenv("ADMM_B200_SCHEDULE")) {
    if (!std::strcmp(env, "twopass")) requested = 1;
    if (!std::strcmp(env, "sweep")) requested = 2;
    if (!std::strcmp(env, "resident")) requested = 4;
    if (!std::strcmp(env, "support")) requested = 5;
  }
  if (skip_cfg_validation || o.batch > 1) requested = 1;  // helper plans / batched scenes
  if (p->dtype == ADMM_C128) {
    build_geometry<double2>(p.get());
    choose_schedule<double2>(p.get(), requested);
  } else {
    build_geometry<float2>(p.get());
    choose_schedule<float2>(p.get(), requested);
  }
  const size_t nb = p->blocks.size();
  upload_desc(p->dblocks, p->blocks.data(), nb * sizeof(BlockDesc));
  upload_desc(p->dgblocks, p->gblocks.data(), p->gblocks.size() * sizeof(BlockDesc));
  p->doutbox.alloc(p->outbox_total * 16);
  p->dscal.alloc(p->Pr * p->Pc * kScalDoubles * sizeof(double));
  upload_desc(p->dhN, p->hN.data(), nb * sizeof(MatDesc));
  upload_desc(p->dhNv, p->hNv.data(), nb * sizeof(MatDesc));
  upload_desc(p->dkN, p->kN.data(), nb * sizeof(MatDesc));
  upload_desc(p->dhH, p->hH.data(), nb * sizeof(MatDesc));
  upload_desc(p->dhHg, p->hHg.data(), nb * sizeof(MatDesc));
  for (DevBuf* d : {&p->dghat, &p->dgij, &p->dr, &p->dq}) d->alloc(p->mvec_total * 16 * p->batch);
  p->ghat_ptr = p->dghat.as<double2>();
  p->outbox_ptr = p->doutbox.as<double2>();
  p->fused_scal = p->Pr == 1 && p->Pc > 1 && p->schedule == 2;
  {  // packed Hermitian K for the per-iteration K apply (the batched schedule uses bgemm)
    p->kpacked = p->batch == 1;
    // keep the packed K in L2 (evict_last) when the H stream cannot evict it: the slab
    // sweep and (two-pass) the GEMVs stream H with evict_first, so a K of <= ~96 MiB stays
    // resident across iterations (config 2: K apply 19 -> 15 us)
    const bool kfits = p->k_elems * p->elem / 2 <= (96ull << 20);
    p->h_evict_first = p->schedule == 1 && kfits;
    p->kkeep = (p->slab_rpl > 0 || p->schedule == 1) && kfits;
  }
  p->scal_ptr = p->fused_scal ? reinterpret_cast<double*>(p->ghat_ptr + p->Mr * p->Nc * p->mpad + p->aoff)
                              : p->dscal.as<double>();
  for (DevBuf* d : {&p->du, &p->ds, &p->dc}) d->alloc(p->vec_total * 16 * p->batch);
  for (DevBuf* d : {&p->dv, &p->dvprev}) d->alloc(p->seg_total * 16 * p->batch);
  p->dg.alloc(p->n_meas * 16 * p->batch);
  p->dparams.alloc(sizeof(Params));
  p->dstate.alloc(sizeof(IterState));
  p->dobj.alloc(sizeof(double));
  p->rgx = (uint32_t)cdiv(p->max_rows, kCtaThreads);
  p->rgx_s = (uint32_t)cdiv(p->max_rows, kRfRows);
  p->zgx = (uint32_t)cdiv(p->max_seg, kCtaThreads);
  p->ogx = (uint32_t)cdiv(p->max_rowblock, kCtaThreads);
  p->nz = p->zgx * (uint32_t)p->Nc;
  p->no = p->ogx * (uint32_t)p->Mr;
  p->dred.alloc((size_t)3 * std::max<uint64_t>(p->nz, p->gS.P) * sizeof(double));
  p->dored.alloc((size_t)std::max<uint32_t>(p->no, p->zgx * (uint32_t)p->Nc) * sizeof(double));
  if (const char* e = std::getenv("ADMM_B200_OBJ")) p->obj_pass = !std::strcmp(e, "pass");
  if (p->Nc > kCtaThreads) p->obj_pass = true;  // the recurrence kernel spreads at most 256 column blocks
  if (p->is_shard) p->obj_pass = false;         // shards: recurrence + gathered A regions only
  if (p->aoff) {
    p->objgx = (uint32_t)cdiv(p->max_rowblock, kCtaThreads);
    p->dobjp.alloc((size_t)p->objgx * p->Mr * sizeof(double));
    p->dl1prev.alloc(sizeof(double));
  }
  if (p->trace_obj && !p->obj_pass) {
    p->dhs.alloc(p->mvec_total * std::max<uint64_t>(1, p->batch) * sizeof(double2));
    while ((1u << p->onp) < p->Nc) ++p->onp;
    p->orgx = (uint32_t)std::max<uint64_t>(1, cdiv(p->max_rowblock, kCtaThreads >> p->onp));
    p->nor = p->orgx * (uint32_t)p->Mr;
    p->drored.alloc((size_t)p->nor * sizeof(double));
  }
  ensure_trace(p.get(), std::max<uint64_t>(cfg.max_iters, 1));

  p->setup_phase[0] = since(t0);
  // In-place scaling of a directly copied H (problem.hpp:59-66) runs after the whole upload:
  // only then are the blocks final, so their Gram launches follow the upload instead of
  // overlapping it.
  const bool direct_scaled = ((h_dtype == ADMM_C128) == (p->dtype == ADMM_C128)) && cfg.scl != 1.0;
  auto setup_dtype = [&](auto tag) {
    using S = decltype(tag);
    GramWork gw;
    gram_begin<S>(p.get(), gw);
    upload_h<S>(p.get(), h, h_dtype, defer_h, [&](size_t b) {
      if (!direct_scaled) gram_blocks<S>(p.get(), gw, b, b + 1);
    });
    h_checked = true;
    if (direct_scaled) gram_blocks<S>(p.get(), gw, 0, p->blocks.size());
    if (p->slab_rpl) build_slab<S>(p.get());
    if (p->schedule == 5) build_support<S>(p.get());
    p->setup_phase[1] = since(t0) - p->setup_phase[0];
    factor_blocks<S>(p.get(), gw);
  };
  if (p->dtype == ADMM_C128)
    setup_dtype(double2{});
  else
    setup_dtype(float2{});
  } catch (const Fail& f) {
    if (defer_h && !h_checked && f.st != ADMM_E_NUMERICAL && !h_finite())
      throw Fail{ADMM_E_NUMERICAL, "SensingProblem: non-finite entries"};
    throw;
  }
  if (p->batch > 1) {
    build_batched(p.get());
    p->schedule = 3;
  }
  upload_g(p.get(), g);
  set_params(p.get());
  reset_state(p.get());
  CK(cudaStreamSynchronize(p->stream));
  p->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return p.release();
}

void check_plan(const admm_plan* p) {
  if (!p) throw Fail{ADMM_E_STATE, "null plan"};
  CK(cudaSetDevice(p->device));
}

// multi-GPU plans (admm_dist.inc)
bool is_dist(const admm_plan* p);
std::vector<admm_plan*> shards_of(admm_plan* p);
void dist_solve(admm_plan* root, double* solution, double* trace, uint64_t* iterations_run, double* objective,
                admm_observer_fn observer, void* user);
void dist_enqueue(admm_plan* root, uint64_t iters);
void dist_reset(const std::vector<admm_plan*>& sh);
void dist_sync(const std::vector<admm_plan*>& sh);
double dist_max_abs_adjoint(admm_plan* root);
void dist_gather_segments(const std::vector<admm_plan*>& sh, int which, double* dst);
void dist_gather_u(const std::vector<admm_plan*>& sh, std::vector<double>& u, std::vector<uint64_t>& off,
                   std::vector<uint64_t>& len);

}  // namespace

// ----------------------------------------------------------------------- C ABI
extern "C" {

int admm_abi_version(void) { return ADMM_B200_ABI_VERSION; }
const char* admm_last_error(void) { return g_last_error.c_str(); }
uint64_t admm_cmat_error_offset(void) { return g_last_offset; }
uint64_t admm_last_good_iteration(void) { return g_last_good; }

admm_status admm_plan_create(const admm_plan_options* opts, const admm_solver_config* cfg, uint64_t n_meas,
                             uint64_t n_pix, const void* h, admm_dtype h_dtype, const double* g,
                             admm_plan** out) {
  return run_guarded([&] {
    if (!opts || !cfg || !out) throw Fail{ADMM_E_STATE, "null argument"};
    *out = nullptr;
    *out = create_plan(*opts, *cfg, n_meas, n_pix, h, h_dtype, g, false);
  });
}

void admm_plan_destroy(admm_plan* plan) {
  if (plan) {
    cudaSetDevice(plan->device);
    if (plan->dtrace_tile.p && plan->slab_rpl) {  // diagnostics: raw slab-sweep timestamps -> file
      const size_t n = plan->gS.P * plan->slab_C * 64 * 8;
      std::vector<unsigned long long> t(n);
      cudaMemcpy(t.data(), plan->dtrace_tile.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      if (FILE* f = std::fopen(std::getenv("ADMM_B200_SLAB_TRACE"), "wb")) {
        std::fwrite(t.data(), sizeof(unsigned long long), n, f);
        std::fclose(f);
      }
    }
    delete plan;
  }
}

admm_status admm_plan_set_g(admm_plan* p, const double* g) {
  return run_guarded([&] {
    check_plan(p);
    if (!g) throw Fail{ADMM_E_STATE, "null g"};
    if (!host_all_finite(g, 2 * p->n_meas * std::max<uint64_t>(1, p->batch)))
      throw Fail{ADMM_E_NUMERICAL, "SensingProblem: non-finite entries"};
    for (admm_plan* s : shards_of(p)) {
      CK(cudaSetDevice(s->device));
      upload_g(s, g);
    }
  });
}

admm_status admm_plan_set_lambda(admm_plan* p, double lambda) {
  return run_guarded([&] {
    check_plan(p);
    if (!(lambda > 0.0)) throw Fail{ADMM_E_PARAMETER, "SolverConfig: lambda must be positive"};
    p->cfg.lambda = lambda;
    for (admm_plan* s : shards_of(p)) {
      CK(cudaSetDevice(s->device));
      s->cfg.lambda = lambda;
      set_params(s);
    }
  });
}

admm_status admm_plan_max_abs_adjoint(admm_plan* p, double* out) {
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p)) {
      *out = dist_max_abs_adjoint(p);
      return;
    }
    const int nb = (int)p->blocks.size();
    const uint32_t gx = p->zgx;
    DevBuf res;
    if (p->Pr * p->Pc != 1) throw Fail{ADMM_E_STATE, "max_abs_adjoint: single-GPU or distributed plans only"};
    res.alloc((size_t)gx * p->N * sizeof(double));
    if (p->dtype == ADMM_C128) {
      gemv_h_kernel<double2, kVH, kEvictNormal><<<(unsigned)p->gG.P, kCtaThreads, 0, p->stream>>>(
          p->dH.as<double2>(), p->dg.as<double2>(), p->dgpart.as<double2>(), p->dhHg.as<MatDesc>(), nb, p->gG.U);
      adjoint_absmax_kernel<chunk_h<double2>()><<<dim3(gx, (unsigned)p->N), kCtaThreads, 0, p->stream>>>(
          p->dgpart.as<double2>(), p->dhHg.as<MatDesc>(), p->dblocks.as<BlockDesc>(), (uint32_t)p->M,
          (uint32_t)p->N, p->gG.U, p->gG.P, res.as<double>());
    } else {
      gemv_h_kernel<float2, kVH, kEvictNormal><<<(unsigned)p->gG.P, kCtaThreads, 0, p->stream>>>(
          p->dH.as<float2>(), p->dg.as<double2>(), p->dgpart.as<double2>(), p->dhHg.as<MatDesc>(), nb, p->gG.U);
      adjoint_absmax_kernel<chunk_h<float2>()><<<dim3(gx, (unsigned)p->N), kCtaThreads, 0, p->stream>>>(
          p->dgpart.as<double2>(), p->dhHg.as<MatDesc>(), p->dblocks.as<BlockDesc>(), (uint32_t)p->M,
          (uint32_t)p->N, p->gG.U, p->gG.P, res.as<double>());
    }
    CK(cudaGetLastError());
    std::vector<double> h((size_t)gx * p->N);
    CK(cudaMemcpyAsync(h.data(), res.p, h.size() * 8, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    double m = 0.0;
    for (double x : h) m = std::max(m, x);
    *out = m;
  });
}

admm_status admm_plan_reset(admm_plan* p) {
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p))
      dist_reset(shards_of(p));
    else
      reset_state(p);
  });
}

admm_status admm_plan_enqueue(admm_plan* p, uint64_t iters) {
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p))
      dist_enqueue(p, iters);
    else
      enqueue_iters(p, iters);
  });
}

admm_status admm_plan_sync(admm_plan* p) {
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p))
      dist_sync(shards_of(p));
    else
      CK(cudaStreamSynchronize(p->stream));
  });
}

void* admm_plan_stream(admm_plan* p) {
  if (!p) return nullptr;
  return !p->subs.empty() ? (void*)p->subs[0]->stream : (void*)p->stream;
}

admm_status admm_plan_set_stream(admm_plan* p, void* stream) {
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p)) throw Fail{ADMM_E_STATE, "set_stream: a distributed plan launches on its own streams"};
    p->stream = stream ? static_cast<cudaStream_t>(stream) : p->own_stream;
  });
}

uint32_t admm_plan_kernel_count(const admm_plan* p) {
  return !p ? 7 : p->schedule == 4 ? 1 : p->schedule == 2 ? 4 : p->schedule == 5 ? 6 : 7;
}

admm_status admm_plan_set_lambdas(admm_plan* p, const double* lambdas) {
  return run_guarded([&] {
    check_plan(p);
    if (p->batch < 2) throw Fail{ADMM_E_STATE, "set_lambdas: not a batched plan"};
    if (!lambdas) throw Fail{ADMM_E_STATE, "null lambdas"};
    for (uint64_t b = 0; b < p->batch; ++b)
      if (!(lambdas[b] > 0.0)) throw Fail{ADMM_E_PARAMETER, "SolverConfig: lambda must be positive"};
    p->lambdas.assign(lambdas, lambdas + p->batch);
    set_params(p);
  });
}

admm_status admm_plan_max_abs_adjoint_batched(admm_plan* p, double* out) {
  return run_guarded([&] {
    check_plan(p);
    if (p->batch < 2) throw Fail{ADMM_E_STATE, "not a batched plan"};
    const uint32_t B = (uint32_t)p->batch;
    if (p->dtype == ADMM_C128)
      launch_bgemm<double2, true>(p, p->stream, p->tG.size(),
          p->dH.as<double2>(), p->dtG.as<BTile>(), p->dg.as<double2>(), p->dz.as<double2>(), B);
    else
      launch_bgemm<float2, true>(p, p->stream, p->tG.size(),
          p->dH.as<float2>(), p->dtG.as<BTile>(), p->dg.as<double2>(), p->dz.as<double2>(), B);
    const unsigned gx = p->pz;
    DevBuf res;
    res.alloc((size_t)gx * kBB * sizeof(double));
    babsmax_kernel<<<gx, kCtaThreads, 0, p->stream>>>(p->dz.as<double2>(), p->dblocks.as<BlockDesc>(),
                                                      (uint32_t)p->Mr, (uint32_t)p->Nc, B, res.as<double>());
    CK(cudaGetLastError());
    std::vector<double> h((size_t)gx * kBB);
    CK(cudaMemcpyAsync(h.data(), res.p, h.size() * 8, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    for (uint32_t b = 0; b < B; ++b) {
      double m = 0.0;
      for (unsigned c = 0; c < gx; ++c) m = std::max(m, h[(size_t)c * kBB + b]);
      out[b] = m;
    }
  });
}

admm_status admm_plan_profile(admm_plan* p, uint64_t iters, const char** names, double* ms) {
  static const char* kNames2[7] = {"gemv_n(H,c)", "rows_finalize(rhs)", "gemv_n(K,r)", "rows_finalize(q)",
                                   "gemv_h(H,q)", "zupdate", "finalize"};
  static const char* kNamesS[4] = {"sweep(H)", "rows_finalize(rhs)+finalize", "gemv_n(K,r)", "rows_finalize(q)"};
  static const char* kNames2P[7] = {"gemv_n(H,c)", "rows_finalize(rhs)", "hemv(Kpacked,r)", "hemv_finalize(q)",
                                    "gemv_h(H,q)", "zupdate", "finalize"};
  static const char* kNamesSP[4] = {"sweep(H)", "rows_finalize(rhs)+finalize", "hemv(Kpacked,r)",
                                    "hemv_finalize(q)"};
  static const char* kNamesB[7] = {"bgemm(H,C)", "brows(rhs)", "bgemm(K,R)", "brows(q)", "bgemm_adj(H,Q)",
                                   "bzupdate", "bfinalize"};
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p)) throw Fail{ADMM_E_STATE, "profile: single-GPU plans only"};
    const int nk = (int)admm_plan_kernel_count(p);
    static const char* kNamesR[1] = {"resident(iteration)"};
    static const char* kNamesU[6] = {"gemv_h(H,q)", "zupdate+support_list", "support_a(Hc,v)",
                                     "support_rows+finalize", "hemv(Kpacked,r)", "hemv_finalize(q)"};
    const char* const* kn = p->schedule == 5   ? kNamesU
                            : p->schedule == 4 ? kNamesR
                            : p->schedule == 2 ? (p->kpacked ? kNamesSP : kNamesS)
                            : p->schedule == 3 ? kNamesB
                                               : (p->kpacked ? kNames2P : kNames2);
    std::vector<cudaEvent_t> ev(nk + 1);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    std::vector<double> acc(nk, 0.0);
    for (uint64_t k = 0; k < iters; ++k) {
      enqueue_iteration_any(p, p->stream, false, &ev);
      CK(cudaEventSynchronize(ev[nk]));
      for (int q = 0; q < nk; ++q) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, ev[q], ev[q + 1]));
        acc[q] += t;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    for (int q = 0; q < nk; ++q) {
      if (names) names[q] = kn[q];
      if (ms) ms[q] = acc[q] / (double)std::max<uint64_t>(iters, 1);
    }
  });
}

admm_status admm_plan_get_info(const admm_plan* p, admm_plan_info* info) {
  return run_guarded([&] {
    if (!p || !info) throw Fail{ADMM_E_STATE, "null argument"};
    if (!p->subs.empty()) {  // single-process multi-GPU plan: its first shard, whole-job fields
      admm_status st = admm_plan_get_info(p->subs[0], info);
      if (st != ADMM_OK) throw Fail{st, g_last_error};
      info->setup_seconds = p->setup_s;
      return;
    }
    admm_plan_info r{};
    r.n_blocks = p->blocks.size();
    uint64_t hb = 0, kb = 0, vb = 0;
    for (const auto& b : p->blocks) {
      hb += (uint64_t)b.rows * b.cols * p->elem;
      kb += (uint64_t)b.rows * b.rows * p->elem;
      vb += (uint64_t)b.cols * 16 * 6 + (uint64_t)b.rows * 16 * 8;
    }
    const uint64_t kb_dense = kb;
    if (p->kpacked) {  // the packed Hermitian tiles actually streamed per iteration
      kb = 0;
      for (const auto& h : p->hv) kb += (uint64_t)h.n_units * kHT * kHT * p->elem;
    }
    r.h_bytes = hb;
    r.k_bytes = kb;
    r.h_stream_bytes_per_iter = 2 * hb;
    r.bytes_per_iter = 2 * hb + kb_dense + vb;  // two-pass algorithmic bytes
    // resident: ONE launch runs all the iterations of an enqueue (reported as 0 per iteration)
    r.launches_per_iter = p->schedule == 5 ? 8 : p->schedule == 4 ? 0 : p->schedule == 3 ? 7 : p->schedule == 2 ? (p->trace_obj ? (p->obj_pass ? 7 : 6) : 4) : (p->trace_obj ? 9 : 7);
    r.schedule = (uint64_t)p->schedule;
    r.grid_sweep = p->gS.P;
    // support schedule: one dense pass + K (+ the data-dependent support columns, admm_plan_read 5)
    r.hbm_bytes_per_iter = p->schedule == 5 ? hb + kb + vb : (p->schedule == 4 ? 0 : p->schedule == 2 ? hb : 2 * hb) + kb + vb;
    r.sweep_variant = p->schedule != 2 ? 0 : p->slab_rpl ? 3 : 1;
    r.slab_cluster = p->slab_rpl ? p->slab_C : 0;
    r.slab_row_bytes = p->slab_rpl ? p->slab_rb : 0;
    r.slab_rows = p->slab_rpl ? (uint64_t)p->slab_rpl * kWarp : 0;
    r.grid_gemv_n = p->gN.P;
    r.grid_gemv_h = p->gH.P;
    r.setup_seconds = p->setup_s;
    r.inner_dim_max = p->max_m;
    for (int k = 0; k < 4; ++k) r.setup_phase_s[k] = p->setup_phase[k];
    r.gram_device_s = p->gram_device_s;
    r.gram_flops = p->gram_flops;
    r.inverse_device_s = p->inverse_device_s;
    r.inverse_flops = p->inverse_flops;
    r.grid_pr = p->Pr;
    r.grid_pc = p->Pc;
    r.n_ranks = p->Pr * p->Pc;
    // bytes this rank RECEIVES per iteration over NCCL (all-gathers: the peers' slots)
    r.exchange_bytes_per_iter = (p->Pc - 1) * p->gslot * 16 +
                                (p->schedule == 2 ? 0 : (p->Pr - 1) * p->Mr * p->Nc * p->npad * 16) +
                                (p->fused_scal ? 0 : (p->Pr * p->Pc - 1) * kScalDoubles * 8);
    *info = r;
  });
}

admm_status admm_plan_read(admm_plan* p, int which, double* dst, uint64_t count) {
  return run_guarded([&] {
    check_plan(p);
    if (!dst) throw Fail{ADMM_E_STATE, "null destination"};
    if (is_dist(p)) {  // whole-problem iterates, identical on every rank
      const auto sh = shards_of(p);
      if (which == 0 || which == 1) {
        if (count < p->n_pix) throw Fail{ADMM_E_DIMENSION, "destination too small"};
        dist_gather_segments(sh, which, dst);
        return;
      }
      if (which == 2) {
        std::vector<double> u;
        std::vector<uint64_t> off, len;
        dist_gather_u(sh, u, off, len);
        if (count < u.size() / 2) throw Fail{ADMM_E_DIMENSION, "destination too small"};
        std::memcpy(dst, u.data(), u.size() * 8);
        return;
      }
      p = sh[0];
      CK(cudaSetDevice(p->device));
    }
    if (which == 0 || which == 1) {
      if (count < p->n_pix * p->batch) throw Fail{ADMM_E_DIMENSION, "destination too small"};
      read_segments(p, which == 0 ? p->dv : p->dvprev, dst);
    } else if (which == 2) {
      uint64_t tot = 0;
      for (auto& b : p->blocks) tot += b.cols;
      if (count < tot) throw Fail{ADMM_E_DIMENSION, "destination too small"};
      std::vector<double> tmp(p->vec_total * 2);
      CK(cudaMemcpyAsync(tmp.data(), p->du.p, p->vec_total * 16, cudaMemcpyDeviceToHost, p->stream));
      CK(cudaStreamSynchronize(p->stream));
      uint64_t o = 0;
      for (auto& b : p->blocks) {
        std::memcpy(dst + 2 * o, tmp.data() + 2 * (uint64_t)b.vec_off, (size_t)b.cols * 16);
        o += b.cols;
      }
    } else if (which == 3) {  // trace of the iterations completed since reset (3 per row)
      const IterState st = read_state(p);
      const uint64_t n = std::min<uint64_t>(st.iter, p->trace_cap);
      if (count < 3 * n) throw Fail{ADMM_E_DIMENSION, "destination too small"};
      CK(cudaMemcpyAsync(dst, p->dtrace.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
      CK(cudaStreamSynchronize(p->stream));
    } else if (which == 9) {  // diagnostics: the resident kernel's clock64 trace (ADMM_B200_RES_TRACE)
      if (p->dres_dbg.p) {
        CK(cudaMemcpyAsync(dst, p->dres_dbg.p, std::min<uint64_t>(count * 8, p->dres_dbg.bytes),
                           cudaMemcpyDeviceToHost, p->stream));
        CK(cudaStreamSynchronize(p->stream));
      }
    } else if (which == 5) {  // support schedule: {iterations completed, support columns summed over them}
      if (count < 2) throw Fail{ADMM_E_DIMENSION, "destination too small"};
      const IterState st = read_state(p);
      unsigned long long tot = 0;
      if (p->dnnz_tot.p) CK(cudaMemcpy(&tot, p->dnnz_tot.p, sizeof(tot), cudaMemcpyDeviceToHost));
      dst[0] = (double)st.iter;
      dst[1] = (double)tot;
    } else if (which == 4) {  // {iterations completed, first non-finite iteration or -1}
      if (count < 2) throw Fail{ADMM_E_DIMENSION, "destination too small"};
      const IterState st = read_state(p);
      dst[0] = (double)st.iter;
      dst[1] = st.first_bad == ~0ull ? -1.0 : (double)st.first_bad;
    } else {
      throw Fail{ADMM_E_PARAMETER, "unknown iterate"};
    }
  });
}

admm_status admm_plan_solve(admm_plan* p, double* solution, double* trace, uint64_t* iterations_run,
                            double* objective, admm_observer_fn observer, void* user) {
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p)) {
      dist_solve(p, solution, trace, iterations_run, objective, observer, user);
      return;
    }
    const uint64_t iters = p->cfg.max_iters;
    ensure_trace(p, iters);
    reset_state(p);
    const bool stepping = observer || p->cfg.eps_pri != 0.0 || p->cfg.eps_dual != 0.0;
    if (p->batch > 1 && observer) throw Fail{ADMM_E_PARAMETER, "batched scenes: no observer"};
    uint64_t done = 0;
    if (!stepping) {
      enqueue_iters(p, iters);
      const IterState st = read_state(p);
      if (st.first_bad != ~0ull)
        throw Fail{ADMM_E_NUMERICAL,
                   "non-finite iterate at iteration " + std::to_string(st.first_bad + 1), st.first_bad};
      done = st.iter;
    } else {
      // per-iteration path: stop_now (admm_core.hpp:52-57) and the observer
      // (solvers.hpp:150-160) need the host after every iteration.
      uint64_t total_u = 0;
      for (auto& b : p->blocks) total_u += b.cols;
      std::vector<const double*> uptr(p->blocks.size());
      std::vector<uint64_t> ulen(p->blocks.size());
      for (uint64_t k = 0; k < iters; ++k) {
        enqueue_iteration_any(p, p->stream, p->trace_obj, nullptr);
        const IterState st = read_state(p);
        if (st.first_bad != ~0ull)
          throw Fail{ADMM_E_NUMERICAL, "non-finite iterate at iteration " + std::to_string(st.first_bad + 1),
                     st.first_bad};
        double tr[3];
        CK(cudaMemcpyAsync(tr, p->dtrace.as<double>() + 3 * k, sizeof(tr), cudaMemcpyDeviceToHost, p->stream));
        CK(cudaStreamSynchronize(p->stream));
        done = k + 1;
        if (observer) {
          p->h_v.resize(2 * p->n_pix);
          p->h_vprev.resize(2 * p->n_pix);
          p->h_u.resize(2 * total_u);
          read_segments(p, p->dv, p->h_v.data());
          read_segments(p, p->dvprev, p->h_vprev.data());
          std::vector<double> tmp(p->vec_total * 2);
          CK(cudaMemcpyAsync(tmp.data(), p->du.p, p->vec_total * 16, cudaMemcpyDeviceToHost, p->stream));
          CK(cudaStreamSynchronize(p->stream));
          uint64_t o = 0;
          for (size_t b = 0; b < p->blocks.size(); ++b) {
            std::memcpy(p->h_u.data() + 2 * o, tmp.data() + 2 * (uint64_t)p->blocks[b].vec_off,
                        (size_t)p->blocks[b].cols * 16);
            uptr[b] = p->h_u.data() + 2 * o;
            ulen[b] = p->blocks[b].cols;
            o += p->blocks[b].cols;
          }
          admm_snapshot snap{};
          snap.iteration = k + 1;
          snap.n_pix = p->n_pix;
          snap.v = p->h_v.data();
          snap.v_prev = p->h_vprev.data();
          snap.n_workers = p->blocks.size();
          snap.replica_u = uptr.data();
          snap.replica_len = ulen.data();
          snap.primal = tr[0];
          snap.dual = tr[1];
          if (observer(&snap, user) != 0) throw Fail{ADMM_E_OBSERVER, "observer stopped the solve"};
        }
        // stop_now: both thresholds 0 never stops; otherwise every enabled one must hold
        const double e1 = p->cfg.eps_pri, e2 = p->cfg.eps_dual;
        if (e1 != 0.0 || e2 != 0.0) {
          const bool pri = e1 == 0.0 || tr[0] <= e1;
          const bool dua = e2 == 0.0 || tr[1] <= e2;
          if (pri && dua) break;
        }
      }
    }
    if (iterations_run) *iterations_run = done;
    double obj = 0.0;
    if (p->batch > 1) {  // per-scene objectives live in the trace; SolveReport.objective is a scalar
      obj = std::numeric_limits<double>::quiet_NaN();
      if (objective) *objective = obj;
      if (trace && p->trace_obj && done > 0) {
        if (p->dtype == ADMM_C128)
          enqueue_bobjective_last<double2>(p, p->stream);
        else
          enqueue_bobjective_last<float2>(p, p->stream);
      }
      if (trace) {
        CK(cudaMemcpyAsync(trace, p->dtrace.p, done * 3 * p->batch * sizeof(double), cudaMemcpyDeviceToHost,
                           p->stream));
        CK(cudaStreamSynchronize(p->stream));
      }
      if (solution) read_segments(p, p->dv, solution);
      return;
    }
    if (p->trace_obj && p->obj_pass) {  // the last iteration's pass already is the final objective
      CK(cudaMemcpyAsync(&obj, p->dtrace.as<double>() + 3 * (done - 1) + 2, 8, cudaMemcpyDeviceToHost, p->stream));
      CK(cudaStreamSynchronize(p->stream));
    } else {  // one exact pass over H for SolveReport::objective (solvers.hpp:163)
      if (p->dtype == ADMM_C128)
        enqueue_objective<double2>(p, p->stream);
      else
        enqueue_objective<float2>(p, p->stream);
      CK(cudaMemcpyAsync(&obj, p->dobj.p, 8, cudaMemcpyDeviceToHost, p->stream));
      CK(cudaStreamSynchronize(p->stream));
    }
    if (objective) *objective = obj;
    if (trace) {
      CK(cudaMemcpyAsync(trace, p->dtrace.p, done * 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
      CK(cudaStreamSynchronize(p->stream));
      // the recurrence fills entry k-1 during iteration k (two-pass) / k (sweep): the last
      // entry is the exact pass either way
      trace[3 * (done - 1) + 2] = obj;
    }
    if (solution) read_segments(p, p->dv, solution);
  });
}

}  // extern "C"

// ---- multi-GPU phases (admm_b200.h) --------------------------------------------
namespace {

// doubles between consecutive ranks' scalar slots
uint64_t scal_stride(const admm_plan* p) { return p->fused_scal ? 2 * p->gslot : kScalDoubles; }

// Objective of a sharded iteration: a_b of the local blocks into the A
// region of the ghat slot; the sweep schedule closes iteration k's objective in iteration
// k (its next w is this iteration's), the two-pass schedule closes iteration k-1's.
void enqueue_arec(admm_plan* p, cudaStream_t s) {
  if (!p->shard_obj) return;
  objective_arec_kernel<<<dim3(p->rgx, (unsigned)p->blocks.size()), kCtaThreads, 0, s>>>(
      row_vecs(p), p->dhs.as<double2>(), p->dblocks.as<BlockDesc>(), p->aoff, p->dstate.as<IterState>(),
      p->schedule == 2 ? 0 : 1);
}
// Rows partials |sum_q a_iq - g_i|^2 of the local row blocks from the gathered A regions.
// count: whether this rank's rows enter the sum (two-pass / final pass: one rank per row
// communicator; sweep: every rank holds all rows and keeps the sum to itself).
void enqueue_grows(admm_plan* p, cudaStream_t s, bool count, uint64_t min_iter) {
  objective_grows_kernel<<<dim3(p->objgx, (unsigned)p->Mr), kCtaThreads, 0, s>>>(
      p->dg.as<double2>(), p->ghat_ptr, p->aoff, p->dgblocks.as<BlockDesc>(), (uint32_t)p->N, (uint32_t)p->i0,
      count ? 1 : 0, p->dstate.as<IterState>(), min_iter, p->dobjp.as<double>());
}

template <typename S>
void enqueue_phase(admm_plan* p, int phase) {
  cudaStream_t s = p->stream;
  const int nb = (int)p->blocks.size();
  if (phase == 1) {
    if (p->schedule == 2) {
      launch_sweep<S>(p, s);
      rows_finalize_sweep_kernel<<<dim3(p->rgx_s, nb), kCtaThreads, 0, s>>>(
          row_vecs(p), p->dwpart_s.as<double2>(), p->dsegs.as<SweepDesc>(), p->dblocks.as<BlockDesc>(),
          p->dgblocks.as<BlockDesc>(), (uint32_t)p->N, (uint32_t)p->n_meas, p->gS.U, p->gS.P, 0, 2,
          p->dred.as<double>(), p->dparams.as<Params>(), p->dtrace.as<double>(), p->trace_cap,
          p->dstate.as<IterState>(), p->scal_ptr + scal_stride(p) * (p->pr * p->Pc + p->pc));
    } else if (p->schedule == 5) {
      // support schedule (admm_sparse.cuh) on a consensus shard: w = H c from the support of the v
      // every rank formed in phase 3 (v = 0 after a reset: empty support, w = 0, r = g)
      support_compact_kernel<<<dim3(p->zgx, (unsigned)p->Nc), kCtaThreads, 0, s>>>(
          p->dv.as<double2>(), p->dblocks.as<BlockDesc>(), p->dnzcnt.as<uint32_t>(), p->zgx, p->dnzlist.as<uint32_t>(),
          p->nzstride, p->dnnz.as<uint32_t>(), p->dnnz_tot.as<unsigned long long>());
      support_a_kernel<S><<<dim3(p->supgx, (unsigned)nb, p->sup_chunks), kSupThreads, 0, s>>>(
          p->dHc.as<S>(), p->dhcoff.as<uint64_t>(), p->dhcld.as<uint32_t>(), p->dblocks.as<BlockDesc>(),
          p->dv.as<double2>(), p->dnzlist.as<uint32_t>(), p->nzstride, p->dnnz.as<uint32_t>(), p->danew.as<double2>(),
          p->mvec_total);
      enqueue_support_rows(p, s, false);
    } else {
      gemv_n_kernel<S, kVN, kEvictNormal><<<(unsigned)p->gN.P, kCtaThreads, 0, s>>>(
          p->dH.as<S>(), p->dc.as<double2>(), p->dwpart.as<double2>(), p->dhN.as<MatDesc>(), nb, p->gN.U);
      rows_finalize_kernel<kRhs><<<dim3(p->rgx, nb), kCtaThreads, 0, s>>>(
          row_vecs(p), p->dwpart.as<double2>(), p->dhN.as<MatDesc>(), p->dblocks.as<BlockDesc>(),
          p->dgblocks.as<BlockDesc>(), (uint32_t)p->N, p->gN.U, p->gN.P, p->dparams.as<Params>());
    }
    enqueue_arec(p, s);  // reads this block's ghat before the K apply replaces it
    enqueue_kapply<S>(p, s);
  } else if (phase == 2) {
    if (p->schedule == 2) throw Fail{ADMM_E_STATE, "phase 2 belongs to the two-pass schedule"};
    gemv_h_kernel<S, kVH, kEvictNormal><<<(unsigned)p->gH.P, kCtaThreads, 0, s>>>(
        p->dH.as<S>(), p->dq.as<double2>(), p->dzpart.as<double2>(), p->dhH.as<MatDesc>(), nb, p->gH.U);
    uupdate_kernel<chunk_h<S>()><<<dim3(p->zgx, nb), kCtaThreads, 0, s>>>(
        col_vecs(p), p->outbox_ptr, p->dzpart.as<double2>(), p->dhH.as<MatDesc>(), p->dblocks.as<BlockDesc>(),
        p->gH.U, p->gH.P, p->dstate.as<IterState>());
  } else if (phase == 3) {
    if (p->schedule == 2) {  // sweep: the iteration's objective rows (all rows are local after the gather)
      if (p->shard_obj) enqueue_grows(p, s, true, 0);
    } else {
      zfinal_kernel<<<dim3(p->zgx, (unsigned)p->Nc), kCtaThreads, 0, s>>>(
          col_vecs(p), p->outbox_ptr, p->dblocks.as<BlockDesc>(), (uint32_t)p->M, (uint32_t)p->Mr,
          (uint32_t)p->Nc, (uint32_t)p->npad, p->pr == 0 ? 1 : 0, p->dparams.as<Params>(), p->dred.as<double>(),
          p->schedule == 5 ? p->dnzcnt.as<uint32_t>() : nullptr);
      if (p->shard_obj) enqueue_grows(p, s, p->pc == 0, 1);  // iteration k-1's rows, one rank per row block
      local_scalars_kernel<<<1, kCtaThreads, 0, s>>>(
          p->dred.as<double>(), p->nz, p->shard_obj ? p->dobjp.as<double>() : nullptr, p->objgx * (uint32_t)p->Mr,
          p->scal_ptr + scal_stride(p) * (p->pr * p->Pc + p->pc), p->dstate.as<IterState>());
    }
  } else if (phase == 4) {
    const int mode = !p->shard_obj ? 0 : p->schedule == 2 ? 2 : 1;
    close_kernel<<<1, kCtaThreads, 0, s>>>(p->scal_ptr, (uint32_t)(p->Pr * p->Pc), scal_stride(p),
                                           p->dparams.as<Params>(), p->dtrace.as<double>(), p->trace_cap,
                                           p->dstate.as<IterState>(), mode, p->dobjp.as<double>(),
                                           p->objgx * (uint32_t)p->Mr, p->dl1prev.as<double>());
  } else {
    throw Fail{ADMM_E_PARAMETER, "unknown phase"};
  }
  CK(cudaGetLastError());
}

}  // namespace

extern "C" {

admm_status admm_plan_create_sharded(const admm_plan_options* opts, const admm_solver_config* cfg, uint64_t n_meas,
                                     uint64_t n_pix, const void* h, admm_dtype h_dtype, const double* g,
                                     const admm_shard* shard, admm_plan** out) {
  return run_guarded([&] {
    if (!opts || !cfg || !out || !shard) throw Fail{ADMM_E_STATE, "null argument"};
    *out = nullptr;
    *out = create_plan(*opts, *cfg, n_meas, n_pix, h, h_dtype, g, false, shard);
  });
}

admm_status admm_plan_exchange_info(const admm_plan* p, int which, uint64_t* total, uint64_t* off, uint64_t* bytes) {
  return run_guarded([&] {
    if (!p) throw Fail{ADMM_E_STATE, "null plan"};
    uint64_t t = 0, o = 0, b = 0;
    if (which == ADMM_X_GHAT) {  // [pc][Mr][Nc][mpad] (+ 4 scalar doubles when fused)
      b = p->gslot * 16;
      t = p->Pc * b;
      o = p->pc * b;
    } else if (which == ADMM_X_OUTBOX) {  // [i = pr*Mr + il][Nc][npad]
      b = p->Mr * p->Nc * p->npad * 16;
      t = p->Pr * b;
      o = p->pr * b;
    } else if (which == ADMM_X_SCAL) {  // [rank][4]; 0 bytes: fused into the ghat exchange
      b = p->fused_scal ? 0 : kScalDoubles * sizeof(double);
      t = p->Pr * p->Pc * b;
      o = (p->pr * p->Pc + p->pc) * b;
    } else {
      throw Fail{ADMM_E_PARAMETER, "unknown exchange buffer"};
    }
    if (total) *total = t;
    if (off) *off = o;
    if (bytes) *bytes = b;
  });
}

admm_status admm_plan_attach(admm_plan* p, int which, void* ptr) {
  return run_guarded([&] {
    check_plan(p);
    if (is_dist(p)) throw Fail{ADMM_E_STATE, "attach: a distributed plan owns its exchange buffers"};
    if (!ptr) throw Fail{ADMM_E_STATE, "null device pointer"};
    if (which == ADMM_X_GHAT) {
      p->ghat_ptr = static_cast<double2*>(ptr);
      if (p->fused_scal) p->scal_ptr = reinterpret_cast<double*>(p->ghat_ptr + p->Mr * p->Nc * p->mpad + p->aoff);
    } else if (which == ADMM_X_OUTBOX) {
      p->outbox_ptr = static_cast<double2*>(ptr);
    } else if (which == ADMM_X_SCAL) {
      if (!p->fused_scal) p->scal_ptr = static_cast<double*>(ptr);
    } else {
      throw Fail{ADMM_E_PARAMETER, "unknown exchange buffer"};
    }
    if (p->exec) {  // captured graphs hold the old pointers
      cudaGraphExecDestroy(p->exec);
      p->exec = nullptr;
    }
  });
}

admm_status admm_plan_run_phase(admm_plan* p, int phase) {
  return run_guarded([&] {
    check_plan(p);
    if (p->dtype == ADMM_C128)
      enqueue_phase<double2>(p, phase);
    else
      enqueue_phase<float2>(p, phase);
  });
}

admm_status admm_plan_schedule(const admm_plan* p, int* schedule) {
  return run_guarded([&] {
    if (!p || !schedule) throw Fail{ADMM_E_STATE, "null argument"};
    *schedule = p->schedule == 2 ? 1 : 2;
  });
}

}  // extern "C"

// ---- L0/L1 operations -------------------------------------------------------

namespace {

__global__ void soft_threshold_kernel(const double2* __restrict__ a, uint64_t n, double kappa,
                                      double2* __restrict__ out) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    out[t] = soft_threshold(a[t], kappa);
}

__global__ void rows_sum_kernel(const double2* __restrict__ part, const MatDesc* __restrict__ mats,
                                uint64_t U, uint64_t P, double2* __restrict__ y) {
  const MatDesc md = mats[0];
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < md.rows) y[row] = sum_rows_part(part, md, row, U, P);
}

template <int CH>
__global__ void cols_sum_kernel(const double2* __restrict__ part, const MatDesc* __restrict__ mats,
                                uint64_t U, uint64_t P, double2* __restrict__ y) {
  const MatDesc md = mats[0];
  const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col < md.cols) y[col] = sum_cols_part<CH>(part, md, col, U, P);
}

admm_plan_options single_block(int device) {
  admm_plan_options o{};
  o.method = ADMM_REFERENCE;
  o.M = o.N = 1;
  o.dtype = ADMM_C128;
  o.device = device;
  return o;
}

}  // namespace

extern "C" {

admm_status admm_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x, double* y, int device) {
  return run_guarded([&] {
    if (!a || !x || !y) throw Fail{ADMM_E_STATE, "null argument"};
    admm_solver_config cfg{1.0, 1.0, 1.0, 1, 0.0, 0.0, 0};
    std::vector<double> g(2 * rows, 0.0);
    std::unique_ptr<admm_plan> p(create_plan(single_block(device), cfg, rows, cols, a, ADMM_C128, g.data(), true));
    std::vector<double> xs(2 * round_up(cols, 4), 0.0);
    std::memcpy(xs.data(), x, cols * 16);
    CK(cudaMemcpyAsync(p->dc.p, xs.data(), cols * 16, cudaMemcpyHostToDevice, p->stream));
    gemv_n_kernel<double2, kVN, kEvictNormal><<<(unsigned)p->gN.P, kCtaThreads, 0, p->stream>>>(
        p->dH.as<double2>(), p->dc.as<double2>(), p->dwpart.as<double2>(), p->dhN.as<MatDesc>(), 1, p->gN.U);
    rows_sum_kernel<<<(unsigned)cdiv(rows, 256), 256, 0, p->stream>>>(p->dwpart.as<double2>(), p->dhN.as<MatDesc>(),
                                                                     p->gN.U, p->gN.P, p->dr.as<double2>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(y, p->dr.p, rows * 16, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  });
}

admm_status admm_adjoint_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x, double* y,
                                int device) {
  return run_guarded([&] {
    if (!a || !x || !y) throw Fail{ADMM_E_STATE, "null argument"};
    admm_solver_config cfg{1.0, 1.0, 1.0, 1, 0.0, 0.0, 0};
    std::vector<double> g(2 * rows, 0.0);
    std::unique_ptr<admm_plan> p(create_plan(single_block(device), cfg, rows, cols, a, ADMM_C128, g.data(), true));
    CK(cudaMemcpyAsync(p->dq.p, x, rows * 16, cudaMemcpyHostToDevice, p->stream));
    gemv_h_kernel<double2, kVH, kEvictNormal><<<(unsigned)p->gH.P, kCtaThreads, 0, p->stream>>>(
        p->dH.as<double2>(), p->dq.as<double2>(), p->dzpart.as<double2>(), p->dhH.as<MatDesc>(), 1, p->gH.U);
    cols_sum_kernel<chunk_h<double2>()><<<(unsigned)cdiv(cols, 256), 256, 0, p->stream>>>(
        p->dzpart.as<double2>(), p->dhH.as<MatDesc>(), p->gH.U, p->gH.P, p->du.as<double2>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(y, p->du.p, cols * 16, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  });
}

admm_status admm_soft_threshold(const double* a, uint64_t n, double kappa, double* out, int device) {
  return run_guarded([&] {
    if (!a || !out) throw Fail{ADMM_E_STATE, "null argument"};
    if (n == 0) return;
    CK(cudaSetDevice(device));
    DevBuf da, db;
    da.alloc(n * 16);
    db.alloc(n * 16);
    CK(cudaMemcpy(da.p, a, n * 16, cudaMemcpyHostToDevice));
    soft_threshold_kernel<<<(unsigned)std::min<uint64_t>(cdiv(n, 256), 4096), 256>>>(da.as<double2>(), n, kappa,
                                                                                    db.as<double2>());
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, db.p, n * 16, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

// GramSolver object (admm_b200.h admm_gram_*): a single-block plan factored once.
//   Woodbury: the plan of H, K = (rho I + H H^H)^-1; solve = one u-update with g = 0:
//             x = c - H^H K H c, c = rhs / rho (gram.hpp:71-77 through the inversion lemma).
//   Direct:   the plan of H^H, whose K = (rho I + H^H H)^-1 is the cols x cols inverse;
//             solve = x = K rhs (dense GEMV of the stored inverse, gram.hpp:68-70).
struct admm_gram {
  std::unique_ptr<admm_plan> plan;
  int strategy = 1;
  uint64_t rows = 0, cols = 0;
  double rho = 1.0;
  std::mutex mu;
};

extern "C" {

admm_status admm_gram_create(const double* h, uint64_t rows, uint64_t cols, double rho, int strategy, int device,
                             admm_gram** out) {
  return run_guarded([&] {
    if (!out) throw Fail{ADMM_E_STATE, "null argument"};
    *out = nullptr;
    if (!h || rows == 0 || cols == 0) throw Fail{ADMM_E_PARAMETER, "GramSolver: empty block"};
    if (!(rho > 0.0)) throw Fail{ADMM_E_PARAMETER, "GramSolver: rho must be positive"};
    if (!host_all_finite(h, 2 * rows * cols)) throw Fail{ADMM_E_NUMERICAL, "GramSolver: non-finite entries in block"};
    auto g = std::make_unique<admm_gram>();
    g->strategy = strategy < 0 ? (rows < cols ? 1 : 0) : (strategy ? 1 : 0);
    g->rows = rows;
    g->cols = cols;
    g->rho = rho;
    admm_solver_config cfg{rho, 1.0, 1.0, 1, 0.0, 0.0, 0};
    if (g->strategy == 1) {
      std::vector<double> z(2 * rows, 0.0);
      g->plan.reset(create_plan(single_block(device), cfg, rows, cols, h, ADMM_C128, z.data(), true));
    } else {  // the plan of H^H (cols x rows): its K is (rho I + H^H H)^-1
      std::vector<double> ht(2 * rows * cols), z(2 * cols, 0.0);
      for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t c = 0; c < cols; ++c) {
          ht[2 * (c * rows + r)] = h[2 * (r * cols + c)];
          ht[2 * (c * rows + r) + 1] = -h[2 * (r * cols + c) + 1];
        }
      admm_plan_options o = single_block(device);
      g->plan.reset(create_plan(o, cfg, cols, rows, ht.data(), ADMM_C128, z.data(), true));
    }
    *out = g.release();
  });
}

admm_status admm_gram_apply(admm_gram* g, const double* rhs, double* x) {
  return run_guarded([&] {
    if (!g || !rhs || !x) throw Fail{ADMM_E_STATE, "null argument"};
    std::lock_guard<std::mutex> lock(g->mu);
    admm_plan* p = g->plan.get();
    CK(cudaSetDevice(p->device));
    if (g->strategy == 1) {
      std::vector<double> c(2 * g->cols);
      for (uint64_t t = 0; t < 2 * g->cols; ++t) c[t] = rhs[t] / g->rho;
      CK(cudaMemcpyAsync(p->dc.p, c.data(), g->cols * 16, cudaMemcpyHostToDevice, p->stream));
      enqueue_iteration_twopass<double2>(p, p->stream, false, nullptr);
      CK(cudaMemcpyAsync(x, p->du.p, g->cols * 16, cudaMemcpyDeviceToHost, p->stream));
    } else {
      CK(cudaMemcpyAsync(p->dr.p, rhs, g->cols * 16, cudaMemcpyHostToDevice, p->stream));
      gemv_n_kernel<double2, kVN, kEvictNormal><<<(unsigned)p->gK.P, kCtaThreads, 0, p->stream>>>(
          p->dK.as<double2>(), p->dr.as<double2>(), p->dqpart.as<double2>(), p->dkN.as<MatDesc>(), 1, p->gK.U);
      rows_sum_kernel<<<(unsigned)cdiv(g->cols, 256), 256, 0, p->stream>>>(p->dqpart.as<double2>(),
                                                                           p->dkN.as<MatDesc>(), p->gK.U, p->gK.P,
                                                                           p->dq.as<double2>());
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(x, p->dq.p, g->cols * 16, cudaMemcpyDeviceToHost, p->stream));
    }
    CK(cudaStreamSynchronize(p->stream));
  });
}

admm_status admm_gram_info(const admm_gram* g, int* strategy, uint64_t* inner_dim) {
  return run_guarded([&] {
    if (!g) throw Fail{ADMM_E_STATE, "null argument"};
    if (strategy) *strategy = g->strategy;
    if (inner_dim) *inner_dim = g->strategy == 1 ? g->rows : g->cols;
  });
}

void admm_gram_destroy(admm_gram* g) {
  if (g) {
    cudaSetDevice(g->plan->device);
    delete g;
  }
}

admm_status admm_gram_solve(const double* h, uint64_t rows, uint64_t cols, double rho, const double* rhs,
                            double* x, int device) {
  return run_guarded([&] {
    if (!h || !rhs || !x) throw Fail{ADMM_E_STATE, "null argument"};
    if (rows == 0 || cols == 0) throw Fail{ADMM_E_PARAMETER, "GramSolver: empty block"};
    if (!(rho > 0.0)) throw Fail{ADMM_E_PARAMETER, "GramSolver: rho must be positive"};
    if (!host_all_finite(h, 2 * rows * cols)) throw Fail{ADMM_E_NUMERICAL, "GramSolver: non-finite entries in block"};
    // (H^H H + rho I)^-1 rhs = c - H^H K H c with c = rhs/rho, K = (rho I + H H^H)^-1:
    // one u-update of the engine with g = 0 (gram.hpp:71-77, inversion lemma).
    admm_solver_config cfg{rho, 1.0, 1.0, 1, 0.0, 0.0, 0};
    std::vector<double> g(2 * rows, 0.0);
    std::unique_ptr<admm_plan> p(create_plan(single_block(device), cfg, rows, cols, h, ADMM_C128, g.data(), true));
    std::vector<double> c(2 * cols);
    for (uint64_t t = 0; t < 2 * cols; ++t) c[t] = rhs[t] / rho;
    CK(cudaMemcpyAsync(p->dc.p, c.data(), cols * 16, cudaMemcpyHostToDevice, p->stream));
    enqueue_iteration_twopass<double2>(p.get(), p->stream, false, nullptr);
    CK(cudaMemcpyAsync(x, p->du.p, cols * 16, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  });
}

}  // extern "C"

// ---- multi-GPU plans with plan-owned NCCL communicators ---------------------------
#include "admm_dist.inc"
