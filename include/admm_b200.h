/* include/admm_b200.h — C ABI of the B200-native ADMM hot path (libadmm_b200.so).
 *
 * Drop-in boundary for the reference library admmsplit (header-only C++20 at
 * /root/reference/proj/include/admmsplit).  Every entry point below names the
 * reference interface it replaces (file:line, relative to that directory).  The
 * C++ shim include/admmgpu/admmgpu.hpp re-exposes these with the reference's own
 * signatures and exception types; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - Complex data are interleaved (re, im) IEEE binary64 (ADMM_C128) or binary32
 *     (ADMM_C64) values; matrices are row-major, exactly the reference's CMatrix layout
 *     (linalg.hpp:21-73) and CMAT payload (cmat_io.hpp:18-24).
 *   - No exceptions cross the ABI.  Every call returns an admm_status; the message of
 *     the last failure on the calling thread is admm_last_error(), and for
 *     ADMM_E_NUMERICAL raised inside the iteration loop admm_last_good_iteration()
 *     carries NumericalError::last_good_iteration() (errors.hpp:33-46).
 *   - A plan owns its device memory, stream and CUDA graph.  Plans are independent;
 *     one plan must not be used from two threads at once (GramSolver-style
 *     reentrancy, gram.hpp:25, is provided by separate plans).
 *   - There is no CPU fallback: without a CUDA device every compute entry point
 *     returns ADMM_E_CUDA.
 */
#ifndef ADMM_B200_H
#define ADMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADMM_B200_ABI_VERSION 3

/* Exception classes of errors.hpp:10-81, in validation order. */
typedef enum {
  ADMM_OK = 0,
  ADMM_E_DIMENSION = 1,   /* DimensionError   errors.hpp:19 */
  ADMM_E_INDEX = 2,       /* IndexError       errors.hpp:25 */
  ADMM_E_NUMERICAL = 3,   /* NumericalError   errors.hpp:31 */
  ADMM_E_SINGULARITY = 4, /* SingularityError errors.hpp:48 */
  ADMM_E_PARTITION = 5,   /* PartitionError   errors.hpp:54 */
  ADMM_E_PARAMETER = 6,   /* ParameterError   errors.hpp:60 */
  ADMM_E_CUDA = 7,        /* device / driver failure (no reference counterpart) */
  ADMM_E_STATE = 8,       /* API misuse (null pointer, wrong plan state) */
  ADMM_E_FORMAT = 9,      /* FormatError      errors.hpp:64 (byte offset: admm_cmat_error_offset) */
  ADMM_E_IO = 10,         /* IoError          errors.hpp:75 */
  ADMM_E_NCCL = 11,       /* NCCL failure in a multi-GPU plan (no reference counterpart) */
  ADMM_E_OBSERVER = 12    /* the observer callback asked to stop (it raised) */
} admm_status;

/* The four solver entry points (reference.hpp:27, solvers.hpp:74,179,306). */
typedef enum {
  ADMM_REFERENCE = 0,  /* lasso_admm_reference: M = N = 1, kappa = lambda/rho */
  ADMM_CONSENSUS = 1,  /* consensus_solve(problem, cfg, m):  M x 1 row split   */
  ADMM_SECTIONING = 2, /* sectioning_solve(problem, cfg, n): 1 x N column split */
  ADMM_HYBRID = 3      /* hybrid_solve(problem, cfg, m, n):  M x N grid         */
} admm_method;

typedef enum {
  ADMM_C128 = 0, /* complex<double> storage of H and K (the reference type) */
  ADMM_C64 = 1   /* complex<float> storage of H and K; iterates stay FP64    */
} admm_dtype;

/* SolverConfig (admm_core.hpp:17-35).  seed is carried but, as in the reference,
 * unused by the solvers. */
typedef struct {
  double rho;
  double lambda;
  double scl;
  uint64_t max_iters;
  double eps_pri;
  double eps_dual;
  uint64_t seed;
} admm_solver_config;

/* Partition + execution options (make_partition partition.hpp:56-65 and
 * SolveOptions report.hpp:42-46; threads has no meaning on the device). */
typedef struct {
  admm_method method;
  uint64_t M;          /* row divisions (consensus m; 1 for sectioning/reference) */
  uint64_t N;          /* column divisions (sectioning n; 1 for consensus/reference) */
  int ragged;          /* SolveOptions::ragged */
  admm_dtype dtype;    /* storage of the streamed matrices */
  int device;          /* CUDA device ordinal */
  int trace_objective; /* 1: objective every iteration (extra H pass, as the reference
                          does at solvers.hpp:146); 0: objective of the final iterate only */
  int schedule;        /* 0 auto, 1 two-pass (H streamed twice per iteration), 2 single-HBM-pass
                          column-strip sweep, 4 resident (small problems: H in SMEM, one
                          persistent kernel per launch), 5 support (one dense pass + the
                          columns in the support of v); env ADMM_B200_SCHEDULE
                          (twopass|sweep|resident|support) overrides */
  uint64_t batch;      /* 0/1: one scene; 2..64: independent scenes sharing H (BASELINE config 5):
                          g is n_meas x batch (scene fastest), solutions n_pix x batch, trace
                          iterations x batch x 3, lambda per scene via admm_plan_set_lambdas */
  double noise_sigma;  /* SensingProblem::noise_sigma: validated (>= 0) after finiteness and
                          before the partition, the order of problem.hpp:35-49 */
} admm_plan_options;

typedef struct admm_plan admm_plan;

/* Per-iteration snapshot (IterateSnapshot, report.hpp:28-35).  Pointers are host
 * buffers owned by the plan, valid during the callback. */
typedef struct {
  uint64_t iteration;          /* 1-based */
  uint64_t n_pix;
  const double* v;             /* n_pix complex */
  const double* v_prev;        /* n_pix complex */
  uint64_t n_workers;          /* M*N, worker id = i*N + j (solvers.hpp:305) */
  const double* const* replica_u; /* n_workers pointers, segment-length complex each */
  const uint64_t* replica_len; /* n_workers */
  double primal, dual;         /* this iteration's residual norms */
} admm_snapshot;
/* Return 0 to continue; any other value stops the solve at once with ADMM_E_OBSERVER
 * (an exception thrown by the reference's observer propagates out of the solver call,
 * solvers.hpp:150-160: the shim and the Python mirror rethrow it). */
typedef int (*admm_observer_fn)(const admm_snapshot* snap, void* user);

/* Setup: validates (cfg -> problem -> partition -> Gram factor, the reference order),
 * uploads the blocks, forms rho I + H_b H_b^H and its inverse on the device.
 * Replaces the setup loops solvers.hpp:92-101 / 197-209 / 325-341 and
 * GramSolver::GramSolver (gram.hpp:48-53).
 *   h: n_meas x n_pix row-major host matrix of type h_dtype; g: n_meas complex128. */
admm_status admm_plan_create(const admm_plan_options* opts, const admm_solver_config* cfg,
                             uint64_t n_meas, uint64_t n_pix, const void* h, admm_dtype h_dtype,
                             const double* g, admm_plan** out);

/* ---- multi-GPU: one plan per GPU over a Pr x Pc process grid -------
 * The plan owns row blocks [pr*M/Pr, (pr+1)*M/Pr) x column blocks [pc*N/Pc, ...).  The
 * caller runs the exchanges (all-gathers) between phases on the plan's stream, over
 * buffers it attaches; the engine never waits on a peer inside a kernel.
 *   iteration (sweep schedule, Pr == 1):  phase 1, X_ghat, X_scal, phase 4
 *   iteration (two-pass schedule):        phase 1, X_ghat, phase 2, X_outbox, phase 3, X_scal, phase 4
 *   (a consensus shard on the support schedule runs the two-pass program: its phase 1 forms
 *   w = H c from the support of the v every rank holds after phase 3 -- one dense pass per rank)
 * X_ghat: all-gather over the row communicator (ranks with the same pr, ordered by pc);
 * X_outbox: all-gather over the column communicator (same pc, ordered by pr);
 * X_scal: all-gather over all Pr*Pc ranks (rank = pr*Pc + pc).  Each rank's slot is
 * [my_offset, my_offset + my_bytes) of a buffer of total_bytes; in-place all-gather. */
typedef struct {
  uint64_t Pr, Pc; /* process grid (Pr | M, Pc | N) */
  uint64_t pr, pc; /* this plan's coordinates */
} admm_shard;
enum { ADMM_X_GHAT = 0, ADMM_X_OUTBOX = 1, ADMM_X_SCAL = 2 };
admm_status admm_plan_create_sharded(const admm_plan_options* opts, const admm_solver_config* cfg,
                                     uint64_t n_meas, uint64_t n_pix, const void* h, admm_dtype h_dtype,
                                     const double* g, const admm_shard* shard, admm_plan** out);
admm_status admm_plan_exchange_info(const admm_plan* plan, int which, uint64_t* total_bytes,
                                    uint64_t* my_offset, uint64_t* my_bytes);
/* Use caller-owned device memory (total_bytes) for exchange buffer `which`. */
admm_status admm_plan_attach(admm_plan* plan, int which, void* device_ptr);
/* Enqueue phase 1..4 of one iteration on the plan's stream (no host sync). */
admm_status admm_plan_run_phase(admm_plan* plan, int phase);
/* 1 = sweep, 2 = two-pass: the phase sequence the caller must drive. */
admm_status admm_plan_schedule(const admm_plan* plan, int* schedule);

/* ---- multi-GPU with plan-owned NCCL communicators ------------------
 * A distributed plan is used exactly like a single-GPU plan (admm_plan_solve, _enqueue,
 * _reset, _set_g, _set_lambda, _max_abs_adjoint, _read, _get_info): each GPU holds the
 * shard of the M x N block grid given by admm_choose_grid, and the plan runs the shard's
 * phases and the NCCL all-gathers of the exchanges (world communicator + row / column
 * communicators split from it) on its own stream(s).  Solutions, traces and errors
 * (NumericalError with last_good_iteration) are complete and identical on every rank and
 * equal to the single-GPU plan's (all-gathers keep the reference's summation order).
 * Replaces the reference's simulated node network (parallel_for + coordinator copies,
 * solvers.hpp:109-166, 211-291, 343-453; its traffic is what CommLedger counts). */
#define ADMM_NCCL_ID_BYTES 128
/* A new NCCL unique id (rank 0 of a multi-process job creates it; the caller broadcasts). */
admm_status admm_nccl_unique_id(unsigned char* id /* ADMM_NCCL_ID_BYTES */);
/* Process grid Pr x Pc for `world` GPUs: consensus shards row blocks (Pr = world),
 * sectioning column blocks (Pc = world), hybrid the grid with the most column ranks. */
admm_status admm_choose_grid(int world, admm_method method, uint64_t M, uint64_t N, uint64_t* Pr, uint64_t* Pc);
/* One process per GPU: rank `rank` of `nranks` (opts->device is this process's GPU).
 * Collective: every rank calls it with the same arguments and id.  Each rank uploads only
 * its own blocks of h. */
admm_status admm_plan_create_dist(const admm_plan_options* opts, const admm_solver_config* cfg, uint64_t n_meas,
                                  uint64_t n_pix, const void* h, admm_dtype h_dtype, const double* g,
                                  const unsigned char* nccl_id, int nranks, int rank, admm_plan** out);
/* One process, n_gpus distinct devices (device_ids, or 0..n_gpus-1 when NULL). */
admm_status admm_plan_create_multi(const admm_plan_options* opts, const admm_solver_config* cfg, uint64_t n_meas,
                                   uint64_t n_pix, const void* h, admm_dtype h_dtype, const double* g, int n_gpus,
                                   const int* device_ids, admm_plan** out);

/* Replace the measurement vector g (H, the partition and the factors are kept). */
admm_status admm_plan_set_g(admm_plan* plan, const double* g);
/* Per-scene lambdas of a batched plan (batch values). */
admm_status admm_plan_set_lambdas(admm_plan* plan, const double* lambdas);
/* Per-scene max_t |(H^H g_b)_t| of a batched plan (batch values). */
admm_status admm_plan_max_abs_adjoint_batched(admm_plan* plan, double* out);
/* Replace lambda (kappa follows). */
admm_status admm_plan_set_lambda(admm_plan* plan, double lambda);
/* max_t |(H^H g)_t| of the (scaled) problem, computed on the device; used for the
 * relative lambda rule of BASELINE.json (lambda = c * max|H^H g|). */
admm_status admm_plan_max_abs_adjoint(admm_plan* plan, double* out);

/* Full solve from u = s = v = 0 (solvers.hpp:108-166 and siblings).
 *   solution: n_pix complex (SolveReport::solution, the final v);
 *   trace:    max_iters x 3 doubles (primal, dual, objective) or NULL;
 *   observer: NULL for the captured-graph fast path. */
admm_status admm_plan_solve(admm_plan* plan, double* solution, double* trace,
                            uint64_t* iterations_run, double* objective, admm_observer_fn observer,
                            void* user);

/* Benchmark entry points: reset the iterates, enqueue `iters` iterations on the
 * plan's stream (CUDA-graph replays, no host sync), and expose that stream. */
admm_status admm_plan_reset(admm_plan* plan);
admm_status admm_plan_enqueue(admm_plan* plan, uint64_t iters);
admm_status admm_plan_sync(admm_plan* plan);
void* admm_plan_stream(admm_plan* plan);
/* Launch on the caller's stream from now on (NULL: back to the plan's own stream); used
 * to capture the phases together with the caller's collectives in one CUDA graph. */
admm_status admm_plan_set_stream(admm_plan* plan, void* stream);

/* Per-kernel device time of one iteration, measured with CUDA events around
 * individually launched kernels on the plan's stream (averaged over `iters`).
 * names/ms: arrays of at least admm_plan_kernel_count() entries. */
uint32_t admm_plan_kernel_count(const admm_plan* plan);
admm_status admm_plan_profile(admm_plan* plan, uint64_t iters, const char** names, double* ms);

typedef struct {
  uint64_t n_blocks;
  uint64_t h_bytes;             /* bytes of H storage (both passes stream it) */
  uint64_t k_bytes;             /* bytes of K storage (one pass per iteration) */
  uint64_t h_stream_bytes_per_iter; /* 2 * H bytes (algorithmic) */
  uint64_t bytes_per_iter;      /* algorithmic HBM bytes per iteration incl. K + vectors */
  uint64_t launches_per_iter;   /* kernels in one captured iteration */
  uint64_t grid_gemv_n, grid_gemv_h;
  double setup_seconds;         /* upload + Gram + inverse (host wall clock) */
  uint64_t inner_dim_max;       /* largest factored dimension */
  uint64_t schedule;            /* 1 two-pass, 2 sweep, 3 batched scenes, 4 resident, 5 support */
  uint64_t grid_sweep;
  uint64_t hbm_bytes_per_iter;  /* compulsory HBM bytes of the chosen schedule */
  uint64_t sweep_variant;       /* schedule 2 kernel: 1 L2 re-read sweep, 2 strip-major tile, 3 slab */
  uint64_t slab_cluster;        /* slab sweep: thread-block cluster size (CTAs per strip) */
  uint64_t slab_row_bytes;      /* slab sweep: bytes per strip row (64 or 32) */
  uint64_t slab_rows;           /* slab sweep: rows per warp slab */
  uint64_t grid_pr, grid_pc;    /* process grid of a multi-GPU plan (1 x 1 on one GPU) */
  uint64_t n_ranks;             /* GPUs of the plan */
  uint64_t exchange_bytes_per_iter; /* NCCL bytes this rank receives per iteration */
  double setup_phase_s[4];      /* setup_seconds split: host validation, upload (+ layout copies; the
                                   Gram launches of the blocks already uploaded run under it), the Gram
                                   time left after the upload, inverse + packing */
  double gram_device_s;         /* device time of the Gram launches (rho I + H_b H_b^H, FP64 tensor cores) */
  double gram_flops;            /* their real FP64 flops: 8 per complex MAC of the lower tiles */
  double inverse_device_s;      /* device time of the blocked Gauss-Jordan inverse */
  double inverse_flops;         /* 8 m^3 per block (rank-64 updates of the whole work matrix) */
} admm_plan_info;
admm_status admm_plan_get_info(const admm_plan* plan, admm_plan_info* info);

/* Current iterate getters (host copies): which = 0 v (n_pix), 1 v_prev (n_pix),
 * 2 u of every worker concatenated in worker order (sum of segment lengths),
 * 3 the trace (3 doubles per completed iteration), 4 {iterations completed,
 * first iteration with a non-finite u or -1}, 5 (support schedule) {iterations completed,
 * support columns of v summed over them}. */
admm_status admm_plan_read(admm_plan* plan, int which, double* dst, uint64_t count);

void admm_plan_destroy(admm_plan* plan);

/* ---- L0/L1 operations on the device (KAT surface of linalg.hpp / prox.hpp / gram.hpp) */
/* y = A x (linalg.hpp:97-111), A rows x cols complex128. */
admm_status admm_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x, double* y,
                        int device);
/* y = A^H x (linalg.hpp:114-127). */
admm_status admm_adjoint_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x,
                                double* y, int device);
/* out = S_kappa(a) element-wise (prox.hpp:21-25). */
admm_status admm_soft_threshold(const double* a, uint64_t n, double kappa, double* out, int device);
/* x = (H^H H + rho I)^-1 rhs (GramSolver::solve, gram.hpp:63-78), one-shot. */
admm_status admm_gram_solve(const double* h, uint64_t rows, uint64_t cols, double rho,
                            const double* rhs, double* x, int device);

/* GramSolver (gram.hpp:26-128) as a device object: validated and factored ONCE at
 * creation (gram.hpp:48-53), then solve() any number of times (serialised internally, so
 * concurrent callers are safe, gram.hpp:25).
 *   strategy: -1 automatic (strategy_for, gram.hpp:32-34: Woodbury iff rows < cols),
 *             0 Direct   ((H^H H + rho I)^-1, cols x cols, applied to rhs),
 *             1 Woodbury ((rho I + H H^H)^-1, rows x rows, through the inversion lemma).
 * Errors in the reference's order: ParameterError (empty block, rho <= 0), NumericalError
 * (non-finite block), SingularityError (factor breakdown). */
typedef struct admm_gram admm_gram;
admm_status admm_gram_create(const double* h, uint64_t rows, uint64_t cols, double rho, int strategy, int device,
                             admm_gram** out);
admm_status admm_gram_apply(admm_gram* g, const double* rhs, double* x);
/* strategy actually used (0 Direct, 1 Woodbury) and the factored dimension (inner_dim). */
admm_status admm_gram_info(const admm_gram* g, int* strategy, uint64_t* inner_dim);
void admm_gram_destroy(admm_gram* g);

/* ---- input tooling (host; not the hot path) */
/* gen_problem (generate.hpp:32-89) with the reference's RNG stream (rng.hpp); H is
 * written as complex128 or complex64 (rounded from the same FP64 values). */
admm_status admm_gen_problem(uint64_t n_meas, uint64_t n_pix, uint64_t k, double snr_db, uint64_t seed,
                             int kind, void* h, admm_dtype h_dtype, double* g, double* truth,
                             double* noise_sigma);
/* CRA-like structured H of BASELINE configs 3/5 (conventions in DESIGN.md). */
admm_status admm_gen_cra(uint64_t n_tx, uint64_t n_freq, uint64_t grid, double spacing, double z0,
                         double aperture, double f0, double f1, uint64_t n_facets, uint64_t seed,
                         void* h, admm_dtype h_dtype);

/* ---- CMAT file I/O (cmat_io.hpp; host, not the hot path) -------------------------
 * "CMX1": the reference format (cmat_io.hpp:18-24), binary64 (re, im) pairs, <= 2^32
 * entries.  "CMF1": the same layout with binary32 pairs (complex64 storage of the c64
 * plans; <= 2^36 entries).  Reads convert to dst_dtype on the fly (round / widen) and
 * validate exactly as read_cmat (cmat_io.hpp:57-105): IoError, FormatError with the
 * byte offset of the defect (admm_cmat_error_offset()).  A vector is a cols == 1 file
 * (read_cvec / write_cvec, cmat_io.hpp:108-125). */
admm_status admm_cmat_info(const char* path, uint64_t* rows, uint64_t* cols, admm_dtype* file_dtype);
/* read_cmat (cmat_io.hpp:57): dst holds capacity_entries complex values of dst_dtype. */
admm_status admm_cmat_read(const char* path, void* dst, uint64_t capacity_entries, admm_dtype dst_dtype);
/* write_cmat (cmat_io.hpp:44): src is rows x cols of src_dtype; file_dtype picks CMX1/CMF1. */
admm_status admm_cmat_write(const char* path, const void* src, uint64_t rows, uint64_t cols, admm_dtype src_dtype,
                            admm_dtype file_dtype);
/* FormatError::byte_offset (errors.hpp:64-73) of the calling thread's last failure. */
uint64_t admm_cmat_error_offset(void);

const char* admm_last_error(void);
uint64_t admm_last_good_iteration(void);
int admm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ADMM_B200_H */
