/* oracle/admm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C99) of the reference admmsplit hot path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker.  It is never linked into, called by, or shipped with the product
 * library (paper_1811_05571_b200/libadmm_b200.so).
 *
 * Parity pin: tests/test_oracle_golden.py checks this restatement BIT-FOR-BIT
 * against fixtures produced by the unmodified reference (oracle/_ref, built from
 * /root/reference by oracle/Makefile; fixtures by tests/golden/make_golden.py).
 *
 * All complex data are interleaved (re, im) binary64, row-major matrices.
 */
#ifndef ADMM_ORACLE_H
#define ADMM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_E_DIMENSION = 1, ORC_E_INDEX = 2, ORC_E_NUMERICAL = 3,
       ORC_E_SINGULARITY = 4, ORC_E_PARTITION = 5, ORC_E_PARAMETER = 6, ORC_E_ALLOC = 7 };
enum { ORC_REFERENCE = 0, ORC_CONSENSUS = 1, ORC_SECTIONING = 2, ORC_HYBRID = 3 };
enum { ORC_KIND_CG = 0, ORC_KIND_RP = 1 };
enum { ORC_STRATEGY_AUTO = -1, ORC_DIRECT = 0, ORC_WOODBURY = 1 };

/* generate.hpp:32-89 + rng.hpp (Xoshiro256++ seeded by SplitMix64, Box-Muller). */
int orc_gen_problem(uint64_t n_meas, uint64_t n_pix, uint64_t k, double snr_db, uint64_t seed,
                    int kind, double* h, double* g, double* truth, double* noise_sigma);
/* testutil::random_matrix / random_vector (tests/support/test_util.hpp:20-34). */
void orc_random_gauss(uint64_t count, uint64_t seed, double* out);

/* FNV-1a 64 (test_util.hpp:109-124). */
uint64_t orc_fnv1a64(const void* data, uint64_t bytes, uint64_t h);
/* linalg.hpp:97-127 */
void orc_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x, double* y);
void orc_adjoint_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x, double* y);
/* prox.hpp:15-25 */
void orc_soft_threshold_vec(const double* a, uint64_t n, double kappa, double* out);
/* gram.hpp:26-128 (+ cholesky.hpp).  strategy: -1 auto (gram.hpp:32-34). */
int orc_gram_solve(const double* h, uint64_t rows, uint64_t cols, double rho, int strategy,
                   const double* rhs, double* x);
/* partition.hpp:34-65.  bounds arrays hold parts+1 entries. */
int orc_split_bounds(uint64_t total, uint64_t parts, int ragged, uint64_t* bounds);
/* admm_core.hpp:60-64 */
double orc_objective(const double* h, uint64_t rows, uint64_t cols, const double* g,
                     const double* v, double lambda);

/* reference.hpp:27 / solvers.hpp:74,179,306.  trace: max_iters x 3 (primal, dual,
 * objective); snapshots (optional): max_iters x n_pix complex v after each iteration;
 * replica_u (optional): max_iters x (n_workers x segment length) flattened per worker. */
int orc_solve(int method, const double* h, const double* g, uint64_t n_meas, uint64_t n_pix,
              uint64_t M, uint64_t N, int ragged, double rho, double lambda, double scl,
              uint64_t max_iters, double eps_pri, double eps_dual, double* solution,
              double* trace, uint64_t* iterations_run, double* objective, uint64_t* last_good,
              double* snapshots);

#ifdef __cplusplus
}
#endif
#endif
