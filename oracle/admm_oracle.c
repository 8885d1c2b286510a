/* oracle/admm_oracle.c — TEST INFRASTRUCTURE ONLY (see admm_oracle.h).
 *
 * A plain-C99 restatement of the reference admmsplit algorithm, written so that
 * every floating-point operation happens in the same order as in the reference
 * (ascending index sums, the same grouping of each update expression, the same
 * libm calls).  Compiled with gcc -O2 -ffp-contract=off this reproduces the
 * reference's bits, which tests/test_oracle_golden.py checks against fixtures made
 * by the unmodified reference (oracle/_ref).
 *
 * Notes on matching libstdc++ std::complex<double> semantics:
 *   - complex*complex uses GCC's __muldc3 path in both C and C++;
 *   - complex*real and complex/real are component-wise in both;
 *   - std::norm(z) for double is re*re + im*im (libstdc++ 13 _Norm_helper<true>);
 *   - std::abs(z) is cabs (hypot).
 */
#include "admm_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* ---------------------------------------------------------------- rng.hpp */
typedef struct { uint64_t s[4]; } xoshiro;

static uint64_t splitmix_next(uint64_t* state) { /* rng.hpp:13-26 */
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static void xo_seed(xoshiro* x, uint64_t seed) { /* rng.hpp:36-39 */
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) x->s[i] = splitmix_next(&sm);
}
static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
static uint64_t xo_next(xoshiro* x) { /* rng.hpp:41-51 */
  uint64_t* s = x->s;
  const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return out;
}
static const double ORC_PI = 3.14159265358979323846;
static double xo_double(xoshiro* x) { return (double)(xo_next(x) >> 11) * 0x1.0p-53; }
static cplx xo_gauss(xoshiro* x) { /* rng.hpp:59-70 Box-Muller */
  const double u1 = 1.0 - xo_double(x);
  const double u2 = xo_double(x);
  const double r = sqrt(-2.0 * log(u1));
  const double th = 2.0 * ORC_PI * u2;
  return CMPLX(r * cos(th), r * sin(th));
}
static cplx xo_phase(xoshiro* x) { /* rng.hpp:73-76 */
  const double th = 2.0 * ORC_PI * xo_double(x);
  return CMPLX(cos(th), sin(th));
}

/* ------------------------------------------------------------- linalg.hpp */
static double cnorm(cplx z) { const double x = creal(z), y = cimag(z); return x * x + y * y; }
static int finite_c(cplx z) { return isfinite(creal(z)) && isfinite(cimag(z)); }
static int all_finite(const cplx* v, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) if (!finite_c(v[i])) return 0;
  return 1;
}
static double sum_sq(const cplx* v, uint64_t n) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc += cnorm(v[i]);
  return acc;
}
static double sum_sq_diff(const cplx* a, const cplx* b, uint64_t n) { /* linalg.hpp:143-148 */
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc += cnorm(a[i] - b[i]);
  return acc;
}
static double norm1(const cplx* v, uint64_t n) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc += cabs(v[i]);
  return acc;
}
static void matvec(const cplx* a, uint64_t rows, uint64_t cols, const cplx* x, cplx* y) {
  for (uint64_t r = 0; r < rows; ++r) { /* linalg.hpp:104-109, ascending column */
    cplx acc = 0.0;
    const cplx* row = a + r * cols;
    for (uint64_t l = 0; l < cols; ++l) acc += row[l] * x[l];
    y[r] = acc;
  }
}
static void adjoint_matvec(const cplx* a, uint64_t rows, uint64_t cols, const cplx* x, cplx* y) {
  for (uint64_t c = 0; c < cols; ++c) { /* linalg.hpp:121-125, ascending row */
    cplx acc = 0.0;
    for (uint64_t k = 0; k < rows; ++k) acc += conj(a[k * cols + c]) * x[k];
    y[c] = acc;
  }
}

void orc_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x, double* y) {
  matvec((const cplx*)a, rows, cols, (const cplx*)x, (cplx*)y);
}
void orc_adjoint_matvec(const double* a, uint64_t rows, uint64_t cols, const double* x, double* y) {
  adjoint_matvec((const cplx*)a, rows, cols, (const cplx*)x, (cplx*)y);
}

/* --------------------------------------------------------------- prox.hpp */
static cplx soft_threshold(cplx a, double kappa) { /* prox.hpp:15-19 */
  const double mag = cabs(a);
  if (mag > kappa) return a * (1.0 - kappa / mag);
  return 0.0;
}
static void soft_vec(const cplx* a, uint64_t n, double kappa, cplx* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = soft_threshold(a[i], kappa);
}
void orc_soft_threshold_vec(const double* a, uint64_t n, double kappa, double* out) {
  soft_vec((const cplx*)a, n, kappa, (cplx*)out);
}

/* ----------------------------------------------------- cholesky.hpp / gram.hpp */
typedef struct {
  const cplx* h;      /* block, rows x cols (borrowed) */
  uint64_t rows, cols;
  double rho;
  int woodbury;
  uint64_t dim;       /* factored dimension */
  cplx* l;            /* dim x dim lower factor */
} gram_solver;

static int cholesky_factor(const cplx* a, uint64_t n, cplx* l) { /* cholesky.hpp:48-74 */
  if (!all_finite(a, n * n)) return ORC_E_NUMERICAL;
  memset(l, 0, n * n * sizeof(cplx));
  for (uint64_t j = 0; j < n; ++j) {
    double d = creal(a[j * n + j]);
    for (uint64_t k = 0; k < j; ++k) d -= cnorm(l[j * n + k]);
    if (!(d > 0.0) || !isfinite(d)) return ORC_E_SINGULARITY;
    const double ljj = sqrt(d);
    l[j * n + j] = CMPLX(ljj, 0.0);
    for (uint64_t i = j + 1; i < n; ++i) {
      cplx acc = a[i * n + j];
      for (uint64_t k = 0; k < j; ++k) acc -= l[i * n + k] * conj(l[j * n + k]);
      l[i * n + j] = acc / ljj;
    }
  }
  return ORC_OK;
}

static void cholesky_solve(const cplx* l, uint64_t n, const cplx* b, cplx* y, cplx* x) {
  for (uint64_t i = 0; i < n; ++i) { /* cholesky.hpp:30-35: L y = b */
    cplx acc = b[i];
    for (uint64_t k = 0; k < i; ++k) acc -= l[i * n + k] * y[k];
    y[i] = acc / creal(l[i * n + i]);
  }
  for (uint64_t ii = n; ii-- > 0;) { /* cholesky.hpp:37-42: L* x = y */
    cplx acc = y[ii];
    for (uint64_t k = ii + 1; k < n; ++k) acc -= conj(l[k * n + ii]) * x[k];
    x[ii] = acc / creal(l[ii * n + ii]);
  }
}

static void gram_free(gram_solver* gs) { free(gs->l); gs->l = NULL; }

/* gram.hpp:48-53 / 81-122 */
static int gram_init(gram_solver* gs, const cplx* h, uint64_t rows, uint64_t cols, double rho,
                     int strategy) {
  memset(gs, 0, sizeof(*gs));
  if (rows == 0 || cols == 0) return ORC_E_PARAMETER;
  if (!(rho > 0.0)) return ORC_E_PARAMETER;
  if (!all_finite(h, rows * cols)) return ORC_E_NUMERICAL;
  gs->h = h; gs->rows = rows; gs->cols = cols; gs->rho = rho;
  gs->woodbury = strategy == ORC_STRATEGY_AUTO ? (rows < cols) : (strategy == ORC_WOODBURY);
  const uint64_t n = gs->woodbury ? rows : cols;
  gs->dim = n;
  cplx* a = (cplx*)calloc(n * n, sizeof(cplx));
  gs->l = (cplx*)malloc(n * n * sizeof(cplx));
  if (!a || !gs->l) { free(a); gram_free(gs); return ORC_E_ALLOC; }
  if (!gs->woodbury) { /* H*H + rho I, gram.hpp:93-106 */
    for (uint64_t r = 0; r < n; ++r)
      for (uint64_t c = 0; c <= r; ++c) {
        cplx acc = 0.0;
        for (uint64_t k = 0; k < rows; ++k) acc += conj(h[k * cols + r]) * h[k * cols + c];
        if (r == c) acc += rho;
        a[r * n + c] = acc;
        a[c * n + r] = conj(acc);
      }
  } else { /* I + (H H^H)/rho, gram.hpp:107-121 */
    for (uint64_t r = 0; r < n; ++r) {
      const cplx* rr = h + r * cols;
      for (uint64_t c = 0; c <= r; ++c) {
        const cplx* rc = h + c * cols;
        cplx acc = 0.0;
        for (uint64_t k = 0; k < cols; ++k) acc += rr[k] * conj(rc[k]);
        acc /= rho;
        if (r == c) acc += 1.0;
        a[r * n + c] = acc;
        a[c * n + r] = conj(acc);
      }
    }
  }
  const int st = cholesky_factor(a, n, gs->l);
  free(a);
  if (st != ORC_OK) gram_free(gs);
  return st;
}

/* gram.hpp:63-78.  scratch: >= 3*dim + cols complex. */
static void gram_solve(const gram_solver* gs, const cplx* rhs, cplx* x, cplx* scratch) {
  const uint64_t n = gs->dim;
  if (!gs->woodbury) {
    cholesky_solve(gs->l, n, rhs, scratch, x);
    return;
  }
  cplx* t = scratch;
  cplx* y1 = scratch + n;
  cplx* y = scratch + 2 * n;
  cplx* z = scratch + 3 * n;
  matvec(gs->h, gs->rows, gs->cols, rhs, t);
  cholesky_solve(gs->l, n, t, y1, y);
  adjoint_matvec(gs->h, gs->rows, gs->cols, y, z);
  const double rho2 = gs->rho * gs->rho;
  for (uint64_t i = 0; i < gs->cols; ++i) x[i] = rhs[i] / gs->rho - z[i] / rho2;
}

int orc_gram_solve(const double* h, uint64_t rows, uint64_t cols, double rho, int strategy,
                   const double* rhs, double* x) {
  gram_solver gs;
  int st = gram_init(&gs, (const cplx*)h, rows, cols, rho, strategy);
  if (st != ORC_OK) return st;
  cplx* scratch = (cplx*)malloc((3 * gs.dim + cols + 1) * sizeof(cplx));
  if (!scratch) { gram_free(&gs); return ORC_E_ALLOC; }
  gram_solve(&gs, (const cplx*)rhs, (cplx*)x, scratch);
  free(scratch);
  gram_free(&gs);
  return ORC_OK;
}

/* ----------------------------------------------------------- partition.hpp */
int orc_split_bounds(uint64_t total, uint64_t parts, int ragged, uint64_t* bounds) {
  if (parts < 1 || parts > total) return ORC_E_PARTITION;          /* partition.hpp:37-40 */
  if (!ragged && total % parts != 0) return ORC_E_PARTITION;       /* partition.hpp:41-45 */
  const uint64_t base = total / parts, rem = total % parts;
  bounds[0] = 0;
  for (uint64_t b = 0; b < parts; ++b) bounds[b + 1] = bounds[b] + base + (b < rem ? 1 : 0);
  return ORC_OK;
}

/* --------------------------------------------------------- admm_core.hpp */
static double objective(const cplx* h, uint64_t rows, uint64_t cols, const cplx* g, const cplx* v,
                        double lambda, cplx* hv) { /* admm_core.hpp:60-64 */
  matvec(h, rows, cols, v, hv);
  return 0.5 * sum_sq_diff(hv, g, rows) + lambda * norm1(v, cols);
}
double orc_objective(const double* h, uint64_t rows, uint64_t cols, const double* g,
                     const double* v, double lambda) {
  cplx* hv = (cplx*)malloc(rows * sizeof(cplx));
  const double o = objective((const cplx*)h, rows, cols, (const cplx*)g, (const cplx*)v, lambda, hv);
  free(hv);
  return o;
}
static int stop_now(double eps_pri, double eps_dual, double rp, double rd) { /* admm_core.hpp:52-57 */
  if (eps_pri == 0.0 && eps_dual == 0.0) return 0;
  const int pri_ok = eps_pri == 0.0 || rp <= eps_pri;
  const int dual_ok = eps_dual == 0.0 || rd <= eps_dual;
  return pri_ok && dual_ok;
}

/* ------------------------------------------------------------ generate.hpp */
int orc_gen_problem(uint64_t n_meas, uint64_t n_pix, uint64_t k, double snr_db, uint64_t seed,
                    int kind, double* h_out, double* g_out, double* truth_out, double* noise_sigma) {
  if (n_meas < 1 || n_pix < 1) return ORC_E_PARAMETER;
  if (k < 1 || k > n_pix) return ORC_E_PARAMETER;
  if (isnan(snr_db)) return ORC_E_PARAMETER;
  if (kind != ORC_KIND_CG && kind != ORC_KIND_RP) return ORC_E_PARAMETER;
  cplx* h = (cplx*)h_out;
  cplx* g = (cplx*)g_out;
  cplx* truth = (cplx*)truth_out;
  xoshiro rng;
  xo_seed(&rng, seed);
  if (kind == ORC_KIND_CG) { /* generate.hpp:50-54 */
    const double scale = 1.0 / sqrt(2.0 * (double)n_meas);
    for (uint64_t i = 0; i < n_meas * n_pix; ++i) h[i] = xo_gauss(&rng) * scale;
  } else { /* generate.hpp:55-59 */
    const double scale = 1.0 / sqrt((double)n_meas);
    for (uint64_t i = 0; i < n_meas * n_pix; ++i) h[i] = xo_phase(&rng) * scale;
  }
  uint64_t* pos = (uint64_t*)malloc(n_pix * sizeof(uint64_t));
  if (!pos) return ORC_E_ALLOC;
  for (uint64_t i = 0; i < n_pix; ++i) pos[i] = i;
  for (uint64_t t = 0; t < k; ++t) { /* partial Fisher-Yates, generate.hpp:64-69 */
    const uint64_t j = t + xo_next(&rng) % (n_pix - t);
    const uint64_t tmp = pos[t]; pos[t] = pos[j]; pos[j] = tmp;
  }
  for (uint64_t i = 0; i < n_pix; ++i) truth[i] = 0.0;
  for (uint64_t t = 0; t < k; ++t) truth[pos[t]] = xo_phase(&rng);
  free(pos);
  matvec(h, n_meas, n_pix, truth, g); /* clean signal */
  *noise_sigma = 0.0;
  if (isfinite(snr_db)) { /* generate.hpp:76-85 */
    cplx* w = (cplx*)malloc(n_meas * sizeof(cplx));
    if (!w) return ORC_E_ALLOC;
    for (uint64_t i = 0; i < n_meas; ++i) w[i] = xo_gauss(&rng);
    const double w_norm = sqrt(sum_sq(w, n_meas));
    const double s_norm = sqrt(sum_sq(g, n_meas));
    const double alpha = w_norm > 0.0 ? s_norm / (w_norm * pow(10.0, snr_db / 20.0)) : 0.0;
    for (uint64_t i = 0; i < n_meas; ++i) g[i] = g[i] + alpha * w[i];
    *noise_sigma = alpha;
    free(w);
  }
  return ORC_OK;
}

void orc_random_gauss(uint64_t count, uint64_t seed, double* out) {
  xoshiro rng;
  xo_seed(&rng, seed);
  cplx* o = (cplx*)out;
  for (uint64_t i = 0; i < count; ++i) o[i] = xo_gauss(&rng);
}

/* --------------------------------------------------------------- solvers */
typedef struct {
  cplx* h;            /* materialised block copy, partition.hpp:79-125 */
  uint64_t rows, cols;
  cplx* g;            /* row-block data (consensus / hybrid) */
  gram_solver gram;
  cplx *hg, *u, *s, *v, *v_prev, *ghat, *inbox_v, *outbox, *rhs, *work, *gj;
  cplx** inbox_ghat;  /* N slots (own unused) */
  double rp2, rd2;
  int ok;
} worker;

typedef struct { void** p; size_t n, cap; } arena;
static void* arena_alloc(arena* a, size_t bytes) {
  if (a->n == a->cap) {
    size_t nc = a->cap ? 2 * a->cap : 64;
    void** np = (void**)realloc(a->p, nc * sizeof(void*));
    if (!np) return NULL;
    a->p = np; a->cap = nc;
  }
  void* q = calloc(1, bytes ? bytes : 1);
  if (q) a->p[a->n++] = q;
  return q;
}
static void arena_free(arena* a) {
  for (size_t i = 0; i < a->n; ++i) free(a->p[i]);
  free(a->p);
}
#define ALLOC(ptr, count, T)                                       \
  do {                                                             \
    (ptr) = (T*)arena_alloc(&ar, (size_t)(count) * sizeof(T));     \
    if (!(ptr)) { st = ORC_E_ALLOC; goto done; }                   \
  } while (0)

int orc_solve(int method, const double* h_in, const double* g_in, uint64_t n_meas, uint64_t n_pix,
              uint64_t M, uint64_t N, int ragged, double rho, double lambda, double scl,
              uint64_t max_iters, double eps_pri, double eps_dual, double* solution,
              double* trace, uint64_t* iterations_run, double* objective_out, uint64_t* last_good,
              double* snapshots) {
  int st = ORC_OK;
  arena ar = {0};
  worker* W = NULL;
  uint64_t nw = 0;
  *iterations_run = 0;
  *last_good = 0;
  /* SolverConfig::validate, admm_core.hpp:26-34 */
  if (!(rho > 0.0) || !(lambda > 0.0) || !(scl > 0.0) || max_iters < 1 || eps_pri < 0.0 ||
      eps_dual < 0.0)
    return ORC_E_PARAMETER;
  /* SensingProblem::validate, problem.hpp:35-49 */
  if (n_meas == 0 || n_pix == 0) return ORC_E_DIMENSION;
  const cplx* H = (const cplx*)h_in;
  const cplx* G = (const cplx*)g_in;
  if (!all_finite(H, n_meas * n_pix) || !all_finite(G, n_meas)) return ORC_E_NUMERICAL;
  if (scl != 1.0) { /* problem.hpp:59-66, then re-validate */
    cplx *hs, *gs;
    ALLOC(hs, n_meas * n_pix, cplx);
    ALLOC(gs, n_meas, cplx);
    for (uint64_t i = 0; i < n_meas * n_pix; ++i) hs[i] = H[i] * scl;
    for (uint64_t i = 0; i < n_meas; ++i) gs[i] = G[i] * scl;
    if (!all_finite(hs, n_meas * n_pix) || !all_finite(gs, n_meas)) { st = ORC_E_NUMERICAL; goto done; }
    H = hs;
    G = gs;
  }
  cplx* sol = (cplx*)solution;
  cplx* snaps = (cplx*)snapshots;
  cplx* hv;
  ALLOC(hv, n_meas, cplx);

  if (method == ORC_REFERENCE) { /* reference.hpp:27-90 */
    const double kappa = lambda / rho;
    gram_solver gs;
    st = gram_init(&gs, H, n_meas, n_pix, rho, ORC_STRATEGY_AUTO);
    if (st != ORC_OK) goto done;
    cplx *hg, *u, *v, *s, *rhs, *w, *vp, *scratch;
    ALLOC(hg, n_pix, cplx); ALLOC(u, n_pix, cplx); ALLOC(v, n_pix, cplx); ALLOC(s, n_pix, cplx);
    ALLOC(rhs, n_pix, cplx); ALLOC(w, n_pix, cplx); ALLOC(vp, n_pix, cplx);
    ALLOC(scratch, 3 * gs.dim + n_pix + 1, cplx);
    adjoint_matvec(H, n_meas, n_pix, G, hg);
    for (uint64_t k = 0; k < max_iters; ++k) {
      for (uint64_t t = 0; t < n_pix; ++t) rhs[t] = hg[t] + rho * (v[t] - s[t]);
      gram_solve(&gs, rhs, u, scratch);
      if (!all_finite(u, n_pix)) { *last_good = k; st = ORC_E_NUMERICAL; gram_free(&gs); goto done; }
      for (uint64_t t = 0; t < n_pix; ++t) w[t] = u[t] + s[t];
      memcpy(vp, v, n_pix * sizeof(cplx));
      soft_vec(w, n_pix, kappa, v);
      for (uint64_t t = 0; t < n_pix; ++t) s[t] = (s[t] + u[t]) - v[t];
      const double rp = sqrt(sum_sq_diff(u, v, n_pix));
      const double dual_sum = sum_sq_diff(v, vp, n_pix);
      const double rd = sqrt(rho * rho * dual_sum);
      const double obj = objective(H, n_meas, n_pix, G, v, lambda, hv);
      trace[3 * k] = rp; trace[3 * k + 1] = rd; trace[3 * k + 2] = obj;
      *iterations_run = k + 1;
      *objective_out = obj;
      if (snaps) memcpy(snaps + k * n_pix, v, n_pix * sizeof(cplx));
      if (stop_now(eps_pri, eps_dual, rp, rd)) break;
    }
    memcpy(sol, v, n_pix * sizeof(cplx));
    gram_free(&gs);
    goto done;
  }

  if (method == ORC_CONSENSUS) N = 1;
  if (method == ORC_SECTIONING) M = 1;
  if (method != ORC_CONSENSUS && method != ORC_SECTIONING && method != ORC_HYBRID) {
    st = ORC_E_PARAMETER;
    goto done;
  }
  uint64_t *rb, *cb;
  ALLOC(rb, M + 1 + 1, uint64_t);
  ALLOC(cb, N + 1 + 1, uint64_t);
  if ((st = orc_split_bounds(n_meas, M, ragged, rb)) != ORC_OK) goto done;
  if ((st = orc_split_bounds(n_pix, N, ragged, cb)) != ORC_OK) goto done;

  nw = M * N;
  W = (worker*)arena_alloc(&ar, nw * sizeof(worker));
  if (!W) { st = ORC_E_ALLOC; goto done; }
  /* setup (solvers.hpp:92-101, 197-209, 325-341): materialised blocks, Gram factor */
  for (uint64_t i = 0; i < M; ++i)
    for (uint64_t j = 0; j < N; ++j) {
      worker* w = &W[i * N + j];
      const uint64_t r0 = rb[i], rows = rb[i + 1] - rb[i];
      const uint64_t c0 = cb[j], cols = cb[j + 1] - cb[j];
      w->rows = rows; w->cols = cols;
      ALLOC(w->h, rows * cols, cplx);
      for (uint64_t r = 0; r < rows; ++r)
        memcpy(w->h + r * cols, H + (r0 + r) * n_pix + c0, cols * sizeof(cplx));
      ALLOC(w->g, rows, cplx);
      memcpy(w->g, G + r0, rows * sizeof(cplx));
      st = gram_init(&w->gram, w->h, rows, cols, rho, ORC_STRATEGY_AUTO);
      if (st != ORC_OK) goto done;
      ALLOC(w->hg, cols, cplx); ALLOC(w->u, cols, cplx); ALLOC(w->s, cols, cplx);
      ALLOC(w->v, cols, cplx); ALLOC(w->v_prev, cols, cplx); ALLOC(w->ghat, rows, cplx);
      ALLOC(w->inbox_v, cols, cplx); ALLOC(w->outbox, cols, cplx); ALLOC(w->rhs, cols, cplx);
      ALLOC(w->work, 3 * w->gram.dim + cols + 1, cplx); ALLOC(w->gj, rows, cplx);
      ALLOC(w->inbox_ghat, N, cplx*);
      for (uint64_t q = 0; q < N; ++q) ALLOC(w->inbox_ghat[q], rows, cplx);
      if (method == ORC_CONSENSUS) adjoint_matvec(w->h, rows, cols, w->g, w->hg); /* solvers.hpp:98 */
    }

  const double kappa = method == ORC_SECTIONING ? lambda / rho : lambda / ((double)M * rho);
  cplx *v, *v_prev, *mean;
  ALLOC(v, n_pix, cplx);       /* segment v_j at cb[j] (consensus: the full v) */
  ALLOC(v_prev, n_pix, cplx);
  ALLOC(mean, n_pix, cplx);

  for (uint64_t k = 0; k < max_iters; ++k) {
    double rp2 = 0.0, dual_sum = 0.0;
    if (method == ORC_SECTIONING) { /* solvers.hpp:217-287 */
      for (uint64_t j = 0; j < N; ++j)
        for (uint64_t q = 0; q < N; ++q)
          if (q != j) memcpy(W[q].inbox_ghat[j], W[j].ghat, n_meas * sizeof(cplx));
      for (uint64_t j = 0; j < N; ++j) {
        worker* w = &W[j];
        memcpy(w->gj, G, n_meas * sizeof(cplx));
        for (uint64_t q = 0; q < N; ++q) {
          if (q == j) continue;
          for (uint64_t t = 0; t < n_meas; ++t) w->gj[t] -= w->inbox_ghat[q][t];
        }
        adjoint_matvec(w->h, w->rows, w->cols, w->gj, w->hg);
        for (uint64_t t = 0; t < w->cols; ++t) w->rhs[t] = w->hg[t] + rho * (w->v[t] - w->s[t]);
        gram_solve(&w->gram, w->rhs, w->u, w->work);
        w->ok = all_finite(w->u, w->cols);
        for (uint64_t t = 0; t < w->cols; ++t) w->outbox[t] = w->u[t] + w->s[t];
        memcpy(w->v_prev, w->v, w->cols * sizeof(cplx));
        soft_vec(w->outbox, w->cols, kappa, w->v);
        for (uint64_t t = 0; t < w->cols; ++t) w->s[t] = (w->s[t] + w->u[t]) - w->v[t];
        matvec(w->h, w->rows, w->cols, w->u, w->ghat);
        w->rp2 = sum_sq_diff(w->u, w->v, w->cols);
        w->rd2 = sum_sq_diff(w->v, w->v_prev, w->cols);
      }
      for (uint64_t j = 0; j < N; ++j)
        if (!W[j].ok) { *last_good = k; st = ORC_E_NUMERICAL; goto done; }
      for (uint64_t j = 0; j < N; ++j) { rp2 += W[j].rp2; dual_sum += W[j].rd2; }
      for (uint64_t j = 0; j < N; ++j) {
        memcpy(v + cb[j], W[j].v, W[j].cols * sizeof(cplx));
        memcpy(v_prev + cb[j], W[j].v_prev, W[j].cols * sizeof(cplx));
      }
      const double rp = sqrt(rp2);
      const double rd = sqrt(rho * rho * dual_sum);
      const double obj = objective(H, n_meas, n_pix, G, v, lambda, hv);
      trace[3 * k] = rp; trace[3 * k + 1] = rd; trace[3 * k + 2] = obj;
      *iterations_run = k + 1;
      *objective_out = obj;
      if (snaps) memcpy(snaps + k * n_pix, v, n_pix * sizeof(cplx));
      if (stop_now(eps_pri, eps_dual, rp, rd)) break;
      continue;
    }

    /* consensus (solvers.hpp:108-162) and hybrid (solvers.hpp:353-449) */
    for (uint64_t id = 0; id < nw; ++id) { /* inbox_v = v_j */
      const uint64_t j = id % N;
      memcpy(W[id].inbox_v, v + cb[j], W[id].cols * sizeof(cplx));
    }
    if (method == ORC_HYBRID) /* row exchange of ghat (previous iteration) */
      for (uint64_t i = 0; i < M; ++i)
        for (uint64_t j = 0; j < N; ++j)
          for (uint64_t q = 0; q < N; ++q)
            if (q != j) memcpy(W[i * N + q].inbox_ghat[j], W[i * N + j].ghat, W[i * N + j].rows * sizeof(cplx));
    for (uint64_t id = 0; id < nw; ++id) {
      worker* w = &W[id];
      const uint64_t j = id % N;
      if (k > 0) /* deferred dual update, admm_core.hpp:87-89 */
        for (uint64_t t = 0; t < w->cols; ++t) w->s[t] = (w->s[t] + w->u[t]) - w->inbox_v[t];
      if (method == ORC_HYBRID) {
        memcpy(w->gj, w->g, w->rows * sizeof(cplx));
        for (uint64_t q = 0; q < N; ++q) {
          if (q == j) continue;
          for (uint64_t t = 0; t < w->rows; ++t) w->gj[t] -= w->inbox_ghat[q][t];
        }
        adjoint_matvec(w->h, w->rows, w->cols, w->gj, w->hg);
      }
      for (uint64_t t = 0; t < w->cols; ++t) w->rhs[t] = w->hg[t] + rho * (w->inbox_v[t] - w->s[t]);
      gram_solve(&w->gram, w->rhs, w->u, w->work);
      w->ok = all_finite(w->u, w->cols);
      for (uint64_t t = 0; t < w->cols; ++t) w->outbox[t] = w->u[t] + w->s[t];
      if (method == ORC_HYBRID) matvec(w->h, w->rows, w->cols, w->u, w->ghat);
    }
    for (uint64_t id = 0; id < nw; ++id)
      if (!W[id].ok) { *last_good = k; st = ORC_E_NUMERICAL; goto done; }
    memcpy(v_prev, v, n_pix * sizeof(cplx));
    for (uint64_t j = 0; j < N; ++j) { /* segment means, ascending replica order */
      const uint64_t len = cb[j + 1] - cb[j];
      cplx* mw = mean + cb[j];
      for (uint64_t t = 0; t < len; ++t) mw[t] = 0.0;
      for (uint64_t i = 0; i < M; ++i) {
        const cplx* o = W[i * N + j].outbox;
        for (uint64_t t = 0; t < len; ++t) mw[t] += o[t];
      }
      for (uint64_t t = 0; t < len; ++t) mw[t] /= (double)M;
      soft_vec(mw, len, kappa, v + cb[j]);
    }
    for (uint64_t i = 0; i < M; ++i)
      for (uint64_t j = 0; j < N; ++j)
        rp2 += sum_sq_diff(W[i * N + j].u, v + cb[j], W[i * N + j].cols);
    if (method == ORC_CONSENSUS) {
      dual_sum = sum_sq_diff(v, v_prev, n_pix);
    } else {
      for (uint64_t j = 0; j < N; ++j)
        dual_sum += sum_sq_diff(v + cb[j], v_prev + cb[j], cb[j + 1] - cb[j]);
    }
    const double rp = sqrt(rp2);
    const double rd = sqrt(rho * rho * (double)M * dual_sum);
    const double obj = objective(H, n_meas, n_pix, G, v, lambda, hv);
    trace[3 * k] = rp; trace[3 * k + 1] = rd; trace[3 * k + 2] = obj;
    *iterations_run = k + 1;
    *objective_out = obj;
    if (snaps) memcpy(snaps + k * n_pix, v, n_pix * sizeof(cplx));
    if (stop_now(eps_pri, eps_dual, rp, rd)) break;
  }
  memcpy(sol, v, n_pix * sizeof(cplx));

done:
  if (W)
    for (uint64_t id = 0; id < nw; ++id) gram_free(&W[id].gram);
  arena_free(&ar);
  return st;
}

/* tests/support/test_util.hpp:109-124 (FNV-1a 64), used to pin generated inputs. */
uint64_t orc_fnv1a64(const void* data, uint64_t bytes, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (uint64_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ULL;
  }
  return h;
}
