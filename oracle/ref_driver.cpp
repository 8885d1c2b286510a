// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin command-line driver around the UNMODIFIED reference library
// (/root/reference/proj/include/admmsplit, header-only C++20).  It is compiled by
// oracle/Makefile into oracle/_ref/admmsplit_ref (git-ignored; it travels to the
// GPU box as a prebuilt binary because /root/reference does not exist there).
//
// Uses:
//   * pins the C restatement in oracle/admm_oracle.c (tests/golden/make_golden.py);
//   * is the CPU baseline ("kind": "reference") timed by bench.py.
//
// Nothing here re-implements solver arithmetic: every number comes from the
// reference's own public entry points
//   gen_problem             generate.hpp:32     (input generation)
//   lasso_admm_reference    reference.hpp:27
//   consensus_solve         solvers.hpp:74
//   sectioning_solve        solvers.hpp:179
//   hybrid_solve            solvers.hpp:306
// and its CMAT I/O (cmat_io.hpp).
//
// Usage (key=value arguments):
//   admmsplit_ref gen   out=DIR m=ROWS n=COLS k=SPARSITY snr=DB|inf seed=S kind=cg|rp
//   admmsplit_ref cmat  in=FILE [vec=0|1]   read_cmat / read_cvec (cmat_io.hpp:57,116):
//                       prints "ok ROWS COLS FNV64" or "error CLASS OFFSET"
//   admmsplit_ref solve in=DIR out=DIR method=reference|consensus|sectioning|hybrid
//                       M=.. N=.. rho=.. lambda=.. [lambda_rel=0|1] scl=.. iters=..
//                       eps_pri=.. eps_dual=.. threads=.. ragged=0|1 snapshots=0|1
// solve writes: solution.cmat, trace.bin (iters x 3 f64: primal, dual, objective),
//   times.bin (f64 observer timestamps, seconds since the solve call),
//   ledger.bin (u64 nodes, u64 iters, then per cell recv, sent_once, sent_link),
//   snapshots.bin (iters x n_pix complex v, when snapshots=1), meta.txt.

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <map>
#include <string>
#include <vector>

#include "admmsplit/admmsplit.hpp"

namespace fs = std::filesystem;
using namespace admmsplit;

namespace {

std::map<std::string, std::string> parse_kv(int argc, char** argv, int first) {
  std::map<std::string, std::string> kv;
  for (int i = first; i < argc; ++i) {
    const char* eq = std::strchr(argv[i], '=');
    if (!eq) {
      std::fprintf(stderr, "bad argument '%s' (expected key=value)\n", argv[i]);
      std::exit(2);
    }
    kv[std::string(argv[i], static_cast<std::size_t>(eq - argv[i]))] = std::string(eq + 1);
  }
  return kv;
}

std::string get(const std::map<std::string, std::string>& kv, const char* key, const char* dflt) {
  auto it = kv.find(key);
  if (it != kv.end()) return it->second;
  if (!dflt) {
    std::fprintf(stderr, "missing argument %s=\n", key);
    std::exit(2);
  }
  return dflt;
}

double to_d(const std::string& s) {
  if (s == "inf") return std::numeric_limits<double>::infinity();
  return std::strtod(s.c_str(), nullptr);
}

std::uint64_t fnv1a64(const void* data, std::size_t bytes, std::uint64_t h) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ULL;
  }
  return h;
}

void write_raw(const fs::path& p, const void* data, std::size_t bytes) {
  std::ofstream out(p, std::ios::binary | std::ios::trunc);
  out.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));
}

int cmd_gen(const std::map<std::string, std::string>& kv) {
  const fs::path out = get(kv, "out", nullptr);
  fs::create_directories(out);
  const std::size_t m = std::stoull(get(kv, "m", nullptr));
  const std::size_t n = std::stoull(get(kv, "n", nullptr));
  const std::size_t k = std::stoull(get(kv, "k", nullptr));
  const double snr = to_d(get(kv, "snr", "inf"));
  const std::uint64_t seed = std::stoull(get(kv, "seed", nullptr));
  const std::string kind = get(kv, "kind", "cg");
  const SensingProblem p =
      gen_problem(m, n, k, snr, seed, kind == "cg" ? ProblemKind::ComplexGaussian : ProblemKind::RandomPhase);
  write_cmat(out / "h.cmat", p.h);
  write_cvec(out / "g.cmat", p.g);
  write_cvec(out / "truth.cmat", *p.truth);
  std::uint64_t h = 0xCBF29CE484222325ULL;
  h = fnv1a64(p.h.data(), p.h.size() * sizeof(Complex), h);
  h = fnv1a64(p.g.data(), p.g.size() * sizeof(Complex), h);
  h = fnv1a64(p.truth->data(), p.truth->size() * sizeof(Complex), h);
  std::FILE* f = std::fopen((out / "meta.txt").c_str(), "w");
  std::fprintf(f, "noise_sigma %.17g\nfnv %016llx\n", p.noise_sigma, (unsigned long long)h);
  std::fclose(f);
  std::printf("fnv %016llx\n", (unsigned long long)h);
  return 0;
}

int cmd_solve(const std::map<std::string, std::string>& kv) {
  const fs::path in = get(kv, "in", nullptr);
  const fs::path out = get(kv, "out", nullptr);
  fs::create_directories(out);
  SensingProblem p;
  p.h = read_cmat(in / "h.cmat");
  p.g = read_cvec(in / "g.cmat");
  if (fs::exists(in / "truth.cmat")) p.truth = read_cvec(in / "truth.cmat");

  const std::string method = get(kv, "method", nullptr);
  const std::size_t M = std::stoull(get(kv, "M", "1"));
  const std::size_t N = std::stoull(get(kv, "N", "1"));
  SolverConfig cfg;
  cfg.rho = to_d(get(kv, "rho", "1"));
  cfg.lambda = to_d(get(kv, "lambda", "1"));
  if (get(kv, "lambda_rel", "0") == "1") cfg.lambda *= norm_inf(adjoint_matvec(p.h, p.g));
  cfg.scl = to_d(get(kv, "scl", "1"));
  cfg.max_iters = std::stoull(get(kv, "iters", "50"));
  cfg.eps_pri = to_d(get(kv, "eps_pri", "0"));
  cfg.eps_dual = to_d(get(kv, "eps_dual", "0"));
  SolveOptions opts;
  opts.threads = std::stoull(get(kv, "threads", "1"));
  opts.ragged = get(kv, "ragged", "0") == "1";
  const bool snapshots = get(kv, "snapshots", "0") == "1";

  std::vector<double> times;
  std::vector<Complex> snaps;
  const auto t0 = std::chrono::steady_clock::now();
  opts.observer = [&](const IterateSnapshot& s) {
    times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    if (snapshots) snaps.insert(snaps.end(), s.v.begin(), s.v.end());
  };

  std::string error = "none";
  std::size_t last_good = 0;
  SolveReport r;
  try {
    if (method == "reference") {
      r = lasso_admm_reference(p, cfg, opts);
    } else if (method == "consensus") {
      r = consensus_solve(p, cfg, M, opts);
    } else if (method == "sectioning") {
      r = sectioning_solve(p, cfg, N, opts);
    } else if (method == "hybrid") {
      r = hybrid_solve(p, cfg, M, N, opts);
    } else {
      std::fprintf(stderr, "unknown method %s\n", method.c_str());
      return 2;
    }
  } catch (const NumericalError& e) {
    error = "NumericalError";
    last_good = e.last_good_iteration();
  } catch (const SingularityError&) {
    error = "SingularityError";
  } catch (const PartitionError&) {
    error = "PartitionError";
  } catch (const DimensionError&) {
    error = "DimensionError";
  } catch (const ParameterError&) {
    error = "ParameterError";
  } catch (const IndexError&) {
    error = "IndexError";
  }
  const double total =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  if (error == "none") {
    write_cvec(out / "solution.cmat", r.solution);
    std::vector<double> tr;
    for (std::size_t k = 0; k < r.trace.size(); ++k) {
      tr.push_back(r.trace.primal[k]);
      tr.push_back(r.trace.dual[k]);
      tr.push_back(r.trace.objective[k]);
    }
    write_raw(out / "trace.bin", tr.data(), tr.size() * sizeof(double));
    std::vector<std::uint64_t> led;
    led.push_back(r.ledger.node_count());
    led.push_back(r.ledger.iteration_count());
    for (std::size_t nd = 0; nd < r.ledger.node_count(); ++nd) {
      for (std::size_t k = 0; k < r.ledger.iteration_count(); ++k) {
        const auto once = r.ledger.counts(nd, k, Convention::SenderOnceBroadcast);
        const auto link = r.ledger.counts(nd, k, Convention::PerLink);
        led.push_back(once.received);
        led.push_back(once.sent);
        led.push_back(link.sent);
      }
    }
    write_raw(out / "ledger.bin", led.data(), led.size() * sizeof(std::uint64_t));
    if (snapshots) write_raw(out / "snapshots.bin", snaps.data(), snaps.size() * sizeof(Complex));
  }
  write_raw(out / "times.bin", times.data(), times.size() * sizeof(double));

  std::FILE* f = std::fopen((out / "meta.txt").c_str(), "w");
  std::fprintf(f, "error %s\nlast_good %zu\niterations_run %zu\nobjective %.17g\nlambda %.17g\n",
               error.c_str(), last_good, r.iterations_run, r.objective, cfg.lambda);
  if (r.metrics) {
    std::fprintf(f, "nmse %.17g\nprecision %.17g\nrecall %.17g\n", r.metrics->nmse,
                 r.metrics->support_precision, r.metrics->support_recall);
  }
  std::fprintf(f, "total_s %.9g\nthreads %zu\n", total, opts.threads);
  if (times.size() >= 2) {
    const double per_iter = (times.back() - times.front()) / double(times.size() - 1);
    std::fprintf(f, "setup_s %.9g\niter_s %.9g\nit_per_s %.9g\n", times.front() - per_iter,
                 per_iter, 1.0 / per_iter);
  }
  std::fclose(f);
  std::printf("error %s iterations_run %zu objective %.17g\n", error.c_str(), r.iterations_run,
              r.objective);
  return 0;
}

// FNV-1a over the payload bytes of a read matrix (what read_cmat returned).
int cmd_cmat(const std::map<std::string, std::string>& kv) {
  const fs::path in = kv.at("in");
  const bool vec = kv.count("vec") && kv.at("vec") == "1";
  try {
    CMatrix a = vec ? CMatrix(1, 1) : read_cmat(in);
    if (vec) {
      const CVector v = read_cvec(in);
      a = CMatrix(v.size(), 1);
      for (std::size_t i = 0; i < v.size(); ++i) a(i, 0) = v[i];
    }
    std::uint64_t h = 0xcbf29ce484222325ULL;
    const unsigned char* b = reinterpret_cast<const unsigned char*>(a.data());
    for (std::size_t i = 0; i < a.size() * sizeof(Complex); ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
    std::printf("ok %zu %zu %016llx\n", a.rows(), a.cols(), static_cast<unsigned long long>(h));
  } catch (const FormatError& e) {
    std::printf("error FormatError %zu\n", e.byte_offset());
  } catch (const IoError&) {
    std::printf("error IoError 0\n");
  } catch (const Error& e) {
    std::printf("error Error 0 %s\n", e.what());
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: admmsplit_ref gen|solve key=value...\n");
    return 2;
  }
  const auto kv = parse_kv(argc, argv, 2);
  const std::string cmd = argv[1];
  if (cmd == "gen") return cmd_gen(kv);
  if (cmd == "solve") return cmd_solve(kv);
  if (cmd == "cmat") return cmd_cmat(kv);
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
