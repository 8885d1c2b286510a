// admmsplit_gpu — the reference's command-line runner with the solvers on a B200.
//
// Same sub-commands, flags, output files and exit codes as the reference CLI
// (/root/reference/proj/tools/admmsplit_main.cpp): `gen` (cmd_gen, :343), `solve`
// (cmd_solve, :353-384: solution.cmat, trace.csv, ledger.csv, metrics.json, optional FNV
// fingerprint), `compare` (cmd_compare, :577-665).  run_method (:296-303) dispatches to the
// admmgpu:: drop-in (include/admmgpu/admmgpu.hpp -> libadmm_b200.so) instead of the host
// loops.  Added flags: --device gpu[:K] (default gpu:0; `cpu` is refused: this library has no
// CPU path, the reference CLI is the CPU runner), --gpus a,b,.. (one shard per listed GPU,
// plan-owned NCCL), --dtype c128|c64 (storage of H and the factor), --no-trace-objective.
// The closed-form `comm` analyser (comm.hpp:128-235) is host arithmetic and stays with the
// reference CLI.
//
// JSON files are written in the reference's layout (nlohmann dump(2): keys in alphabetical
// order, shortest round-trip doubles); CSV doubles are %.17g as in fmt_double (:41-45).
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "admmgpu/admmgpu.hpp"

namespace fs = std::filesystem;
using namespace admmgpu;

namespace {

constexpr const char* kSchemaVersion = "1";
constexpr int kExitUsage = 2;
constexpr int kExitNumerical = 3;

std::string fmt_double(double x) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", x);
  return buf;
}

// nlohmann's number format: shortest digits that round-trip; fixed notation while the
// decimal point position n satisfies -4 < n <= 15, else d[.ddd]e+XX; integral values get ".0".
std::string json_double(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), std::fabs(x), std::chars_format::scientific);
  std::string s(buf, r.ptr);  // d[.ddd]e[+-]XX
  const auto epos = s.find('e');
  std::string digits = s.substr(0, epos);
  const int e10 = std::stoi(s.substr(epos + 1));
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int len = (int)digits.size(), n = e10 + 1;  // value = 0.digits * 10^n
  std::string out = x < 0 ? "-" : "";
  if (len <= n && n <= 15) {
    out += digits + std::string(n - len, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (len > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', std::abs(e));
    out += eb;
  }
  return out;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

// An object with pre-rendered values, printed with sorted keys at a given indent.
struct JObject {
  std::map<std::string, std::string> kv;
  void num(const std::string& k, double v) { kv[k] = json_double(v); }
  void integer(const std::string& k, std::uint64_t v) { kv[k] = std::to_string(v); }
  void str(const std::string& k, const std::string& v) { kv[k] = json_string(v); }
  void null(const std::string& k) { kv[k] = "null"; }
  void raw(const std::string& k, const std::string& v) { kv[k] = v; }
  std::string dump(int indent, int step = 2) const {
    if (kv.empty()) return "{}";
    std::string pad(indent + step, ' '), o = "{\n";
    bool first = true;
    for (const auto& [k, v] : kv) {
      if (!first) o += ",\n";
      first = false;
      o += pad + json_string(k) + ": " + v;
    }
    return o + "\n" + std::string(indent, ' ') + "}";
  }
  std::string compact() const {
    std::string o = "{";
    bool first = true;
    for (const auto& [k, v] : kv) {
      if (!first) o += ",";
      first = false;
      o += json_string(k) + ":" + v;
    }
    return o + "}";
  }
};

std::uint64_t fnv1a_bytes(const void* data, std::size_t n, std::uint64_t h) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ULL;
  }
  return h;
}

std::uint64_t fnv1a_file(const fs::path& path, std::uint64_t h) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path.string() + " for fingerprinting");
  char buf[4096];
  while (in.read(buf, sizeof(buf)) || in.gcount() > 0) {
    h = fnv1a_bytes(buf, static_cast<std::size_t>(in.gcount()), h);
    if (!in) break;
  }
  return h;
}

std::string hex64(std::uint64_t v) {
  char buf[20];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(v));
  return buf;
}

// ---- flags ---------------------------------------------------------------------------
struct GenFlags {
  std::size_t nm = 0, np = 0, k = 0;
  double snr_db = std::numeric_limits<double>::infinity();
  std::uint64_t seed = 0;
  std::string kind = "complex-gaussian";
};

int parse_kind(const std::string& name) {
  if (name == "complex-gaussian") return 0;
  if (name == "random-phase") return 1;
  throw ParameterError("unknown problem kind: " + name);
}

SensingProblem generate_from_flags(const GenFlags& f) {  // gen_problem, generate.hpp:32-89
  const int kind = parse_kind(f.kind);
  SensingProblem p;
  p.h = CMatrix(f.nm, f.np);
  p.g = zeros(f.nm);
  CVector truth = zeros(f.np);
  double sigma = 0.0;
  check(admm_gen_problem(f.nm, f.np, f.k, f.snr_db, f.seed, kind, p.h.data(), ADMM_C128,
                         reinterpret_cast<double*>(p.g.data()), reinterpret_cast<double*>(truth.data()), &sigma));
  p.truth = std::move(truth);
  p.noise_sigma = sigma;
  p.kind = kind == 0 ? ProblemKind::ComplexGaussian : ProblemKind::RandomPhase;
  return p;
}

void write_text(const fs::path& path, const std::string& text) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw IoError("cannot write " + path.string());
  out << text;
}

void write_problem_dir(const fs::path& dir, const SensingProblem& p, const GenFlags& f) {
  fs::create_directories(dir);
  write_cmat((dir / "H.cmat").string(), p.h);
  write_cvec((dir / "g.cmat").string(), p.g);
  if (p.truth) write_cvec((dir / "truth.cmat").string(), *p.truth);
  JObject m;
  m.str("schema_version", kSchemaVersion);
  m.str("kind", f.kind);
  m.integer("nm", f.nm);
  m.integer("np", f.np);
  m.integer("k", f.k);
  if (std::isfinite(f.snr_db))
    m.num("snr_db", f.snr_db);
  else
    m.str("snr_db", "inf");
  m.integer("seed", f.seed);
  m.num("noise_sigma", p.noise_sigma);
  write_text(dir / "manifest.json", m.dump(0) + "\n");
}

SensingProblem load_problem_dir(const fs::path& dir) {
  SensingProblem p;
  p.h = read_cmat((dir / "H.cmat").string());
  p.g = read_cvec((dir / "g.cmat").string());
  if (fs::exists(dir / "truth.cmat")) p.truth = read_cvec((dir / "truth.cmat").string());
  p.kind = ProblemKind::FromFile;
  if (fs::exists(dir / "manifest.json")) {
    std::ifstream in(dir / "manifest.json");
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string t = ss.str();
    const auto k = t.find("\"noise_sigma\"");
    if (k != std::string::npos) {
      const auto c = t.find(':', k);
      if (c != std::string::npos) p.noise_sigma = std::strtod(t.c_str() + c + 1, nullptr);
    }
  }
  return p;  // validated by the solver entry (problem.hpp:35-49 order)
}

struct ProblemSource {
  std::string problem_dir;
  GenFlags gen;
  bool seed_given = false, any_gen_flag = false;
  SensingProblem resolve() const {
    if (!problem_dir.empty() && any_gen_flag)
      throw ParameterError("give either --problem or generation flags (--nm/--np/--k/--seed/...), not both");
    if (!problem_dir.empty()) return load_problem_dir(problem_dir);
    if (!any_gen_flag) throw ParameterError("no problem source: pass --problem DIR or --nm/--np/--k/--seed");
    if (gen.nm == 0 || gen.np == 0 || gen.k == 0) throw ParameterError("inline generation needs --nm, --np and --k");
    if (!seed_given) throw ParameterError("--seed is mandatory when generating (reproducibility)");
    return generate_from_flags(gen);
  }
};

struct SolverFlags {
  double rho = 1e5, lambda = 1e-2, scl = 1.0;
  std::size_t iters = 50;
  double eps_pri = 0.0, eps_dual = 0.0;
  std::string preset;
  std::size_t threads = 1;
  bool ragged = false, scl_given = false;
  // B200
  std::string device = "gpu";
  std::string gpus;
  std::string dtype = "c128";
  bool trace_objective = true;

  SolverConfig config(std::uint64_t seed) const {
    SolverConfig cfg;
    cfg.rho = rho;
    cfg.lambda = lambda;
    cfg.scl = (preset == "paper" && !scl_given) ? 1e-4 : scl;
    cfg.max_iters = iters;
    cfg.eps_pri = eps_pri;
    cfg.eps_dual = eps_dual;
    cfg.seed = seed;
    cfg.validate();
    return cfg;
  }
  SolveOptions options() const {
    SolveOptions o;
    o.threads = threads;
    o.ragged = ragged;
    o.trace_objective = trace_objective;
    if (dtype == "c64")
      o.dtype = ADMM_C64;
    else if (dtype != "c128")
      throw ParameterError("--dtype must be c128 or c64");
    if (device == "cpu")
      throw ParameterError("--device cpu: libadmm_b200 has no CPU path (use the reference CLI for host runs)");
    if (device.rfind("gpu", 0) != 0) throw ParameterError("--device must be gpu or gpu:K");
    if (device.size() > 3) {
      if (device[3] != ':') throw ParameterError("--device must be gpu or gpu:K");
      o.device = std::stoi(device.substr(4));
    }
    if (!gpus.empty()) {
      std::stringstream ss(gpus);
      std::string item;
      while (std::getline(ss, item, ',')) o.devices.push_back(std::stoi(item));
    }
    return o;
  }
};

struct MethodSpec {
  std::string method;
  std::size_t m = 0, n = 0;
};

SolveReport run_method(const MethodSpec& s, const SensingProblem& p, const SolverConfig& cfg, const SolveOptions& o) {
  if (s.method == "reference") return lasso_admm_reference(p, cfg, o);
  if (s.method == "consensus") return consensus_solve(p, cfg, s.m, o);
  if (s.method == "sectioning") return sectioning_solve(p, cfg, s.n, o);
  if (s.method == "hybrid") return hybrid_solve(p, cfg, s.m, s.n, o);
  throw ParameterError("unknown method: " + s.method);
}

void check_method_divisions(const MethodSpec& s) {
  const bool has_m = s.m > 0, has_n = s.n > 0;
  if (s.method == "reference" && (has_m || has_n)) throw ParameterError("reference takes neither --m nor --n");
  if (s.method == "consensus" && (!has_m || has_n)) throw ParameterError("consensus takes --m only");
  if (s.method == "sectioning" && (has_m || !has_n)) throw ParameterError("sectioning takes --n only");
  if (s.method == "hybrid" && (!has_m || !has_n)) throw ParameterError("hybrid takes both --m and --n");
}

// per_node_elements (comm.hpp:128-148), the one closed form `compare` reports.
std::optional<std::uint64_t> method_per_node_elements(const MethodSpec& s, const SensingProblem& p) {
  if (s.method == "reference") return std::nullopt;
  const std::uint64_t np = p.n_pix(), nm = p.n_meas();
  auto divides = [](std::uint64_t d, std::uint64_t total, const char* what) {
    if (total % d != 0)
      throw PartitionError("per_node_elements: " + std::to_string(d) + " does not divide " + std::to_string(total) +
                           " " + what);
  };
  if (s.method == "consensus") {
    divides(s.m, nm, "rows");
    return 2 * np;
  }
  if (s.method == "sectioning") {
    divides(s.n, np, "columns");
    return (std::uint64_t)s.n * nm;
  }
  divides(s.m, nm, "rows");
  divides(s.n, np, "columns");
  return (std::uint64_t)s.n * (nm / s.m) + 2 * (np / s.n);
}

// ---- report writers (admmsplit_main.cpp:145-195) -----------------------------------------
void write_trace_csv(const fs::path& path, const ResidualTrace& t) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw IoError("cannot write " + path.string());
  out << "iteration,primal_norm,dual_norm,objective\n";
  for (std::size_t k = 0; k < t.size(); ++k)
    out << (k + 1) << ',' << fmt_double(t.primal[k]) << ',' << fmt_double(t.dual[k]) << ',' << fmt_double(t.objective[k])
        << '\n';
}

void write_ledger_csv(const fs::path& path, const CommLedger& ledger) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw IoError("cannot write " + path.string());
  out << "node_id,iteration,received,sent,convention\n";
  for (std::size_t node = 0; node < ledger.node_count(); ++node)
    for (std::size_t k = 0; k < ledger.iteration_count(); ++k) {
      const auto c = ledger.counts(node, k, Convention::SenderOnceBroadcast);
      out << node << ',' << (k + 1) << ',' << c.received << ',' << c.sent << ",sender_once_broadcast\n";
    }
}

JObject metrics_json(const SolveReport& r) {
  JObject j;
  j.str("schema_version", kSchemaVersion);
  if (r.metrics) {
    j.num("nmse", r.metrics->nmse);
    j.num("support_precision", r.metrics->support_precision);
    j.num("support_recall", r.metrics->support_recall);
  } else {
    j.null("nmse");
    j.null("support_precision");
    j.null("support_recall");
  }
  j.integer("iterations_run", r.iterations_run);
  j.num("objective", r.objective);
  return j;
}

int cmd_gen(const GenFlags& f, const std::string& out_dir) {
  const SensingProblem p = generate_from_flags(f);
  write_problem_dir(out_dir, p, f);
  std::cout << "wrote " << out_dir << ": H " << f.nm << "x" << f.np << ", k=" << f.k << ", kind=" << f.kind
            << ", seed=" << f.seed << "\n";
  return 0;
}

int cmd_solve(const ProblemSource& src, const MethodSpec& spec, const SolverFlags& flags, const std::string& out_dir,
              bool fingerprint) {
  check_method_divisions(spec);
  const SolveOptions opts = flags.options();
  const SensingProblem problem = src.resolve();
  const SolverConfig cfg = flags.config(src.gen.seed);
  const SolveReport report = run_method(spec, problem, cfg, opts);

  fs::create_directories(out_dir);
  const fs::path dir(out_dir);
  write_cvec((dir / "solution.cmat").string(), report.solution);
  write_trace_csv(dir / "trace.csv", report.trace);
  write_ledger_csv(dir / "ledger.csv", report.ledger);
  write_text(dir / "metrics.json", metrics_json(report).dump(0) + "\n");

  std::cout << "method=" << spec.method << " iterations=" << report.iterations_run
            << " objective=" << fmt_double(report.objective) << " primal=" << fmt_double(report.trace.primal.back())
            << " dual=" << fmt_double(report.trace.dual.back());
  if (report.metrics) std::cout << " nmse=" << fmt_double(report.metrics->nmse);
  std::cout << "\n";
  if (fingerprint) {
    std::uint64_t h = 0xCBF29CE484222325ULL;
    for (const char* name : {"solution.cmat", "trace.csv", "ledger.csv", "metrics.json"}) h = fnv1a_file(dir / name, h);
    std::cout << "fingerprint " << hex64(h) << "\n";
  }
  return 0;
}

std::vector<MethodSpec> parse_method_specs(const std::string& text) {
  std::vector<MethodSpec> specs;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) {
    if (item.empty()) continue;
    MethodSpec s;
    const auto colon = item.find(':');
    s.method = item.substr(0, colon);
    if (colon != std::string::npos) {
      const std::string arg = item.substr(colon + 1);
      try {
        if (s.method == "hybrid") {
          const auto x = arg.find('x');
          if (x == std::string::npos) throw std::invalid_argument("need MxN");
          s.m = std::stoull(arg.substr(0, x));
          s.n = std::stoull(arg.substr(x + 1));
        } else if (s.method == "consensus") {
          s.m = std::stoull(arg);
        } else if (s.method == "sectioning") {
          s.n = std::stoull(arg);
        } else {
          throw std::invalid_argument("reference takes no divisions");
        }
      } catch (const std::exception& e) {
        throw ParameterError("bad method spec '" + item + "': " + e.what());
      }
    }
    check_method_divisions(s);
    specs.push_back(s);
  }
  if (specs.empty()) throw ParameterError("no methods given");
  return specs;
}

std::string spec_label(const MethodSpec& s) {
  std::string label = s.method;
  if (s.method == "consensus") label += ":" + std::to_string(s.m);
  if (s.method == "sectioning") label += ":" + std::to_string(s.n);
  if (s.method == "hybrid") label += ":" + std::to_string(s.m) + "x" + std::to_string(s.n);
  return label;
}

struct CompareEntry {
  JObject j;
  std::string label;
  std::map<std::string, std::optional<double>> val;  // keys the winners table ranks
};

int cmd_compare(const ProblemSource& src, const std::string& methods_text, const SolverFlags& flags,
                const std::string& out_path, bool fingerprint) {
  const std::vector<MethodSpec> specs = parse_method_specs(methods_text);
  const SolveOptions opts = flags.options();
  const SensingProblem problem = src.resolve();
  const SolverConfig cfg = flags.config(src.gen.seed);

  std::vector<CompareEntry> entries;
  for (const MethodSpec& spec : specs) {
    const auto start = std::chrono::steady_clock::now();
    const SolveReport report = run_method(spec, problem, cfg, opts);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
    CompareEntry e;
    e.label = spec_label(spec);
    e.j.str("method", spec.method);
    e.j.str("label", e.label);
    if (spec.m > 0) e.j.integer("m", spec.m); else e.j.null("m");
    if (spec.n > 0) e.j.integer("n", spec.n); else e.j.null("n");
    e.j.num("objective", report.objective);
    e.j.num("final_primal", report.trace.primal.back());
    e.j.num("final_dual", report.trace.dual.back());
    e.j.integer("iterations_run", report.iterations_run);
    e.val["objective"] = report.objective;
    e.val["final_primal"] = report.trace.primal.back();
    if (report.metrics) {
      e.j.num("nmse", report.metrics->nmse);
      e.val["nmse"] = report.metrics->nmse;
    } else {
      e.j.null("nmse");
      e.val["nmse"] = std::nullopt;
    }
    const auto elems = method_per_node_elements(spec, problem);
    if (elems) e.j.integer("per_node_elements", *elems); else e.j.null("per_node_elements");
    e.val["per_node_elements"] = elems ? std::optional<double>((double)*elems) : std::nullopt;
    e.j.num("wall_clock_ms", ms);
    e.val["wall_clock_ms"] = ms;
    entries.push_back(std::move(e));
  }
  auto winner = [&](const char* key, bool skip_null) -> std::string {
    std::string best = "null";
    double best_value = 0.0;
    for (const auto& e : entries) {
      const auto& v = e.val.at(key);
      if (!v) {
        if (skip_null) continue;
        return "null";
      }
      if (best == "null" || *v < best_value) {
        best = json_string(e.label);
        best_value = *v;
      }
    }
    return best;
  };
  auto render = [&](bool canonical, int indent) {
    JObject out, prob, conf, win;
    out.str("schema_version", kSchemaVersion);
    prob.integer("nm", problem.n_meas());
    prob.integer("np", problem.n_pix());
    conf.num("rho", cfg.rho);
    conf.num("lambda", cfg.lambda);
    conf.num("scl", cfg.scl);
    conf.integer("max_iters", cfg.max_iters);
    conf.num("eps_pri", cfg.eps_pri);
    conf.num("eps_dual", cfg.eps_dual);
    win.raw("objective", winner("objective", false));
    win.raw("nmse", winner("nmse", true));
    win.raw("final_primal", winner("final_primal", false));
    win.raw("communication", winner("per_node_elements", true));
    if (!canonical) win.raw("wall_clock", winner("wall_clock_ms", false));
    std::string arr = canonical ? "[" : "[\n";
    for (std::size_t i = 0; i < entries.size(); ++i) {
      JObject e = entries[i].j;
      if (canonical) e.kv.erase("wall_clock_ms");
      if (canonical)
        arr += (i ? "," : "") + e.compact();
      else
        arr += std::string(indent + 4, ' ') + e.dump(indent + 4) + (i + 1 < entries.size() ? ",\n" : "\n");
    }
    arr += canonical ? "]" : std::string(indent + 2, ' ') + "]";
    if (canonical) {
      out.raw("problem", prob.compact());
      out.raw("config", conf.compact());
      out.raw("winners", win.compact());
      out.raw("entries", arr);
      return out.compact();
    }
    out.raw("problem", prob.dump(indent + 2));
    out.raw("config", conf.dump(indent + 2));
    out.raw("winners", win.dump(indent + 2));
    out.raw("entries", arr);
    return out.dump(indent);
  };
  write_text(out_path, render(false, 0) + "\n");
  std::cout << "wrote " << out_path << " (" << entries.size() << " entries)\n";
  for (const auto& e : entries) {
    std::cout << "  " << e.label << " objective=" << fmt_double(*e.val.at("objective"));
    if (e.val.at("nmse")) std::cout << " nmse=" << fmt_double(*e.val.at("nmse"));
    std::cout << "\n";
  }
  if (fingerprint) {
    const std::string text = render(true, 0);
    std::cout << "fingerprint " << hex64(fnv1a_bytes(text.data(), text.size(), 0xCBF29CE484222325ULL)) << "\n";
  }
  return 0;
}

// ---- argument parsing (the reference uses CLI11; same option names and defaults) -----------
struct Args {
  std::map<std::string, std::string> opt;
  std::map<std::string, bool> flag;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
};

[[noreturn]] void usage(const std::string& msg) {
  std::cerr << msg << "\n"
            << "usage: admmsplit_gpu gen --nm N --np N --k N --seed S [--snr dB] [--kind K] --out DIR\n"
               "       admmsplit_gpu solve --method reference|consensus|sectioning|hybrid [--m M] [--n N]\n"
               "                     (--problem DIR | --nm --np --k --seed [--snr] [--kind]) [--rho] [--lambda] [--scl]\n"
               "                     [--iters] [--eps-pri] [--eps-dual] [--preset paper] [--threads] [--ragged]\n"
               "                     [--device gpu[:K]] [--gpus a,b,..] [--dtype c128|c64] [--no-trace-objective]\n"
               "                     --out DIR [--fingerprint]\n"
               "       admmsplit_gpu compare --methods reference,consensus:M,sectioning:N,hybrid:MxN (problem / solver\n"
               "                     flags as for solve) [--out compare.json] [--fingerprint]\n";
  std::exit(kExitUsage);
}

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& options,
                const std::vector<std::string>& flags) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string t = argv[i];
    std::string val;
    bool has_val = false;
    const auto eq = t.find('=');
    if (t.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = t.substr(eq + 1);
      t = t.substr(0, eq);
      has_val = true;
    }
    if (std::find(flags.begin(), flags.end(), t) != flags.end()) {
      a.flag[t] = true;
    } else if (std::find(options.begin(), options.end(), t) != options.end()) {
      if (!has_val) {
        if (i + 1 >= argc) usage(t + ": 1 required TEXT missing");
        val = argv[++i];
      }
      a.opt[t] = val;
    } else {
      usage("The following argument was not expected: " + t);
    }
  }
  return a;
}

std::uint64_t to_u64(const Args& a, const std::string& k, std::uint64_t dflt) {
  if (!a.has(k)) return dflt;
  try {
    std::size_t pos = 0;
    const std::uint64_t v = std::stoull(a.opt.at(k), &pos);
    if (pos != a.opt.at(k).size() || a.opt.at(k)[0] == '-') throw std::invalid_argument("");
    return v;
  } catch (const std::exception&) {
    usage("Could not convert: " + k + " = " + a.opt.at(k));
  }
}

double to_f64(const Args& a, const std::string& k, double dflt) {
  if (!a.has(k)) return dflt;
  const std::string& s = a.opt.at(k);
  if (s == "inf" || s == "+inf") return std::numeric_limits<double>::infinity();
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (end == s.c_str() || *end) usage("Could not convert: " + k + " = " + s);
  return v;
}

const std::vector<std::string> kProblemOpts = {"--problem", "--nm", "--np", "--k", "--snr", "--seed", "--kind"};
const std::vector<std::string> kSolverOpts = {"--rho", "--lambda", "--scl", "--iters", "--eps-pri", "--eps-dual",
                                              "--preset", "--threads", "--device", "--gpus", "--dtype"};

void fill_source(const Args& a, ProblemSource& src) {
  src.problem_dir = a.has("--problem") ? a.opt.at("--problem") : "";
  src.gen.nm = to_u64(a, "--nm", 0);
  src.gen.np = to_u64(a, "--np", 0);
  src.gen.k = to_u64(a, "--k", 0);
  src.gen.snr_db = to_f64(a, "--snr", std::numeric_limits<double>::infinity());
  src.gen.seed = to_u64(a, "--seed", 0);
  if (a.has("--kind")) {
    src.gen.kind = a.opt.at("--kind");
    if (src.gen.kind != "complex-gaussian" && src.gen.kind != "random-phase")
      usage("--kind: " + src.gen.kind + " not in {complex-gaussian,random-phase}");
  }
  src.seed_given = a.has("--seed");
  for (const char* k : {"--nm", "--np", "--k", "--snr", "--seed", "--kind"}) src.any_gen_flag |= a.has(k);
}

void fill_solver(const Args& a, SolverFlags& f) {
  f.rho = to_f64(a, "--rho", f.rho);
  f.lambda = to_f64(a, "--lambda", f.lambda);
  f.scl = to_f64(a, "--scl", f.scl);
  f.scl_given = a.has("--scl");
  f.iters = to_u64(a, "--iters", f.iters);
  f.eps_pri = to_f64(a, "--eps-pri", 0.0);
  f.eps_dual = to_f64(a, "--eps-dual", 0.0);
  if (a.has("--preset")) {
    f.preset = a.opt.at("--preset");
    if (f.preset != "paper") usage("--preset: " + f.preset + " not in {paper}");
  }
  f.threads = to_u64(a, "--threads", 1);
  f.ragged = a.flag.count("--ragged") != 0;
  if (a.has("--device")) f.device = a.opt.at("--device");
  if (a.has("--gpus")) f.gpus = a.opt.at("--gpus");
  if (a.has("--dtype")) f.dtype = a.opt.at("--dtype");
  f.trace_objective = a.flag.count("--no-trace-objective") == 0;
}

std::vector<std::string> join(std::initializer_list<std::vector<std::string>> lists) {
  std::vector<std::string> o;
  for (const auto& l : lists) o.insert(o.end(), l.begin(), l.end());
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) usage("A subcommand is required");
  const std::string cmd = argv[1];
  try {
    if (cmd == "gen") {
      const Args a = parse_args(argc, argv, 2, {"--nm", "--np", "--k", "--snr", "--seed", "--kind", "--out"}, {});
      for (const char* k : {"--nm", "--np", "--k", "--seed", "--out"})
        if (!a.has(k)) usage(std::string(k) + " is required");
      ProblemSource src;
      fill_source(a, src);
      return cmd_gen(src.gen, a.opt.at("--out"));
    }
    if (cmd == "solve") {
      const Args a = parse_args(argc, argv, 2, join({kProblemOpts, kSolverOpts, {"--method", "--m", "--n", "--out"}}),
                                {"--ragged", "--fingerprint", "--no-trace-objective"});
      for (const char* k : {"--method", "--out"})
        if (!a.has(k)) usage(std::string(k) + " is required");
      MethodSpec spec;
      spec.method = a.opt.at("--method");
      if (spec.method != "reference" && spec.method != "consensus" && spec.method != "sectioning" &&
          spec.method != "hybrid")
        usage("--method: " + spec.method + " not in {reference,consensus,sectioning,hybrid}");
      spec.m = to_u64(a, "--m", 0);
      spec.n = to_u64(a, "--n", 0);
      ProblemSource src;
      fill_source(a, src);
      SolverFlags flags;
      fill_solver(a, flags);
      return cmd_solve(src, spec, flags, a.opt.at("--out"), a.flag.count("--fingerprint") != 0);
    }
    if (cmd == "compare") {
      const Args a = parse_args(argc, argv, 2, join({kProblemOpts, kSolverOpts, {"--methods", "--out"}}),
                                {"--ragged", "--fingerprint", "--no-trace-objective"});
      if (!a.has("--methods")) usage("--methods is required");
      ProblemSource src;
      fill_source(a, src);
      SolverFlags flags;
      fill_solver(a, flags);
      return cmd_compare(src, a.opt.at("--methods"), flags, a.has("--out") ? a.opt.at("--out") : "compare.json",
                         a.flag.count("--fingerprint") != 0);
    }
    if (cmd == "comm") usage("comm: the closed-form analyser is host arithmetic; use the reference CLI");
    if (cmd == "--help" || cmd == "-h") usage("admmsplit_gpu: the admmsplit runner on a B200");
    usage("unknown subcommand: " + cmd);
  } catch (const NumericalError& e) {
    std::cerr << "numerical failure: " << e.what() << " (last good iteration: " << e.last_good_iteration() << ")\n";
    return kExitNumerical;
  } catch (const SingularityError& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return kExitNumerical;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
  return 0;
}
