// admm_generate.cpp — synthetic inputs for the benchmark configs (host C++).
//
// Input tooling, not the hot path.  Two families:
//   * admm_gen_problem: the reference's seeded generator (generate.hpp:32-89 with the
//     Xoshiro256++/SplitMix64/Box-Muller stream of rng.hpp:13-84), reproduced
//     bit-for-bit (tests/test_generate.py pins its FNV hash against fixtures made by
//     the unmodified reference).  The RNG stream is drawn sequentially; the
//     Box-Muller / unit-phase transforms run on all host cores.
//   * admm_gen_cra: the CRA-like structured sensing matrix of BASELINE.json
//     configs 3 and 5 (no reference counterpart — the paper's measured CRA operator
//     was never published; conventions are fixed in DESIGN.md §Inputs).
// Compiled with -O2 -ffp-contract=off so the FP64 arithmetic matches the reference.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "admm_b200.h"

namespace {

struct SplitMix64 {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
};

struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    SplitMix64 sm{seed};
    for (auto& w : s) w = sm.next();
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
};

constexpr double kPi = 3.14159265358979323846;

inline void box_muller(uint64_t a, uint64_t b, double& re, double& im) {
  const double u1 = 1.0 - (double)(a >> 11) * 0x1.0p-53;
  const double u2 = (double)(b >> 11) * 0x1.0p-53;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double th = 2.0 * kPi * u2;
  re = r * std::cos(th);
  im = r * std::sin(th);
}

inline void unit_phase(uint64_t a, double& re, double& im) {
  const double th = 2.0 * kPi * ((double)(a >> 11) * 0x1.0p-53);
  re = std::cos(th);
  im = std::sin(th);
}

template <typename F>
void parallel_rows(uint64_t n, F&& f) {
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 64) nt = 1;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (uint64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) f(i);
    });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

// generate.hpp:32-89.  kind 0 = complex-gaussian (x+iy)/sqrt(2 m), 1 = random-phase
// e^{i theta}/sqrt(m).  h_dtype selects the host output of H (ADMM_C128: double
// pairs, ADMM_C64: the same values rounded to float pairs); g and truth are FP64, and
// g is formed from the FP64 H exactly as the reference does.
admm_status admm_gen_problem(uint64_t n_meas, uint64_t n_pix, uint64_t k, double snr_db, uint64_t seed,
                             int kind, void* h_out, admm_dtype h_dtype, double* g, double* truth,
                             double* noise_sigma) {
  if (n_meas < 1 || n_pix < 1 || k < 1 || k > n_pix || std::isnan(snr_db) || (kind != 0 && kind != 1))
    return ADMM_E_PARAMETER;
  Xoshiro rng(seed);
  const uint64_t total = n_meas * n_pix;
  const double scale = kind == 0 ? 1.0 / std::sqrt(2.0 * (double)n_meas) : 1.0 / std::sqrt((double)n_meas);
  // H, drawn row-major (draw order is part of the reproducibility contract,
  // generate.hpp:30-31).  Raw words are drawn sequentially in row slabs, the
  // transcendental transforms of each slab run in parallel.
  const uint64_t per = kind == 0 ? 2 : 1;
  const uint64_t slab_rows = std::max<uint64_t>(1, (1ull << 24) / n_pix);
  std::vector<uint64_t> raw;
  std::vector<double> hrow_keep;  // FP64 copy of the support columns, for g
  double* h64 = h_dtype == ADMM_C128 ? static_cast<double*>(h_out) : nullptr;
  float* h32 = h_dtype == ADMM_C64 ? static_cast<float*>(h_out) : nullptr;
  if (!h64 && !h32) return ADMM_E_PARAMETER;
  // full FP64 H is needed for g = H truth; for c64 output keep FP64 values of the
  // support columns only (the support is drawn after H, so buffer all of H's FP64
  // values per slab and gather the support columns once it is known: instead,
  // recompute g from the raw stream below).
  std::vector<double> slab;
  for (uint64_t r0 = 0; r0 < n_meas; r0 += slab_rows) {
    const uint64_t nr = std::min(slab_rows, n_meas - r0);
    raw.resize(nr * n_pix * per);
    for (auto& w : raw) w = rng.next();
    if (h64) {
      double* dst = h64 + 2 * r0 * n_pix;
      parallel_rows(nr, [&](uint64_t r) {
        for (uint64_t c = 0; c < n_pix; ++c) {
          const uint64_t e = r * n_pix + c;
          double re, im;
          if (kind == 0)
            box_muller(raw[2 * e], raw[2 * e + 1], re, im);
          else
            unit_phase(raw[e], re, im);
          dst[2 * e] = re * scale;
          dst[2 * e + 1] = im * scale;
        }
      });
    } else {
      float* dst = h32 + 2 * r0 * n_pix;
      parallel_rows(nr, [&](uint64_t r) {
        for (uint64_t c = 0; c < n_pix; ++c) {
          const uint64_t e = r * n_pix + c;
          double re, im;
          if (kind == 0)
            box_muller(raw[2 * e], raw[2 * e + 1], re, im);
          else
            unit_phase(raw[e], re, im);
          dst[2 * e] = (float)(re * scale);
          dst[2 * e + 1] = (float)(im * scale);
        }
      });
    }
  }
  // support: partial Fisher-Yates (generate.hpp:64-69), values unit phase (70-71)
  std::vector<uint64_t> pos(n_pix);
  for (uint64_t i = 0; i < n_pix; ++i) pos[i] = i;
  for (uint64_t t = 0; t < k; ++t) {
    const uint64_t j = t + rng.next() % (n_pix - t);
    std::swap(pos[t], pos[j]);
  }
  std::memset(truth, 0, n_pix * 16);
  for (uint64_t t = 0; t < k; ++t) unit_phase(rng.next(), truth[2 * pos[t]], truth[2 * pos[t] + 1]);
  std::vector<uint64_t> supp(pos.begin(), pos.begin() + (std::ptrdiff_t)k);
  std::sort(supp.begin(), supp.end());
  // clean = H truth (linalg.hpp:97-111).  Zero entries of truth only add signed
  // zeros, so summing the support in ascending column order gives the reference's
  // bits.  For c64 output H is regenerated in FP64 for the support columns.
  std::vector<double> hs(2 * n_meas * k);
  if (h64) {
    parallel_rows(n_meas, [&](uint64_t r) {
      for (uint64_t t = 0; t < k; ++t) {
        hs[2 * (r * k + t)] = h64[2 * (r * n_pix + supp[t])];
        hs[2 * (r * k + t) + 1] = h64[2 * (r * n_pix + supp[t]) + 1];
      }
    });
  } else {
    Xoshiro rr(seed);
    for (uint64_t r = 0; r < n_meas; ++r) {
      uint64_t t = 0;
      for (uint64_t c = 0; c < n_pix; ++c) {
        double re = 0.0, im = 0.0;
        if (kind == 0) {
          const uint64_t a = rr.next(), b = rr.next();
          if (t < k && supp[t] == c) box_muller(a, b, re, im);
        } else {
          const uint64_t a = rr.next();
          if (t < k && supp[t] == c) unit_phase(a, re, im);
        }
        if (t < k && supp[t] == c) {
          hs[2 * (r * k + t)] = re * scale;
          hs[2 * (r * k + t) + 1] = im * scale;
          ++t;
        }
      }
    }
  }
  parallel_rows(n_meas, [&](uint64_t r) {
    double ar = 0.0, ai = 0.0;
    for (uint64_t t = 0; t < k; ++t) {
      const double a = hs[2 * (r * k + t)], b = hs[2 * (r * k + t) + 1];
      const double c = truth[2 * supp[t]], d = truth[2 * supp[t] + 1];
      ar += a * c - b * d;
      ai += a * d + b * c;
    }
    g[2 * r] = ar;
    g[2 * r + 1] = ai;
  });
  *noise_sigma = 0.0;
  if (std::isfinite(snr_db)) {  // exact-SNR noise, generate.hpp:76-85
    std::vector<double> w(2 * n_meas);
    for (uint64_t i = 0; i < n_meas; ++i) {
      const uint64_t a = rng.next();  // u1 then u2: draw order matters (rng.hpp:59-65)
      const uint64_t b = rng.next();
      box_muller(a, b, w[2 * i], w[2 * i + 1]);
    }
    double ws = 0.0, ss = 0.0;
    for (uint64_t i = 0; i < n_meas; ++i) ws += w[2 * i] * w[2 * i] + w[2 * i + 1] * w[2 * i + 1];
    for (uint64_t i = 0; i < n_meas; ++i) ss += g[2 * i] * g[2 * i] + g[2 * i + 1] * g[2 * i + 1];
    const double w_norm = std::sqrt(ws), s_norm = std::sqrt(ss);
    const double alpha = w_norm > 0.0 ? s_norm / (w_norm * std::pow(10.0, snr_db / 20.0)) : 0.0;
    for (uint64_t i = 0; i < n_meas; ++i) {
      g[2 * i] = g[2 * i] + alpha * w[2 * i];
      g[2 * i + 1] = g[2 * i + 1] + alpha * w[2 * i + 1];
    }
    *noise_sigma = alpha;
  }
  return ADMM_OK;
}

// CRA-like structured sensing matrix (BASELINE.json configs 3 and 5).
//   n_tx transceivers at uniform-random (x, y) on [-a/2, a/2]^2, z = 0;
//   n_freq frequencies linspace(f0, f1); row = t * n_freq + f;
//   voxels on a g^3 grid, spacing d, centred at (0, 0, z0); v = (ix*g + iy)*g + iz,
//   r_v = ((ix-(g-1)/2) d, (iy-(g-1)/2) d, z0 + (iz-(g-1)/2) d);
//   H[(t,f), v] = exp(-j 2 k_f |x_t - r_v| + j phi[t, f, v mod n_facets]) / |x_t - r_v|^2,
//   k_f = 2 pi f / c, phi ~ U[0, 2 pi); each row is normalised to unit L2 norm.
// Draws (one Xoshiro256++ stream): transceiver x, y (t ascending), then phi (t, f,
// facet ascending).  Output H as complex64 or complex128 (values computed in FP64).
admm_status admm_gen_cra(uint64_t n_tx, uint64_t n_freq, uint64_t grid, double spacing, double z0,
                         double aperture, double f0, double f1, uint64_t n_facets, uint64_t seed,
                         void* h_out, admm_dtype h_dtype) {
  if (!n_tx || !n_freq || !grid || !n_facets || !h_out) return ADMM_E_PARAMETER;
  Xoshiro rng(seed);
  std::vector<double> tx(2 * n_tx);
  for (uint64_t t = 0; t < n_tx; ++t) {
    tx[2 * t] = (rng.unit() - 0.5) * aperture;
    tx[2 * t + 1] = (rng.unit() - 0.5) * aperture;
  }
  std::vector<double> phi(n_tx * n_freq * n_facets);
  for (auto& x : phi) x = 2.0 * kPi * rng.unit();
  const uint64_t n_vox = grid * grid * grid, rows = n_tx * n_freq;
  const double c0 = 299792458.0, half = 0.5 * (double)(grid - 1);
  parallel_rows(rows, [&](uint64_t row) {
    const uint64_t t = row / n_freq, f = row % n_freq;
    const double freq = n_freq == 1 ? f0 : f0 + (f1 - f0) * (double)f / (double)(n_freq - 1);
    const double kf = 2.0 * kPi * freq / c0;
    std::vector<double> val(2 * n_vox);
    double nrm = 0.0;
    for (uint64_t v = 0; v < n_vox; ++v) {
      const uint64_t ix = v / (grid * grid), iy = (v / grid) % grid, iz = v % grid;
      const double dx = ((double)ix - half) * spacing - tx[2 * t];
      const double dy = ((double)iy - half) * spacing - tx[2 * t + 1];
      const double dz = z0 + ((double)iz - half) * spacing;
      const double d = std::sqrt(dx * dx + dy * dy + dz * dz);
      const double ph = -2.0 * kf * d + phi[(t * n_freq + f) * n_facets + v % n_facets];
      const double a = 1.0 / (d * d);
      val[2 * v] = a * std::cos(ph);
      val[2 * v + 1] = a * std::sin(ph);
      nrm += a * a;
    }
    const double inv = 1.0 / std::sqrt(nrm);
    if (h_dtype == ADMM_C128) {
      double* dst = static_cast<double*>(h_out) + 2 * row * n_vox;
      for (uint64_t e = 0; e < 2 * n_vox; ++e) dst[e] = val[e] * inv;
    } else {
      float* dst = static_cast<float*>(h_out) + 2 * row * n_vox;
      for (uint64_t e = 0; e < 2 * n_vox; ++e) dst[e] = (float)(val[e] * inv);
    }
  });
  return ADMM_OK;
}

}  // extern "C"
