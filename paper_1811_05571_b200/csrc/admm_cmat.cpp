// admm_cmat.cpp — CMAT file I/O for the input pipeline (host C++; not the hot path).
//
// The reference's format (cmat_io.hpp:18-24): magic "CMX1", rows and cols as
// little-endian u64, then rows*cols row-major complex entries, each two IEEE binary64
// values (re, im).  This file adds a complex64 variant, magic "CMF1", identical except
// that each entry is two binary32 values — half the bytes, and the storage type the
// c64 plans stream (a config-4 H is 32 GiB as CMF1 instead of 64 GiB as CMX1).
//
// Reading converts on the fly to the destination type the caller asks for (a CMX1 file
// into a float2 buffer rounds each value once, exactly like admm_gen_problem's c64
// output; a CMF1 file into a double2 buffer widens exactly), so a c64 plan can be fed
// from a reference-written FP64 file without a full FP64 host copy.
//
// Validation and error classes follow read_cmat / write_cmat (cmat_io.hpp:44-116)
// check for check, including FormatError's byte offset (errors.hpp:64-73), which
// admm_cmat_error_offset() returns:
//   cannot open -> IoError; file < 20 bytes -> FormatError(file size); bad magic ->
//   FormatError(0); zero dimension / rows*cols overflow / implausible count ->
//   FormatError(4); payload short -> FormatError(file size); trailing bytes ->
//   FormatError(expected size); non-finite entry i -> FormatError(20 + i * entry size);
//   write of an empty matrix -> ParameterError; of non-finite entries -> NumericalError.
// The reference caps CMX1 at 2^32 entries (cmat_io.hpp:84-86) and so do we for CMX1;
// CMF1 allows 2^36 (config 4's 2^32-entry H fits either).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "admm_b200.h"
#include "admm_host.h"

namespace {

constexpr char kMagic128[4] = {'C', 'M', 'X', '1'};
constexpr char kMagic64[4] = {'C', 'M', 'F', '1'};
constexpr uint64_t kHeader = 20;
constexpr uint64_t kChunk = 1u << 22;  // entries per streamed chunk

struct CmatFail {
  admm_status st;
  std::string msg;
  uint64_t offset;
};

struct File {
  std::FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

uint64_t entry_bytes(admm_dtype t) { return t == ADMM_C128 ? 16 : 8; }

struct Header {
  uint64_t rows, cols, file_size;
  admm_dtype dtype;
};

// cmat_io.hpp:57-105 up to (not including) the payload scan.
Header open_and_check(File& fh, const char* path) {
  const std::string p = path ? path : "";
  fh.f = std::fopen(p.c_str(), "rb");
  if (!fh.f) throw CmatFail{ADMM_E_IO, "read_cmat: cannot open " + p, 0};
  std::fseek(fh.f, 0, SEEK_END);
  const long long end = std::ftell(fh.f);
  std::fseek(fh.f, 0, SEEK_SET);
  const uint64_t size = end < 0 ? 0 : (uint64_t)end;
  if (size < kHeader)
    throw CmatFail{ADMM_E_FORMAT,
                   "read_cmat: truncated header in " + p + " (file ends at byte " + std::to_string(size) +
                       ", header needs 20)",
                   size};
  unsigned char h[kHeader];
  if (std::fread(h, 1, kHeader, fh.f) != kHeader) throw CmatFail{ADMM_E_IO, "read_cmat: read failed for " + p, 0};
  admm_dtype t;
  if (std::memcmp(h, kMagic128, 4) == 0)
    t = ADMM_C128;
  else if (std::memcmp(h, kMagic64, 4) == 0)
    t = ADMM_C64;
  else
    throw CmatFail{ADMM_E_FORMAT, "read_cmat: bad magic in " + p, 0};
  uint64_t rows = 0, cols = 0;
  std::memcpy(&rows, h + 4, 8);
  std::memcpy(&cols, h + 12, 8);
  if (rows == 0 || cols == 0) throw CmatFail{ADMM_E_FORMAT, "read_cmat: zero dimension declared in " + p, 4};
  if (rows > UINT64_MAX / cols) throw CmatFail{ADMM_E_FORMAT, "read_cmat: dimension overflow in " + p, 4};
  const uint64_t entries = rows * cols;
  const uint64_t cap = t == ADMM_C128 ? (1ull << 32) : (1ull << 36);
  if (entries > cap) throw CmatFail{ADMM_E_FORMAT, "read_cmat: implausible element count in " + p, 4};
  const uint64_t expected = kHeader + entries * entry_bytes(t);
  if (size < expected)
    throw CmatFail{ADMM_E_FORMAT,
                   "read_cmat: declared " + std::to_string(entries) + " entries but " + p + " ends at byte " +
                       std::to_string(size) + " (expected " + std::to_string(expected) + ")",
                   size};
  if (size > expected) throw CmatFail{ADMM_E_FORMAT, "read_cmat: trailing bytes after payload in " + p, expected};
  return Header{rows, cols, size, t};
}

template <typename F>
admm_status guarded(F&& f) {
  try {
    admm_host_set_error("", 0);
    f();
    return ADMM_OK;
  } catch (const CmatFail& e) {
    admm_host_set_error(e.msg.c_str(), e.offset);
    return e.st;
  } catch (const std::exception& e) {
    admm_host_set_error(e.what(), 0);
    return ADMM_E_IO;
  }
}

template <typename Src, typename Dst>
void convert_chunk(const Src* s, Dst* d, uint64_t n_reals, uint64_t first_entry, const std::string& p) {
  for (uint64_t k = 0; k < n_reals; ++k) {
    if (!std::isfinite(s[k])) {
      const uint64_t e = first_entry + k / 2;
      throw CmatFail{ADMM_E_FORMAT, "read_cmat: non-finite entry " + std::to_string(e) + " in " + p,
                     kHeader + e * 2 * sizeof(Src)};
    }
    d[k] = (Dst)s[k];
  }
}

template <typename Src, typename Dst>
void read_payload(File& fh, const Header& h, Dst* dst, const std::string& p) {
  const uint64_t entries = h.rows * h.cols;
  std::vector<Src> buf;
  if (!std::is_same<Src, Dst>::value) buf.resize(2 * std::min(entries, kChunk));
  for (uint64_t e0 = 0; e0 < entries; e0 += kChunk) {
    const uint64_t n = std::min(kChunk, entries - e0);
    Src* s = std::is_same<Src, Dst>::value ? reinterpret_cast<Src*>(dst + 2 * e0) : buf.data();
    if (std::fread(s, sizeof(Src), 2 * n, fh.f) != 2 * n)
      throw CmatFail{ADMM_E_IO, "read_cmat: read failed for " + p, 0};
    convert_chunk<Src, Dst>(s, dst + 2 * e0, 2 * n, e0, p);
  }
}

}  // namespace

extern "C" {

admm_status admm_cmat_info(const char* path, uint64_t* rows, uint64_t* cols, admm_dtype* dtype) {
  return guarded([&] {
    File fh;
    const Header h = open_and_check(fh, path);
    if (rows) *rows = h.rows;
    if (cols) *cols = h.cols;
    if (dtype) *dtype = h.dtype;
  });
}

admm_status admm_cmat_read(const char* path, void* dst, uint64_t capacity_entries, admm_dtype dst_dtype) {
  return guarded([&] {
    if (!dst) throw CmatFail{ADMM_E_STATE, "read_cmat: null destination", 0};
    if (dst_dtype != ADMM_C128 && dst_dtype != ADMM_C64) throw CmatFail{ADMM_E_PARAMETER, "read_cmat: dtype", 0};
    File fh;
    const Header h = open_and_check(fh, path);
    if (h.rows * h.cols > capacity_entries)
      throw CmatFail{ADMM_E_DIMENSION,
                     "read_cmat: " + std::string(path) + " holds " + std::to_string(h.rows * h.cols) +
                         " entries, destination has room for " + std::to_string(capacity_entries),
                     0};
    const std::string p = path;
    if (h.dtype == ADMM_C128 && dst_dtype == ADMM_C128)
      read_payload<double, double>(fh, h, static_cast<double*>(dst), p);
    else if (h.dtype == ADMM_C128)
      read_payload<double, float>(fh, h, static_cast<float*>(dst), p);
    else if (dst_dtype == ADMM_C128)
      read_payload<float, double>(fh, h, static_cast<double*>(dst), p);
    else
      read_payload<float, float>(fh, h, static_cast<float*>(dst), p);
  });
}

admm_status admm_cmat_write(const char* path, const void* src, uint64_t rows, uint64_t cols, admm_dtype src_dtype,
                            admm_dtype file_dtype) {
  return guarded([&] {
    if (rows == 0 || cols == 0 || !src) throw CmatFail{ADMM_E_PARAMETER, "write_cmat: empty matrix", 0};
    if (rows > UINT64_MAX / cols) throw CmatFail{ADMM_E_PARAMETER, "write_cmat: dimension overflow", 0};
    if ((src_dtype != ADMM_C128 && src_dtype != ADMM_C64) || (file_dtype != ADMM_C128 && file_dtype != ADMM_C64))
      throw CmatFail{ADMM_E_PARAMETER, "write_cmat: dtype", 0};
    const uint64_t n = 2 * rows * cols;
    // all_finite check first (cmat_io.hpp:45-46); rounding to binary32 may overflow to
    // inf, which is equally non-finite in the written file
    for (uint64_t k = 0; k < n; ++k) {
      const double x = src_dtype == ADMM_C128 ? static_cast<const double*>(src)[k] : static_cast<const float*>(src)[k];
      if (!std::isfinite(x) || (file_dtype == ADMM_C64 && !std::isfinite((float)x)))
        throw CmatFail{ADMM_E_NUMERICAL, "write_cmat: non-finite entries", 0};
    }
    const std::string p = path ? path : "";
    File fh;
    fh.f = std::fopen(p.c_str(), "wb");
    if (!fh.f) throw CmatFail{ADMM_E_IO, "write_cmat: cannot open " + p, 0};
    bool ok = std::fwrite(file_dtype == ADMM_C128 ? kMagic128 : kMagic64, 1, 4, fh.f) == 4 &&
              std::fwrite(&rows, 8, 1, fh.f) == 1 && std::fwrite(&cols, 8, 1, fh.f) == 1;
    if (ok && file_dtype == src_dtype) {
      ok = std::fwrite(src, (size_t)entry_bytes(src_dtype) / 2, n, fh.f) == n;
    } else if (ok) {
      std::vector<unsigned char> buf(2 * kChunk * 8);
      for (uint64_t k0 = 0; ok && k0 < n; k0 += 2 * kChunk) {
        const uint64_t m = std::min<uint64_t>(2 * kChunk, n - k0);
        if (file_dtype == ADMM_C64) {
          float* d = reinterpret_cast<float*>(buf.data());
          for (uint64_t k = 0; k < m; ++k) d[k] = (float)static_cast<const double*>(src)[k0 + k];
          ok = std::fwrite(d, 4, m, fh.f) == m;
        } else {
          double* d = reinterpret_cast<double*>(buf.data());
          for (uint64_t k = 0; k < m; ++k) d[k] = (double)static_cast<const float*>(src)[k0 + k];
          ok = std::fwrite(d, 8, m, fh.f) == m;
        }
      }
    }
    ok = ok && std::fflush(fh.f) == 0;
    if (!ok) throw CmatFail{ADMM_E_IO, "write_cmat: write failed for " + p, 0};
  });
}

}  // extern "C"
