// fftmv/vector_io.hpp -- FMV1 vector persistence (SPEC.md cli module,
// save_vector / load_vector). The reference specifies the
// format but ships no implementation; this is it, bit-exact to the spec:
//   "FMV1" (4 bytes), then little-endian u64 space_extent, time_extent,
//   layout code (0 SOTI, 1 TOSI), precision code (0 f64, 1 f32), domain code
//   (0 time, 1 frequency), then the raw little-endian scalars
//   (space*time scalars, x2 for the frequency domain's complex elements).
// load(save(v)) is bitwise identical. Errors name the defect: bad magic,
// truncated file, code out of range, truncated/oversized payload.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "block_vector.hpp"

namespace fftmv {

namespace detail {
static_assert(sizeof(double) == 8 && sizeof(float) == 4, "IEEE binary64/binary32 expected");
inline void put_u64(std::string& s, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) s.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}
inline std::uint64_t get_u64(const unsigned char* p) {
  std::uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
template <class T>
void put_scalars(std::string& s, const std::vector<T>& v) {  // little-endian, host assumed LE (x86/ARM)
  const std::size_t off = s.size();
  s.resize(off + v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(s.data() + off, v.data(), v.size() * sizeof(T));
}
}  // namespace detail

inline std::string encode_vector(const BlockVector& v) {
  if (v.precision == Precision::Half) throw std::invalid_argument("FMV1: fp16 vectors have no precision code");
  v.validate();
  std::string s = "FMV1";
  detail::put_u64(s, v.space_extent);
  detail::put_u64(s, v.time_extent);
  detail::put_u64(s, v.layout == Layout::SOTI ? 0 : 1);
  detail::put_u64(s, v.precision == Precision::Double ? 0 : 1);
  detail::put_u64(s, v.domain == Domain::Time ? 0 : 1);
  if (v.precision == Precision::Double) detail::put_scalars(s, v.f64);
  else detail::put_scalars(s, v.f32);
  return s;
}

inline BlockVector decode_vector(const std::string& bytes) {
  if (bytes.size() < 4 || std::memcmp(bytes.data(), "FMV1", 4) != 0) throw std::invalid_argument("FMV1: bad magic");
  if (bytes.size() < 44) throw std::invalid_argument("FMV1: truncated file (header)");
  const auto* p = reinterpret_cast<const unsigned char*>(bytes.data()) + 4;
  BlockVector v;
  v.space_extent = detail::get_u64(p);
  v.time_extent = detail::get_u64(p + 8);
  const std::uint64_t lay = detail::get_u64(p + 16), prec = detail::get_u64(p + 24), dom = detail::get_u64(p + 32);
  if (lay > 1) throw std::invalid_argument("FMV1: layout code out of range (" + std::to_string(lay) + ")");
  if (prec > 1) throw std::invalid_argument("FMV1: precision code out of range (" + std::to_string(prec) + ")");
  if (dom > 1) throw std::invalid_argument("FMV1: domain code out of range (" + std::to_string(dom) + ")");
  v.layout = lay == 0 ? Layout::SOTI : Layout::TOSI;
  v.precision = prec == 0 ? Precision::Double : Precision::Single;
  v.domain = dom == 0 ? Domain::Time : Domain::Frequency;
  const std::size_t es = prec == 0 ? 8 : 4;
  const std::size_t scalars = v.space_extent * v.time_extent * (dom == 1 ? 2 : 1);
  const std::size_t have = bytes.size() - 44;
  if (v.space_extent == 0 || v.time_extent == 0 || scalars / v.time_extent / (dom == 1 ? 2 : 1) != v.space_extent ||
      have != scalars * es)
    throw std::invalid_argument("FMV1: truncated/oversized payload (" + std::to_string(have) + " bytes for " +
                                std::to_string(scalars) + " scalars of " + std::to_string(es) + " bytes)");
  if (prec == 0) {
    v.f64.resize(scalars);
    std::memcpy(v.f64.data(), bytes.data() + 44, have);
  } else {
    v.f32.resize(scalars);
    std::memcpy(v.f32.data(), bytes.data() + 44, have);
  }
  return v;
}

inline void save_vector(const std::string& path, const BlockVector& v) {
  const std::string s = encode_vector(v);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw std::runtime_error("save_vector: cannot open " + path);
  f.write(s.data(), static_cast<std::streamsize>(s.size()));
  if (!f) throw std::runtime_error("save_vector: write failed: " + path);
}

inline BlockVector load_vector(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("load_vector: cannot open " + path);
  std::string s((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  return decode_vector(s);
}

}  // namespace fftmv
