// Forced-include prefix for compiling /root/reference/proj/include/fftmv/partition.hpp
// unmodified (TEST INFRASTRUCTURE ONLY).
//
// partition.hpp:92 and :106 call detail::cast_to before its declaration at
// :109-122, and cast_to<double>(std::vector<float>) matches neither template.
// Two-phase lookup rejects that under g++ 13. Declaring the two reference
// templates up front plus the missing float->double overload makes the header
// compile as written; the overload does exactly what :117-121 intends.
#pragma once
#include <span>
#include <vector>

#include "fftmv/precision.hpp"

namespace fftmv::detail {
template <class T>
std::vector<T> cast_to(const std::vector<double>& v);
template <class T>
std::vector<double> cast_to(const std::vector<T>& v);
template <class T>
std::vector<double> cast_to(const std::vector<float>& v) {
  return cast_buffer<double>(std::span<const float>(v));
}
}  // namespace fftmv::detail
