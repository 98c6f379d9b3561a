// Fixed-width integer types and integral_constant for the headers that are
// also compiled at run time by NVRTC (vd_jit.cu), which has no standard
// library headers: under __CUDACC_RTC__ the few std names the device code
// uses are declared here; everywhere else the real headers are included.
#pragma once

#ifdef __CUDACC_RTC__
namespace std {
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long size_t;
typedef long ptrdiff_t;
typedef unsigned long uintptr_t;
template <class T, T V>
struct integral_constant {
  static constexpr T value = V;
};
}  // namespace std
#else
#include <cstddef>
#include <cstdint>
#include <type_traits>
#endif
