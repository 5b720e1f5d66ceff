// Device helpers shared by the SIMT kernel translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace stn {
namespace dev {


template <class R>
struct Cx;
template <>
struct Cx<float> {
  using T = float2;
};
template <>
struct Cx<double> {
  using T = double2;
};
template <class R>
using cx_t = typename Cx<R>::T;

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// acc += a * b
template <bool EXACT, class T>
__device__ __forceinline__ void cmac(T &acc, const T a, const T b) {
  if constexpr (EXACT) {
    auto re = sub_rn(mul_rn(a.x, b.x), mul_rn(a.y, b.y));
    auto im = add_rn(mul_rn(a.x, b.y), mul_rn(a.y, b.x));
    acc.x = add_rn(acc.x, re);
    acc.y = add_rn(acc.y, im);
  } else {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
  }
}

inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b > max_blocks) b = max_blocks;
  if (b < 1) b = 1;
  return int(b);
}

}  // namespace dev
}  // namespace stn
