// rowops.cuh — per-row helpers shared by the fused GAT kernels (gat.cu) and the unfused
// primitives (prims.cu): int8 row loads, exact int8->fp32 conversion, IDP4A dots, the chunked sum.
#pragma once
#include "kernels.h"

namespace tango {

template <int VPL>
struct Row {
  uint32_t w[(VPL + 3) / 4];
};
template <int VPL>
__device__ __forceinline__ Row<VPL> load_row(const int8_t* p) {
  Row<VPL> r;
  if constexpr (VPL == 16) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    r.w[0] = v.x; r.w[1] = v.y; r.w[2] = v.z; r.w[3] = v.w;
  } else if constexpr (VPL == 8) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    r.w[0] = v.x; r.w[1] = v.y;
  } else if constexpr (VPL == 4) {
    r.w[0] = __ldg(reinterpret_cast<const unsigned*>(p));
  } else if constexpr (VPL == 2) {
    r.w[0] = (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p));
  } else {
    r.w[0] = (uint32_t)__ldg(reinterpret_cast<const unsigned char*>(p));
  }
  return r;
}
template <int VPL>
__device__ __forceinline__ float row_f(const Row<VPL>& r, int k) {
  return i8_to_f(r.w[k >> 2], k & 3);
}
template <int VPL>
__device__ __forceinline__ int row_dot(const Row<VPL>& a, const Row<VPL>& b) {
  int acc = 0;
  if constexpr (VPL >= 4) {
#pragma unroll
    for (int i = 0; i < VPL / 4; ++i) acc = __dp4a((int)a.w[i], (int)b.w[i], acc);
  } else {
#pragma unroll
    for (int k = 0; k < VPL; ++k)
      acc += (int)(int8_t)((a.w[0] >> (8 * k)) & 0xFF) * (int)(int8_t)((b.w[0] >> (8 * k)) & 0xFF);
  }
  return acc;
}
__device__ __forceinline__ float i8f(int8_t v) { return __int2float_rn((int)v); }

// Chunked sum state (reading R14): partial sums restart every C_E list elements.
struct CSum {
  float total, part;
  bool folded;
  __device__ __forceinline__ void init() { total = 0.0f; part = 0.0f; folded = false; }
  __device__ __forceinline__ void fold() {
    total = folded ? __fadd_rn(total, part) : part;
    part = 0.0f;
    folded = true;
  }
  __device__ __forceinline__ float finish(int64_t len) const {
    if (len == 0) return 0.0f;
    return folded ? __fadd_rn(total, part) : part;
  }
};

// e_pre for edge (u -> v), head h (reading: two rn multiplies, one rn add, order a + b)
__device__ __forceinline__ float sddmm_add1(int8_t qs, float sS, int8_t qd, float sD) {
  return __fadd_rn(__fmul_rn(i8f(qs), sS), __fmul_rn(i8f(qd), sD));
}

inline int rows_grid(int64_t rows) {
  int64_t g = (rows + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace tango
