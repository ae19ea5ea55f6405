// Shared helpers for the sm_100a kernels behind include/pdg_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/pdg_b200.h"

namespace pdg {

// Thread-local last-error text for pdg_last_error().
void set_error(const char* fmt, ...);

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PDG_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return PDG_ECUDA;
}

// After a <<<>>> launch: report configuration errors without syncing.
inline int launch_status(const char* what) {
  return cuda_status(cudaGetLastError(), what);
}

int sm_count();

constexpr unsigned kFull = 0xffffffffu;

// ---- exact float64 helpers (never contracted into FMA) --------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Exact int -> double / u16 -> float without the XU conversion pipe.
__device__ __forceinline__ double small_int_to_double(int j) {   // 0 <= j < 2^31
  return dsub(__hiloint2double(0x43300000, j), 4503599627370496.0);
}
__device__ __forceinline__ float u16_to_float(uint32_t c) {       // c < 2^23
  return __int_as_float(0x4B000000u | c) - 8388608.f;
}

// Bucket midpoint exactly as distributions.py:103,131 evaluates it:
//   ((lo + j*w) + (lo + (j+1)*w)) / 2.0      (each op rounded separately)
__device__ __forceinline__ double bucket_mid(double lo, double w, int j) {
  const double jd = small_int_to_double(j);
  double a = dadd(lo, dmul(jd, w));
  double b = dadd(lo, dmul(dadd(jd, 1.0), w));
  return dmul(dadd(a, b), 0.5);
}

// ---- warp primitives -------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

}  // namespace pdg
