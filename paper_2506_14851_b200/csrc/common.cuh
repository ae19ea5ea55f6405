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

// Per (kernel, block size, dynamic shared memory, device): sets the kernel's
// max dynamic shared memory and returns its resident blocks per SM.  Cached,
// so the per-call cost of a launch is the launch alone.
int launch_setup(const void* kern, int threads, size_t smem, int* per_sm);

// K5's one-kernel stable radix sort (sort.cu), shared by pdg_order, the
// cross-rank exchange and the dispatch planner: bits [begin_bit, end_bit) of
// the u64 keys, u32 payload optional (slots_in = slots_out = nullptr).
size_t order_temp_bytes(int64_t n);
int order_sort(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* slots_in,
               uint32_t* slots_out, int64_t n, int begin_bit, int end_bit, void* temp,
               size_t temp_bytes, cudaStream_t stream);

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
// u32 inclusive scan: shfl.up's validity predicate guards the add, so no
// per-step lane compare or select (the engine runs one per unit visit)
template <int O>
__device__ __forceinline__ void scan_up_add(uint32_t& v) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
      "shfl.sync.up.b32 t|p, %0, %1, 0x0, 0xffffffff;\n\t"
      "@p add.u32 %0, %0, t;\n\t}"
      : "+r"(v)
      : "n"(O));
}
__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v) {
  scan_up_add<1>(v);
  scan_up_add<2>(v);
  scan_up_add<4>(v);
  scan_up_add<8>(v);
  scan_up_add<16>(v);
  return v;
}

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

// ---- TMA bulk copies (cp.async.bulk) completing on shared-memory mbarriers --
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// make barrier inits visible to the async (TMA) proxy
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order this thread's earlier generic-proxy shared accesses before later
// async-proxy writes into the same buffer (WAR on a reused staging slot)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned, bytes % 16 == 0), completion
// counted in bytes on `bar`; the source is read once, so it is evicted first
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

}  // namespace pdg
