// numpy-compatible PCG64 (XSL-RR 128/64) + SeedSequence on the device, with
// O(1) jump-ahead from constant tables, so every warp lane can produce the
// word at any stream position of numpy.random.default_rng(seed).
//
// numpy semantics reproduced (numpy/random/src/pcg64, bit_generator.pyx):
//   state' = state * M + inc  (mod 2^128);  out = rotr64(hi ^ lo, hi >> 58)
//   default_rng(seed) -> SeedSequence(seed).generate_state(4, uint64)
//                     -> srandom(initstate = w0:w1, initseq = w2:w3)
//   random()          -> (word >> 11) * 2^-53
//   next_uint32       -> low half of a fresh word, high half buffered
#pragma once

#include <stdint.h>

namespace pdg {

struct U128 {
  uint64_t lo, hi;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  asm("add.cc.u64 %0, %2, %4;\n\taddc.u64 %1, %3, %5;"
      : "=l"(r.lo), "=l"(r.hi)
      : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
  return r;
}

// XSL-RR output: rotr64(hi ^ lo, hi >> 58), as two 32-bit funnel shifts
__device__ __forceinline__ uint64_t pcg_out(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const uint32_t r = uint32_t(s.hi >> 58);
  const uint32_t xl = uint32_t(x), xh = uint32_t(x >> 32);
  const bool sw = r & 32u;
  const uint32_t a = sw ? xh : xl, b = sw ? xl : xh;   // rotate by 32 first
  const uint32_t lo = __funnelshift_r(a, b, r), hi = __funnelshift_r(b, a, r);
  return (uint64_t(hi) << 32) | lo;
}

constexpr uint64_t kMultLo = 0x4385DF649FCCF645ull;
constexpr uint64_t kMultHi = 0x2360ED051FC65DA4ull;

__device__ __forceinline__ U128 pcg_step(U128 s, U128 inc) {
  return add128(mul128(s, U128{kMultLo, kMultHi}), inc);
}

// 32 steps at once: s -> A_32 * s + c32 with c32 = G_32 * inc (per stream)
constexpr uint64_t kA32Lo = 0x82B631BA6B261781ull;
constexpr uint64_t kA32Hi = 0x2C82901AD1CB0CD1ull;

__device__ __forceinline__ U128 pcg_stride32(U128 s, U128 c32) {
  return add128(mul128(s, U128{kA32Lo, kA32Hi}), c32);
}

// Jump tables: jt[(level*1024 + j)*4 + {A.lo, A.hi, G.lo, G.hi}];
// after j steps: s -> A_j * s + inc * G_j.  Level 1 holds j = 1024*q.
__device__ __forceinline__ U128 jump_apply(const uint64_t* __restrict__ jt, int level,
                                           uint32_t j, U128 s, U128 inc) {
  const ulonglong2* e = reinterpret_cast<const ulonglong2*>(jt) + 2 * (level * 1024 + j);
  const ulonglong2 a = __ldg(e), g = __ldg(e + 1);
  return add128(mul128(s, U128{a.x, a.y}), mul128(inc, U128{g.x, g.y}));
}

// State after j more steps (j < 2^20).
__device__ __forceinline__ U128 pcg_jump(const uint64_t* __restrict__ jt, U128 s, U128 inc,
                                         uint32_t j) {
  if (j & 1023u) s = jump_apply(jt, 0, j & 1023u, s, inc);
  if (j >> 10) s = jump_apply(jt, 1, j >> 10, s, inc);
  return s;
}

// ---- SeedSequence -> PCG64 initial state -----------------------------------
__device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931E8875u;
  v *= hc;
  return v ^ (v >> 16);
}

__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
  return r ^ (r >> 16);
}

// seed: non-negative integer entropy (< 2^64), as np.random.default_rng(seed)
__device__ __forceinline__ void pcg_seed(uint64_t seed, U128& state, U128& inc) {
  const uint32_t ent0 = uint32_t(seed), ent1 = uint32_t(seed >> 32);
  const int ne = ent1 ? 2 : 1;
  uint32_t hc = 0x43B0D7E5u;
  uint32_t pool[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i == 0 ? ent0 : (i == 1 && ne > 1 ? ent1 : 0u), hc);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  uint32_t hb = 0x8B51F9DDu, st[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58F38DEDu;
    v *= hb;
    st[i] = v ^ (v >> 16);
  }
  const uint64_t w0 = uint64_t(st[0]) | (uint64_t(st[1]) << 32);
  const uint64_t w1 = uint64_t(st[2]) | (uint64_t(st[3]) << 32);
  const uint64_t w2 = uint64_t(st[4]) | (uint64_t(st[5]) << 32);
  const uint64_t w3 = uint64_t(st[6]) | (uint64_t(st[7]) << 32);
  const U128 initstate{w1, w0}, initseq{w3, w2};
  inc.lo = (initseq.lo << 1) | 1ull;
  inc.hi = (initseq.hi << 1) | (initseq.lo >> 63);
  U128 s = inc;                       // step from state 0
  s = add128(s, initstate);
  state = pcg_step(s, inc);
}

// Lemire bounded draw on one 32-bit half (numpy buffered_bounded_lemire_uint32);
// P > 1.  Sets rej when numpy would reject this half and draw again.
// the rare branch (low word < P, probability P / 2^32) is kept out of line:
// the modulo would otherwise be inlined at every draw site of the large
// kernels and crowd their instruction cache
__device__ __noinline__ uint32_t lemire_thr_cold(uint32_t P) { return (0u - P) % P; }
// numpy's rejection threshold (2^32 - P) mod P for a pool of P > 1 values
// (0 for P <= 1: nothing is drawn); out of line, computed once per unit
__device__ __forceinline__ uint32_t lemire_thr_of(uint32_t P) {
  return P > 1 ? lemire_thr_cold(P) : 0u;
}

__device__ __forceinline__ uint32_t lemire(uint32_t h, uint32_t P, bool& rej) {
  const uint64_t m = uint64_t(h) * P;
  const uint32_t left = uint32_t(m);
  if (left < P) {
    if (left < lemire_thr_cold(P)) rej = true;
  }
  return uint32_t(m >> 32);
}

// lemire() with the threshold precomputed: branch-free (rejection iff the
// low product word < thr, which implies < P)
__device__ __forceinline__ uint32_t lemire_t(uint32_t h, uint32_t P, uint32_t thr, bool& rej) {
  const uint64_t m = uint64_t(h) * P;
  rej |= uint32_t(m) < thr;
  return uint32_t(m >> 32);
}

__device__ __forceinline__ double u53_double(uint64_t w) {
  return __dmul_rn(__ull2double_rn(w >> 11), 1.0 / 9007199254740992.0);
}

// Sequential generator (rare serial paths).
struct SeqGen {
  U128 s, inc;
  bool pend;
  uint32_t pv;
  __device__ __forceinline__ uint64_t next64() {
    s = pcg_step(s, inc);
    return pcg_out(s);
  }
  __device__ __forceinline__ uint32_t next32() {
    if (pend) { pend = false; return pv; }
    const uint64_t w = next64();
    pend = true;
    pv = uint32_t(w >> 32);
    return uint32_t(w);
  }
  __device__ __forceinline__ uint32_t bounded(uint32_t P) {   // choice index, P >= 1
    if (P <= 1) return 0;
    uint64_t m = uint64_t(next32()) * P;
    uint32_t left = uint32_t(m);
    if (left < P) {
      const uint32_t thr = (0u - P) % P;
      while (left < thr) {
        m = uint64_t(next32()) * P;
        left = uint32_t(m);
      }
    }
    return uint32_t(m >> 32);
  }
};

}  // namespace pdg
