// K1: Gittins-rank scorers for sm_100a.
//
// Reference: pdgsim.sched.gittins_rank_batch (sched.py:102-129) and the
// batched refresh around it (sched.py:271-305).  For one row with support
// values v_j (ascending), masses p_j and attained service a:
//   d_j = v_j - a,  alive_j = d_j > 0,  m_j = alive_j ? p_j : 0,  Z = sum m
//   rank = min over alive j with S_j > 0 of (P_j + d_j * T_j) / S_j
// where S_j = sum_{k<=j} m_k, P_j = sum_{k<=j} m_k d_k, T_j = Z - S_j.  This is
// the reference's num/cum_p with the 1/Z normalisation cancelled; exhausted
// rows (Z <= 0) give NaN, or age*penalty in the fused refresh.
//
// Two kernels:
//   K1a gittins_f64_kernel  -- drop-in for gittins_rank_batch on arbitrary
//        float64 rows: everything in float64, same formula order as numpy.
//   K1b gittins_hist_kernel -- the device-resident queue: one warp per app,
//        u16 bucket counts (exact: p_j = count_j / n), d_j formed bit-exactly
//        in float64 at the alive boundary, scans in int32 (S, T exact) and
//        float32 (P); HBM-bound, 128-bit loads of 8 counts per lane.
#include <cstring>

#include "common.cuh"

namespace pdg {

// ---------------------------------------------------------------------------
// K1a
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gittins_f64_kernel(
    const double* __restrict__ V, const double* __restrict__ P,
    const double* __restrict__ A, int64_t N, int B, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = gw; r < N; r += nw) {
    const double* v = V + r * B;
    const double* p = P + r * B;
    const double age = A[r];
    double z = 0.0;
    for (int j = lane; j < B; j += 32) {
      double d = dsub(v[j], age);
      if (d > 0.0) z = dadd(z, p[j]);
    }
    z = warp_sum(z);
    if (!(z > 0.0)) {                      // sched.py:117-118,129
      if (lane == 0) out[r] = __longlong_as_double(0x7ff8000000000000ll);
      continue;
    }
    double cp_carry = 0.0, cpv_carry = 0.0, best = __longlong_as_double(0x7ff0000000000000ll);
    for (int base = 0; base < B; base += 32) {
      const int j = base + lane;
      double dl = 0.0, c = 0.0;
      bool live = false;
      if (j < B) {
        double d = dsub(v[j], age);
        live = d > 0.0;
        if (live) {
          dl = d;
          c = __ddiv_rn(p[j], z);         // cond = mass / z  (sched.py:120)
        }
      }
      double cp = dadd(warp_incl_scan(c, lane), cp_carry);
      double cpv = dadd(warp_incl_scan(dmul(c, dl), lane), cpv_carry);
      double num = dadd(cpv, dmul(dl, dsub(1.0, cp)));   // sched.py:124
      if (live && cp > 0.0) best = fmin(best, __ddiv_rn(num, cp));
      cp_carry = __shfl_sync(kFull, cp, 31);
      cpv_carry = __shfl_sync(kFull, cpv, 31);
    }
    best = warp_min(best);
    if (lane == 0) out[r] = best;
  }
}

// ---------------------------------------------------------------------------
// K1b
// ---------------------------------------------------------------------------
struct HistArgs {
  const double* __restrict__ lo;
  const double* __restrict__ width;
  const double* __restrict__ est;
  const int32_t* __restrict__ nbins;
  const uint16_t* __restrict__ counts;
  int64_t stride;
  const double* __restrict__ age;
  int64_t n;
  double penalty;
  float* __restrict__ out_f32;
  uint8_t* __restrict__ out_flags;
  const uint32_t* __restrict__ tiebreak;
  uint64_t* __restrict__ out_key;
  const int32_t* __restrict__ row_idx;   // optional: score only these rows
};

// Exact d = fl(fl(mid_j + est) - age), as sched.py:179 then sched.py:114.
__device__ __forceinline__ double exact_d(double lo, double w, double est,
                                          double age, int j) {
  return dsub(dadd(bucket_mid(lo, w, j), est), age);
}

// One lane's segment of 8 consecutive buckets starting at j0.  Produces float
// masses (integer counts, exact) and float32 offsets d for the alive buckets.
// Values ascend, so the alive buckets are a suffix; its first bucket i0 is
// located with bit-exact float64 tests and d_i = d_{i0} + (i - i0)*w is then a
// sum of positive terms, which float32 carries to ~1e-7 relative accuracy.
__device__ __forceinline__ void lane_segment(const uint4 raw, int j0, int k,
                                             double lo, double w, double est,
                                             double age, float (&m)[8],
                                             float (&d)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) { m[i] = 0.f; d[i] = 0.f; }
  if (j0 >= k) return;
  const int last = min(7, k - 1 - j0);
  int i0 = 8;
  double d0 = 0.0;
  const double ef = exact_d(lo, w, est, age, j0);
  if (ef > 0.0) {
    i0 = 0;
    d0 = ef;
  } else if (exact_d(lo, w, est, age, j0 + last) > 0.0) {
#pragma unroll 1
    for (int i = 1; i <= last; ++i) {
      const double e = exact_d(lo, w, est, age, j0 + i);
      if (e > 0.0) { i0 = i; d0 = e; break; }
    }
  }
  if (i0 == 8) return;
  // buckets past the row's last real bucket are excluded (they would be
  // zero-mass padding in the reference, sched.py:282-291)
  const float df = float(d0), wf = float(w), fi0 = float(i0);
  const uint32_t wd[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float c = u16_to_float((wd[i >> 1] >> (16 * (i & 1))) & 0xffffu);
    const bool on = (i >= i0) && (i <= last);
    m[i] = on ? c : 0.f;
    d[i] = on ? fmaf(float(i) - fi0, wf, df) : 0.f;
  }
}

// Gittins key of one row held as CH chunks of 8 buckets per lane (chunk c,
// lane l owns buckets 256c + 8l .. +7).  Masses are integer-valued floats, so
// S (prefix mass), Z and T = Z - S are exact; P (prefix of m*d) is a float32
// sum of positive terms.  The min over buckets of (P + d*T)/S is tracked as a
// fraction (cross-multiplied compares) so each lane divides once.
template <int CH>
__device__ __forceinline__ float row_key(const float (&m)[CH][8], const float (&d)[CH][8],
                                         int lane, bool& exhausted) {
  float lm[CH], lp[CH], z = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    float sm = 0.f, sp = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) { sm += m[c][i]; sp = fmaf(m[c][i], d[c][i], sp); }
    lm[c] = sm;
    lp[c] = sp;
    z += sm;
  }
  const float Z = warp_sum(z);
  exhausted = !(Z > 0.f);
  if (exhausted) return 0.f;
  float s_carry = 0.f, p_carry = 0.f, bn = 1.f, bd = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const float s_incl = warp_incl_scan(lm[c], lane);
    const float p_incl = warp_incl_scan(lp[c], lane);
    float S = s_carry + (s_incl - lm[c]);
    float P = p_carry + (p_incl - lp[c]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float mi = m[c][i];
      S += mi;
      P = fmaf(mi, d[c][i], P);
      // zero-mass buckets never beat the previous positive one (and give
      // +inf before any mass), so only positive-mass buckets are candidates
      const float num = fmaf(d[c][i], Z - S, P);
      const bool take = (mi > 0.f) && (num * bd < bn * S);
      bn = take ? num : bn;
      bd = take ? S : bd;
    }
    s_carry += __shfl_sync(kFull, s_incl, 31);
    p_carry += __shfl_sync(kFull, p_incl, 31);
  }
  const float r = bd > 0.f ? __fdiv_rn(bn, bd) : __int_as_float(0x7f800000);
  return warp_min(r);
}

template <int CH>   // row holds up to 256*CH buckets
__global__ void __launch_bounds__(256, (CH == 1 ? 4 : 2)) gittins_hist_kernel(HistArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  if (gw >= a.n) return;

  // software pipeline: counts of the next row are in flight while the current
  // row is scored
  uint4 nxt[CH];
  int knxt;
  auto row_of = [&](int64_t i) -> int64_t { return a.row_idx ? int64_t(__ldg(a.row_idx + i)) : i; };
  auto load = [&](int64_t i, uint4 (&dst)[CH], int& kk) {
    const int64_t r = row_of(i);
    const uint4* row = reinterpret_cast<const uint4*>(a.counts + r * a.stride);
    kk = __ldg(a.nbins + r);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int j0 = 256 * c + 8 * lane;
      dst[c] = (j0 < kk) ? __ldcs(row + 32 * c + lane) : make_uint4(0, 0, 0, 0);
    }
  };
  load(gw, nxt, knxt);
  for (int64_t i = gw; i < a.n; i += nw) {
    const int64_t r = row_of(i);
    uint4 cur[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) cur[c] = nxt[c];
    const int k = knxt;
    const double lo = __ldg(a.lo + r), w = __ldg(a.width + r);
    const double est = __ldg(a.est + r), age = __ldg(a.age + r);
    if (i + nw < a.n) load(i + nw, nxt, knxt);

    float m[CH][8], d[CH][8];
#pragma unroll
    for (int c = 0; c < CH; ++c)
      lane_segment(cur[c], 256 * c + 8 * lane, k, lo, w, est, age, m[c], d[c]);
    bool exhausted;
    float key = row_key<CH>(m, d, lane, exhausted);
    uint8_t flags = 0;
    if (exhausted) {                                 // sched.py:295-300
      key = float(dmul(age, a.penalty));
      flags = PDG_FLAG_OVERRUN;
    }
    if (lane == 0) {
      if (!(key > 0.f)) key = 0.f;                   // canonical +0 for the sort key
      if (a.out_f32) a.out_f32[r] = key;
      if (a.out_flags) a.out_flags[r] = flags;
      if (a.out_key) {
        const uint32_t tb = a.tiebreak ? a.tiebreak[r] : uint32_t(r);
        a.out_key[r] = (uint64_t(__float_as_uint(key)) << 32) | tb;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1b, pair form for the queue's layout (rows of <= 256 buckets, 16-byte
// aligned, zero counts past nbins).  Two lanes score one row: lane
// l = 16g + r works on row r of a 16-row tile and owns two 64-bucket segments
// of it, x = [64g, 64g+64) and y = [128+64g, 192+64g), which it scans
// together as the two halves of packed f32x2 registers (sm_100 FADD2 / FFMA2 /
// FMUL2: one issue slot per bucket pair).  (Four lanes per row were tried:
// the per-row work -- j0, segment sums, prefix -- then dominates.)
//
// Staging: each warp stages its tile in shared memory with TMA bulk copies
// (cp.async.bulk, one 2*stride-byte copy per row issued by lanes 0..15)
// completing on an mbarrier; STAGES > 1 rings prefetch tiles ahead, but one
// stage with 24 warps per SM measured faster (the other warps hide the copy).
// Rows are 528 B apart (33 x 16 B), so the eight lanes of a quarter-warp
// (same g, eight consecutive rows) read eight different bank groups.
//
// Per row (sched.py:102-129 with the 1/Z normalisation cancelled):
//  * the first alive bucket j0 (d_j = fl(fl(mid_j + est) - age) > 0, values
//    ascend) is bracketed by a float32 estimate and confirmed by four exact
//    float64 tests, two per lane of the row (binary search if the estimate
//    misses); counts of dead buckets are zeroed;
//  * each segment's alive mass and its weighted mass sum_k (k - j0) m_k come
//    from IADD3 / IDP2A over the packed u16 counts; a prefix over the row's
//    four segments (one shuffle across g) gives every segment its start state;
//  * with t = j - j0, d_j = d0 + t*w, S_j the alive prefix mass and
//    T_j = Z - S_j, the numerator P_j + d_j*T_j is exactly d0*Z + w*I_j with
//    I_j = I_{j-1} + T_{j-1} (integer-valued floats, exact), so a bucket is
//    I += T, T -= m, S = Z - T, one FFMA, one MUFU reciprocal, one FMUL and a
//    min.  Dead and massless buckets give S = 0 -> |num| * inf (or NaN),
//    which never wins; zero-mass buckets after mass never beat the previous
//    positive one.
// I, T and S are exact, so the key equals the warp-per-row kernel's
// (gittins_hist_kernel) up to its own float32 rounding of P.
// ---------------------------------------------------------------------------
constexpr int kPairPitchU4 = 33;                      // 528 B per staged row
constexpr int kPairTileU4 = 16 * kPairPitchU4;         // 16 rows per tile
#ifndef PDG_PAIR_WARPS
#define PDG_PAIR_WARPS 4
#endif
#ifndef PDG_PAIR_STAGES
#define PDG_PAIR_STAGES 1
#endif
#ifndef PDG_PAIR_MINB
#define PDG_PAIR_MINB 6
#endif
constexpr int kPairWarps = PDG_PAIR_WARPS;
constexpr int kPairStages = PDG_PAIR_STAGES;
#ifndef PDG_PAIR_MIN_ROWS
#define PDG_PAIR_MIN_ROWS 4736                          // 148 SMs x 32 rows
#endif
constexpr int64_t kPairMinRows = PDG_PAIR_MIN_ROWS;      // smaller batches: warp per row

__device__ __forceinline__ float rcp_approx(float x) {    // MUFU.RCP, ~1 ulp; rcp(0) = +inf
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// packed f32x2 arithmetic (sm_100)
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ uint64_t f2_pack_bits(uint32_t lo, uint32_t hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(hi));
  return d;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <uint32_t SEL>
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b) {   // selector immediate
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL));
  return d;
}

struct QuadHdr {
  double lo, w, est, age;
  int64_t r;                        // < 0: no row (past the end)
  int k;
  uint32_t tb;
};

// smallest j in [0, k] with exact_d(j) > 0 (k: nothing alive)
__device__ __forceinline__ int first_alive_search(double lo, double w, double est, double age,
                                                  int k) {
  int l = 0, hi = k;
  while (l < hi) {
    const int mid = (l + hi) >> 1;
    if (exact_d(lo, w, est, age, mid) > 0.0) hi = mid; else l = mid + 1;
  }
  return l;
}

template <int W, int STAGES>
__global__ void __launch_bounds__(W * 32, PDG_PAIR_MINB) gittins_pair_kernel(HistArgs a) {
  extern __shared__ __align__(128) uint4 stage[];
  __shared__ uint64_t bars[W * STAGES];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int r = lane & 15, g = lane >> 4;             // row of the tile, half of the row
  uint4* tiles = stage + size_t(wib) * STAGES * kPairTileU4;
  uint64_t* bar = bars + wib * STAGES;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(bar + s, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const int64_t ntiles = (a.n + 15) >> 4;
  const int64_t gw = int64_t(blockIdx.x) * W + wib;
  const int64_t nw = int64_t(gridDim.x) * W;
  const unsigned row_bytes = unsigned(a.stride) * 2u;     // <= 512, multiple of 16
  const int kmax = int(a.stride);
  const int nu4 = int(a.stride >> 3);                     // uint4 per row
  const uint64_t policy = l2_evict_first_policy();

  // one tile into ring slot `slot`: lanes 0..15 copy rows 0..15; every lane
  // loads its row's header
  auto issue = [&](int64_t t, int slot, QuadHdr& h) {
    const int64_t i = t * 16 + r;
    const bool valid = i < a.n;
    const int64_t rg = valid ? (a.row_idx ? int64_t(__ldg(a.row_idx + i)) : i) : -1;
    const int64_t left = a.n - t * 16;
    const unsigned nvalid = left < 16 ? unsigned(left) : 16u;
    fence_proxy_async_smem();                        // earlier reads of the slot first
    if (lane == 0) mbar_arrive_expect_tx(bar + slot, nvalid * row_bytes);
    __syncwarp();
    if (g == 0 && valid)
      bulk_g2s(tiles + slot * kPairTileU4 + r * kPairPitchU4, a.counts + rg * a.stride,
               row_bytes, bar + slot, policy);
    h.r = rg;
    if (valid) {
      h.lo = __ldg(a.lo + rg);
      h.w = __ldg(a.width + rg);
      h.est = __ldg(a.est + rg);
      h.age = __ldg(a.age + rg);
      h.k = min(__ldg(a.nbins + rg), kmax);
      h.tb = a.tiebreak ? __ldg(a.tiebreak + rg) : uint32_t(rg);
    } else {
      h.lo = 0.0;
      h.w = 1.0;
      h.est = 0.0;
      h.age = 1.0;
      h.k = 0;
      h.tb = 0;
    }
  };

  QuadHdr h[STAGES];
#pragma unroll
  for (int s = 0; s + 1 < STAGES; ++s)
    if (gw + s * nw < ntiles) issue(gw + s * nw, s, h[s]);
  uint32_t q = 0;
  for (int64_t t = gw; t < ntiles; t += nw, ++q) {
    const int64_t tn = t + int64_t(STAGES - 1) * nw;
    if (tn < ntiles) issue(tn, int((q + STAGES - 1) % STAGES), h[STAGES - 1]);
    const int s = int(q % STAGES);
    const QuadHdr hd = h[0];
#pragma unroll
    for (int j = 0; j + 1 < STAGES; ++j) h[j] = h[j + 1];
    const double lo = hd.lo, w = hd.w, est = hd.est, age = hd.age;
    const int k = hd.k;

    // ---- first alive bucket: float32 estimate, four exact tests per row
    int j0;
    {
      const float x = __fdividef(float(dsub(dsub(age, est), lo)), float(w)) - 0.5f;
      int c;
      if (!(x > -1.0e9f)) c = 0;                        // NaN / -inf / far below
      else if (!(x < 1.0e9f)) c = k;
      else c = min(max(__float2int_rd(x) + 1, 0), k);
      auto test = [&](int j) {
        return j >= k ? true : (j < 0 ? false : exact_d(lo, w, est, age, j) > 0.0);
      };
      const bool a0 = test(c - 2 + 2 * g), a1 = test(c - 1 + 2 * g);   // j = c-2 .. c+1
      const unsigned b0 = __ballot_sync(kFull, a0) >> r, b1 = __ballot_sync(kFull, a1) >> r;
      const unsigned bits = (b0 & 1u) | ((b1 & 1u) << 1) | ((b0 >> 14) & 4u) |
                            ((b1 >> 13) & 8u);
      if (!(bits & 1u) && (bits & 8u)) j0 = c - 3 + __ffs(bits);
      else j0 = first_alive_search(lo, w, est, age, k);   // estimate missed (rare)
    }
    mbar_wait(bar + s, (q / STAGES) & 1u);
    uint4* row = tiles + s * kPairTileU4 + r * kPairPitchU4;
    const int c0 = j0 >> 3, e0 = j0 & 7;
    // zero the dead counts of the uint4 holding j0 (its owner, in place; also
    // when nothing is alive, j0 = k, and k is not a multiple of 8)
    if (e0 != 0 && c0 < nu4 && g == ((c0 >> 3) & 1)) {
      uint4 v = row[c0];
      const uint64_t m_lo = e0 >= 4 ? 0ull : (~0ull << (16 * e0));
      const uint64_t m_hi = e0 >= 4 ? (~0ull << (16 * (e0 - 4))) : ~0ull;
      v.x &= uint32_t(m_lo);
      v.y &= uint32_t(m_lo >> 32);
      v.z &= uint32_t(m_hi);
      v.w &= uint32_t(m_hi >> 32);
      row[c0] = v;
    }
    __syncwarp();
    // segment x = uint4 [8g, 8g+8), y = [16+8g, 16+8g+8); dead and past-the-row
    // uint4 read as zero
    auto ld = [&](int u) {
      return (u >= c0 && u < nu4) ? row[u] : make_uint4(0, 0, 0, 0);
    };

    // ---- segment sums: packed u16 mass (IADD3), weighted mass (IDP2A)
    uint32_t sx = 0, sy = 0, wx = 0, wy = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 X = ld(8 * g + i), Y = ld(16 + 8 * g + i);
      const uint32_t xs[4] = {X.x, X.y, X.z, X.w};
      const uint32_t ys[4] = {Y.x, Y.y, Y.z, Y.w};
      sx += (xs[0] + xs[1]) + (xs[2] + xs[3]);
      sy += (ys[0] + ys[1]) + (ys[2] + ys[3]);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int b = 2 * (4 * i + p);                   // bucket offset in the segment
        const uint32_t wt = uint32_t(b | ((b + 1) << 8));
        wx = __dp2a_lo(xs[p], wt, wx);
        wy = __dp2a_lo(ys[p], wt, wy);
      }
    }
    const int mx = int((sx & 0xffffu) + (sx >> 16)), my = int((sy & 0xffffu) + (sy >> 16));
    const int bx = 64 * g, by = 128 + 64 * g;              // segment starts
    // alive mass and sum_k (k - j0) m_k (>= 0: dead counts are zero) per
    // segment; the row's other half is lane ^ 16
    const int kx = int(wx) + (bx - j0) * mx, ky = int(wy) + (by - j0) * my;
    const int omx = __shfl_xor_sync(kFull, mx, 16), okx = __shfl_xor_sync(kFull, kx, 16);
    const int omy = __shfl_xor_sync(kFull, my, 16), oky = __shfl_xor_sync(kFull, ky, 16);
    const int zx = mx + omx, kxt = kx + okx;
    const int Z = zx + my + omy;
    float key;
    uint8_t flags = 0;
    if (Z == 0) {                                          // exhausted: sched.py:295-300
      key = float(dmul(age, a.penalty));
      flags = PDG_FLAG_OVERRUN;
    } else {
      // segment start state (after bucket b - 1): T = Z - S_before,
      // I = K_before + (b - 1 - j0) T
      const int sbx = g ? omx : 0, kbx = g ? okx : 0;
      const int sby = zx + (g ? omy : 0), kby = kxt + (g ? oky : 0);
      const int Tx = Z - sbx, Ty = Z - sby;
      const int Ix = kbx + (bx - 1 - j0) * Tx, Iy = kby + (by - 1 - j0) * Ty;
      const double d0 = exact_d(lo, w, est, age, j0);
      const float af = float(dmul(d0, double(Z))), bf = float(w);
      const uint64_t A2 = f2_pack(af, af), B2 = f2_pack(bf, bf);
      const uint64_t Z2 = f2_pack(float(Z), float(Z));
      const uint64_t bias2 = f2_pack(-8388608.f, -8388608.f);
      uint64_t I2 = f2_pack(float(Ix), float(Iy)), T2 = f2_pack(float(Tx), float(Ty));
      float bestx = __int_as_float(0x7f800000), besty = bestx;
      // 0x4B00 in a register (kmax <= 256), so that ptxas keeps the PRMT
      // selectors as immediates instead of re-materialising them
      const uint32_t magic = 0x4B00u | (uint32_t(kmax) >> 16);
      auto step = [&](uint32_t xw, uint32_t yw, auto sel) {
        constexpr uint32_t S = decltype(sel)::value;
        const uint64_t m2 = f2_add(f2_pack_bits(prmt<S>(xw, magic), prmt<S>(yw, magic)), bias2);
        I2 = f2_add(I2, T2);                               // exact (integer-valued)
        T2 = f2_sub(T2, m2);
        float sxf, syf;
        f2_unpack(f2_sub(Z2, T2), sxf, syf);
        const uint64_t q2 =
            f2_mul(f2_fma(B2, I2, A2), f2_pack(rcp_approx(sxf), rcp_approx(syf)));
        float qx, qy;
        f2_unpack(q2, qx, qy);
        bestx = fminf(bestx, fabsf(qx));
        besty = fminf(besty, fabsf(qy));
      };
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 X = ld(8 * g + i), Y = ld(16 + 8 * g + i);
        const uint32_t xs[4] = {X.x, X.y, X.z, X.w};
        const uint32_t ys[4] = {Y.x, Y.y, Y.z, Y.w};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          step(xs[p], ys[p], std::integral_constant<uint32_t, 0x5410u>{});
          step(xs[p], ys[p], std::integral_constant<uint32_t, 0x5432u>{});
        }
      }
      key = fminf(bestx, besty);
    }
    key = fminf(key, __shfl_xor_sync(kFull, key, 16));
    __syncwarp();                                          // slot reads done before reuse
    if (g == 0 && hd.r >= 0) {
      const int64_t rg = hd.r;
      if (!(key > 0.f)) key = 0.f;                         // canonical +0 for the sort key
      if (a.out_f32) a.out_f32[rg] = key;
      if (a.out_flags) a.out_flags[rg] = flags;
      if (a.out_key) a.out_key[rg] = (uint64_t(__float_as_uint(key)) << 32) | hd.tb;
    }
  }
}

}  // namespace pdg

using namespace pdg;

extern "C" int pdg_gittins_rank_f64(const double* values, const double* probs,
                                    const double* ages, int64_t n_rows,
                                    int32_t n_bins, double* out_rank,
                                    void* stream) {
  if (n_rows < 0 || n_bins <= 0 || (n_rows > 0 && (!values || !probs || !ages || !out_rank))) {
    set_error("pdg_gittins_rank_f64: invalid arguments");
    return PDG_EINVAL;
  }
  if (n_rows == 0) return PDG_OK;
  const int threads = 256;
  int64_t warps_needed = n_rows;
  int64_t blocks = (warps_needed * 32 + threads - 1) / threads;
  const int64_t cap = int64_t(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  gittins_f64_kernel<<<unsigned(blocks), threads, 0, (cudaStream_t)stream>>>(
      values, probs, ages, n_rows, n_bins, out_rank);
  return launch_status("gittins_f64_kernel");
}

// Host-buffer form for scheduler-sized batches (the drop-in refresh): one
// packed upload into a pinned staging area, the kernel, one download, all on
// the caller's stream inside the library -- no per-call allocation.
namespace {
struct HostStage {
  double* h = nullptr;     // pinned host
  double* d = nullptr;     // device
  size_t cap = 0;          // doubles
  double* zh = nullptr;    // mapped pinned host (small batches: read in place by the kernel)
  double* zd = nullptr;    // its device alias
  size_t zcap = 0;
};
thread_local HostStage g_stage;
#ifndef PDG_ZERO_COPY_MAX
#define PDG_ZERO_COPY_MAX (1u << 17)   // doubles (1 MiB): batches up to this skip the copies
#endif
}  // namespace

extern "C" int pdg_gittins_rank_f64_host(const double* values, const double* probs,
                                         const double* ages, int64_t n_rows, int32_t n_bins,
                                         double* out_rank, void* stream) {
  using namespace pdg;
  if (n_rows < 0 || n_bins <= 0 || (n_rows > 0 && (!values || !probs || !ages || !out_rank))) {
    set_error("pdg_gittins_rank_f64_host: invalid arguments");
    return PDG_EINVAL;
  }
  if (n_rows == 0) return PDG_OK;
  const size_t nb = size_t(n_rows) * size_t(n_bins);
  const size_t need = 2 * nb + 2 * size_t(n_rows);
  HostStage& st = g_stage;
  if (need <= PDG_ZERO_COPY_MAX) {
    // scheduler-sized batch: the kernel reads the rows from mapped pinned
    // memory and writes the ranks back there -- one launch and one sync, no
    // copy calls on the latency path
    if (!st.zh) {
      cudaError_t e = cudaHostAlloc(&st.zh, PDG_ZERO_COPY_MAX * sizeof(double),
                                    cudaHostAllocMapped);
      if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host cudaHostAlloc");
      e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&st.zd), st.zh, 0);
      if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host map");
      st.zcap = PDG_ZERO_COPY_MAX;
    }
    std::memcpy(st.zh, values, nb * sizeof(double));
    std::memcpy(st.zh + nb, probs, nb * sizeof(double));
    std::memcpy(st.zh + 2 * nb, ages, size_t(n_rows) * sizeof(double));
    const size_t in = 2 * nb + size_t(n_rows);
    int rc = pdg_gittins_rank_f64(st.zd, st.zd + nb, st.zd + 2 * nb, n_rows, n_bins,
                                  st.zd + in, stream);
    if (rc != PDG_OK) return rc;
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host sync");
    std::memcpy(out_rank, st.zh + in, size_t(n_rows) * sizeof(double));
    return PDG_OK;
  }
  if (need > st.cap) {
    size_t cap = 4096;
    while (cap < need) cap <<= 1;
    if (st.h) cudaFreeHost(st.h);
    if (st.d) cudaFree(st.d);
    st.h = nullptr;
    st.d = nullptr;
    st.cap = 0;
    cudaError_t e = cudaMallocHost(&st.h, cap * sizeof(double));
    if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host cudaMallocHost");
    e = cudaMalloc(&st.d, cap * sizeof(double));
    if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host cudaMalloc");
    st.cap = cap;
  }
  std::memcpy(st.h, values, nb * sizeof(double));
  std::memcpy(st.h + nb, probs, nb * sizeof(double));
  std::memcpy(st.h + 2 * nb, ages, size_t(n_rows) * sizeof(double));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t in = 2 * nb + size_t(n_rows);
  cudaError_t e = cudaMemcpyAsync(st.d, st.h, in * sizeof(double), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host upload");
  int rc = pdg_gittins_rank_f64(st.d, st.d + nb, st.d + 2 * nb, n_rows, n_bins, st.d + in,
                                stream);
  if (rc != PDG_OK) return rc;
  e = cudaMemcpyAsync(st.h + in, st.d + in, size_t(n_rows) * sizeof(double),
                      cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host download");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_f64_host sync");
  std::memcpy(out_rank, st.h + in, size_t(n_rows) * sizeof(double));
  return PDG_OK;
}

extern "C" int pdg_gittins_score_hist(const pdg_hist_rows* rows, const double* age,
                                      int64_t n, double penalty, float* out_key_f32,
                                      uint8_t* out_flags, const uint32_t* tiebreak,
                                      uint64_t* out_key, const int32_t* row_idx,
                                      void* stream) {
  if (!rows || n < 0 || (n > 0 && (!age || !rows->lo || !rows->width || !rows->est_age ||
                                   !rows->nbins || !rows->counts))) {
    set_error("pdg_gittins_score_hist: invalid arguments");
    return PDG_EINVAL;
  }
  if (rows->stride % 8 != 0 || (reinterpret_cast<uintptr_t>(rows->counts) & 15)) {
    set_error("pdg_gittins_score_hist: counts must be 16-byte aligned, stride %% 8 == 0");
    return PDG_EINVAL;
  }
  if (n == 0) return PDG_OK;
  HistArgs a{rows->lo, rows->width, rows->est_age, rows->nbins, rows->counts,
             rows->stride, age, n, penalty, out_key_f32, out_flags, tiebreak, out_key,
             row_idx};
  const int threads = 256;
  int64_t blocks = (n * 32 + threads - 1) / threads;
  const int64_t cap = int64_t(sm_count()) * 4;
  if (blocks > cap) blocks = cap;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t maxb = rows->stride;   // buckets per row are bounded by the stride
  // quad tiles pay off once every SM has tiles to stream; small
  // (incremental) batches take the warp-per-row kernel's lower latency
  if (maxb <= 256 && n >= kPairMinRows) {
    auto kern = gittins_pair_kernel<kPairWarps, kPairStages>;
    const size_t smem = size_t(kPairWarps) * kPairStages * kPairTileU4 * sizeof(uint4);
    int per_sm = 0;
    if (int r = launch_setup(reinterpret_cast<const void*>(kern), kPairWarps * 32, smem, &per_sm))
      return r;
    const int64_t tiles = (n + 15) / 16;
    int64_t nb = (tiles + kPairWarps - 1) / kPairWarps;
    if (nb > int64_t(per_sm) * sm_count()) nb = int64_t(per_sm) * sm_count();
    kern<<<unsigned(nb), kPairWarps * 32, smem, s>>>(a);
    return launch_status("gittins_pair_kernel");
  }
  if (maxb <= 256) gittins_hist_kernel<1><<<unsigned(blocks), threads, 0, s>>>(a);
  else if (maxb <= 512) gittins_hist_kernel<2><<<unsigned(blocks), threads, 0, s>>>(a);
  else if (maxb <= 1024) gittins_hist_kernel<4><<<unsigned(blocks), threads, 0, s>>>(a);
  else {
    set_error("pdg_gittins_score_hist: more than 1024 buckets per row");
    return PDG_EUNSUPPORTED;
  }
  return launch_status("gittins_hist_kernel");
}

// ---------------------------------------------------------------------------
// K1a, sample form (sched.py:51-85): one CTA per distribution; the tail
// {s - age : s > age} (+inf padding) is bitonic-sorted in shared memory, then
// one thread replays the reference's scan: prefix sums in sorted order, one
// candidate per group of equal values, (prefix + d*(n-j)) / j.
// ---------------------------------------------------------------------------
namespace pdg {
__global__ void __launch_bounds__(256) gittins_samples_kernel(
    const double* __restrict__ samples, const int64_t* __restrict__ off,
    const int32_t* __restrict__ len, const double* __restrict__ ages, int64_t n_rows,
    int npow2, double* __restrict__ out) {
  extern __shared__ double tail[];
  __shared__ int cnt;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const double* s = samples + off[r];
    const int n = len[r];
    const double age = ages[r];
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    int live = 0;
    for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
      const bool on = i < n && s[i] > age;
      tail[i] = on ? dsub(s[i], age) : inf;
      live += on;
    }
    if (live) atomicAdd(&cnt, live);
    for (int k = 2; k <= npow2; k <<= 1) {             // bitonic sort, ascending
      for (int j = k >> 1; j > 0; j >>= 1) {
        __syncthreads();
        for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
          const int p = i ^ j;
          if (p > i) {
            const double x = tail[i], y = tail[p];
            const bool up = (i & k) == 0;
            if (up ? x > y : x < y) { tail[i] = y; tail[p] = x; }
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int m = cnt;
      double best;
      if (m == 0) {
        best = __longlong_as_double(0x7ff8000000000000ll);           // exhausted
      } else if (tail[0] == tail[m - 1]) {
        best = tail[0];                                               // degenerate
      } else {
        best = inf;
        double prefix = 0.0;
        int i = 0;
        while (i < m) {
          int j = i;
          while (j < m && tail[j] == tail[i]) prefix = dadd(prefix, tail[j++]);
          const double d = tail[i];
          const double num = dadd(prefix, dmul(d, double(m - j)));
          const double ratio = __ddiv_rn(num, double(j));
          if (ratio < best) best = ratio;
          i = j;
        }
      }
      out[r] = best;
    }
    __syncthreads();
  }
}
}  // namespace pdg

extern "C" int pdg_gittins_rank_samples(const double* samples, const int64_t* off,
                                        const int32_t* len, const double* ages, int64_t n_rows,
                                        int32_t max_len, double* out_rank, void* stream) {
  using namespace pdg;
  if (n_rows < 0 || max_len < 0 || max_len > PDG_SAMPLES_MAX ||
      (n_rows > 0 && (!samples || !off || !len || !ages || !out_rank))) {
    set_error("pdg_gittins_rank_samples: invalid arguments (max_len <= %d)", PDG_SAMPLES_MAX);
    return PDG_EINVAL;
  }
  if (n_rows == 0) return PDG_OK;
  int npow2 = 1;
  while (npow2 < max_len) npow2 <<= 1;
  const size_t smem = size_t(npow2) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gittins_samples_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(PDG_SAMPLES_MAX * sizeof(double)));
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(gittins_samples_kernel)");
    attr = true;
  }
  const int64_t blocks = n_rows < int64_t(sm_count()) * 8 ? n_rows : int64_t(sm_count()) * 8;
  gittins_samples_kernel<<<unsigned(blocks), 256, smem, (cudaStream_t)stream>>>(
      samples, off, len, ages, n_rows, npow2, out_rank);
  return launch_status("gittins_samples_kernel");
}

extern "C" int pdg_gittins_rank_samples_host(const double* samples, int32_t n, double age,
                                             double* out_rank, void* stream) {
  using namespace pdg;
  if (n < 0 || n > PDG_SAMPLES_MAX || (n > 0 && !samples) || !out_rank) {
    set_error("pdg_gittins_rank_samples_host: invalid arguments (n <= %d)", PDG_SAMPLES_MAX);
    return PDG_EINVAL;
  }
  HostStage& st = g_stage;
  if (!st.zh) {
    cudaError_t e = cudaHostAlloc(&st.zh, PDG_ZERO_COPY_MAX * sizeof(double),
                                  cudaHostAllocMapped);
    if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_samples_host cudaHostAlloc");
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&st.zd), st.zh, 0);
    if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_samples_host map");
    st.zcap = PDG_ZERO_COPY_MAX;
  }
  // [samples | age | out | off (int64) | len (int32)]
  std::memcpy(st.zh, samples, size_t(n) * sizeof(double));
  st.zh[n] = age;
  int64_t* offp = reinterpret_cast<int64_t*>(st.zh + n + 2);
  int32_t* lenp = reinterpret_cast<int32_t*>(st.zh + n + 3);
  *offp = 0;
  *lenp = n;
  int rc = pdg_gittins_rank_samples(st.zd, reinterpret_cast<const int64_t*>(st.zd + n + 2),
                                    reinterpret_cast<const int32_t*>(st.zd + n + 3), st.zd + n,
                                    1, n, st.zd + n + 1, stream);
  if (rc != PDG_OK) return rc;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "pdg_gittins_rank_samples_host sync");
  *out_rank = st.zh[n + 1];
  return PDG_OK;
}

// pdg_order (K5) lives in sort.cu

// ---------------------------------------------------------------------------
// a4 standalone: equal-width bucketing of sample rows (distributions.py:79-105)
// one warp per row; the engine fuses the same epilogue.
// ---------------------------------------------------------------------------
namespace pdg {
__global__ void __launch_bounds__(128) bucketize_kernel(const double* __restrict__ samples,
                                                        int64_t rows, int n, int k,
                                                        double* lo_out, double* w_out,
                                                        int32_t* nb_out, uint16_t* counts,
                                                        int64_t stride) {
  extern __shared__ uint32_t bcnt[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* cnt = bcnt + size_t(wib) * k;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = gw; r < rows; r += nw) {
    const double* s = samples + r * int64_t(n);
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    for (int i = lane; i < n; i += 32) { lo = fmin(lo, s[i]); hi = fmax(hi, s[i]); }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(kFull, lo, o));
      hi = fmax(hi, __shfl_xor_sync(kFull, hi, o));
    }
    const int kk = lo == hi ? 1 : k;
    const double w = lo == hi ? 0.0 : __ddiv_rn(dsub(hi, lo), small_int_to_double(k));
    for (int b = lane; b < kk; b += 32) cnt[b] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      int idx = 0;
      if (kk > 1) {
        idx = __double2int_rz(__ddiv_rn(dsub(s[i], lo), w));
        idx = idx < kk - 1 ? idx : kk - 1;
      }
      atomicAdd(&cnt[idx], 1u);
    }
    __syncwarp();
    for (int b = lane; b < stride; b += 32)
      counts[r * stride + b] = b < kk ? uint16_t(cnt[b]) : uint16_t(0);
    if (lane == 0) { lo_out[r] = lo; w_out[r] = w; nb_out[r] = kk; }
    __syncwarp();
  }
}
}  // namespace pdg

extern "C" int pdg_bucketize(const double* samples, int64_t rows, int32_t n, int32_t k,
                             double* lo, double* width, int32_t* nbins, uint16_t* counts,
                             int64_t stride, void* stream) {
  if (rows < 0 || n < 1 || n > 65535 || k < 1 || k > 1024 || stride < k ||
      (rows > 0 && (!samples || !lo || !width || !nbins || !counts))) {
    set_error("pdg_bucketize: invalid arguments (n <= 65535, 1 <= k <= stride, k <= 1024)");
    return PDG_EINVAL;
  }
  if (rows == 0) return PDG_OK;
  int64_t blocks = (rows * 32 + 127) / 128;
  const int64_t cap = int64_t(sm_count()) * 16;
  if (blocks > cap) blocks = cap;
  bucketize_kernel<<<unsigned(blocks), 128, 4 * k * sizeof(uint32_t), (cudaStream_t)stream>>>(
      samples, rows, n, k, lo, width, nbins, counts, stride);
  return launch_status("bucketize_kernel");
}

// ---------------------------------------------------------------------------
// K1c: SRPT-mean and LSTF keys over the queue (sched.py:216-224, 132-140);
// elementwise, HBM-bound (5 x 8 B in, 16 B out per row)
// ---------------------------------------------------------------------------
namespace pdg {
// order-preserving uint64 image of a float64 (negative keys included)
__device__ __forceinline__ uint64_t orderable(double x) {
  const uint64_t b = uint64_t(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(256) policy_keys_kernel(
    int policy, const double* __restrict__ mean, const double* __restrict__ worst,
    const double* __restrict__ est_age, const double* __restrict__ age,
    const double* __restrict__ deadline, double now, int64_t n,
    const int32_t* __restrict__ row_idx, double* __restrict__ out_f64,
    uint64_t* __restrict__ out_key) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = row_idx ? row_idx[i] : i;
    double key;
    if (policy == PDG_POLICY_SRPT_MEAN) {
      key = dsub(mean[r], dsub(age[r], est_age[r]));
    } else {
      key = dsub(dsub(deadline[r], now), dsub(dadd(worst[r], est_age[r]), age[r]));
    }
    if (out_f64) out_f64[r] = key;
    if (out_key) out_key[r] = orderable(key);
  }
}
}  // namespace pdg

extern "C" int pdg_policy_keys(int32_t policy, const double* mean, const double* worst,
                               const double* est_age, const double* age,
                               const double* deadline, double now, int64_t n,
                               const int32_t* row_idx, double* out_key_f64, uint64_t* out_key,
                               void* stream) {
  using namespace pdg;
  const bool srpt = policy == PDG_POLICY_SRPT_MEAN, lstf = policy == PDG_POLICY_LSTF;
  if (n < 0 || !(srpt || lstf) || !est_age || !age || (srpt && !mean) ||
      (lstf && (!worst || !deadline)) || (!out_key_f64 && !out_key)) {
    set_error("pdg_policy_keys: invalid arguments");
    return PDG_EINVAL;
  }
  if (n == 0) return PDG_OK;
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = int64_t(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  policy_keys_kernel<<<unsigned(blocks), 256, 0, (cudaStream_t)stream>>>(
      policy, mean, worst, est_age, age, deadline, now, n, row_idx, out_key_f64, out_key);
  return launch_status("policy_keys_kernel");
}

// K5b (pdg_order_update) lives in sort.cu
