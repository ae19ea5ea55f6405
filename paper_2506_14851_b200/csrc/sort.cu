// K5: the global order -- stable LSD radix sort of packed 64-bit keys with a
// u32 payload (the queue slot), in ONE cooperative kernel.
//
// Reference: the scheduler's ordering of applications by (key, arrival)
// (sched.py:191-192 sort key, simcore.py:339-344 _task_sort_key, 636-640
// the refresh order).  Keys are (float32 key bits << 32 | tiebreak), so a
// stable sort of bits [begin_bit, 64) is the reference order (begin_bit = 32
// when the input is already in tiebreak order).
//
// Why one kernel: the queue is 1e5-1e6 keys, where a library radix sort is
// launch- and latency-bound (histogram kernel + scan kernel + one kernel per
// 8-bit digit).  Here a persistent grid of co-resident CTAs (cooperative
// launch) runs every digit pass with grid barriers in between:
//   A  per-CTA digit histogram of its contiguous chunk (shared atomics),
//      written digit-major: H[d * G + cta]
//   B  exclusive scan of H: each CTA scans one 256-entry segment in place
//      and publishes the segment total
//   C  each CTA scans the G segment totals in shared memory, forms its 256
//      digit offsets, and scatters its chunk tile by tile: inside a tile
//      every warp ranks its 128 consecutive keys with __match_any_sync (peer
//      groups = equal digits), warps are combined per digit through a
//      shared-memory count table, so equal digits keep input order (stable).
// Three grid barriers per pass; 4 passes for begin_bit = 32, 8 for 0.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace pdg {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortSteps = 4;                           // keys per lane per tile
constexpr int kSortTile = kSortThreads * kSortSteps;    // 1024 keys
constexpr int kSortWarpKeys = 32 * kSortSteps;          // 128 consecutive keys per warp

struct SortArgs {
  const uint64_t* kin;
  const uint32_t* sin;
  uint64_t* kout;
  uint32_t* sout;
  uint64_t* ktmp;
  uint32_t* stmp;
  uint32_t* H;        // [256 * G] digit-major counts, then in-segment exclusive prefixes
  uint32_t* S;        // [G] segment totals
  int64_t n;
  int64_t chunk;      // keys per CTA (multiple of kSortTile)
  int begin_bit;
  int passes;
};

// exclusive scan of one value per thread over the CTA; returns the total
__device__ __forceinline__ uint32_t cta_excl_scan(uint32_t v, uint32_t& excl, uint32_t* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < kSortWarps ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < kSortWarps; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kSortWarps) wsum[lane] = t;              // inclusive warp totals
  }
  __syncthreads();
  const uint32_t total = wsum[kSortWarps - 1];
  excl = x - v + (w > 0 ? wsum[w - 1] : 0u);
  __syncthreads();                                      // wsum reusable
  return total;
}

__global__ void __launch_bounds__(kSortThreads) order_sort_kernel(SortArgs a) {
  extern __shared__ uint32_t sS[];                      // [G] segment prefixes
  __shared__ uint32_t hist[256];
  __shared__ uint32_t off[256];
  __shared__ uint32_t cnt[kSortWarps][256];
  __shared__ uint32_t wsum[kSortWarps];
  cg::grid_group grid = cg::this_grid();
  const int G = int(gridDim.x), b = int(blockIdx.x), t = int(threadIdx.x);
  const int lane = t & 31, w = t >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t c0 = int64_t(b) * a.chunk;
  const int64_t c1 = c0 + a.chunk < a.n ? c0 + a.chunk : a.n;

  for (int p = 0; p < a.passes; ++p) {
    const uint64_t* kr = p == 0 ? a.kin : ((p & 1) ? a.ktmp : a.kout);
    const uint32_t* sr = p == 0 ? a.sin : ((p & 1) ? a.stmp : a.sout);
    uint64_t* kw = (p & 1) ? a.kout : a.ktmp;
    uint32_t* sw = (p & 1) ? a.sout : a.stmp;
    const int shift = a.begin_bit + 8 * p;

    // A: digit histogram of this CTA's chunk
    hist[t] = 0u;
    __syncthreads();
    for (int64_t i = c0 + t; i < c1; i += kSortThreads)
      atomicAdd(&hist[uint32_t(__ldcg(kr + i) >> shift) & 255u], 1u);
    __syncthreads();
    a.H[size_t(t) * G + b] = hist[t];
    grid.sync();

    // B: in-place exclusive scan of segment b (256 entries) + its total
    {
      const size_t idx = size_t(b) * 256 + t;
      const uint32_t v = __ldcg(a.H + idx);
      uint32_t ex;
      const uint32_t tot = cta_excl_scan(v, ex, wsum);
      a.H[idx] = ex;
      if (t == 0) a.S[b] = tot;
    }
    grid.sync();

    // C: segment prefixes -> this CTA's digit offsets, then the scatter
    {
      uint32_t carry = 0;
      for (int base = 0; base < G; base += kSortThreads) {
        const int i = base + t;
        const uint32_t v = i < G ? __ldcg(a.S + i) : 0u;
        uint32_t ex;
        const uint32_t tot = cta_excl_scan(v, ex, wsum);
        if (i < G) sS[i] = carry + ex;
        carry += tot;
      }
      __syncthreads();
      const size_t fi = size_t(t) * G + b;
      off[t] = sS[fi >> 8] + __ldcg(a.H + fi);
    }
    for (int64_t tb = c0; tb < c1; tb += kSortTile) {
#pragma unroll
      for (int k = lane; k < 256; k += 32) cnt[w][k] = 0u;
      __syncwarp();
      uint64_t key[kSortSteps];
      uint32_t slot[kSortSteps], dig[kSortSteps], rnk[kSortSteps];
#pragma unroll
      for (int s = 0; s < kSortSteps; ++s) {
        const int64_t i = tb + int64_t(w) * kSortWarpKeys + 32 * s + lane;
        const bool valid = i < c1;
        key[s] = valid ? __ldcg(kr + i) : 0ull;
        slot[s] = valid ? __ldcg(sr + i) : 0u;
        const uint32_t d = valid ? uint32_t(key[s] >> shift) & 255u : 0x100u + lane;
        dig[s] = d;
        const unsigned peers = __match_any_sync(kFull, d);
        uint32_t v = 0;
        if (valid) v = cnt[w][d];
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) cnt[w][d] = v + __popc(peers);
        __syncwarp();
        rnk[s] = v + __popc(peers & lt);
      }
      __syncthreads();
      uint32_t run = 0;                                // digit t: exclusive over warps
#pragma unroll
      for (int ww = 0; ww < kSortWarps; ++ww) {
        const uint32_t c = cnt[ww][t];
        cnt[ww][t] = run;
        run += c;
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < kSortSteps; ++s) {
        const uint32_t d = dig[s];
        if (d < 256u) {
          const uint32_t pos = off[d] + cnt[w][d] + rnk[s];
          kw[pos] = key[s];
          sw[pos] = slot[s];
        }
      }
      __syncthreads();
      off[t] += run;
      __syncthreads();
    }
    if (p + 1 < a.passes) grid.sync();
  }
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// upper bound of the cooperative grid (8 CTAs of 256 threads per SM)
static int sort_grid_cap() { return sm_count() * (2048 / kSortThreads); }

}  // namespace pdg

using namespace pdg;

extern "C" size_t pdg_order_temp_bytes(int64_t n) {
  if (n < 0) n = 0;
  const size_t G = size_t(sort_grid_cap());
  return align256(size_t(n) * 8) + align256(size_t(n) * 4) + align256(256 * G * 4) +
         align256(G * 4);
}

extern "C" int pdg_order(const uint64_t* keys_in, uint64_t* keys_out,
                         const uint32_t* slots_in, uint32_t* slots_out, int64_t n,
                         int32_t begin_bit, void* temp, size_t temp_bytes,
                         void* stream) {
  if (n < 0 || (n > 0 && (!keys_in || !keys_out || !slots_in || !slots_out || !temp))) {
    set_error("pdg_order: invalid arguments");
    return PDG_EINVAL;
  }
  if (begin_bit != 0 && begin_bit != 32) {
    set_error("pdg_order: begin_bit must be 0 or 32");
    return PDG_EINVAL;
  }
  if (n > (int64_t(1) << 32) - 1) {
    set_error("pdg_order: more than 2^32 - 1 keys");
    return PDG_EUNSUPPORTED;
  }
  if (n == 0) return PDG_OK;
  const size_t need = pdg_order_temp_bytes(n);
  if (temp_bytes < need) {
    set_error("pdg_order: temp_bytes %zu < %zu", temp_bytes, need);
    return PDG_EINVAL;
  }
  const int gcap = sort_grid_cap();
  int per_sm = 0;
  const size_t dsmem = size_t(gcap) * 4;
  if (int r = launch_setup(reinterpret_cast<const void*>(order_sort_kernel), kSortThreads,
                           dsmem, &per_sm))
    return r;
  int64_t G = int64_t(per_sm) * sm_count();
  if (G > gcap) G = gcap;
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  if (G > tiles) G = tiles;
  SortArgs a;
  char* tp = static_cast<char*>(temp);
  a.kin = keys_in;
  a.sin = slots_in;
  a.kout = keys_out;
  a.sout = slots_out;
  a.ktmp = reinterpret_cast<uint64_t*>(tp);
  tp += align256(size_t(n) * 8);
  a.stmp = reinterpret_cast<uint32_t*>(tp);
  tp += align256(size_t(n) * 4);
  a.H = reinterpret_cast<uint32_t*>(tp);
  tp += align256(256 * size_t(gcap) * 4);
  a.S = reinterpret_cast<uint32_t*>(tp);
  a.n = n;
  a.chunk = ((tiles + G - 1) / G) * kSortTile;
  G = (n + a.chunk - 1) / a.chunk;                       // no CTA without keys
  a.begin_bit = begin_bit;
  a.passes = (64 - begin_bit) / 8;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(order_sort_kernel),
                                              dim3(unsigned(G)), dim3(kSortThreads), args,
                                              size_t(G) * 4, (cudaStream_t)stream);
  return cuda_status(e, "pdg_order (order_sort_kernel)");
}
