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
// Three grid barriers per pass; 4 passes for begin_bit = 32, 8 for 0.  The
// same kernel sorts the all-gathered keys of pdg_rank_allgather_sort and the
// three stable passes of the dispatch planner (K6).
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
  int end_bit;
  int passes;         // ceil((end_bit - begin_bit) / 8); the last one writes kout
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

  const bool payload = a.sin != nullptr;
  for (int p = 0; p < a.passes; ++p) {
    // pass p writes kout when (passes - 1 - p) is even, so the last one does
    const bool to_out = ((a.passes - 1 - p) & 1) == 0;
    const uint64_t* kr = p == 0 ? a.kin : (to_out ? a.ktmp : a.kout);
    const uint32_t* sr = p == 0 ? a.sin : (to_out ? a.stmp : a.sout);
    uint64_t* kw = to_out ? a.kout : a.ktmp;
    uint32_t* sw = to_out ? a.sout : a.stmp;
    const int shift = a.begin_bit + 8 * p;
    const uint32_t dmask = a.end_bit - shift >= 8 ? 255u : (1u << (a.end_bit - shift)) - 1u;

    // A: digit histogram of this CTA's chunk
    hist[t] = 0u;
    __syncthreads();
    for (int64_t tb = c0; tb < c1; tb += kSortTile) {   // a tile's loads in flight together
      uint64_t x[kSortSteps];
#pragma unroll
      for (int s = 0; s < kSortSteps; ++s) {
        const int64_t i = tb + t + int64_t(s) * kSortThreads;
        x[s] = i < c1 ? __ldcg(kr + i) : 0ull;
      }
#pragma unroll
      for (int s = 0; s < kSortSteps; ++s)
        if (tb + t + int64_t(s) * kSortThreads < c1)
          atomicAdd(&hist[uint32_t(x[s] >> shift) & dmask], 1u);
    }
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
      // all of the lane's loads in flight before the first ranking step (the
      // warp syncs between steps would otherwise serialise them)
#pragma unroll
      for (int s = 0; s < kSortSteps; ++s) {
        const int64_t i = tb + int64_t(w) * kSortWarpKeys + 32 * s + lane;
        const bool valid = i < c1;
        key[s] = valid ? __ldcg(kr + i) : 0ull;
        slot[s] = (valid && payload) ? __ldcg(sr + i) : 0u;
      }
#pragma unroll
      for (int s = 0; s < kSortSteps; ++s) {
        const int64_t i = tb + int64_t(w) * kSortWarpKeys + 32 * s + lane;
        const bool valid = i < c1;
        const uint32_t d = valid ? uint32_t(key[s] >> shift) & dmask : 0x100u + lane;
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
          if (payload) sw[pos] = slot[s];
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

size_t order_temp_bytes(int64_t n) {
  if (n < 0) n = 0;
  const size_t G = size_t(sort_grid_cap());
  return align256(size_t(n) * 8) + align256(size_t(n) * 4) + align256(256 * G * 4) +
         align256(G * 4);
}

// Stable LSD radix sort of keys_in on bits [begin_bit, end_bit) into
// keys_out, carrying slots (optional: both null for keys only).
int order_sort(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* slots_in,
               uint32_t* slots_out, int64_t n, int begin_bit, int end_bit, void* temp,
               size_t temp_bytes, cudaStream_t stream) {
  if (n == 0 || end_bit <= begin_bit) {
    if (n > 0) {                                        // nothing to sort on: copy
      cudaError_t e = cudaMemcpyAsync(keys_out, keys_in, size_t(n) * 8,
                                      cudaMemcpyDeviceToDevice, stream);
      if (e == cudaSuccess && slots_in)
        e = cudaMemcpyAsync(slots_out, slots_in, size_t(n) * 4, cudaMemcpyDeviceToDevice,
                            stream);
      return cuda_status(e, "order_sort copy");
    }
    return PDG_OK;
  }
  const size_t need = order_temp_bytes(n);
  if (temp_bytes < need) {
    set_error("order_sort: temp_bytes %zu < %zu", temp_bytes, need);
    return PDG_EINVAL;
  }
  const int gcap = sort_grid_cap();
  int per_sm = 0;
  if (int r = launch_setup(reinterpret_cast<const void*>(order_sort_kernel), kSortThreads,
                           size_t(gcap) * 4, &per_sm))
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
  a.end_bit = end_bit;
  a.passes = (end_bit - begin_bit + 7) / 8;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(order_sort_kernel),
                                              dim3(unsigned(G)), dim3(kSortThreads), args,
                                              size_t(G) * 4, stream);
  return cuda_status(e, "order_sort_kernel");
}

}  // namespace pdg

using namespace pdg;

extern "C" size_t pdg_order_temp_bytes(int64_t n) { return order_temp_bytes(n); }

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
  return order_sort(keys_in, keys_out, slots_in, slots_out, n, begin_bit, 64, temp,
                    temp_bytes, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// K5b: incremental order after re-scoring m rows (config 4), ONE cooperative
// kernel instead of mark / select / sort / merge library passes.  With the
// previous order O (n sorted unique keys + slots), the re-scored rows R and
// their new keys B (unique too):
//   P0  mark R; gather B (key, row)
//   P1  per 1024-key tile of O: keep = !mark[slot], kept count per tile
//   P2  unmark R; tile prefixes of the kept counts; rank B by counting
//       (m <= kUpdRankMax: every CTA ranks a share of B against all of B in
//       shared memory; larger batches arrive pre-sorted by order_sort)
//   P3  a kept key k of O goes to (#kept before it) + (#B < k); the j-th
//       smallest b of B goes to j + (#kept < b) = j + kept_prefix(lower_bound(O, b)),
//       the prefix finished by one warp over the tile's keep bytes.
// Same result as a full sort of the updated keys (all keys are unique).
// ---------------------------------------------------------------------------
namespace pdg {

constexpr int kUpdTile = 1024;
constexpr int kUpdRankMax = 4096;

struct UpdArgs {
  const uint64_t* keys;     // every row's packed key (new keys of R)
  const uint64_t* ski;      // previous order
  const uint32_t* ssi;
  int64_t n;
  const int32_t* rows;
  int64_t m;
  uint8_t* mark;
  uint64_t* sko;
  uint32_t* sso;
  uint8_t* keep;
  uint64_t* bk;             // gathered batch
  uint32_t* bs;
  uint64_t* bk2;            // sorted batch
  uint32_t* bs2;
  uint32_t* tc;             // kept per tile, then exclusive tile prefixes
  uint32_t* S;              // kept per CTA
  int64_t chunk;            // keys of O per CTA (multiple of kUpdTile)
  int presorted;            // bk2 / bs2 given (m > kUpdRankMax)
};

__global__ void __launch_bounds__(kSortThreads) order_update_kernel(UpdArgs a) {
  extern __shared__ __align__(16) unsigned char usm[];     // [G] u32 | batch keys
  __shared__ uint32_t wsum[kSortWarps];
  cg::grid_group grid = cg::this_grid();
  const int G = int(gridDim.x), b = int(blockIdx.x), t = int(threadIdx.x);
  const int lane = t & 31, w = t >> 5;
  const int64_t gt = int64_t(b) * kSortThreads + t, gstride = int64_t(G) * kSortThreads;
  const int64_t c0 = int64_t(b) * a.chunk;
  const int64_t c1 = c0 + a.chunk < a.n ? c0 + a.chunk : a.n;
  uint32_t* sS = reinterpret_cast<uint32_t*>(usm);
  uint64_t* sB = reinterpret_cast<uint64_t*>(usm + ((size_t(G) * 4 + 15) & ~size_t(15)));

  // P0
  for (int64_t j = gt; j < a.m; j += gstride) {
    const int32_t r = a.rows[j];
    a.mark[r] = 1;
    if (!a.presorted) {
      a.bk[j] = a.keys[r];
      a.bs[j] = uint32_t(r);
    }
  }
  grid.sync();

  // P1: keep flags and kept count per tile (4 keys per thread per tile)
  uint32_t cta_kept = 0;
  for (int64_t tb = c0; tb < c1; tb += kUpdTile) {
    uint32_t c = 0;
#pragma unroll
    for (int s = 0; s < kUpdTile / kSortThreads; ++s) {
      const int64_t i = tb + int64_t(s) * kSortThreads + t;
      if (i < c1) {
        const uint8_t k = a.mark[__ldcg(a.ssi + i)] ? 0 : 1;
        a.keep[i] = k;
        c += k;
      }
    }
    uint32_t ex;
    const uint32_t tot = cta_excl_scan(c, ex, wsum);
    if (t == 0) a.tc[tb / kUpdTile] = tot;
    cta_kept += tot;
  }
  if (t == 0) a.S[b] = cta_kept;
  grid.sync();

  // P2: unmark; tile prefixes; rank the batch
  for (int64_t j = gt; j < a.m; j += gstride) a.mark[a.rows[j]] = 0;
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
    if (t == 0) {
      uint32_t run = sS[b];
      for (int64_t tb = c0; tb < c1; tb += kUpdTile) {
        const uint32_t c = __ldcg(a.tc + tb / kUpdTile);
        a.tc[tb / kUpdTile] = run;
        run += c;
      }
    }
  }
  if (!a.presorted && a.m > 0) {
    for (int64_t j = t; j < a.m; j += kSortThreads) sB[j] = __ldcg(a.bk + j);
    __syncthreads();
    for (int64_t j = gt; j < a.m; j += gstride) {
      const uint64_t x = sB[j];
      uint32_t rank = 0;
      for (int64_t i = 0; i < a.m; ++i) rank += sB[i] < x ? 1u : 0u;
      a.bk2[rank] = x;
      a.bs2[rank] = __ldcg(a.bs + j);
    }
  }
  grid.sync();

  // P3: scatter the kept keys of O ...
  // (a batch ranked here is staged back into shared memory once, so the
  // per-key binary searches over it cost shared-memory, not L2, latency)
  const bool bsm = !a.presorted && a.m > 0;
  if (bsm) {
    for (int64_t j = t; j < a.m; j += kSortThreads) sB[j] = __ldcg(a.bk2 + j);
    __syncthreads();
  }
  for (int64_t tb = c0; tb < c1; tb += kUpdTile) {
    const uint32_t base = __ldcg(a.tc + tb / kUpdTile);
    const int64_t i0 = tb + int64_t(t) * (kUpdTile / kSortThreads);   // 4 consecutive keys
    uint32_t c = 0;
    uint8_t kp[kUpdTile / kSortThreads];
#pragma unroll
    for (int s = 0; s < kUpdTile / kSortThreads; ++s) {
      kp[s] = (i0 + s < c1) ? __ldcg(a.keep + i0 + s) : 0;
      c += kp[s];
    }
    uint32_t ex;
    cta_excl_scan(c, ex, wsum);
    uint64_t kk[kUpdTile / kSortThreads];
    uint32_t ks[kUpdTile / kSortThreads];
#pragma unroll
    for (int s = 0; s < kUpdTile / kSortThreads; ++s) {   // loads in flight together
      kk[s] = kp[s] ? __ldcg(a.ski + i0 + s) : 0ull;
      ks[s] = kp[s] ? __ldcg(a.ssi + i0 + s) : 0u;
    }
#pragma unroll
    for (int s = 0; s < kUpdTile / kSortThreads; ++s) {
      if (!kp[s]) continue;
      const uint64_t k = kk[s];
      int64_t lo = 0, hi = a.m;                          // #B < k
      if (bsm) {
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (sB[mid] < k) lo = mid + 1; else hi = mid;
        }
      } else {
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (__ldcg(a.bk2 + mid) < k) lo = mid + 1; else hi = mid;
        }
      }
      const uint64_t pos = uint64_t(base) + ex + uint64_t(lo);
      a.sko[pos] = k;
      a.sso[pos] = ks[s];
      ++ex;
    }
  }
  // ... and the batch: one warp per batch key
  const int64_t gw = int64_t(b) * kSortWarps + w, nwarps = int64_t(G) * kSortWarps;
  for (int64_t j = gw; j < a.m; j += nwarps) {
    const uint64_t x = __ldcg(a.bk2 + j);
    // L = #O < x by a 32-way search: every round the warp probes 32 evenly
    // spaced keys of the candidate range [lo, hi] and keeps the gap the
    // ballot points at (4 dependent rounds for 1M keys instead of 20)
    int64_t lo = 0, hi = a.n;
    while (hi > lo) {
      const int64_t step = (hi - lo + 31) / 32;
      const int64_t q = lo + int64_t(lane + 1) * step - 1;
      const bool below = q < hi && __ldcg(a.ski + q) < x;
      const int c = __popc(__ballot_sync(kFull, below));   // probes below x: a prefix
      const int64_t nlo = lo + int64_t(c) * step;
      const int64_t qc = lo + int64_t(c + 1) * step - 1;   // first probe >= x, if any
      hi = qc < hi ? qc : hi;
      lo = nlo < hi ? nlo : hi;
    }
    const int64_t tile = lo / kUpdTile, ts = tile * kUpdTile;
    uint32_t c = 0;                                      // kept in [ts, lo)
    for (int64_t i = ts + lane; i < lo; i += 32) c += __ldcg(a.keep + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    // (lo = n: every key of O is below x, so all n - m kept ones are)
    const uint32_t before = lo < a.n ? __ldcg(a.tc + tile) + c : uint32_t(a.n - a.m);
    if (lane == 0) {
      const uint64_t pos = uint64_t(j) + before;
      a.sko[pos] = x;
      a.sso[pos] = __ldcg(a.bs2 + j);
    }
  }
}

__global__ void gather_batch_kernel(const int32_t* __restrict__ rows, int64_t m,
                                    const uint64_t* __restrict__ keys, uint64_t* __restrict__ k,
                                    uint32_t* __restrict__ s) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = rows[i];
    k[i] = keys[r];
    s[i] = uint32_t(r);
  }
}

static size_t update_temp_bytes(int64_t n, int64_t m) {
  const size_t nn = size_t(n > 0 ? n : 1), mm = size_t(m > 0 ? m : 1);
  const size_t tiles = (nn + kUpdTile - 1) / kUpdTile;
  const size_t G = size_t(sort_grid_cap());
  return align256(nn) + 2 * align256(mm * 8) + 2 * align256(mm * 4) + align256(tiles * 4) +
         align256(G * 4) + (m > kUpdRankMax ? order_temp_bytes(m) : 0) + 256;
}

}  // namespace pdg

extern "C" size_t pdg_order_update_temp_bytes(int64_t n, int64_t m) {
  return update_temp_bytes(n, m);
}

extern "C" int pdg_order_update(const uint64_t* keys, const uint64_t* sorted_keys_in,
                                const uint32_t* sorted_slots_in, int64_t n,
                                const int32_t* rows, int64_t m, uint8_t* mark,
                                uint64_t* sorted_keys_out, uint32_t* sorted_slots_out,
                                void* temp, size_t temp_bytes, void* stream) {
  if (n < 0 || m < 0 || m > n || n > (int64_t(1) << 32) - 1 ||
      (n > 0 && (!keys || !sorted_keys_in || !sorted_slots_in || !mark || !sorted_keys_out ||
                 !sorted_slots_out)) ||
      (m > 0 && !rows) || !temp) {
    set_error("pdg_order_update: invalid arguments");
    return PDG_EINVAL;
  }
  if (temp_bytes < update_temp_bytes(n, m)) {
    set_error("pdg_order_update: temp_bytes %zu too small", temp_bytes);
    return PDG_EINVAL;
  }
  if (n == 0) return PDG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nn = size_t(n), mm = size_t(m > 0 ? m : 1);
  const size_t tiles = (nn + kUpdTile - 1) / kUpdTile;
  const int gcap = sort_grid_cap();
  char* p = static_cast<char*>(temp);
  UpdArgs a;
  a.keys = keys;
  a.ski = sorted_keys_in;
  a.ssi = sorted_slots_in;
  a.n = n;
  a.rows = rows;
  a.m = m;
  a.mark = mark;
  a.sko = sorted_keys_out;
  a.sso = sorted_slots_out;
  a.keep = reinterpret_cast<uint8_t*>(p);   p += align256(nn);
  a.bk = reinterpret_cast<uint64_t*>(p);    p += align256(mm * 8);
  a.bk2 = reinterpret_cast<uint64_t*>(p);   p += align256(mm * 8);
  a.bs = reinterpret_cast<uint32_t*>(p);    p += align256(mm * 4);
  a.bs2 = reinterpret_cast<uint32_t*>(p);   p += align256(mm * 4);
  a.tc = reinterpret_cast<uint32_t*>(p);    p += align256(tiles * 4);
  a.S = reinterpret_cast<uint32_t*>(p);     p += align256(size_t(gcap) * 4);
  a.presorted = m > kUpdRankMax ? 1 : 0;
  if (a.presorted) {                        // large batch: gather + one-kernel sort first
    gather_batch_kernel<<<unsigned(sm_count()) * 4, 256, 0, st>>>(rows, m, keys, a.bk, a.bs);
    if (int r = launch_status("gather_batch_kernel")) return r;
    if (int r = order_sort(a.bk, a.bk2, a.bs, a.bs2, m, 0, 64, p, order_temp_bytes(m), st))
      return r;
  }
  const size_t dsmem = ((size_t(gcap) * 4 + 15) & ~size_t(15)) +
                       (a.presorted ? 0 : size_t(m) * 8);
  int per_sm = 0;
  if (int r = launch_setup(reinterpret_cast<const void*>(order_update_kernel), kSortThreads,
                           dsmem, &per_sm))
    return r;
  int64_t G = int64_t(per_sm) * sm_count();
  if (G > gcap) G = gcap;
  const int64_t need_tiles = int64_t(tiles);
  if (G > need_tiles) G = need_tiles;
  a.chunk = ((need_tiles + G - 1) / G) * kUpdTile;
  G = (n + a.chunk - 1) / a.chunk;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(order_update_kernel),
                                              dim3(unsigned(G)), dim3(kSortThreads), args,
                                              dsmem, st);
  return cuda_status(e, "pdg_order_update (order_update_kernel)");
}
