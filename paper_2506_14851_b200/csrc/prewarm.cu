// K4: backend-prewarm estimator for sm_100a.
//
// K4a prewarm_plan_kernel -- batched, bit-exact pdgsim.prewarm.plan_prewarm
//     (prewarm.py:42-96): one warp per (application, successor) job.  The
//     completion samples are conditioned on "still running" (> now, else
//     all), bucketed (distributions.py:79-105); the candidate triggers are
//     max(boundary - t_p, now) and now; the plan takes the latest candidate t_s
//     with p_s * survival(t_s + t_p) >= K, survival(x) = #{s >= x} / n
//     (distributions.py:73-77).  p_e is monotone in t_s, so "first hit in
//     descending order" == "largest satisfying candidate": every lane scores
//     its candidates independently and a warp max picks the trigger.
//
// K4b prewarm_need_kernel -- the per-backend-type need probability over a
//     window grid (BASELINE config 5): for each queued application and window
//     edge W_k, need[a, type(v), k] = sum over successors v of the current
//     unit of p_s(v) * P(completion < now + W_k), with the completion time
//     distribution of the current unit taken exactly as _plan_prewarms builds
//     it (simcore.py:450-487: now + unconditioned service samples, then the
//     "> now" conditioning of plan_prewarm).  One warp per application, one
//     lane per window; the sorted service pools make each survival a binary
//     search.  Output need[N, T, K] (float32) is the HBM-bound part.
//     prewarm_need_batched_kernel is the production form (packed unit
//     records + window index): two consecutive applications per warp with
//     their load chains interleaved, per-warp aggregates without atomics.
#include "common.cuh"

namespace pdg {

struct PlanArgs {
  const double* pool;       // completion samples (absolute times)
  const int32_t* off;       // [J]
  const int32_t* len;       // [J]
  const int32_t* bucket_count;
  const double* p_s;
  const double* t_p;
  const double* knob;
  const double* now;
  int64_t n_jobs;
  uint8_t* has_plan;
  double* trigger;
  double* p_e;
  double* scratch;          // per-warp conditioned samples
  int scratch_per_warp;
  const double* shift;      // optional [J]: samples are relative, completion = shift + s
};

// count of cond samples >= x (cond = samples > now, or all if none)
__device__ __forceinline__ int count_ge(const double* s, int n, double now, bool all, double x,
                                       int lane, bool rel = false, double sh = 0.0) {
  int c = 0;
  for (int i = lane; i < n; i += 32) {
    const double v = rel ? dadd(sh, s[i]) : s[i];
    c += ((all || v > now) && v >= x) ? 1 : 0;
  }
  return warp_sum(c);
}

__global__ void __launch_bounds__(128) prewarm_plan_kernel(PlanArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = gw; j < a.n_jobs; j += nw) {
    const double* s = a.pool + a.off[j];
    const int n = a.len[j];
    const double now = a.now[j], p_s = a.p_s[j], t_p = a.t_p[j], knob = a.knob[j];
    const bool rel = a.shift != nullptr;             // completion = shift + sample (simcore.py:455)
    const double sh = rel ? a.shift[j] : 0.0;
    if (p_s < knob || n <= 0) {                      // prewarm.py:63-64
      // (n < 0: a slot the trigger setup flagged; its has_plan stays)
      if (lane == 0) { if (n >= 0) a.has_plan[j] = 0; a.trigger[j] = 0.0; a.p_e[j] = 0.0; }
      continue;
    }
    // relative pools are sorted (the prewarm tables) and shift + s is
    // monotone in s: conditioned samples and those >= x are suffixes
    auto first_ge = [&](double y, bool strict) {
      int lo_i = 0, hi_i = n;
      while (lo_i < hi_i) {
        const int mid = (lo_i + hi_i) >> 1;
        const double v = dadd(sh, s[mid]);
        if (strict ? v > y : v >= y) hi_i = mid; else lo_i = mid + 1;
      }
      return lo_i;
    };
    // conditioning on "still running" (prewarm.py:65-67)
    int live = 0;
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    int start_gt = 0;                                // first sample > now (sorted pools)
    if (rel) {
      start_gt = first_ge(now, true);
      live = n - start_gt;
    } else {
      for (int i = lane; i < n; i += 32) live += s[i] > now ? 1 : 0;
      live = warp_sum(live);
    }
    const bool all = live == 0;
    const int m = all ? n : live;
    if (rel) {                                       // sorted: the suffix's ends
      lo = dadd(sh, s[all ? 0 : start_gt]);
      hi = dadd(sh, s[n - 1]);
    } else {
      for (int i = lane; i < n; i += 32) {
        const double v = s[i];
        if (all || v > now) { lo = fmin(lo, v); hi = fmax(hi, v); }
      }
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(kFull, lo, o));
        hi = fmax(hi, __shfl_xor_sync(kFull, hi, o));
      }
    }
    // bucket boundaries (distributions.py:120-126): [lo] if degenerate, else
    // lo + j*w for j = 0..k with w = (hi - lo)/k
    const int k = a.bucket_count[j];
    const bool degen = lo == hi;
    const double w = degen ? 0.0 : __ddiv_rn(dsub(hi, lo), small_int_to_double(k));
    const int nb = degen ? 1 : k + 1;
    // candidates: max(b - t_p, now) for each boundary, plus now
    double best_ts = -__longlong_as_double(0x7ff0000000000000ll), best_pe = 0.0;
    bool any = false;
    for (int c = lane; c <= nb; c += 32) {
      double ts;
      if (c == nb) {
        ts = now;
      } else {
        const double b = c == 0 ? lo : dadd(lo, dmul(small_int_to_double(c), w));
        const double t = dsub(b, t_p);
        ts = t > now ? t : now;
      }
      const double x = dadd(ts, t_p);
      int cnt = 0;
      if (rel) {                                     // one binary search, not a scan
        const int start = all ? 0 : start_gt;
        const int from = first_ge(x, false);
        cnt = n - (from > start ? from : start);
      } else {
        for (int i = 0; i < n; ++i) {
          const double v = s[i];
          cnt += ((all || v > now) && v >= x) ? 1 : 0;
        }
      }
      const double pe = dmul(p_s, __ddiv_rn(small_int_to_double(cnt), small_int_to_double(m)));
      if (pe >= knob && ts > best_ts) { best_ts = ts; best_pe = pe; any = true; }
    }
    const bool anyw = __any_sync(kFull, any);
    // warp arg-max of the satisfying trigger
    for (int o = 16; o > 0; o >>= 1) {
      const double ots = __shfl_xor_sync(kFull, best_ts, o);
      const double ope = __shfl_xor_sync(kFull, best_pe, o);
      if (ots > best_ts) { best_ts = ots; best_pe = ope; }
    }
    if (!anyw) {                                     // prewarm.py:87-96
      const double x = dadd(now, t_p);
      const int cnt = count_ge(s, n, now, all, x, lane, rel, sh);
      best_ts = now;
      best_pe = dmul(p_s, __ddiv_rn(small_int_to_double(cnt), small_int_to_double(m)));
    }
    if (lane == 0) { a.has_plan[j] = 1; a.trigger[j] = best_ts; a.p_e[j] = best_pe; }
  }
}

// ---------------------------------------------------------------------------
struct NeedArgs {
  const double* svc_sorted;     // unconditioned service samples, ascending, per unit
  const int32_t* svc_off;       // [U] per global unit
  const int32_t* svc_len;
  const int32_t* graph_base;    // [G]
  const int32_t* succ_off;      // [U]
  const int32_t* succ_len;      // [U]
  const int32_t* succ_nxt;      // local unit index
  const double* succ_p;         // branch probability (pdgraph.py:182-194)
  const int32_t* unit_type;     // [U] backend type (warm content), -1 none
  const int32_t* graph;         // [N] job graph
  const int32_t* unit;          // [N] current unit (local)
  const double* now;            // [N]
  const double* windows;        // [K] window edges W_k (relative)
  int n_types, n_windows;
  int64_t n;
  float* need;                  // [N, T, K] optional
  double* agg;                  // [T, K] optional, sum over applications
  const int32_t* win_idx;       // [U, K] optional: lower_bound(svc[u], W_k)
  int stage_n;                  // service samples staged per warp (0 with win_idx)
  const int4* unit_rec;         // [U, 3] optional packed unit record (see header)
};

// first index i in the ascending array with now + s[i] >= x  (exact f64)
__device__ __forceinline__ int lower_bound_abs(const double* s, int n, double now, double x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (dadd(now, s[mid]) >= x) hi = mid; else lo = mid + 1;
  }
  return lo;
}

constexpr int kNeedWarps = 8;
constexpr int kNeedStage = 256;       // service samples staged in shared memory per warp

__global__ void __launch_bounds__(kNeedWarps * 32) prewarm_need_kernel(NeedArgs a) {
  // per warp: staged service samples + a private [T][K] aggregate (each lane
  // owns window column k, so no atomics until the block reduction)
  extern __shared__ double nsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int TK = a.n_types * a.n_windows;
  double* stage = nsm + size_t(wib) * a.stage_n;
  double* cagg = nsm + size_t(kNeedWarps) * a.stage_n;   // [T][K] of this CTA
  if (a.agg) {
    for (int i = threadIdx.x; i < TK; i += blockDim.x) cagg[i] = 0.0;
    __syncthreads();
  }
  const int64_t gw = int64_t(blockIdx.x) * kNeedWarps + wib;
  const int64_t nw = int64_t(gridDim.x) * kNeedWarps;
  const int kwin = lane < a.n_windows ? lane : -1;
  const double wk = kwin >= 0 ? a.windows[kwin] : 0.0;
  for (int64_t app = gw; app < a.n; app += nw) {
    const int gbase = a.graph_base[a.graph[app]];
    const int u = gbase + a.unit[app];
    const double now = a.now[app];
    // one 48-byte record per unit when available (fewer dependent loads)
    int4 r0 = make_int4(0, 0, 0, 0), r1 = r0, r2 = r0;
    if (a.unit_rec) {
      r0 = a.unit_rec[3 * int64_t(u)];
      r1 = a.unit_rec[3 * int64_t(u) + 1];
      r2 = a.unit_rec[3 * int64_t(u) + 2];
    }
    const int n = a.unit_rec ? r0.y : a.svc_len[u];
    const double* gsrc = a.svc_sorted + (a.unit_rec ? r0.x : a.svc_off[u]);
    const double* s = gsrc;
    if (n <= a.stage_n) {                            // coalesced stage, then LDS searches
      for (int i = lane; i < n; i += 32) stage[i] = gsrc[i];
      __syncwarp();
      s = stage;
    }
    // completion = now + s; conditioned on > now (all if none).  Samples
    // ascend; the common case (every sample finishes after now) is one test.
    int first_live = 0;
    if (n > 0 && !(dadd(now, s[0]) > now))
      first_live = lower_bound_abs(s, n, now, __longlong_as_double(
          __double_as_longlong(now) + 1));           // smallest value > now
    const int live = n - first_live;
    const int base = live > 0 ? first_live : 0;
    const int m = live > 0 ? live : n;
    float pneed = 0.f;                               // P(completion < now + W_k)
    if (kwin >= 0 && m > 0) {
      const double x = dadd(now, wk);
      int j;
      if (a.win_idx) {
        // samples >= W_k complete at >= now + W_k (rounding is monotone); a
        // sample just below W_k can round up onto it: walk back over those
        j = a.win_idx[int64_t(u) * a.n_windows + kwin];
        while (j > 0 && dadd(now, s[j - 1]) >= x) --j;
        j = j > base ? j : base;
      } else {
        j = base + lower_bound_abs(s + base, n - base, now, x);
      }
      pneed = 1.f - __fdiv_rn(float(n - j), float(m));
    }
    // up to 4 successors; successors of equal type are merged first
    int t0 = -1, t1 = -1, t2 = -1, t3 = -1;
    float f0 = 0.f, f1 = 0.f, f2 = 0.f, f3 = 0.f;
    if (a.unit_rec) {                                // types -1 beyond the successors
      t0 = r0.z; t1 = r0.w; t2 = r1.x; t3 = r1.y;
      f0 = __int_as_float(r1.z) * pneed;
      f1 = __int_as_float(r1.w) * pneed;
      f2 = __int_as_float(r2.x) * pneed;
      f3 = __int_as_float(r2.y) * pneed;
    } else {
      const int so = a.succ_off[u];
      const int ns = a.succ_len[u] < 4 ? a.succ_len[u] : 4;
      if (ns > 0) { t0 = a.unit_type[gbase + a.succ_nxt[so]];     f0 = float(a.succ_p[so]) * pneed; }
      if (ns > 1) { t1 = a.unit_type[gbase + a.succ_nxt[so + 1]]; f1 = float(a.succ_p[so + 1]) * pneed; }
      if (ns > 2) { t2 = a.unit_type[gbase + a.succ_nxt[so + 2]]; f2 = float(a.succ_p[so + 2]) * pneed; }
      if (ns > 3) { t3 = a.unit_type[gbase + a.succ_nxt[so + 3]]; f3 = float(a.succ_p[so + 3]) * pneed; }
    }
    if (t1 >= 0 && t1 == t0) { f0 += f1; t1 = -1; }
    if (t2 >= 0 && t2 == t0) { f0 += f2; t2 = -1; }
    if (t2 >= 0 && t2 == t1) { f1 += f2; t2 = -1; }
    if (t3 >= 0 && t3 == t0) { f0 += f3; t3 = -1; }
    if (t3 >= 0 && t3 == t1) { f1 += f3; t3 = -1; }
    if (t3 >= 0 && t3 == t2) { f2 += f3; t3 = -1; }
    // successors 4.. (no unit records): merged into the first four by type,
    // or written once per further type (its first occurrence sums the rest)
    const int ns_all = a.unit_rec ? 0 : a.succ_len[u];
    auto succ_type = [&](int i) {
      const int ty = a.unit_type[gbase + a.succ_nxt[a.succ_off[u] + i]];
      return ty < a.n_types ? ty : -1;               // no need row for that type
    };
    for (int i = 4; i < ns_all; ++i) {
      const int ty = succ_type(i);
      const float f = float(a.succ_p[a.succ_off[u] + i]) * pneed;
      if (ty < 0) continue;
      if (ty == t0) f0 += f;
      else if (ty == t1) f1 += f;
      else if (ty == t2) f2 += f;
      else if (ty == t3) f3 += f;
    }
    t0 = t0 < a.n_types ? t0 : -1;
    t1 = t1 < a.n_types ? t1 : -1;
    t2 = t2 < a.n_types ? t2 : -1;
    t3 = t3 < a.n_types ? t3 : -1;
    if (a.need && (TK & 3) == 0) {                   // dense row: 16-B zero stores ...
      float4* row4 = reinterpret_cast<float4*>(a.need + app * int64_t(TK));
      for (int i = lane; i < (TK >> 2); i += 32) __stcs(row4 + i, make_float4(0.f, 0.f, 0.f, 0.f));
      __syncwarp();                                  // ... ordered before the values
    }
    if (kwin >= 0) {
      if (a.need && (TK & 3) == 0) {                 // the <= 4 non-zero types
        float* row = a.need + app * int64_t(TK) + kwin;
        if (t0 >= 0) __stcs(row + t0 * a.n_windows, f0);
        if (t1 >= 0) __stcs(row + t1 * a.n_windows, f1);
        if (t2 >= 0) __stcs(row + t2 * a.n_windows, f2);
        if (t3 >= 0) __stcs(row + t3 * a.n_windows, f3);
      } else if (a.need) {                           // dense row, each element once
        float* row = a.need + app * int64_t(TK) + kwin;
        for (int t = 0; t < a.n_types; ++t) {
          const float v = t == t0 ? f0 : t == t1 ? f1 : t == t2 ? f2 : t == t3 ? f3 : 0.f;
          __stcs(row + t * a.n_windows, v);
        }
      }
      if (a.agg) {
        if (t0 >= 0) atomicAdd(cagg + t0 * a.n_windows + kwin, double(f0));
        if (t1 >= 0) atomicAdd(cagg + t1 * a.n_windows + kwin, double(f1));
        if (t2 >= 0) atomicAdd(cagg + t2 * a.n_windows + kwin, double(f2));
        if (t3 >= 0) atomicAdd(cagg + t3 * a.n_windows + kwin, double(f3));
      }
    }
    if (ns_all > 4) {                                // types beyond the first four
      __syncwarp();                                  // after the zero fill and the stores
      for (int i = 4; i < ns_all; ++i) {
        const int ty = succ_type(i);
        if (ty < 0 || ty == t0 || ty == t1 || ty == t2 || ty == t3) continue;
        bool first = true;
        for (int k = 4; k < i; ++k) first = first && succ_type(k) != ty;
        if (!first) continue;
        float f = 0.f;
        for (int k = i; k < ns_all; ++k)
          if (succ_type(k) == ty) f += float(a.succ_p[a.succ_off[u] + k]) * pneed;
        if (kwin >= 0) {
          if (a.need) __stcs(a.need + app * int64_t(TK) + ty * a.n_windows + kwin, f);
          if (a.agg) atomicAdd(cagg + ty * a.n_windows + kwin, double(f));
        }
      }
    }
    __syncwarp();
  }
  if (a.agg) {
    __syncthreads();
    for (int i = threadIdx.x; i < TK; i += blockDim.x)
      if (cagg[i] != 0.0) atomicAdd(a.agg + i, cagg[i]);
  }
}

// The same computation for the common layout (packed unit records, window
// index, dense rows of 4k floats), NB applications per warp at a time: the
// per-application chain of dependent loads (job -> graph base -> unit record
// -> window index / samples) is issued for all NB applications before any of
// them is consumed, so NB chains are in flight per warp instead of one.
#ifndef PDG_NEED_CONSEC
#define PDG_NEED_CONSEC 1
#endif
#ifndef PDG_NEED_STCS
#define PDG_NEED_STCS 1
#endif

template <typename T>
__device__ __forceinline__ void need_st(T* p, T v) {
#if PDG_NEED_STCS
  __stcs(p, v);
#else
  *p = v;
#endif
}

template <int NB>
__global__ void __launch_bounds__(kNeedWarps * 32) prewarm_need_batched_kernel(NeedArgs a) {
  extern __shared__ double nsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int TK = a.n_types * a.n_windows, K = a.n_windows;
  // per warp [T][K] aggregate: lane k owns column k, so plain read-add-write
  double* cagg = nsm + size_t(wib) * TK;
  if (a.agg) {
    for (int i = lane; i < TK; i += 32) cagg[i] = 0.0;
    __syncwarp();
  }
  const int64_t gw = int64_t(blockIdx.x) * kNeedWarps + wib;
  const int64_t nw = int64_t(gridDim.x) * kNeedWarps;
  const int kwin = lane < K ? lane : -1;
  const double wk = kwin >= 0 ? a.windows[kwin] : 0.0;
  // warp-consecutive applications: a warp's rows form one contiguous run
  for (int64_t app0 = PDG_NEED_CONSEC ? gw * NB : gw; app0 < a.n; app0 += NB * nw) {
    int64_t app[NB];
    int g[NB], un[NB], u[NB], j[NB];
    double now[NB], s0[NB], sj[NB];
    int4 r0[NB], r1[NB], r2[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      app[b] = PDG_NEED_CONSEC ? app0 + b : app0 + b * nw;
      const int64_t q = app[b] < a.n ? app[b] : app0;
      g[b] = __ldg(a.graph + q);
      un[b] = __ldg(a.unit + q);
      now[b] = __ldg(a.now + q);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) u[b] = __ldg(a.graph_base + g[b]) + un[b];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      r0[b] = __ldg(a.unit_rec + 3 * int64_t(u[b]));
      r1[b] = __ldg(a.unit_rec + 3 * int64_t(u[b]) + 1);
      r2[b] = __ldg(a.unit_rec + 3 * int64_t(u[b]) + 2);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const double* s = a.svc_sorted + r0[b].x;
      s0[b] = r0[b].y > 0 ? __ldg(s) : 0.0;
      j[b] = kwin >= 0 ? __ldg(a.win_idx + int64_t(u[b]) * K + kwin) : 0;
    }
#pragma unroll
    for (int b = 0; b < NB; ++b)
      sj[b] = j[b] > 0 ? __ldg(a.svc_sorted + r0[b].x + j[b] - 1) : 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (app[b] >= a.n) break;                      // warp-uniform
      const int n = r0[b].y;
      const double* s = a.svc_sorted + r0[b].x;
      const double nw_ = now[b];
      int first_live = 0;
      if (n > 0 && !(dadd(nw_, s0[b]) > nw_))
        first_live = lower_bound_abs(s, n, nw_, __longlong_as_double(
            __double_as_longlong(nw_) + 1));         // smallest value > now
      const int live = n - first_live;
      const int base = live > 0 ? first_live : 0;
      const int m = live > 0 ? live : n;
      float pneed = 0.f;
      if (kwin >= 0 && m > 0) {
        const double x = dadd(nw_, wk);
        int jj = j[b];
        if (jj > 0 && dadd(nw_, sj[b]) >= x) {       // rounding walk-back (rare)
          --jj;
          while (jj > 0 && dadd(nw_, s[jj - 1]) >= x) --jj;
        }
        jj = jj > base ? jj : base;
        pneed = 1.f - __fdiv_rn(float(n - jj), float(m));
      }
      int t0 = r0[b].z, t1 = r0[b].w, t2 = r1[b].x, t3 = r1[b].y;
      float f0 = __int_as_float(r1[b].z) * pneed;
      float f1 = __int_as_float(r1[b].w) * pneed;
      float f2 = __int_as_float(r2[b].x) * pneed;
      float f3 = __int_as_float(r2[b].y) * pneed;
      if (t1 >= 0 && t1 == t0) { f0 += f1; t1 = -1; }
      if (t2 >= 0 && t2 == t0) { f0 += f2; t2 = -1; }
      if (t2 >= 0 && t2 == t1) { f1 += f2; t2 = -1; }
      if (t3 >= 0 && t3 == t0) { f0 += f3; t3 = -1; }
      if (t3 >= 0 && t3 == t1) { f1 += f3; t3 = -1; }
      if (t3 >= 0 && t3 == t2) { f2 += f3; t3 = -1; }
      {
        float4* row4 = reinterpret_cast<float4*>(a.need + app[b] * int64_t(TK));
#pragma unroll 4
        for (int i = lane; i < (TK >> 2); i += 32)
          need_st(row4 + i, make_float4(0.f, 0.f, 0.f, 0.f));
        __syncwarp();
        if (kwin >= 0) {
          float* row = a.need + app[b] * int64_t(TK) + kwin;
          if (t0 >= 0) need_st(row + t0 * K, f0);
          if (t1 >= 0) need_st(row + t1 * K, f1);
          if (t2 >= 0) need_st(row + t2 * K, f2);
          if (t3 >= 0) need_st(row + t3 * K, f3);
        }
      }
      if (kwin >= 0) {
        if (a.agg) {
          double* c = cagg + kwin;
          if (t0 >= 0) c[t0 * K] += double(f0);
          if (t1 >= 0) c[t1 * K] += double(f1);
          if (t2 >= 0) c[t2 * K] += double(f2);
          if (t3 >= 0) c[t3 * K] += double(f3);
        }
      }
      __syncwarp();
    }
  }
  if (a.agg) {                                       // warps -> CTA -> global
    __syncthreads();
    for (int i = threadIdx.x; i < TK; i += blockDim.x) {
      double v = 0.0;
      for (int w = 0; w < kNeedWarps; ++w) v += nsm[size_t(w) * TK + i];
      if (v != 0.0) atomicAdd(a.agg + i, v);
    }
  }
}

#ifndef PDG_NEED_BATCH
#define PDG_NEED_BATCH 2
#endif

}  // namespace pdg

using namespace pdg;

extern "C" int pdg_plan_prewarm(const double* pool, const int32_t* off, const int32_t* len,
                                const int32_t* bucket_count, const double* p_s,
                                const double* t_p, const double* knob, const double* now,
                                int64_t n_jobs, uint8_t* has_plan, double* trigger,
                                double* p_e, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && (!pool || !off || !len || !bucket_count || !p_s || !t_p ||
                                    !knob || !now || !has_plan || !trigger || !p_e))) {
    set_error("pdg_plan_prewarm: invalid arguments");
    return PDG_EINVAL;
  }
  if (n_jobs == 0) return PDG_OK;
  PlanArgs a{pool, off, len, bucket_count, p_s, t_p, knob, now, n_jobs, has_plan, trigger, p_e,
             nullptr, 0, nullptr};
  int64_t blocks = (n_jobs * 32 + 127) / 128;
  const int64_t cap = int64_t(sm_count()) * 16;
  if (blocks > cap) blocks = cap;
  prewarm_plan_kernel<<<unsigned(blocks), 128, 0, (cudaStream_t)stream>>>(a);
  return launch_status("prewarm_plan_kernel");
}

__global__ void window_index_kernel(const double* __restrict__ svc, const int32_t* __restrict__ off,
                                    const int32_t* __restrict__ len, int32_t n_units,
                                    const double* __restrict__ windows, int32_t k,
                                    int32_t* __restrict__ out) {
  const int64_t total = int64_t(n_units) * k;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int u = int(i / k), w = int(i % k);
    const double* s = svc + off[u];
    const double x = windows[w];
    int lo = 0, hi = len[u];
    while (lo < hi) {                                // first s >= W_k
      const int mid = (lo + hi) >> 1;
      if (s[mid] >= x) hi = mid; else lo = mid + 1;
    }
    out[i] = lo;
  }
}

extern "C" int pdg_prewarm_window_index(const pdg_prewarm_tables* t, int32_t n_units,
                                        const double* windows, int32_t n_windows,
                                        int32_t* out, void* stream) {
  if (!t || n_units < 0 || n_windows < 1 || n_windows > 32 || !windows || !out) {
    set_error("pdg_prewarm_window_index: invalid arguments");
    return PDG_EINVAL;
  }
  if (n_units == 0) return PDG_OK;
  int64_t blocks = (int64_t(n_units) * n_windows + 255) / 256;
  const int64_t cap = int64_t(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  window_index_kernel<<<unsigned(blocks), 256, 0, (cudaStream_t)stream>>>(
      t->svc_sorted, t->svc_off, t->svc_len, n_units, windows, n_windows, out);
  return launch_status("window_index_kernel");
}

extern "C" int pdg_prewarm_need(const pdg_prewarm_tables* t, const int32_t* graph,
                                const int32_t* unit, const double* now, int64_t n,
                                const double* windows, int32_t n_windows, int32_t n_types,
                                float* need, double* agg, void* stream) {
  if (!t || n < 0 || n_windows < 1 || n_windows > 32 || n_types < 1 || n_types > 64 ||
      (n > 0 && (!graph || !unit || !now || !windows))) {
    set_error("pdg_prewarm_need: invalid arguments (1 <= windows <= 32, 1 <= types <= 64)");
    return PDG_EINVAL;
  }
  if (n == 0) return PDG_OK;
  NeedArgs a{t->svc_sorted, t->svc_off, t->svc_len, t->graph_base, t->succ_off, t->succ_len,
             t->succ_nxt, t->succ_p, t->unit_type, graph, unit, now, windows, n_types,
             n_windows, n, need, agg, t->win_idx, t->win_idx ? 0 : kNeedStage,
             reinterpret_cast<const int4*>(t->unit_rec)};
  if (t->unit_rec && t->win_idx && need && ((n_types * n_windows) & 3) == 0) {
    auto kern = prewarm_need_batched_kernel<PDG_NEED_BATCH>;
    const size_t smem = agg ? sizeof(double) * size_t(kNeedWarps) * n_types * n_windows : 0;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(prewarm_need_batched)");
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNeedWarps * 32, smem);
    int64_t blocks = (n + kNeedWarps * PDG_NEED_BATCH - 1) / (kNeedWarps * PDG_NEED_BATCH);
    const int64_t cap = int64_t(sm_count()) * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    kern<<<unsigned(blocks), kNeedWarps * 32, smem, (cudaStream_t)stream>>>(a);
    return launch_status("prewarm_need_batched_kernel");
  }
  const size_t smem = sizeof(double) * (size_t(kNeedWarps) * a.stage_n +
                                        (agg ? size_t(n_types) * n_windows : 0));
  cudaError_t e = cudaFuncSetAttribute(prewarm_need_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(prewarm_need_kernel)");
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prewarm_need_kernel, kNeedWarps * 32, smem);
  int64_t blocks = (n + kNeedWarps - 1) / kNeedWarps;
  const int64_t cap = int64_t(sm_count()) * (per_sm > 0 ? per_sm : 1);
  if (blocks > cap) blocks = cap;
  prewarm_need_kernel<<<unsigned(blocks), kNeedWarps * 32, smem, (cudaStream_t)stream>>>(a);
  return launch_status("prewarm_need_kernel");
}

// ---------------------------------------------------------------------------
// Config 5 triggers: plan_prewarm for every (application, successor slot) of
// a queue, straight from the prewarm tables -- the completion distribution is
// now + the current unit's service samples (simcore.py:450-478), so the
// sorted pool serves as the relative sample list (plan_prewarm only uses
// order-free statistics of it).  A setup kernel lays out the K4a jobs.
// ---------------------------------------------------------------------------
namespace pdg {
__global__ void trigger_jobs_kernel(pdg_prewarm_tables t, const int32_t* __restrict__ graph,
                                    const int32_t* __restrict__ unit,
                                    const double* __restrict__ now, int64_t n, int32_t slots,
                                    const double* __restrict__ warmup, int32_t n_types,
                                    double knob, int32_t bucket_count, int32_t* off,
                                    int32_t* len, int32_t* bc, double* p_s, double* t_p,
                                    double* kn, double* nw, uint8_t* has_plan) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < int64_t(slots) * n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t app = j / slots;
    const int slot = int(j - app * slots);
    const int gb = t.graph_base[graph[app]];
    const int u = gb + unit[app];
    const int ns = t.succ_len[u];
    int ty = -1;
    double p = 0.0;
    if (slot < ns) {
      const int so = t.succ_off[u] + slot;
      ty = t.unit_type[gb + t.succ_nxt[so]];
      p = t.succ_p[so];
    }
    // successors without warm content: no plan (simcore.py:462-464); a fan-out
    // wider than the output or a type without a warmup entry is flagged
    const uint8_t flag = ns > slots ? uint8_t(PDG_PLAN_OVERFLOW)
                       : ty >= n_types ? uint8_t(PDG_PLAN_BAD_TYPE) : uint8_t(0);
    const bool ok = ty >= 0 && flag == 0;
    off[j] = t.svc_off[u];
    len[j] = ok ? t.svc_len[u] : -1;                 // -1: the plan kernel leaves has_plan
    bc[j] = bucket_count;
    p_s[j] = p;
    t_p[j] = ok ? warmup[ty] : 0.0;
    kn[j] = knob;
    nw[j] = now[app];
    if (!ok) has_plan[j] = flag;
  }
}
}  // namespace pdg

extern "C" size_t pdg_prewarm_triggers_temp_bytes(int64_t n, int32_t slots) {
  return size_t(slots > 0 ? slots : 0) * size_t(n) * (4 * 3 + 8 * 4) + 256;
}

extern "C" int pdg_prewarm_triggers(const pdg_prewarm_tables* t, const int32_t* graph,
                                    const int32_t* unit, const double* now, int64_t n,
                                    int32_t slots, const double* warmup_by_type,
                                    int32_t n_types, double knob, int32_t bucket_count,
                                    uint8_t* has_plan, double* trigger, double* p_e,
                                    void* temp, size_t temp_bytes, void* stream) {
  if (!t || n < 0 || slots < 1 || slots > 64 || n_types < 1 || bucket_count < 1 ||
      !(knob >= 0.0 && knob <= 1.0) ||
      (n > 0 && (!graph || !unit || !now || !warmup_by_type || !has_plan || !trigger || !p_e ||
                 !temp))) {
    set_error("pdg_prewarm_triggers: invalid arguments (1 <= slots <= 64, knob in [0, 1], "
              "bucket_count >= 1)");
    return PDG_EINVAL;
  }
  if (n == 0) return PDG_OK;
  if (temp_bytes < pdg_prewarm_triggers_temp_bytes(n, slots)) {
    set_error("pdg_prewarm_triggers: temp_bytes %zu < %zu", temp_bytes,
              pdg_prewarm_triggers_temp_bytes(n, slots));
    return PDG_EINVAL;
  }
  const int64_t J = int64_t(slots) * n;
  char* b = static_cast<char*>(temp);
  double* p_s = reinterpret_cast<double*>(b);
  double* t_p = p_s + J;
  double* kn = t_p + J;
  double* nw = kn + J;
  int32_t* off = reinterpret_cast<int32_t*>(nw + J);
  int32_t* len = off + J;
  int32_t* bc = len + J;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t blocks = (J + 255) / 256;
  const int64_t cap = int64_t(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  trigger_jobs_kernel<<<unsigned(blocks), 256, 0, st>>>(*t, graph, unit, now, n, slots,
                                                        warmup_by_type, n_types, knob,
                                                        bucket_count, off, len, bc, p_s, t_p,
                                                        kn, nw, has_plan);
  int rc = launch_status("trigger_jobs_kernel");
  if (rc != PDG_OK) return rc;
  PlanArgs a{t->svc_sorted, off, len, bc, p_s, t_p, kn, nw, J, has_plan, trigger, p_e,
             nullptr, 0, nw};
  int64_t pb = (J * 32 + 127) / 128;
  const int64_t pcap = int64_t(sm_count()) * 16;
  if (pb > pcap) pb = pcap;
  prewarm_plan_kernel<<<unsigned(pb), 128, 0, st>>>(a);
  return launch_status("prewarm_plan_kernel");
}
