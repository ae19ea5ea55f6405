// K2 + K3 + a4: the PDGraph demand engine for sm_100a.
//
// Replaces estimator.monte_carlo_remaining_demand (estimator.py:305-362) with
// its per-unit sampler (236-286), one-hop conditioning (155-233, 289-302) and
// ApplicationInstance.set_remaining's bucketing (sched.py:170-181,
// distributions.py:79-105).  Output samples are bit-identical to the
// reference for the same (graph, current unit, observations, n, seed): the
// kernels evaluate the reference's numpy PCG64 stream *by position*.
//
// The reference walk is vectorised per (step, unit): at each outer step the
// occupied-unit set is frozen, units are visited in ascending index order,
// and every walk sitting on the unit *at that moment* draws
//   choice(A, m) [, choice(B, m) | per-input-bucket choice(pool_b, m_b)],
//   then random(m)                                 (estimator.py:343-353)
// so each draw's position in the stream is (visit base) + (rank of the walk
// among the unit's members).  One warp per application in both kernels:
//
//   mc_walk_kernel (n <= 512, the production path; design at its definition
//     below): walk membership as per-unit bitsets in shared memory, the
//     visit's stream segment decoded lane-strided (lane l reads words l,
//     l+32, ..., one multiply-add per 32-word stride).
//   mc_engine_kernel (512 < n): active-walk and member compaction per visit,
//     lane-contiguous rank blocks, one PCG64 jump per lane and draw group.
//
// numpy's Lemire rejection (probability < P/2^32 per draw) shifts every later
// position.  A warp vote detects it; the application is then abandoned by the
// fast kernel and recomputed from scratch by mc_serial_kernel, which runs the
// reference algorithm with the sequential generator (one lane per app).
#include <type_traits>

#include "common.cuh"
#include "pcg64.cuh"

#ifndef PDG_UNROLL_B
#define PDG_UNROLL_B 1       // unroll of the bounded-word decode loop
#endif
#ifndef PDG_UNROLL_U
#define PDG_UNROLL_U 2       // unroll of the uniform-word loop
#endif

namespace pdg {

constexpr int kUnrollB = PDG_UNROLL_B;
constexpr int kUnrollU = PDG_UNROLL_U;
constexpr int kWarps = 4;            // apps per CTA
constexpr int kSmemWalks = 512;      // walks kept in shared memory per warp

enum : int32_t {
  F_LLM = 1, F_OWN = 2, F_ANYMASK = 4, F_IUI = 8, F_IUO = 16, F_OUO = 32, F_PUP = 64
};

struct __align__(16) UnitDesc {      // graphs.UNIT_DTYPE (64 B)
  int32_t flags, a_off, a_len, b_off, b_len, succ_off, succ_len, pool_off, ib_k, cond_off;
  double ib_lo, ib_hi;
  int32_t cond_len, pad;
};
static_assert(sizeof(UnitDesc) == 64, "unit descriptor layout");

struct __align__(16) CondDesc {      // graphs.COND_DTYPE
  int32_t up_local, pair_off, pair_len, pad;
  double lo[3], hi[3];
  int32_t k[3], ok[3], pad2[2];
};

struct __align__(8) PairRec {        // graphs.PAIR_DTYPE
  int32_t bk[3], pad;
  double in, out;
};

struct EngineArgs {
  pdg_graph_bank b;
  pdg_mc_jobs j;
  pdg_mc_out o;
  int64_t n_jobs;
  int n;             // samples per app
  int cap;           // visit cap
  int k_out;         // bucket_count of the output histogram
  int counters;      // u32 counters per warp in smem
  int max_unit_k;    // largest unit input-bucket count (own-input sampling)
  int max_pairs;     // K3 scratch per warp
  char* scratch;     // global scratch base
  size_t scratch_per_warp;
  int32_t* serial_list;   // [n_jobs] apps left to mc_serial_kernel
  int32_t* serial_count;  // [1]
  int32_t* job_next;      // [1] dynamic job counter (mc_walk_kernel)
  int32_t* redo_next;     // [1] dynamic counter over serial_list (careful mc_walk_kernel)
  const int32_t* order;   // [n_jobs] longest-first job order (NULL: queue order)
};

// distributions.py:107-118 with (lo, hi = last bucket edge, k)
__device__ __forceinline__ int bucket_of(double v, double lo, double hi, int k) {
  if (hi == lo || v <= lo) return 0;
  if (v >= hi) return k - 1;
  const double q = __ddiv_rn(dsub(v, lo), __ddiv_rn(dsub(hi, lo), small_int_to_double(k)));
  int i = __double2int_rz(q);
  return i < k - 1 ? i : k - 1;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// unit sets: 32-bit masks for graphs of <= 32 units, 64-bit above
__device__ __forceinline__ int mask_ffs(uint32_t m) { return __ffs(m); }
__device__ __forceinline__ int mask_ffs(uint64_t m) { return __ffsll((long long)m); }
__device__ __forceinline__ uint32_t warp_or(uint32_t v) { return __reduce_or_sync(kFull, v); }
__device__ __forceinline__ uint64_t warp_or(uint64_t v) {
  return (uint64_t(__reduce_or_sync(kFull, uint32_t(v >> 32))) << 32) |
         __reduce_or_sync(kFull, uint32_t(v));
}

struct Pools {            // the draw pools of one unit visit
  const double* A;
  int pa;
  const double* B;
  int pb;
};

// Per-warp stream state (warp-uniform): base state after the consumed words,
// plus the buffered high half of numpy's next_uint32.
struct Stream {
  U128 s, inc;
  bool pend;
  uint32_t pv;
  bool redrawn;     // a Lemire rejection was redrawn inside a visit (flags bit 3)
};

// Reads words forward from a base state: word q is the output after q+1 steps.
struct Cursor {
  U128 st;
  uint32_t q;      // index of the word held in w (0xffffffff: st is the base)
  uint64_t w;
};

__device__ __forceinline__ uint64_t cursor_word(Cursor& c, const uint64_t* jt, const U128& inc,
                                                uint32_t q) {
  if (q != c.q) {
    const uint32_t d = q - c.q;
    if (d == 1) c.st = pcg_step(c.st, inc);
    else c.st = pcg_jump(jt, c.st, inc, d);
    c.q = q;
    c.w = pcg_out(c.st);
  }
  return c.w;
}

// R-th 32-bit half of the bounded-draw stream (R = 0 is the buffered half).
__device__ __forceinline__ uint32_t cursor_half(Cursor& c, const uint64_t* jt, const Stream& g,
                                                uint32_t R) {
  if (g.pend) {
    if (R == 0) return g.pv;
    --R;
  }
  const uint64_t w = cursor_word(c, jt, g.inc, R >> 1);
  return (R & 1) ? uint32_t(w >> 32) : uint32_t(w);
}

template <typename Idx>
struct WarpState {
  double* tot;      // [n] accumulated remaining demand per walk
  Idx* act;         // [n] active walks, ascending
  Idx* mem;         // [n] members of the visited unit, ascending (= rank order)
  int8_t* cur;      // [n] current unit per walk (-1 = terminated)
  uint32_t* cnt;    // [counters]
  double* tmp;      // [n] own-input path: input draw / stage time per rank (global)
  uint16_t* bkt;    // [n] own-input path: input bucket per rank (global)
  Idx* osrt;        // [n] own-input path: ranks sorted by bucket (global)
  double* kin;      // [max_pairs] K3 kept inputs
  double* kout;     // [max_pairs] K3 kept outputs
};

// ---------------------------------------------------------------------------
// K3: conditioned draw pools for the current unit (estimator.py:155-233)
// ---------------------------------------------------------------------------
__device__ bool condition(const EngineArgs& a, int gbase, int cur_unit, int obs_up,
                          const double* obs, double* kin_buf, double* kout_buf, Pools& ovp,
                          bool& conditioned, int lane) {
  const UnitDesc d = reinterpret_cast<const UnitDesc*>(a.b.units)[gbase + cur_unit];
  if (obs_up < 0 || !(d.flags & F_ANYMASK)) return false;   // no override
  const CondDesc* cd = reinterpret_cast<const CondDesc*>(a.b.conds) + d.cond_off;
  int ci = -1;
  for (int q = 0; q < d.cond_len; ++q)
    if (cd[q].up_local == obs_up) ci = q;
  ovp.A = a.b.vals + d.a_off;
  ovp.pa = d.a_len;
  ovp.B = a.b.vals + d.b_off;
  ovp.pb = d.b_len;
  conditioned = false;
  if (ci < 0) return true;            // override exists, nothing joins: priors
  const CondDesc& c = cd[ci];
  int ob[3];
#pragma unroll
  for (int t = 0; t < 3; ++t)
    ob[t] = c.ok[t] ? bucket_of(obs[t], c.lo[t], c.hi[t], c.k[t]) : -2;
  // which upstream variables condition which target (estimator.py:209-221)
  const bool iui = d.flags & F_IUI, iuo = d.flags & F_IUO;
  const bool ouo = d.flags & F_OUO, pup = d.flags & F_PUP;
  const PairRec* pr = reinterpret_cast<const PairRec*>(a.b.pairs) + c.pair_off;
  const unsigned lt = lanemask_lt();
  uint32_t nin = 0, nout = 0, npar = 0;
  const int plen = c.pair_len;
  for (int base = 0; base < plen; base += 32) {
    const int p = base + lane;
    bool kn = false, ko = false, kp = false;
    double rin = 0.0, rout = 0.0;
    if (p < plen) {
      const PairRec rec = pr[p];
      rin = rec.in;
      rout = rec.out;
      // a condition on an empty upstream distribution never matches
      kn = (iui || iuo) && (!iui || (ob[0] >= 0 && rec.bk[0] == ob[0])) &&
           (!iuo || (ob[1] >= 0 && rec.bk[1] == ob[1]));
      ko = ouo && ob[1] >= 0 && rec.bk[1] == ob[1];
      kp = pup && ob[2] >= 0 && rec.bk[2] == ob[2];
    }
    const unsigned bi = __ballot_sync(kFull, kn), bo = __ballot_sync(kFull, ko);
    if (kn) kin_buf[nin + __popc(bi & lt)] = rin;
    if (ko) kout_buf[nout + __popc(bo & lt)] = rout;
    nin += __popc(bi);
    nout += __popc(bo);
    npar += __popc(__ballot_sync(kFull, kp));
  }
  __syncwarp();
  const int capu = a.b.unit_capacity ? a.b.unit_capacity[gbase + cur_unit] : 1000;
  constexpr uint32_t kMin = 5;          // MIN_CONDITIONAL_SAMPLES (estimator.py:25)
  if ((iui || iuo) && nin >= kMin) {    // FIFO cap keeps the last `capacity` kept values
    const uint32_t keep = nin > uint32_t(capu) ? uint32_t(capu) : nin;
    ovp.A = kin_buf + (nin - keep);
    ovp.pa = int(keep);
    conditioned = true;
  }
  if (ouo && nout >= kMin) {
    const uint32_t keep = nout > uint32_t(capu) ? uint32_t(capu) : nout;
    ovp.B = kout_buf + (nout - keep);
    ovp.pb = int(keep);
    conditioned = true;
  }
  if (pup && npar >= kMin) conditioned = true;
  return true;
}

__device__ __forceinline__ Pools pools_for(const EngineArgs& a, const UnitDesc& d, bool ov,
                                           const Pools& ovp) {
  Pools pl;
  if ((d.flags & F_LLM) && ov) {
    pl = ovp;
  } else {
    pl.A = a.b.vals + d.a_off;
    pl.pa = d.a_len;
    pl.B = a.b.vals + d.b_off;
    pl.pb = d.b_len;
  }
  return pl;
}

// successor index of a uniform draw: searchsorted(cum, u, side="right")
__device__ __forceinline__ int next_unit(const EngineArgs& a, const UnitDesc& d, double uu) {
  const double* cum = a.b.succ_cum + d.succ_off;
  int idx = 0;
  while (idx < d.succ_len && __ldg(cum + idx) <= uu) ++idx;
  return __ldg(a.b.succ_nxt + d.succ_off + idx);
}

// the first three successors of a unit held in registers for a whole visit
struct SuccCache {
  double c0, c1, c2;
  int n0, n1, n2, n3, ns;
  __device__ __forceinline__ void load(const EngineArgs& a, const UnitDesc& d) {
    const double* cum = a.b.succ_cum + d.succ_off;
    const int32_t* nxt = a.b.succ_nxt + d.succ_off;
    ns = d.succ_len;
    c0 = ns > 0 ? __ldg(cum) : 2.0;                // cumulative probabilities <= 1
    c1 = ns > 1 ? __ldg(cum + 1) : 2.0;
    c2 = ns > 2 ? __ldg(cum + 2) : 2.0;
    n0 = __ldg(nxt);
    n1 = ns > 0 ? __ldg(nxt + 1) : -1;
    n2 = ns > 1 ? __ldg(nxt + 2) : -1;
    n3 = ns > 2 ? __ldg(nxt + 3) : -1;
  }
  __device__ __forceinline__ int next(const EngineArgs& a, const UnitDesc& d, double uu) const {
    if (ns > 3) return next_unit(a, d, uu);
    return !(c0 <= uu) ? n0 : !(c1 <= uu) ? n1 : !(c2 <= uu) ? n2 : n3;
  }
};

// close a bounded-draw group of C halves: the word holding the last fresh half
// was read by some lane (the largest word index a cursor holds)
__device__ __forceinline__ void close_group(Stream& g, uint32_t C, const Cursor& ca,
                                            const Cursor& cb) {
  if (C == 0) return;
  const uint32_t F = C - (g.pend ? 1u : 0u);
  if (F & 1u) {
    const uint32_t qlast = (F - 1) >> 1;
    const bool own_a = ca.q == qlast, own_b = cb.q == qlast;
    const unsigned who = __ballot_sync(kFull, own_a || own_b);
    const uint64_t wv = own_a ? ca.w : cb.w;
    g.pv = uint32_t(__shfl_sync(kFull, wv, __ffs(who) - 1) >> 32);
    g.pend = true;
  } else {
    g.pend = false;
  }
}

// ---------------------------------------------------------------------------
// one (step, unit) visit; returns false if a Lemire rejection was seen (the
// application must then be recomputed by mc_serial_kernel)
// ---------------------------------------------------------------------------
template <typename Idx>
__device__ bool visit_unit(const EngineArgs& a, int gbase, int u, const Pools& ovp,
                           bool has_ov, int cur_unit, const WarpState<Idx>& ws, uint32_t na,
                           Stream& g, int lane) {
  const uint64_t* jt = a.b.jump;
  const unsigned lt = lanemask_lt();
  const UnitDesc d = reinterpret_cast<const UnitDesc*>(a.b.units)[gbase + u];
  const bool llm = d.flags & F_LLM;
  const Pools pl = pools_for(a, d, has_ov && u == cur_unit, ovp);
  const bool own = llm && (d.flags & F_OWN) && !(has_ov && u == cur_unit);
  SuccCache sc;
  sc.load(a, d);
  // members of this visit, in walk order: list position == rank
  uint32_t m = 0;
  for (uint32_t base = 0; base < na; base += 32) {
    const uint32_t idx = base + lane;
    bool is = false;
    Idx w = 0;
    if (idx < na) {
      w = ws.act[idx];
      is = ws.cur[w] == u;
    }
    const unsigned bal = __ballot_sync(kFull, is);
    if (is) ws.mem[m + __popc(bal & lt)] = w;
    m += __popc(bal);
  }
  __syncwarp();
  const uint32_t per = (m + 31) >> 5;
  const uint32_t k0 = min(lane * per, m), k1 = min(k0 + per, m);
  const uint32_t c1 = pl.pa > 1 ? m : 0u;
  const double pre = a.b.prefill_rate, dec = a.b.decode_rate;
  bool rej = false;
  Cursor ca{g.s, 0xffffffffu, 0}, cb{g.s, 0xffffffffu, 0};
  uint32_t words;
  if (!own) {
    const uint32_t C = c1 + ((llm && pl.pb > 1) ? m : 0u);
    const uint32_t F = C == 0 ? 0u : C - (g.pend ? 1u : 0u);
    words = (F + 1) >> 1;
    Cursor cd{g.s, 0xffffffffu, 0};
    for (uint32_t k = k0; k < k1; ++k) {
      const uint32_t ia = pl.pa > 1 ? lemire(cursor_half(ca, jt, g, k), uint32_t(pl.pa), rej) : 0u;
      double t = pl.A[ia];
      if (llm) {
        const uint32_t ib =
            pl.pb > 1 ? lemire(cursor_half(cb, jt, g, c1 + k), uint32_t(pl.pb), rej) : 0u;
        t = dadd(__ddiv_rn(t, pre), __ddiv_rn(pl.B[ib], dec));
      }
      // random(m) word of member k, then the successor jump (estimator.py:350-353)
      const double uu = u53_double(cursor_word(cd, jt, g.inc, words + k));
      const Idx w = ws.mem[k];
      ws.cur[w] = int8_t(sc.next(a, d, uu));
      ws.tot[w] = dadd(ws.tot[w], t);
    }
    if (__any_sync(kFull, rej)) return false;
    close_group(g, C, ca, cb);
    const unsigned last_lane = (m - 1) / per;   // it drew the last uniform
    g.s.lo = __shfl_sync(kFull, cd.st.lo, last_lane);
    g.s.hi = __shfl_sync(kFull, cd.st.hi, last_lane);
    __syncwarp();
    return true;
  }
  // ---- own-input sampling: outputs drawn per input bucket, buckets
  // ascending, walks in order within a bucket (estimator.py:275-283)
  const int K = d.ib_k;
  uint32_t* cnt = ws.cnt;
  uint32_t* start = ws.cnt + a.max_unit_k;
  uint32_t* effo = ws.cnt + 2 * a.max_unit_k;
  for (int b = lane; b < K; b += 32) cnt[b] = 0;
  __syncwarp();
  for (uint32_t k = k0; k < k1; ++k) {
    const uint32_t ia = pl.pa > 1 ? lemire(cursor_half(ca, jt, g, k), uint32_t(pl.pa), rej) : 0u;
    const double iv = pl.A[ia];
    ws.tmp[k] = iv;
    const int bb = bucket_of(iv, d.ib_lo, d.ib_hi, K);
    ws.bkt[k] = uint16_t(bb);
    atomicAdd(&cnt[bb], 1u);
  }
  __syncwarp();
  const int perb = (K + 31) >> 5;
  uint32_t la = 0, le = 0;
  for (int q = 0; q < perb; ++q) {
    const int bb = lane * perb + q;
    if (bb < K) {
      const int pln = a.b.pool_len[d.pool_off + bb];
      const int P = pln > 0 ? pln : pl.pb;
      la += cnt[bb];
      le += P > 1 ? cnt[bb] : 0u;
    }
  }
  const uint32_t ia_incl = warp_incl_scan(la, lane), ie_incl = warp_incl_scan(le, lane);
  const uint32_t eff_total = __shfl_sync(kFull, ie_incl, 31);
  uint32_t ra = ia_incl - la, re = ie_incl - le;
  __syncwarp();
  for (int q = 0; q < perb; ++q) {
    const int bb = lane * perb + q;
    if (bb < K) {
      const int pln = a.b.pool_len[d.pool_off + bb];
      const int P = pln > 0 ? pln : pl.pb;
      const uint32_t c = cnt[bb];
      start[bb] = ra;
      effo[bb] = re;
      cnt[bb] = ra;                        // cursor of the counting sort
      ra += c;
      re += P > 1 ? c : 0u;
    }
  }
  __syncwarp();
  // stable counting sort of member ranks by bucket (rank order = round order)
  for (uint32_t base = 0; base < m; base += 32) {
    const uint32_t k = base + lane;
    const bool valid = k < m;
    const int bb = valid ? int(ws.bkt[k]) : (0x10000 + lane);
    const unsigned peers = __match_any_sync(kFull, bb);
    uint32_t dest = 0;
    if (valid) dest = cnt[bb];
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == lane) cnt[bb] = dest + __popc(peers);
    __syncwarp();
    if (valid) ws.osrt[dest + __popc(peers & lt)] = Idx(k);
  }
  __syncwarp();
  for (uint32_t j = k0; j < k1; ++j) {
    const uint32_t k = ws.osrt[j];
    const int bb = ws.bkt[k];
    const int pln = a.b.pool_len[d.pool_off + bb];
    const double* pool = pln > 0 ? a.b.vals + a.b.pool_off[d.pool_off + bb] : pl.B;
    const uint32_t P = uint32_t(pln > 0 ? pln : pl.pb);
    const uint32_t pos = c1 + effo[bb] + (j - start[bb]);
    const uint32_t ob = P > 1 ? lemire(cursor_half(cb, jt, g, pos), P, rej) : 0u;
    ws.tmp[k] = dadd(__ddiv_rn(ws.tmp[k], pre), __ddiv_rn(pool[ob], dec));
  }
  if (__any_sync(kFull, rej)) return false;
  const uint32_t C = c1 + eff_total;
  const uint32_t F = C == 0 ? 0u : C - (g.pend ? 1u : 0u);
  words = (F + 1) >> 1;
  close_group(g, C, ca, cb);
  __syncwarp();
  Cursor cd{g.s, 0xffffffffu, 0};
  for (uint32_t k = k0; k < k1; ++k) {
    const double uu = u53_double(cursor_word(cd, jt, g.inc, words + k));
    const Idx w = ws.mem[k];
    ws.cur[w] = int8_t(sc.next(a, d, uu));
    ws.tot[w] = dadd(ws.tot[w], ws.tmp[k]);
  }
  const unsigned last_lane = (m - 1) / per;
  g.s.lo = __shfl_sync(kFull, cd.st.lo, last_lane);
  g.s.hi = __shfl_sync(kFull, cd.st.hi, last_lane);
  __syncwarp();
  return true;
}

// ---------------------------------------------------------------------------
// shared epilogue: samples out, capped count, bucketing (distributions.py:79-105)
// ---------------------------------------------------------------------------
// RemainingDemand.mean() = sum(samples) / n (estimator.py:55-56) with CPython
// >= 3.12 sum(): Neumaier-compensated, in sample order.  Both running sums are
// sequential float64 chains; with a buffer `sb` of n doubles the warp splits
// the work: lane 0 runs the sum chain (partial sums -> sb), all lanes form the
// compensation terms, lane 0 runs the compensation chain (same operations in
// the same order, so the same bits).  tot is overwritten in that case.
__device__ double neumaier_mean(double* tot, int n, double* sb, int lane) {
  double f = 0.0;
  if (!sb) {                                     // one lane, one pass
    if (lane == 0) {
      double c = 0.0;
      f = tot[0];
#pragma unroll 1
      for (int w = 1; w < n; ++w) {
        const double x = tot[w];
        const double t = dadd(f, x);
        c = fabs(f) >= fabs(x) ? dadd(c, dadd(dsub(f, t), x)) : dadd(c, dadd(dsub(x, t), f));
        f = t;
      }
      if (c != 0.0 && isfinite(c)) f = dadd(f, c);
    }
    return f;
  }
  if (lane == 0) {                               // pairs: 16-byte loads / stores
    const double2* t2 = reinterpret_cast<const double2*>(tot);
    double2* s2 = reinterpret_cast<double2*>(sb);
    f = tot[0];
    sb[0] = f;
    if (n > 1) sb[1] = f = dadd(f, tot[1]);
#pragma unroll 4
    for (int i = 1; i < n / 2; ++i) {
      const double2 y = t2[i];
      const double f0 = dadd(f, y.x);
      f = dadd(f0, y.y);
      s2[i] = make_double2(f0, f);
    }
    if ((n & 1) && n > 1) sb[n - 1] = f = dadd(f, tot[n - 1]);
  }
  __syncwarp();
  for (int w = lane + 1; w < n; w += 32) {       // compensation term of sample w
    const double p = sb[w - 1], t = sb[w], x = tot[w];
    tot[w] = fabs(p) >= fabs(x) ? dadd(dsub(p, t), x) : dadd(dsub(x, t), p);
  }
  __syncwarp();
  if (lane == 0) {
    const double2* e2 = reinterpret_cast<const double2*>(tot);
    double c = 0.0;
    if (n > 1) c = dadd(c, tot[1]);
#pragma unroll 4
    for (int i = 1; i < n / 2; ++i) {
      const double2 e = e2[i];
      c = dadd(dadd(c, e.x), e.y);
    }
    if ((n & 1) && n > 1) c = dadd(c, tot[n - 1]);
    if (c != 0.0 && isfinite(c)) f = dadd(f, c);
  }
  return f;
}

__device__ void write_result(const EngineArgs& a, int64_t job, double* tot,
                             const int8_t* cur, uint32_t* cnt, bool conditioned, bool has_ov,
                             bool replayed, int lane, int capped_walks = -1,
                             double* mean_buf = nullptr, bool redrawn = false) {
  const int n = a.n;
  int capped = 0;
  double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
#pragma unroll 1
  for (int w = lane; w < n; w += 32) {
    if (cur) capped += cur[w] >= 0;
    const double sv = tot[w];
    lo = fmin(lo, sv);
    hi = fmax(hi, sv);
    if (a.o.samples) a.o.samples[job * a.o.samples_stride + w] = sv;
  }
  capped = cur ? warp_sum(capped) : capped_walks;
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(kFull, lo, o));
    hi = fmax(hi, __shfl_xor_sync(kFull, hi, o));
  }
  const int64_t row = a.o.slot ? a.o.slot[job] : job;
  int k = a.k_out;
  double width = 0.0;
  if (lo == hi) k = 1;
  else width = __ddiv_rn(dsub(hi, lo), small_int_to_double(k));
#pragma unroll 1
  for (int b = lane; b < k; b += 32) cnt[b] = 0;
  __syncwarp();
#pragma unroll 1
  for (int w = lane; w < n; w += 32) {
    int idx = 0;
    if (k > 1) {
      idx = __double2int_rz(__ddiv_rn(dsub(tot[w], lo), width));
      idx = idx < k - 1 ? idx : k - 1;
    }
    atomicAdd(&cnt[idx], 1u);
  }
  __syncwarp();
  if (a.o.counts) {
    uint16_t* crow = a.o.counts + row * a.o.stride;
#pragma unroll 1
    for (int b = lane; b < a.o.stride; b += 32) crow[b] = b < k ? uint16_t(cnt[b]) : 0;
  }
  if (a.o.mean) {
    const double f = neumaier_mean(tot, n, mean_buf, lane);
    if (lane == 0) a.o.mean[row] = __ddiv_rn(f, small_int_to_double(n));
  }
  if (lane == 0) {
    if (a.o.worst) a.o.worst[row] = hi;
    if (a.o.lo) a.o.lo[row] = lo;
    if (a.o.width) a.o.width[row] = width;
    if (a.o.nbins) a.o.nbins[row] = k;
    if (a.o.nsamp) a.o.nsamp[row] = n;
    if (a.o.capped) a.o.capped[job] = capped;
    if (a.o.flags)
      a.o.flags[job] = (conditioned ? 1 : 0) | (has_ov ? 2 : 0) | (replayed ? 4 : 0) |
                       (redrawn ? 8 : 0);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// per-warp footprints
// ---------------------------------------------------------------------------
template <typename Idx>
__host__ __device__ constexpr size_t smem_walk_bytes() { return 8 + 2 * sizeof(Idx) + 1; }
template <typename Idx>
__host__ __device__ constexpr size_t gmem_walk_bytes() {   // own-input arrays
  return 8 + 2 + sizeof(Idx);
}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename Idx>
__device__ WarpState<Idx> carve(unsigned char* walk_base, unsigned char* gbase, int nw,
                                uint32_t* cnt, int max_pairs) {
  WarpState<Idx> ws;
  ws.tot = reinterpret_cast<double*>(walk_base);
  ws.act = reinterpret_cast<Idx*>(ws.tot + nw);
  ws.mem = ws.act + nw;
  ws.cur = reinterpret_cast<int8_t*>(ws.mem + nw);
  ws.cnt = cnt;
  ws.tmp = reinterpret_cast<double*>(gbase);
  ws.bkt = reinterpret_cast<uint16_t*>(ws.tmp + nw);
  ws.osrt = reinterpret_cast<Idx*>(ws.bkt + nw);
  ws.kin = reinterpret_cast<double*>(gbase + align16(size_t(nw) * gmem_walk_bytes<Idx>()));
  ws.kout = ws.kin + max_pairs;
  return ws;
}

__device__ __forceinline__ void job_obs(const EngineArgs& a, int64_t job, int& obs_up,
                                        double (&obs)[3]) {
  obs_up = a.j.obs_unit ? a.j.obs_unit[job] : -1;
  obs[0] = obs[1] = obs[2] = 0.0;
  if (obs_up >= 0) {
    obs[0] = a.j.obs_val[3 * job];
    obs[1] = a.j.obs_val[3 * job + 1];
    obs[2] = a.j.obs_val[3 * job + 2];
  }
}

template <typename Idx>
__global__ void __launch_bounds__(kWarps * 32, 5) mc_engine_kernel(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = a.n;
  const bool in_smem = n <= kSmemWalks;
  const int nw = in_smem ? kSmemWalks : ((n + 15) & ~15);
  const size_t cnt_bytes = align16(size_t(a.counters) * 4);
  const size_t per_warp_smem =
      cnt_bytes + (in_smem ? size_t(kSmemWalks) * smem_walk_bytes<Idx>() : 0);
  unsigned char* sb = smem + per_warp_smem * wib;
  const int64_t gwarp = int64_t(blockIdx.x) * kWarps + wib;
  unsigned char* gs =
      reinterpret_cast<unsigned char*>(a.scratch) + size_t(gwarp) * a.scratch_per_warp;
  unsigned char* gown = gs + (in_smem ? 0 : align16(size_t(nw) * smem_walk_bytes<Idx>()));
  const WarpState<Idx> ws = carve<Idx>(in_smem ? sb + cnt_bytes : gs, gown, nw,
                                       reinterpret_cast<uint32_t*>(sb), a.max_pairs);
  const unsigned lt = lanemask_lt();
  const int64_t stride = int64_t(gridDim.x) * kWarps;
  for (int64_t job = gwarp; job < a.n_jobs; job += stride) {
    const int gbase = a.b.graph_base[a.j.graph[job]];
    const int u0 = a.j.unit[job];
    Stream g;
    pcg_seed(a.j.seed[job], g.s, g.inc);
    g.pend = false;
    g.pv = 0;
    Pools ovp{nullptr, 0, nullptr, 0};
    bool conditioned = false;
    int obs_up;
    double obs[3];
    job_obs(a, job, obs_up, obs);
    const bool has_ov =
        condition(a, gbase, u0, obs_up, obs, ws.kin, ws.kout, ovp, conditioned, lane);
    for (int w = lane; w < n; w += 32) {
      ws.cur[w] = int8_t(u0);
      ws.tot[w] = 0.0;
      ws.act[w] = Idx(w);
    }
    __syncwarp();
    uint32_t na = uint32_t(n);
    bool ok = true;
    for (int step = 0; step < a.cap && ok; ++step) {
      // compact the still-active walks (order kept) and collect occupied units
      uint64_t occ = 0;
      uint32_t nn = 0;
      for (uint32_t base = 0; base < na; base += 32) {
        const uint32_t idx = base + lane;
        Idx w = 0;
        int c = -1;
        if (idx < na) {
          w = ws.act[idx];
          c = ws.cur[w];
        }
        const unsigned bal = __ballot_sync(kFull, c >= 0);
        if (c >= 0) {
          ws.act[nn + __popc(bal & lt)] = w;
          occ |= 1ull << c;
        }
        nn += __popc(bal);
      }
      na = nn;
      occ = warp_or(occ);
      __syncwarp();
      if (!occ) break;
      while (occ && ok) {
        const int u = mask_ffs(occ) - 1;
        occ &= occ - 1;
        ok = visit_unit<Idx>(a, gbase, u, ovp, has_ov, u0, ws, na, g, lane);
      }
    }
    if (!ok) {                     // Lemire rejection: leave it to mc_serial_kernel
      if (lane == 0) a.serial_list[atomicAdd(a.serial_count, 1)] = int32_t(job);
      __syncwarp();
      continue;
    }
    write_result(a, job, ws.tot, ws.cur, ws.cnt, conditioned, has_ov, false, lane);
  }
}

// ---------------------------------------------------------------------------
// Sequential reference walk for the apps the fast kernel gave up on (lane 0
// computes, the warp helps with conditioning and the epilogue).  Walk state
// lives in global scratch; numpy's generator is stepped one word at a time.
// ---------------------------------------------------------------------------
__host__ __device__ inline size_t serial_bytes(int nw) { return align16(size_t(nw) * 19); }

__global__ void __launch_bounds__(32) mc_serial_kernel(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int n = a.n;
  const int nw = (n + 15) & ~15;
  unsigned char* gs =
      reinterpret_cast<unsigned char*>(a.scratch) + size_t(blockIdx.x) * a.scratch_per_warp;
  double* tot = reinterpret_cast<double*>(gs);
  double* tmp = tot + nw;
  uint16_t* bkt = reinterpret_cast<uint16_t*>(tmp + nw);
  int8_t* cur = reinterpret_cast<int8_t*>(bkt + nw);
  double* kin = reinterpret_cast<double*>(gs + serial_bytes(nw));
  double* kout = kin + a.max_pairs;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
  const int total = *a.serial_count;
  for (int li = blockIdx.x; li < total; li += gridDim.x) {
    const int64_t job = a.serial_list[li];
    if (job < 0) continue;                       // finished by the careful walk kernel
    const int gbase = a.b.graph_base[a.j.graph[job]];
    const int u0 = a.j.unit[job];
    Pools ovp{nullptr, 0, nullptr, 0};
    bool conditioned = false;
    int obs_up;
    double obs[3];
    job_obs(a, job, obs_up, obs);
    const bool has_ov = condition(a, gbase, u0, obs_up, obs, kin, kout, ovp, conditioned, lane);
    if (lane == 0) {
      SeqGen sg;
      pcg_seed(a.j.seed[job], sg.s, sg.inc);
      sg.pend = false;
      sg.pv = 0;
      for (int w = 0; w < n; ++w) { cur[w] = int8_t(u0); tot[w] = 0.0; }
      const double pre = a.b.prefill_rate, dec = a.b.decode_rate;
      for (int step = 0; step < a.cap; ++step) {
        uint64_t occ = 0;
        for (int w = 0; w < n; ++w)
          if (cur[w] >= 0) occ |= 1ull << cur[w];
        if (!occ) break;
        while (occ) {
          const int u = mask_ffs(occ) - 1;
          occ &= occ - 1;
          const UnitDesc d = reinterpret_cast<const UnitDesc*>(a.b.units)[gbase + u];
          const bool ov = has_ov && u == u0;
          const Pools pl = pools_for(a, d, ov, ovp);
          const bool llm = d.flags & F_LLM;
          const bool own = llm && (d.flags & F_OWN) && !ov;
          for (int w = 0; w < n; ++w)
            if (cur[w] == u) tmp[w] = pl.A[sg.bounded(uint32_t(pl.pa))];
          if (llm && !own) {
            for (int w = 0; w < n; ++w)
              if (cur[w] == u)
                tmp[w] = dadd(__ddiv_rn(tmp[w], pre),
                              __ddiv_rn(pl.B[sg.bounded(uint32_t(pl.pb))], dec));
          } else if (own) {
            const int K = d.ib_k;
            for (int w = 0; w < n; ++w)
              if (cur[w] == u) bkt[w] = uint16_t(bucket_of(tmp[w], d.ib_lo, d.ib_hi, K));
            for (int bb = 0; bb < K; ++bb) {
              const int pln = a.b.pool_len[d.pool_off + bb];
              const double* pool = pln > 0 ? a.b.vals + a.b.pool_off[d.pool_off + bb] : pl.B;
              const uint32_t P = uint32_t(pln > 0 ? pln : pl.pb);
              for (int w = 0; w < n; ++w)
                if (cur[w] == u && bkt[w] == bb)
                  tmp[w] = dadd(__ddiv_rn(tmp[w], pre), __ddiv_rn(pool[sg.bounded(P)], dec));
            }
          }
          for (int w = 0; w < n; ++w) {
            if (cur[w] != u) continue;
            const double uu = u53_double(sg.next64());
            tot[w] = dadd(tot[w], tmp[w]);
            cur[w] = int8_t(next_unit(a, d, uu));
          }
        }
      }
    }
    __syncwarp();
    write_result(a, job, tot, cur, cnt, conditioned, has_ov, true, lane);
  }
}

// ===========================================================================
// mc_walk_kernel: the demand engine for n <= kSmemWalks walks per application
// (larger n: mc_engine_kernel above).
//
// Walk membership is one bitset per unit in shared memory (bit w set = walk w
// sits on the unit).  A unit visit extracts its members in ascending walk
// order (list position = rank = draw index inside the reference's
// choice()/random() calls), clears the bitset, draws, and moves every member
// by setting its bit in the successor's bitset -- a walk entering a later
// unit of the same step is visited again in that step, exactly as the
// reference's `cur == ui` test at visit time does (estimator.py:343-353).
//
// The visit's stream segment is wb words of 32-bit bounded halves (A draws
// for ranks 0..mA-1, then B draws), then m words of random(m).  For duration
// units (the common case) lane l owns a contiguous run of bounded words: word
// j holds the draws of ranks 2j+pin and 2j+pin+1, whose uniforms are words
// wb+2j+pin and wb+2j+pin+1, so a lane walks two LCG cursors forward in
// lock-step with its neighbours (one jump each per visit, then single
// steps) and finishes its members in registers.  Uniform -> successor uses
// integer thresholds ceil(cum * 2^53) against word >> 11, which is exact.
// LLM units use per-member cursors over the A/B/U groups; own-input units
// (draw order depends on the drawn inputs) add a counting sort by bucket.
// ===========================================================================
constexpr int kWalkWords = kSmemWalks / 32;

struct WalkState {
  double* tot;       // [kSmemWalks] accumulated remaining demand per walk
  uint16_t* mem;     // [kSmemWalks] members of the visited unit, ascending
  uint32_t* bits;    // [kWalkUnits][kWalkWords] walks per unit
  uint32_t* cnt;     // [counters] histogram / own-input bucket counters
  uint16_t* ia;      // [kSmemWalks] staged A-draw index per rank (over cnt)
  uint16_t* ib;      // [kSmemWalks] staged B-draw index per rank
  void* uc;          // [max_units] the application's unit descriptors (UnitCacheOf)
  double* tmp;       // own-input path (global scratch)
  uint16_t* bkt;
  uint16_t* osrt;
  double* kin;       // [max_pairs] K3 kept inputs / outputs (global scratch)
  double* kout;
  double* kin_d;     // [max_pairs] the same divided by prefill / decode rate
  double* kout_d;
};

// pool values as the stage time uses them: LLM inputs / prefill_rate, LLM
// outputs / decode_rate (divided once, exactly as estimator.py:286 divides
// each draw), durations unchanged -- the same offsets in a.b.vals_div
__device__ __forceinline__ Pools pools_div(const EngineArgs& a, const UnitDesc& d, bool ov,
                                           const Pools& ovd) {
  Pools pl;
  if ((d.flags & F_LLM) && ov) {
    pl = ovd;
  } else {
    pl.A = a.b.vals_div + d.a_off;
    pl.pa = d.a_len;
    pl.B = a.b.vals_div + d.b_off;
    pl.pb = d.b_len;
  }
  return pl;
}

// shared memory per warp: [counters | LLM staging] [tot] [mem] [bitsets of
// max_units units]
// (banks without LLM units stage no B draws: the staging area is ia only)
// (+64 B: the uniform loop prefetches the draw index one stride ahead,
// ia[k + 32] / ib[k + 32] for k < m; past the last rank it reads this
// slack -- value discarded -- instead of the tot array other lanes write)
__host__ __device__ inline size_t walk_union_bytes(int counters, bool llm = true) {
  const size_t c = size_t(counters) * 4, s = size_t(kSmemWalks) * (llm ? 4 : 2) + 64;
  return align16(c > s ? c : s);
}
// (+ for LLM banks: the own-input visit's input bucket and sort order per
// member, 2 x 512 u16, after the unit cache)
__host__ __device__ inline size_t walk_smem_bytes(int counters, int units, bool llm = true) {
  return walk_union_bytes(counters, llm) + size_t(kSmemWalks) * 10 +
         size_t(units) * kWalkWords * 4 + size_t(units) * (llm ? 112 : 64) +
         (llm ? size_t(kSmemWalks) * 4 : 0);
}
// global scratch per warp: [own-input arrays] [K3 pairs]
__host__ __device__ inline size_t walk_gmem_bytes() {
  return align16(size_t(kSmemWalks) * gmem_walk_bytes<uint16_t>());
}

// the threshold form of searchsorted(cum, u, "right") for u = k * 2^-53,
// k = word >> 11: the successor is the first i with k < t_i (t_i =
// ceil(cum_i * 2^53) >= 1), i.e. word <= T_i with T_i = t_i * 2^11 - 1 (all
// ones for t_i >= 2^53) -- compared on the raw 64-bit word, no shift
__device__ __forceinline__ uint64_t word_threshold(uint64_t t) {
  return t >= (1ull << 53) ? ~0ull : (t << 11) - 1ull;
}

struct SuccTab {
  uint64_t t0, t1, t2;     // word thresholds T_i
  int n0, n1, n2, n3, ns;
  __device__ __forceinline__ void load(const EngineArgs& a, const UnitDesc& d) {
    const uint64_t* thr = a.b.succ_thr + d.succ_off;
    const int32_t* nxt = a.b.succ_nxt + d.succ_off;
    ns = d.succ_len;
    constexpr uint64_t always = ~0ull;              // absent slot: taken by every word
    t0 = ns > 0 ? word_threshold(__ldg(thr)) : always;
    t1 = ns > 1 ? word_threshold(__ldg(thr + 1)) : always;
    t2 = ns > 2 ? word_threshold(__ldg(thr + 2)) : always;
    n0 = __ldg(nxt);
    n1 = ns > 0 ? __ldg(nxt + 1) : -1;
    n2 = ns > 1 ? __ldg(nxt + 2) : -1;
    n3 = ns > 2 ? __ldg(nxt + 3) : -1;
  }
  // successor of the uniform carried by a raw 64-bit word (<= 3 successors)
  __device__ __forceinline__ int next3(uint64_t w) const {
    return w <= t0 ? n0 : w <= t1 ? n1 : w <= t2 ? n2 : n3;
  }
  // successor of the uniform carried by a raw 64-bit word
  __device__ __forceinline__ int next(const EngineArgs& a, const UnitDesc& d, uint64_t w) const {
    if (ns > 3) return next_unit(a, d, u53_double(w));
    return next3(w);
  }
};

// an application's unit, staged in shared memory once per application
struct __align__(16) UnitCache {
  UnitDesc d;
  uint64_t t0, t1, t2;
  int32_t ns;
  int8_t n[4];
  uint32_t thr_a, thr_b;   // Lemire rejection thresholds of the unit's A / B pools
};
static_assert(sizeof(UnitCache) == 112, "unit cache layout");

// the same for banks without LLM units: only what a duration visit reads
struct __align__(16) UnitCacheLean {
  uint64_t t0, t1, t2;
  const double* pa;        // the unit's rate-divided A pool (vals_div + a_off)
  int32_t a_len, succ_off;
  int16_t flags, ns;
  uint32_t thr_a;          // Lemire rejection threshold of the A pool
  int32_t n[4];            // successor units, one 16-byte load (no sign-extension per visit)
};
static_assert(sizeof(UnitCacheLean) == 64, "lean unit cache layout");

template <bool LLM>
struct UnitCacheOf { using type = UnitCache; };
template <>
struct UnitCacheOf<false> { using type = UnitCacheLean; };

__host__ __device__ constexpr size_t unit_cache_bytes(bool llm) {
  return llm ? sizeof(UnitCache) : sizeof(UnitCacheLean);
}

__device__ __forceinline__ UnitDesc desc_of(const UnitCache& c) { return c.d; }
__device__ __forceinline__ UnitDesc desc_of(const UnitCacheLean& c) {
  UnitDesc d{};
  d.flags = c.flags;
  d.a_len = c.a_len;
  d.succ_off = c.succ_off;
  d.succ_len = c.ns;
  return d;
}
// a visit's rate-divided pools: the lean cache holds the A pool's address
// (duration units: no B pool, no override); the full one goes through the
// descriptor and the K3 override
__device__ __forceinline__ Pools pools_of(const EngineArgs& a, const UnitCache& c,
                                          const UnitDesc& d, bool ov, const Pools& ovd) {
  return pools_div(a, d, ov, ovd);
}
__device__ __forceinline__ Pools pools_of(const EngineArgs&, const UnitCacheLean& c,
                                          const UnitDesc&, bool, const Pools&) {
  return Pools{c.pa, c.a_len, nullptr, 0};
}

__device__ __forceinline__ uint32_t thr_a_of(const UnitCache& c) { return c.thr_a; }
__device__ __forceinline__ uint32_t thr_a_of(const UnitCacheLean& c) { return c.thr_a; }
__device__ __forceinline__ uint32_t thr_b_of(const UnitCache& c) { return c.thr_b; }
__device__ __forceinline__ uint32_t thr_b_of(const UnitCacheLean&) { return 0u; }

__device__ __forceinline__ SuccTab succ_of(const UnitCache& c) {
  SuccTab s;
  s.t0 = c.t0;
  s.t1 = c.t1;
  s.t2 = c.t2;
  s.ns = c.ns;
  const char4 n = *reinterpret_cast<const char4*>(c.n);
  s.n0 = n.x;
  s.n1 = n.y;
  s.n2 = n.z;
  s.n3 = n.w;
  return s;
}
__device__ __forceinline__ SuccTab succ_of(const UnitCacheLean& c) {
  SuccTab s;
  s.t0 = c.t0;
  s.t1 = c.t1;
  s.t2 = c.t2;
  s.ns = c.ns;
  const int4 n = *reinterpret_cast<const int4*>(c.n);
  s.n0 = n.x;
  s.n1 = n.y;
  s.n2 = n.z;
  s.n3 = n.w;
  return s;
}

template <typename M>
__device__ __forceinline__ void arrive(const WalkState& ws, uint32_t w, int v, M& targets) {
  if (v >= 0) {
    atomicOr(ws.bits + v * kWalkWords + (w >> 5), 1u << (w & 31));
    targets |= M(1) << v;
  }
}

// members of unit u in ascending walk order -> ws.mem; clears the bitset
__device__ __forceinline__ uint32_t take_members(const WalkState& ws, int u, int lane) {
  uint32_t* bu = ws.bits + u * kWalkWords;
  // kSmemWalks = 512: one 16-bit slice per lane
  uint32_t x = (bu[lane >> 1] >> ((lane & 1) << 4)) & 0xffffu;
  const uint32_t c = __popc(x);
  const uint32_t incl = warp_incl_scan_u32(c);
  uint32_t o = incl - c;
  while (x) {
    const int b = __ffs(x) - 1;
    x &= x - 1;
    ws.mem[o++] = uint16_t(lane * 16 + b);
  }
  __syncwarp();
  if (lane < kWalkWords) bu[lane] = 0u;
  __syncwarp();
  return __shfl_sync(kFull, incl, 31);
}

// per-application stride constants: lane l starts one stride before word l
// of a visit's segment (state A'_l s + cl) and advances 32 words at a time
struct LaneConst {
  U128 cl;     // K_l * inc
  U128 c32;    // G_32 * inc
};

// Lane l decodes the words of the application's stream whose absolute
// position is l mod 32, whatever visit they belong to: its chain state `st`
// is the state of the last such word it decoded, so every visit simply
// continues the chain one 32-word stride at a time.  P = words consumed.
struct LaneStream {
  U128 st;
  uint32_t P;
};

__device__ __forceinline__ LaneConst lane_const(const uint64_t* jt, const U128& inc, int lane) {
  const ulonglong2* l2 = reinterpret_cast<const ulonglong2*>(jt) + 2 * 2048;
  const ulonglong2 k = __ldg(l2 + 2 * lane + 1), g32 = __ldg(l2 + 2 * 32 + 1);
  LaneConst c;
  c.cl = mul128(U128{k.x, k.y}, inc);
  c.c32 = mul128(U128{g32.x, g32.y}, inc);
  return c;
}

// a unit visit without own-input sampling: lane l decodes words l, l+32, ...
// of the segment [wb bounded words | m uniforms]; bounded halves stage the
// draw indices per rank, the uniform of rank k then adds the stage time and
// moves the walk
// numpy's Lemire rejection inside a visit's bounded draws: the rejected half
// is replaced by the next one, which shifts every later half of the visit.
// Lane 0 redraws the visit's C bounded values with the sequential generator,
// from the visit's first word P0 (state jumped from the application's seed),
// and returns the number of words they consumed plus numpy's buffered half.
// Out of line: it runs for ~1 visit in 10^6 and stays out of the hot code.
// Returns words | pend << 31 | buffered half << 32.
__device__ __noinline__ uint64_t redo_bounded(const EngineArgs& a, int job, uint32_t P0,
                                              bool pin, uint32_t pv, uint32_t pa, uint32_t pb,
                                              uint32_t mA, uint32_t C, uint16_t* ia,
                                              uint16_t* ib) {
  U128 st, inc;
  pcg_seed(a.j.seed[job], st, inc);
  if (P0) st = pcg_jump(a.b.jump, st, inc, P0);        // the next step yields word P0
  bool pend = pin;
  uint32_t hv = pv, words = 0;
  auto next32 = [&]() -> uint32_t {                    // numpy next_uint32
    if (pend) {
      pend = false;
      return hv;
    }
    st = pcg_step(st, inc);
    ++words;
    const uint64_t w = pcg_out(st);
    pend = true;
    hv = uint32_t(w >> 32);
    return uint32_t(w);
  };
  for (uint32_t j = 0; j < C; ++j) {                   // buffered_bounded_lemire_uint32
    const uint32_t P = j < mA ? pa : pb;
    uint64_t mm = uint64_t(next32()) * P;
    uint32_t left = uint32_t(mm);
    if (left < P) {
      const uint32_t thr = (0u - P) % P;
      while (left < thr) {
        mm = uint64_t(next32()) * P;
        left = uint32_t(mm);
      }
    }
    if (j < mA) ia[j] = uint16_t(mm >> 32);
    else ib[j - mA] = uint16_t(mm >> 32);
  }
  return uint64_t(words) | (pend ? (1ull << 31) : 0ull) | (uint64_t(hv) << 32);
}

// SPEC: per-successor-count specialised, unrolled uniform loops (the lean
// duration-only kernel); the multi-kind kernels take one generic loop, whose
// smaller code keeps them out of instruction-cache misses
template <bool LLM, typename M, bool SPEC, bool CAREFUL>
__device__ bool visit_strided(const EngineArgs& a, int job, const UnitDesc& d, const SuccTab& sc,
                              const Pools& pl, uint32_t thr_a, uint32_t thr_b,
                              const WalkState& ws, uint32_t m, Stream& g, LaneStream& ls,
                              const LaneConst& lc, M& targets, int lane) {
  constexpr bool llm = LLM;
  // pool bases kept opaque, so that a draw's address is one IMAD.WIDE of the
  // 32-bit index instead of a re-associated 64-bit offset chain
  const double* PA = pl.A;
  const double* PB = pl.B;
  asm("" : "+l"(PA));
  if (LLM) asm("" : "+l"(PB));
  const uint32_t mA = pl.pa > 1 ? m : 0u;
  const uint32_t C = mA + ((llm && pl.pb > 1) ? m : 0u);
  const uint32_t pin = g.pend ? 1u : 0u;
  uint32_t wb = C ? (C - pin + 1) >> 1 : 0u;
  U128& st = ls.st;                               // one stride before word q
  bool rej = false;
  // duration units: the smallest low product word of the visit's draws; a
  // rejection happened iff it is below the threshold (one VIMNMX per half)
  uint32_t min_left = 0xffffffffu;
  uint32_t pend_hi = 0;
  uint32_t q = (uint32_t(lane) - ls.P) & 31u;
#pragma unroll kUnrollB
  for (; q < wb; q += 32) {                       // bounded halves -> draw indices
    st = pcg_stride32(st, lc.c32);
    const uint64_t wd = pcg_out(st);
    const uint32_t R = 2u * q + pin;
    if (!LLM) {                                   // every low half is an A draw
      const uint64_t m0 = uint64_t(uint32_t(wd)) * uint32_t(pl.pa);
      const uint64_t m1 = uint64_t(uint32_t(wd >> 32)) * uint32_t(pl.pa);
      ws.ia[R] = uint16_t(m0 >> 32);
      // the high half of the visit's last word may be numpy's buffered half
      // rather than a draw: it is still stored (into the staging slack) and
      // still counted -- a false alarm costs a careful-pass redo, nothing else
      ws.ia[R + 1] = uint16_t(m1 >> 32);
      min_left = min(min_left, min(uint32_t(m0), uint32_t(m1)));
      pend_hi = uint32_t(wd >> 32);
    } else {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint32_t r = R + t, h = t ? uint32_t(wd >> 32) : uint32_t(wd);
        if (r < mA) ws.ia[r] = uint16_t(lemire_t(h, uint32_t(pl.pa), thr_a, rej));
        else if (r < C) ws.ib[r - mA] = uint16_t(lemire_t(h, uint32_t(pl.pb), thr_b, rej));
        else pend_hi = h;
      }
    }
  }
  if (pin && C && lane == 0) {                    // half 0 is numpy's buffered half
    if (mA) ws.ia[0] = uint16_t(lemire_t(g.pv, uint32_t(pl.pa), thr_a, rej));
    else ws.ib[0] = uint16_t(lemire_t(g.pv, uint32_t(pl.pb), thr_b, rej));
  }
  if (!LLM) rej |= min_left < thr_a;
  __syncwarp();
  bool redone = false;
  uint64_t rd = 0;
  if (__any_sync(kFull, rej)) {                   // a Lemire rejection shifted the halves
    if constexpr (!CAREFUL) return false;        // the careful kernel redoes this app
    if (lane == 0)
      rd = redo_bounded(a, job, ls.P, pin != 0, g.pv, uint32_t(pl.pa), uint32_t(pl.pb), mA, C,
                        ws.ia, ws.ib);
    __syncwarp();
    rd = __shfl_sync(kFull, rd, 0);
    const uint32_t w2 = uint32_t(rd) & 0x7fffffffu;
    for (; q < w2; q += 32) st = pcg_stride32(st, lc.c32);   // skip the extra words
    wb = w2;
    redone = true;
    g.redrawn = true;
  }
  const uint32_t W = wb + m;
  const bool hb = C > mA;
  // random(m): stage time + successor; the pool loads of the next word are
  // issued before the current word is finished
  // (reads past the last rank hit the staging area's slack and are clamped
  // into the pool)
  const uint32_t la = mA ? uint32_t(pl.pa - 1) : 0u, lb = hb ? uint32_t(pl.pb - 1) : 0u;
  uint32_t k = q - wb;
  double xa = __ldg(PA + min(uint32_t(ws.ia[k]), la)), xb = 0.0;
  if (LLM) xb = __ldg(PB + min(uint32_t(ws.ib[k]), lb));
  auto uniform = [&](auto few_succ) {             // one 32-word stride
    const double ca = xa, cb = xb;
    xa = __ldg(PA + min(uint32_t(ws.ia[k + 32]), la));
    if (LLM) xb = __ldg(PB + min(uint32_t(ws.ib[k + 32]), lb));
    st = pcg_stride32(st, lc.c32);
    const uint64_t wd = pcg_out(st);
    // successor decided by as many threshold compares as the unit has
    constexpr int NS = decltype(few_succ)::value;
    const int v = NS == 0 ? sc.n0
                : NS == 1 ? (wd <= sc.t0 ? sc.n0 : sc.n1)
                : NS == 2 ? (wd <= sc.t0 ? sc.n0 : wd <= sc.t1 ? sc.n1 : sc.n2)
                : NS == 3 ? sc.next3(wd) : sc.next(a, d, wd);
    const uint32_t w = ws.mem[k];
    const double t = LLM ? dadd(ca, cb) : ca;      // pools hold i/prefill, o/decode
    ws.tot[w] = dadd(ws.tot[w], t);
    arrive(ws, w, v, targets);
    k += 32;
  };
  if constexpr (SPEC) {        // one unrolled loop per successor count
    auto uniforms = [&](auto few_succ) {
#pragma unroll kUnrollU
      for (; q < W; q += 32) uniform(few_succ);
    };
    switch (sc.ns) {
      case 0: uniforms(std::integral_constant<int, 0>{}); break;
      case 1: uniforms(std::integral_constant<int, 1>{}); break;
      case 2: uniforms(std::integral_constant<int, 2>{}); break;
      case 3: uniforms(std::integral_constant<int, 3>{}); break;
      default: uniforms(std::integral_constant<int, 4>{}); break;
    }
  } else {                     // one generic loop: less code in the big variants
#pragma unroll 1
    for (; q < W; q += 32) uniform(std::integral_constant<int, 4>{});
  }
  const uint32_t pv = __shfl_sync(kFull, pend_hi, (ls.P + wb - 1) & 31u);
  ls.P += W;
  if (redone) {
    g.pend = (rd >> 31) & 1u;
    g.pv = uint32_t(rd >> 32);
  } else if (C) {
    g.pend = ((pin + C) & 1u) != 0;
    if (g.pend) g.pv = pv;
  }
  __syncwarp();
  return true;
}

// The own-input visit's bounded draws after a Lemire rejection: lane 0
// redraws them with the sequential generator from the visit's first word,
// in numpy's order (estimator.py:275-283): every input index, then per input
// bucket ascending the output indices of that bucket's members in walk order.
// Rewrites tmp (i / prefill + o / decode) and bkt; returns words | pend << 31
// | buffered half << 32.  Out of line, careful pass only.
__device__ __noinline__ uint64_t redo_own(const EngineArgs& a, int job, uint32_t P0, bool pin,
                                          uint32_t pv, const UnitDesc& d, const Pools& pl,
                                          const Pools& pd, uint32_t m, double* tmp,
                                          uint16_t* bkt) {
  U128 st, inc;
  pcg_seed(a.j.seed[job], st, inc);
  if (P0) st = pcg_jump(a.b.jump, st, inc, P0);
  bool pend = pin;
  uint32_t hv = pv, words = 0;
  auto next32 = [&]() -> uint32_t {
    if (pend) {
      pend = false;
      return hv;
    }
    st = pcg_step(st, inc);
    ++words;
    const uint64_t w = pcg_out(st);
    pend = true;
    hv = uint32_t(w >> 32);
    return uint32_t(w);
  };
  auto bounded = [&](uint32_t P) -> uint32_t {        // buffered_bounded_lemire_uint32
    if (P <= 1) return 0u;
    uint64_t mm = uint64_t(next32()) * P;
    uint32_t left = uint32_t(mm);
    if (left < P) {
      const uint32_t thr = (0u - P) % P;
      while (left < thr) {
        mm = uint64_t(next32()) * P;
        left = uint32_t(mm);
      }
    }
    return uint32_t(mm >> 32);
  };
  const int K = d.ib_k;
  const double blo = d.ib_lo, bhi = d.ib_hi;
  const double bw = __ddiv_rn(dsub(bhi, blo), small_int_to_double(K));
  auto bucket = [&](double v) -> int {
    if (bhi == blo || v <= blo) return 0;
    if (v >= bhi) return K - 1;
    const int i = __double2int_rz(__ddiv_rn(dsub(v, blo), bw));
    return i < K - 1 ? i : K - 1;
  };
  for (uint32_t k = 0; k < m; ++k) {                  // choice(inputs, m)
    const uint32_t ia = bounded(uint32_t(pl.pa));
    tmp[k] = pd.A[ia];
    bkt[k] = uint16_t(bucket(pl.A[ia]));
  }
  for (int bb = 0; bb < K; ++bb) {                     // per bucket: choice(pool_b, m_b)
    const int pln = a.b.pool_len[d.pool_off + bb];
    const double* pool = pln > 0 ? a.b.vals_div + a.b.pool_off[d.pool_off + bb] : pd.B;
    const uint32_t P = uint32_t(pln > 0 ? pln : pl.pb);
    for (uint32_t k = 0; k < m; ++k)
      if (bkt[k] == bb) tmp[k] = dadd(tmp[k], pool[bounded(P)]);
  }
  return uint64_t(words) | (pend ? (1ull << 31) : 0ull) | (uint64_t(hv) << 32);
}

// own-input LLM unit: outputs drawn per input bucket, buckets ascending,
// walks in order within a bucket (estimator.py:275-283).  The segment is
// [A halves | B halves in (bucket, rank) order | uniforms]; lanes decode it
// strided like visit_strided, in three phases: the A words (input draws,
// their buckets and bucket counts), a counting sort that maps each B half to
// its member, the B words, then the uniforms.  The half shared by the last A
// word and the first B draw, and numpy's buffered half, are placed by lane 0.
template <typename M, bool CAREFUL>
__device__ bool visit_own(const EngineArgs& a, int job, const UnitDesc& d, const SuccTab& sc,
                          const Pools& pl, const Pools& pd, const WalkState& ws, uint32_t m,
                          Stream& g, LaneStream& ls, const LaneConst& lc, M& targets,
                          int lane) {
  const unsigned lt = lanemask_lt();
  const int K = d.ib_k;
  uint32_t* cnt = ws.cnt;
  uint32_t* start = ws.cnt + a.max_unit_k;
  uint32_t* effo = ws.cnt + 2 * a.max_unit_k;
  uint16_t* effl = ws.osrt;                       // B position -> member rank
  const uint32_t mA = pl.pa > 1 ? m : 0u;
  const uint32_t pin = g.pend ? 1u : 0u;
  const uint32_t wA = mA ? (mA - pin + 1) >> 1 : 0u;
  // bucket_index of an input draw (distributions.py:107-118), bucket width hoisted
  const double blo = d.ib_lo, bhi = d.ib_hi;
  const double bw = __ddiv_rn(dsub(bhi, blo), small_int_to_double(K));
  auto bucket = [&](double v) -> int {
    if (bhi == blo || v <= blo) return 0;
    if (v >= bhi) return K - 1;
    const int i = __double2int_rz(__ddiv_rn(dsub(v, blo), bw));
    return i < K - 1 ? i : K - 1;
  };
  bool rej = false;
  auto a_draw = [&](uint32_t r, uint32_t h) {
    const uint32_t ia = lemire(h, uint32_t(pl.pa), rej);
    ws.tmp[r] = pd.A[ia];                         // i / prefill_rate
    const int bb = bucket(pl.A[ia]);              // the raw input picks the bucket
    ws.bkt[r] = uint16_t(bb);
    atomicAdd(&cnt[bb], 1u);
  };
  for (int b = lane; b < K; b += 32) cnt[b] = 0;
  __syncwarp();
  U128& st = ls.st;                               // one stride before word q
  uint32_t pend_hi = 0;
  uint32_t q = (uint32_t(lane) - ls.P) & 31u;
  for (; q < wA; q += 32) {                       // phase A: input draws
    st = pcg_stride32(st, lc.c32);
    const uint64_t wd = pcg_out(st);
    const uint32_t R = 2u * q + pin;
    a_draw(R, uint32_t(wd));
    if (R + 1 < mA) a_draw(R + 1, uint32_t(wd >> 32));
    else pend_hi = uint32_t(wd >> 32);            // half mA: first B draw or leftover
  }
  if (mA && pin && lane == 0) a_draw(0, g.pv);
  if (!mA) {                                      // single-value input pool
    const int bb = bucket(pl.A[0]);
    for (uint32_t k = lane; k < m; k += 32) {
      ws.tmp[k] = pd.A[0];
      ws.bkt[k] = uint16_t(bb);
    }
    if (lane == 0) cnt[bb] = m;
  }
  __syncwarp();
  // per input bucket: its output pool (own pool or the unit's B pool) and
  // size, staged once per visit (the draws below read them from shared memory)
  uint32_t* bsize = ws.cnt + 3 * a.max_unit_k;
  const double** bpool = reinterpret_cast<const double**>(ws.cnt + 4 * a.max_unit_k);
  // bucket layout: all members by bucket (start), drawing members (effo)
  const int perb = (K + 31) >> 5;
  uint32_t la = 0, le = 0;
  for (int t = 0; t < perb; ++t) {
    const int bb = lane * perb + t;
    if (bb < K) {
      const int pln = a.b.pool_len[d.pool_off + bb];
      const int P = pln > 0 ? pln : pl.pb;
      bsize[bb] = uint32_t(P);
      bpool[bb] = pln > 0 ? a.b.vals_div + a.b.pool_off[d.pool_off + bb] : pd.B;
      la += cnt[bb];
      le += P > 1 ? cnt[bb] : 0u;
    }
  }
  const uint32_t ia_incl = warp_incl_scan(la, lane), ie_incl = warp_incl_scan(le, lane);
  const uint32_t eff_total = __shfl_sync(kFull, ie_incl, 31);
  uint32_t ra = ia_incl - la, re = ie_incl - le;
  __syncwarp();
  for (int t = 0; t < perb; ++t) {
    const int bb = lane * perb + t;
    if (bb < K) {
      const uint32_t P = bsize[bb];
      const uint32_t c = cnt[bb];
      start[bb] = ra;
      effo[bb] = re;
      cnt[bb] = ra;
      ra += c;
      re += P > 1 ? c : 0u;
    }
  }
  __syncwarp();
  // stable counting sort by bucket: drawing members get their B position,
  // members of single-value pools take value 0 now
  for (uint32_t base = 0; base < m; base += 32) {
    const uint32_t k = base + lane;
    const bool valid = k < m;
    const int bb = valid ? int(ws.bkt[k]) : (0x10000 + lane);
    const unsigned peers = __match_any_sync(kFull, bb);
    uint32_t dest = 0;
    if (valid) dest = cnt[bb];
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == lane) cnt[bb] = dest + __popc(peers);
    __syncwarp();
    if (valid) {
      if (bsize[bb] > 1u) effl[effo[bb] + dest + __popc(peers & lt) - start[bb]] = uint16_t(k);
      else ws.tmp[k] = dadd(ws.tmp[k], bpool[bb][0]);
    }
  }
  __syncwarp();
  const uint32_t C = mA + eff_total;
  uint32_t wb = C ? (C - pin + 1) >> 1 : 0u;
  auto b_draw = [&](uint32_t j, uint32_t h) {
    const uint32_t k = effl[j];
    const int bb = ws.bkt[k];
    ws.tmp[k] = dadd(ws.tmp[k], bpool[bb][lemire(h, bsize[bb], rej)]);   // + o / decode_rate
  };
  const uint32_t sh = __shfl_sync(kFull, pend_hi, (ls.P + wA - 1) & 31u);
  for (; q < wb; q += 32) {                       // phase B: output draws
    st = pcg_stride32(st, lc.c32);
    const uint64_t wd = pcg_out(st);
    const uint32_t R = 2u * q + pin;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t r = R + t, h = t ? uint32_t(wd >> 32) : uint32_t(wd);
      if (r < C) b_draw(r - mA, h);
      else pend_hi = h;
    }
  }
  if (eff_total && lane == 0) {                   // B draw 0 on a half decoded earlier
    if (!mA && pin) b_draw(0, g.pv);
    else if (mA && ((mA - pin) & 1u)) b_draw(0, sh);
  }
  bool redone = false;
  uint64_t rd = 0;
  if (__any_sync(kFull, rej)) {                   // a Lemire rejection shifted the halves
    if constexpr (!CAREFUL) return false;        // the careful kernel redoes this app
    __syncwarp();
    if (lane == 0) rd = redo_own(a, job, ls.P, pin != 0, g.pv, d, pl, pd, m, ws.tmp, ws.bkt);
    __syncwarp();
    rd = __shfl_sync(kFull, rd, 0);
    const uint32_t w2 = uint32_t(rd) & 0x7fffffffu;
    for (; q < w2; q += 32) st = pcg_stride32(st, lc.c32);   // skip the extra words
    wb = w2;
    redone = true;
    g.redrawn = true;
  }
  __syncwarp();
  const uint32_t W = wb + m;
  for (; q < W; q += 32) {                        // random(m): successor + total
    st = pcg_stride32(st, lc.c32);
    const uint32_t k = q - wb;
    const int v = sc.ns <= 3 ? sc.next3(pcg_out(st)) : sc.next(a, d, pcg_out(st));
    const uint32_t w = ws.mem[k];
    ws.tot[w] = dadd(ws.tot[w], ws.tmp[k]);
    arrive(ws, w, v, targets);
  }
  const uint32_t pv = __shfl_sync(kFull, pend_hi, (ls.P + wb - 1) & 31u);
  ls.P += W;
  if (redone) {
    g.pend = (rd >> 31) & 1u;
    g.pv = uint32_t(rd >> 32);
  } else if (C) {
    g.pend = ((pin + C) & 1u) != 0;
    if (g.pend) g.pv = pv;
  }
  __syncwarp();
  return true;
}

#ifndef PDG_WALK_MINB
#define PDG_WALK_MINB 5      // resident CTAs per SM the register budget is cut for
#endif
#ifndef PDG_WALK_WARPS
#define PDG_WALK_WARPS 4     // applications (warps) per CTA
#endif
constexpr int kWalkWarps = PDG_WALK_WARPS;

#ifndef PDG_WALK_MINB_LEAN
#define PDG_WALK_MINB_LEAN 7 // the same for banks without LLM / own-input / K3 units
#endif

// FEAT: the unit kinds the bank holds (F_LLM, F_OWN, F_ANYMASK bits; the
// host reads them from pdg_graph_bank.features).  Paths for kinds a bank does
// not hold are compiled out -- their registers otherwise cost the plain
// duration walk a resident CTA per SM.  A job that needs a compiled-out path
// anyway (features understated by the caller) is handed to mc_serial_kernel,
// so FEAT only ever affects speed.
// M: unit-set mask (uint64_t: > 32 units).  CAREFUL: the second pass over
// the applications the first pass handed back (serial_list): a visit whose
// bounded draws hit a numpy Lemire rejection is redrawn in place with the
// sequential generator (redo_bounded) instead of abandoning the application;
// what it cannot finish (own-input visits, compiled-out paths) stays in the
// list for mc_serial_kernel.  Keeping the redo out of the first pass keeps its
// registers and code out of the hot kernel.
template <int FEAT, typename M = uint32_t, bool CAREFUL = false>
__global__ void __launch_bounds__(kWalkWarps * 32,
                                  FEAT == 0 ? PDG_WALK_MINB_LEAN : PDG_WALK_MINB)
mc_walk_kernel(EngineArgs a) {
  constexpr bool kLLM = FEAT & F_LLM, kOwn = FEAT & F_OWN, kCond = FEAT & F_ANYMASK;
  constexpr bool kSpec = FEAT == 0;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = a.n;
  unsigned char* sb = smem + walk_smem_bytes(a.counters, a.b.max_units, kLLM) * wib;
  const int64_t gwarp = int64_t(blockIdx.x) * kWalkWarps + wib;
  unsigned char* gs =
      reinterpret_cast<unsigned char*>(a.scratch) + size_t(gwarp) * a.scratch_per_warp;
  WalkState ws;
  ws.cnt = reinterpret_cast<uint32_t*>(sb);
  ws.ia = reinterpret_cast<uint16_t*>(sb);
  ws.ib = ws.ia + kSmemWalks;
  ws.tot = reinterpret_cast<double*>(sb + walk_union_bytes(a.counters, kLLM));
  ws.mem = reinterpret_cast<uint16_t*>(ws.tot + kSmemWalks);
  ws.bits = reinterpret_cast<uint32_t*>(ws.mem + kSmemWalks);
  using Cache = typename UnitCacheOf<kLLM>::type;
  Cache* const uc = reinterpret_cast<Cache*>(ws.bits + a.b.max_units * kWalkWords);
  ws.uc = uc;
  ws.tmp = reinterpret_cast<double*>(gs);
  if constexpr (kLLM) {                          // own-input staging in shared memory
    ws.bkt = reinterpret_cast<uint16_t*>(
        reinterpret_cast<unsigned char*>(uc) + size_t(a.b.max_units) * sizeof(Cache));
  } else {
    ws.bkt = reinterpret_cast<uint16_t*>(ws.tmp + kSmemWalks);
  }
  ws.osrt = ws.bkt + kSmemWalks;
  ws.kin = reinterpret_cast<double*>(gs + walk_gmem_bytes());
  ws.kout = ws.kin + a.max_pairs;
  ws.kin_d = ws.kout + a.max_pairs;
  ws.kout_d = ws.kin_d + a.max_pairs;
  for (;;) {
    int job = 0, li = 0;
    if constexpr (CAREFUL) {
      if (lane == 0) li = atomicAdd(a.redo_next, 1);
      li = __shfl_sync(kFull, li, 0);
      if (li >= *a.serial_count) break;
      job = a.serial_list[li];
    } else {
      if (lane == 0) {
        job = atomicAdd(a.job_next, 1);
        if (a.order && job < a.n_jobs) job = a.order[job];
      }
      job = __shfl_sync(kFull, job, 0);
      if (job >= a.n_jobs) break;
    }
    // hand the application on (first pass: to the careful pass; careful pass:
    // leave it in the list for mc_serial_kernel)
    auto hand_on = [&]() {
      if (!CAREFUL && lane == 0) a.serial_list[atomicAdd(a.serial_count, 1)] = int32_t(job);
      __syncwarp();
    };
    const int gi = a.j.graph[job];
    const int gbase = a.b.graph_base[gi];
    const int gn = a.b.graph_n[gi];
    const int u0 = a.j.unit[job];
    Stream g;
    pcg_seed(a.j.seed[job], g.s, g.inc);
    g.pend = false;
    g.pv = 0;
    g.redrawn = false;
    Pools ovp{nullptr, 0, nullptr, 0};
    bool conditioned = false;
    int obs_up;
    double obs[3];
    job_obs(a, job, obs_up, obs);
    if (!kCond && obs_up >= 0 &&
        (reinterpret_cast<const UnitDesc*>(a.b.units)[gbase + u0].flags & F_ANYMASK)) {
      hand_on();
      continue;                                  // K3 compiled out: serial path
    }
    const bool has_ov = kCond &&
        condition(a, gbase, u0, obs_up, obs, ws.kin, ws.kout, ovp, conditioned, lane);
    Pools ovd = ovp;                             // the override pools, divided
    if (kCond && has_ov) {
      const double pre = a.b.prefill_rate, dec = a.b.decode_rate;
      auto divide = [&](const double* p, int len, const double* buf, double* dbuf,
                        double rate) -> const double* {
        if (p >= buf && p < buf + a.max_pairs) {   // kept records: divide them
          const int off = int(p - buf);
          for (int i = lane; i < len; i += 32) dbuf[off + i] = __ddiv_rn(buf[off + i], rate);
          return dbuf + off;
        }
        return a.b.vals_div + (p - a.b.vals);     // prior pool
      };
      ovd.A = divide(ovp.A, ovp.pa, ws.kin, ws.kin_d, pre);
      ovd.B = divide(ovp.B, ovp.pb, ws.kout, ws.kout_d, dec);
      __syncwarp();
    }
    const LaneConst lc = lane_const(a.b.jump, g.inc, lane);
    LaneStream ls;                               // lane l: words l, l+32, ... of the stream
    {
      const ulonglong2 ap =
          __ldg(reinterpret_cast<const ulonglong2*>(a.b.jump) + 2 * (2048 + lane));
      ls.st = add128(mul128(g.s, U128{ap.x, ap.y}), lc.cl);   // one stride before word lane
      ls.P = 0;
    }
    for (int ul = lane; ul < gn; ul += 32) {     // stage the unit descriptors
      Cache c;
      const UnitDesc d = reinterpret_cast<const UnitDesc*>(a.b.units)[gbase + ul];
      if constexpr (kLLM) {
        c.d = d;
      } else {
        c.pa = a.b.vals_div + d.a_off;
        c.a_len = d.a_len;
        c.succ_off = d.succ_off;
        c.flags = int16_t(d.flags);
      }
      const SuccTab t = [&] { SuccTab x; x.load(a, d); return x; }();
      c.t0 = t.t0;
      c.t1 = t.t1;
      c.t2 = t.t2;
      c.ns = t.ns;
      c.thr_a = lemire_thr_of(uint32_t(d.a_len));
      if constexpr (kLLM) c.thr_b = lemire_thr_of(uint32_t(d.b_len));
      c.n[0] = t.n0;
      c.n[1] = t.n1;
      c.n[2] = t.n2;
      c.n[3] = t.n3;
      uc[ul] = c;
    }
    for (int i = lane; i < gn * kWalkWords; i += 32) {
      const int u = i / kWalkWords, wi = i - u * kWalkWords;
      const int rem = n - 32 * wi;
      ws.bits[i] = (u != u0 || rem <= 0) ? 0u : (rem >= 32 ? 0xffffffffu : (1u << rem) - 1u);
    }
    for (int w = lane; w < n; w += 32) ws.tot[w] = 0.0;
    __syncwarp();
    M pending = M(1) << u0;                      // units holding walks
    bool ok = true;
    for (int step = 0; step < a.cap && ok && pending; ++step) {
      M occ = pending;                           // frozen occupied set of the step
      while (occ && ok) {
        const int u = mask_ffs(occ) - 1;
        occ &= occ - 1;
        const uint32_t m = take_members(ws, u, lane);
        pending &= ~(M(1) << u);
        const UnitDesc d = desc_of(uc[u]);
        const bool ov = has_ov && u == u0;
        const Pools pd = pools_of(a, uc[u], d, ov, ovd);
        M targets = 0;
        if (!(d.flags & F_LLM))
          ok = visit_strided<false, M, kSpec, CAREFUL>(a, job, d, succ_of(uc[u]), pd, thr_a_of(uc[u]), 0u,
                                              ws, m, g, ls, lc, targets, lane);
        else if (!kLLM)
          ok = false;                            // compiled out: serial path
        else if ((d.flags & F_OWN) && !ov)
          ok = kOwn && visit_own<M, CAREFUL>(a, job, d, succ_of(uc[u]), pools_for(a, d, ov, ovp), pd, ws, m,
                                 g, ls, lc, targets, lane);
        else {                                   // override pools: thresholds here
          const uint32_t ta = ov ? lemire_thr_of(uint32_t(pd.pa)) : thr_a_of(uc[u]);
          const uint32_t tb = ov ? lemire_thr_of(uint32_t(pd.pb)) : thr_b_of(uc[u]);
          ok = visit_strided<true, M, kSpec, CAREFUL>(a, job, d, succ_of(uc[u]), pd, ta, tb, ws, m, g, ls,
                                             lc, targets, lane);
        }
        pending |= warp_or(targets);
      }
    }
    if (!ok) {                     // Lemire rejection: careful pass / mc_serial_kernel
      hand_on();
      continue;
    }
    if (CAREFUL && lane == 0) a.serial_list[li] = -1;   // done here
    int capped = 0;
    for (int i = lane; i < gn * kWalkWords; i += 32) capped += __popc(ws.bits[i]);
    capped = warp_sum(capped);
    write_result(a, job, ws.tot, nullptr, ws.cnt, conditioned, has_ov, false, lane, capped,
                 ws.tmp, g.redrawn);
  }
}

// Longest-first job order (pdg_graph_bank.unit_class): a job's class is its
// start unit's expected remaining walk length; the dynamic job counter then
// hands out the long applications first, so the last applications to start
// are short ones and the warps finish together (~3 % of a 100k-app launch).
// Order within a class is arbitrary: every application's result depends only
// on its own stream.  Two passes: class counts, then warp-aggregated slots.
__device__ __forceinline__ int job_class(const EngineArgs& a, int64_t i) {
  return a.b.unit_class[a.b.graph_base[a.j.graph[i]] + a.j.unit[i]] & 15;
}

__global__ void job_class_count_kernel(EngineArgs a, int32_t* counts) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n_jobs;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int c = job_class(a, i);
    const unsigned same = __match_any_sync(__activemask(), c);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(counts + c, __popc(same));
  }
}

__global__ void job_order_kernel(EngineArgs a, const int32_t* counts, int32_t* cursor,
                                 int32_t* order) {
  __shared__ int32_t base[16];
  if (threadIdx.x < 16) {                        // classes 15, 14, ... first
    int32_t s = 0;
    for (int c = 15; c > int(threadIdx.x); --c) s += counts[c];
    base[threadIdx.x] = s;
  }
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n_jobs;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int c = job_class(a, i);
    const unsigned same = __match_any_sync(__activemask(), c);
    const int leader = __ffs(same) - 1;
    int32_t slot = 0;
    if (int(lane) == leader) slot = atomicAdd(cursor + c, __popc(same));
    slot = __shfl_sync(same, slot, leader) + __popc(same & ((1u << lane) - 1u));
    order[base[c] + slot] = int32_t(i);
  }
}

}  // namespace pdg

using namespace pdg;

#ifndef PDG_ORDER_MAX_APPS_PER_SM
#define PDG_ORDER_MAX_APPS_PER_SM 2048
#endif

static bool small_idx(int n) { return n <= 65535; }

static size_t walk_scratch(int n) {
  const size_t nw = size_t((n + 15) & ~15);
  const bool si = small_idx(n);
  const size_t smem_part = n <= kSmemWalks ? 0
      : align16(nw * (si ? smem_walk_bytes<uint16_t>() : smem_walk_bytes<uint32_t>()));
  const size_t own = align16(nw * (si ? gmem_walk_bytes<uint16_t>() : gmem_walk_bytes<uint32_t>()));
  const size_t fast = smem_part + own;
  const size_t serial = serial_bytes(int(nw));
  const size_t walk = n <= kSmemWalks ? walk_gmem_bytes() : 0;
  const size_t r = fast > serial ? fast : serial;
  return r > walk ? r : walk;
}

static size_t scratch_per_warp(int n, int max_pairs) {
  // kept-pool buffers kin/kout, plus their rate-divided copies (walk kernel)
  return (walk_scratch(n) + align16(size_t(max_pairs) * 32) + 64 + 255) & ~size_t(255);
}

// scratch = per-warp regions + 256 B (serial counter) + one int per job
extern "C" size_t pdg_mc_scratch_bytes(int32_t n_samples, int32_t max_pairs, int32_t grid_warps) {
  return scratch_per_warp(n_samples, max_pairs) * size_t(grid_warps) + 256;
}

extern "C" int pdg_mc_grid_warps(void) { return sm_count() * 8 * kWarps; }

extern "C" int pdg_mc_remaining_demand(const pdg_graph_bank* bank, const pdg_mc_jobs* jobs,
                                       int64_t n_jobs, int32_t n_samples, int32_t visit_cap,
                                       int32_t bucket_count, int32_t max_unit_k,
                                       int32_t max_pairs, const pdg_mc_out* out,
                                       void* scratch, size_t scratch_bytes, void* stream) {
  if (!bank || !jobs || !out || n_jobs < 0 || n_jobs > INT32_MAX || n_samples < 1 ||
      n_samples > (1 << 19) || visit_cap < 0 || bucket_count < 1 || bucket_count > 1024 ||
      max_unit_k < 0 || max_unit_k > 1024 || max_pairs < 0) {
    set_error("pdg_mc_remaining_demand: invalid arguments");
    return PDG_EINVAL;
  }
  if (bank->max_units > 64) {
    set_error("pdg_mc_remaining_demand: graphs of more than 64 units are not supported");
    return PDG_EUNSUPPORTED;
  }
  if (n_samples <= kSmemWalks && !bank->vals_div) {
    set_error("pdg_mc_remaining_demand: graph bank without vals_div");
    return PDG_EINVAL;
  }
  if (out->counts && out->stride < bucket_count) {
    set_error("pdg_mc_remaining_demand: histogram stride < bucket_count");
    return PDG_EINVAL;
  }
  if (n_jobs == 0) return PDG_OK;
  const int grid_warps = pdg_mc_grid_warps();
  const size_t need = pdg_mc_scratch_bytes(n_samples, max_pairs, grid_warps) +
                      size_t(n_jobs) * sizeof(int32_t);
  if (scratch_bytes < need || !scratch) {
    set_error("pdg_mc_remaining_demand: scratch %zu < %zu bytes", scratch_bytes, need);
    return PDG_EINVAL;
  }
  EngineArgs a;
  a.b = *bank;
  a.j = *jobs;
  a.o = *out;
  a.n_jobs = n_jobs;
  a.n = n_samples;
  a.cap = visit_cap;
  a.k_out = bucket_count;
  a.max_unit_k = max_unit_k;
  // counters per warp: the output histogram, or the own-input visit's
  // per-bucket count / start / offset / pool size (u32) and pool address (u64)
  const int c = bucket_count > 6 * max_unit_k ? bucket_count : 6 * max_unit_k;
  a.counters = (c + 3) & ~3;
  a.max_pairs = max_pairs;
  a.scratch = static_cast<char*>(scratch);
  a.scratch_per_warp = scratch_per_warp(n_samples, max_pairs);
  char* tail = static_cast<char*>(scratch) + a.scratch_per_warp * size_t(grid_warps);
  a.serial_count = reinterpret_cast<int32_t*>(tail);
  a.job_next = reinterpret_cast<int32_t*>(tail + 4);
  a.redo_next = reinterpret_cast<int32_t*>(tail + 8);
  a.serial_list = reinterpret_cast<int32_t*>(tail + 256);
  a.order = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  const bool sm = n_samples <= kSmemWalks;
  // longest-first order: a hint, used when the bank has classes and the
  // scratch has room for it
  // (above ~2k applications per SM the tail is amortised and the queue
  // order's graph locality is worth more: 1M apps measured 20.61 vs 20.67 ms)
  const bool ordered = sm && bank->unit_class && n_jobs > 1 &&
                       n_jobs <= int64_t(sm_count()) * PDG_ORDER_MAX_APPS_PER_SM &&
                       scratch_bytes >= need + size_t(n_jobs) * sizeof(int32_t);
  int32_t* cls_counts = reinterpret_cast<int32_t*>(tail + 64);
  int32_t* cls_cursor = reinterpret_cast<int32_t*>(tail + 128);
  cudaError_t e = cudaMemsetAsync(a.serial_count, 0, ordered ? 192 : 3 * sizeof(int32_t), st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(serial_count)");
  if (ordered) {
    int32_t* ord = reinterpret_cast<int32_t*>(tail + 256 + size_t(n_jobs) * sizeof(int32_t));
    int64_t blocks = (n_jobs + 255) / 256;
    const int64_t capb = int64_t(sm_count()) * 8;
    if (blocks > capb) blocks = capb;
    job_class_count_kernel<<<unsigned(blocks), 256, 0, st>>>(a, cls_counts);
    if (int rc = launch_status("job_class_count_kernel")) return rc;
    job_order_kernel<<<unsigned(blocks), 256, 0, st>>>(a, cls_counts, cls_cursor, ord);
    if (int rc = launch_status("job_order_kernel")) return rc;
    a.order = ord;
  }
  const size_t cnt_bytes = align16(size_t(a.counters) * 4);
  // sequential completion of rejected apps (normally none: every block exits
  // after reading the counter)
  auto finish = [&]() -> int {
    int rc = launch_status("mc_engine_kernel");
    if (rc != PDG_OK) return rc;
    const unsigned sblocks = unsigned(grid_warps < n_jobs ? grid_warps : n_jobs);
    mc_serial_kernel<<<sblocks, 32, cnt_bytes, st>>>(a);
    return launch_status("mc_serial_kernel");
  };
  // persistent grid: exactly the resident CTAs (a second partial wave of
  // grid-stride CTAs would leave SMs idle at the tail)
  auto launch = [&](auto kern, int warps, size_t smem) -> int {
    int64_t blocks = (n_jobs + warps - 1) / warps;
    const int64_t capb = grid_warps / warps;
    if (blocks > capb) blocks = capb;
    int per_sm = 0;
    if (int r = launch_setup(reinterpret_cast<const void*>(kern), warps * 32, smem, &per_sm))
      return r;
    int64_t nb = int64_t(per_sm) * sm_count();
    if (nb > capb) nb = capb;
    if (nb > blocks) nb = blocks;
    kern<<<unsigned(nb), warps * 32, smem, st>>>(a);
    return PDG_OK;
  };
  if (sm) {
    const int mu = bank->max_units < 1 ? 1 : bank->max_units;
    // unit kinds present (pdg_graph_bank.features; VALID bit clear: assume all)
    int feat = (bank->features & PDG_BANK_FEATURES_VALID) ? (bank->features & 7) : 7;
    if (!jobs->obs_unit) feat &= ~F_ANYMASK;     // no observations: no K3
    const size_t smem = size_t(kWalkWarps) * walk_smem_bytes(a.counters, mu);
    const size_t smem_plain = size_t(kWalkWarps) * walk_smem_bytes(a.counters, mu, false);
    int r = PDG_OK;
    // the careful second pass over the handed-back applications: one CTA per
    // SM, warps fetch list entries dynamically and exit at once when the
    // first pass handed back nothing
    auto careful = [&](auto kern, size_t sm_bytes) -> int {
      int per_sm = 0;
      if (int rc = launch_setup(reinterpret_cast<const void*>(kern), kWalkWarps * 32, sm_bytes,
                                &per_sm))
        return rc;
      kern<<<unsigned(sm_count()), kWalkWarps * 32, sm_bytes, st>>>(a);
      return launch_status("mc_walk_kernel (careful pass)");
    };
    // the careful pass always runs the full variant: it handles every unit
    // kind and redraws every rejection, so nothing is left for the
    // sequential replay kernel on this path
    if (mu > 32) {                               // 64-bit unit sets, every unit kind
      r = launch(mc_walk_kernel<7, uint64_t>, kWalkWarps, smem);
      if (!r) r = careful(mc_walk_kernel<7, uint64_t, true>, smem);
      return r;
    }
    switch (feat) {
      case 0: r = launch(mc_walk_kernel<0>, kWalkWarps, smem_plain); break;
      case 1: r = launch(mc_walk_kernel<1>, kWalkWarps, smem); break;
      case 4: r = launch(mc_walk_kernel<4>, kWalkWarps, smem_plain); break;
      case 5: r = launch(mc_walk_kernel<5>, kWalkWarps, smem); break;
      default: r = launch(mc_walk_kernel<7>, kWalkWarps, smem); break;
    }
    if (!r) r = careful(mc_walk_kernel<7, uint32_t, true>, smem);
    return r;
  } else if (small_idx(n_samples)) {
    if (int r = launch(mc_engine_kernel<uint16_t>, kWarps, size_t(kWarps) * cnt_bytes)) return r;
  } else {
    if (int r = launch(mc_engine_kernel<uint32_t>, kWarps, size_t(kWarps) * cnt_bytes)) return r;
  }
  return finish();
}
