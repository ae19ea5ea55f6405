// K2 + K3 + a4: the PDGraph demand engine for sm_100a.
//
// Replaces estimator.monte_carlo_remaining_demand (estimator.py:305-362) with
// its per-unit sampler (236-286), one-hop conditioning (155-233, 289-302) and
// ApplicationInstance.set_remaining's bucketing (sched.py:170-181,
// distributions.py:79-105).  Output samples are bit-identical to the
// reference for the same (graph, current unit, observations, n, seed): the
// kernel evaluates the reference's numpy PCG64 stream *by position*.
//
// Mapping: one warp per application; walk w lives on lane w % 32 (round
// w / 32).  The reference walk is vectorised per (step, unit): at each outer
// step the occupied-unit set is frozen, units are visited in ascending index
// order, and every walk sitting on the unit *at that moment* draws
//   choice(A, m) [, choice(B, m) | per-input-bucket choice(pool_b, m_b)],
//   then random(m)                                 (estimator.py:343-353)
// so each draw's position in the stream is (group base) + (rank of the walk
// among the unit's members), computed with ballots; each lane jumps the
// PCG64 state straight to its position (pcg64.cuh).  numpy's Lemire rejection
// (probability < P/2^32 per draw) is detected by a warp vote and the affected
// unit visit is then replayed sequentially by lane 0 with the exact
// sequential generator.
#include "common.cuh"
#include "pcg64.cuh"

namespace pdg {

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
static_assert(sizeof(CondDesc) == 88 || sizeof(CondDesc) == 96, "cond descriptor layout");

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
  int max_pairs;     // K3 scratch per warp
  char* scratch;     // global scratch base
  size_t scratch_per_warp;
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

struct Pools {            // the draw pools of one unit visit
  const double* A;
  int pa;
  const double* B;
  int pb;
};

// Per-warp stream state (warp-uniform).
struct Stream {
  U128 s, inc;
  bool pend;
  uint32_t pv;
};

__device__ __forceinline__ uint32_t half_at(const uint64_t* jt, const Stream& g, uint32_t R) {
  if (g.pend) {
    if (R == 0) return g.pv;
    R -= 1;
  }
  const uint64_t w = pcg_out(pcg_jump(jt, g.s, g.inc, (R >> 1) + 1));
  return (R & 1) ? uint32_t(w >> 32) : uint32_t(w);
}

// C halves (positions 0..C-1) of the u32 stream were consumed.
__device__ __forceinline__ void close_u32(const uint64_t* jt, Stream& g, uint32_t C) {
  if (C == 0) return;
  const uint32_t F = C - (g.pend ? 1u : 0u);
  if (F & 1u) {
    const uint64_t w = pcg_out(pcg_jump(jt, g.s, g.inc, ((F - 1) >> 1) + 1));
    g.pv = uint32_t(w >> 32);
    g.pend = true;
  } else {
    g.pend = false;
  }
  g.s = pcg_jump(jt, g.s, g.inc, (F + 1) >> 1);
}

struct WarpState {
  double* tot;      // [n] accumulated remaining demand per walk
  double* tmp;      // [n] this visit's stage time per walk
  int8_t* cur;      // [n] current unit per walk (-1 = terminated)
  uint16_t* bkt;    // [n] input bucket per walk (own-input sampling)
  uint32_t* cnt;    // [counters]
  double* kin;      // [max_pairs] K3 kept inputs
  double* kout;     // [max_pairs] K3 kept outputs
};

// ---------------------------------------------------------------------------
// Sequential replay of one unit visit (lane 0) -- exact on Lemire rejections.
// ---------------------------------------------------------------------------
__device__ void serial_visit(const EngineArgs& a, const UnitDesc& d, const Pools& pl,
                             bool own, int u, const WarpState& ws, Stream& g) {
  SeqGen sg{g.s, g.inc, g.pend, g.pv};
  const int n = a.n;
  const double* V = a.b.vals;
  const bool llm = d.flags & F_LLM;
  for (int w = 0; w < n; ++w)
    if (ws.cur[w] == u) ws.tmp[w] = pl.A[sg.bounded(uint32_t(pl.pa))];
  if (llm) {
    if (!own) {
      for (int w = 0; w < n; ++w)
        if (ws.cur[w] == u)
          ws.tmp[w] = dadd(__ddiv_rn(ws.tmp[w], a.b.prefill_rate),
                           __ddiv_rn(pl.B[sg.bounded(uint32_t(pl.pb))], a.b.decode_rate));
    } else {
      const int k = d.ib_k;
      for (int w = 0; w < n; ++w)
        if (ws.cur[w] == u) ws.bkt[w] = uint16_t(bucket_of(ws.tmp[w], d.ib_lo, d.ib_hi, k));
      for (int bb = 0; bb < k; ++bb) {
        const int pln = a.b.pool_len[d.pool_off + bb];
        const double* pool = pln > 0 ? V + a.b.pool_off[d.pool_off + bb] : pl.B;
        const uint32_t P = uint32_t(pln > 0 ? pln : pl.pb);
        for (int w = 0; w < n; ++w)
          if (ws.cur[w] == u && ws.bkt[w] == bb)
            ws.tmp[w] = dadd(__ddiv_rn(ws.tmp[w], a.b.prefill_rate),
                             __ddiv_rn(pool[sg.bounded(P)], a.b.decode_rate));
      }
    }
  }
  g.s = sg.s;
  g.pend = sg.pend;
  g.pv = sg.pv;
}

// ---------------------------------------------------------------------------
// one (step, unit) visit of the vectorised walk
// ---------------------------------------------------------------------------
__device__ void visit_unit(const EngineArgs& a, int gbase, int u, const Pools& ovp,
                           bool has_ov, int cur_unit, const WarpState& ws, Stream& g,
                           int lane) {
  const uint64_t* jt = a.b.jump;
  const int n = a.n;
  const int W = (n + 31) >> 5;
  const unsigned lt = lanemask_lt();
  const UnitDesc d = reinterpret_cast<const UnitDesc*>(a.b.units)[gbase + u];
  const bool llm = d.flags & F_LLM;
  const bool ov = has_ov && u == cur_unit;
  Pools pl;
  if (llm && ov) {
    pl = ovp;
  } else {
    pl.A = a.b.vals + d.a_off;
    pl.pa = d.a_len;
    pl.B = a.b.vals + d.b_off;
    pl.pb = d.b_len;
  }
  const bool own = llm && (d.flags & F_OWN) && !ov;
  // members
  uint32_t m = 0;
  for (int i = 0; i < W; ++i) {
    const int w = i * 32 + lane;
    m += __popc(__ballot_sync(kFull, w < n && ws.cur[w] == u));
  }
  const uint32_t c1 = pl.pa > 1 ? m : 0u;
  bool rej = false;
  uint32_t C = 0;
  if (!own) {
    uint32_t R = 0;
    for (int i = 0; i < W; ++i) {
      const int w = i * 32 + lane;
      const bool mem = w < n && ws.cur[w] == u;
      const unsigned bal = __ballot_sync(kFull, mem);
      if (mem) {
        const uint32_t r = R + __popc(bal & lt);
        const uint32_t ia = pl.pa > 1 ? lemire(half_at(jt, g, r), uint32_t(pl.pa), rej) : 0u;
        double t = pl.A[ia];
        if (llm) {
          const uint32_t ib = pl.pb > 1 ? lemire(half_at(jt, g, c1 + r), uint32_t(pl.pb), rej) : 0u;
          t = dadd(__ddiv_rn(t, a.b.prefill_rate), __ddiv_rn(pl.B[ib], a.b.decode_rate));
        }
        ws.tmp[w] = t;
      }
      R += __popc(bal);
    }
    C = c1 + ((llm && pl.pb > 1) ? m : 0u);
  } else {
    // own-input sampling: outputs drawn per input bucket, buckets ascending,
    // walks in order within a bucket (estimator.py:275-283)
    const int k = d.ib_k;
    for (int b = lane; b < k; b += 32) ws.cnt[b] = 0;
    __syncwarp();
    uint32_t R = 0;
    for (int i = 0; i < W; ++i) {
      const int w = i * 32 + lane;
      const bool mem = w < n && ws.cur[w] == u;
      const unsigned bal = __ballot_sync(kFull, mem);
      if (mem) {
        const uint32_t r = R + __popc(bal & lt);
        const uint32_t ia = pl.pa > 1 ? lemire(half_at(jt, g, r), uint32_t(pl.pa), rej) : 0u;
        const double iv = pl.A[ia];
        ws.tmp[w] = iv;
        const int bb = bucket_of(iv, d.ib_lo, d.ib_hi, k);
        ws.bkt[w] = uint16_t(bb);
        atomicAdd(&ws.cnt[bb], 1u);
      }
      R += __popc(bal);
    }
    __syncwarp();
    // exclusive offsets over buckets that consume stream halves (pool > 1)
    const int per = (k + 31) >> 5;
    uint32_t loc = 0;
    for (int q = 0; q < per; ++q) {
      const int bb = lane * per + q;
      if (bb < k) {
        const int pln = a.b.pool_len[d.pool_off + bb];
        const int P = pln > 0 ? pln : pl.pb;
        loc += P > 1 ? ws.cnt[bb] : 0u;
      }
    }
    const uint32_t incl = warp_incl_scan(loc, lane);
    const uint32_t eff_total = __shfl_sync(kFull, incl, 31);
    uint32_t run = incl - loc;
    __syncwarp();
    for (int q = 0; q < per; ++q) {
      const int bb = lane * per + q;
      if (bb < k) {
        const int pln = a.b.pool_len[d.pool_off + bb];
        const int P = pln > 0 ? pln : pl.pb;
        const uint32_t c = ws.cnt[bb];
        ws.cnt[bb] = run;                 // becomes the running position cursor
        run += P > 1 ? c : 0u;
      }
    }
    __syncwarp();
    for (int i = 0; i < W; ++i) {
      const int w = i * 32 + lane;
      const bool mem = w < n && ws.cur[w] == u;
      const int bb = mem ? int(ws.bkt[w]) : (0x10000 + lane);
      const unsigned peers = __match_any_sync(kFull, bb);
      uint32_t base = 0;
      if (mem) base = ws.cnt[bb];
      __syncwarp();
      if (mem && (__ffs(peers) - 1) == lane) ws.cnt[bb] = base + __popc(peers);
      __syncwarp();
      if (mem) {
        const int pln = a.b.pool_len[d.pool_off + bb];
        const double* pool = pln > 0 ? a.b.vals + a.b.pool_off[d.pool_off + bb] : pl.B;
        const uint32_t P = uint32_t(pln > 0 ? pln : pl.pb);
        const uint32_t pos = c1 + base + __popc(peers & lt);
        const uint32_t ob = P > 1 ? lemire(half_at(jt, g, pos), P, rej) : 0u;
        ws.tmp[w] = dadd(__ddiv_rn(ws.tmp[w], a.b.prefill_rate),
                         __ddiv_rn(pool[ob], a.b.decode_rate));
      }
    }
    C = c1 + eff_total;
  }
  if (__any_sync(kFull, rej)) {
    __syncwarp();
    if (lane == 0) serial_visit(a, d, pl, own, u, ws, g);
    __syncwarp();
    g.s.lo = __shfl_sync(kFull, g.s.lo, 0);
    g.s.hi = __shfl_sync(kFull, g.s.hi, 0);
    g.pend = __shfl_sync(kFull, int(g.pend), 0);
    g.pv = __shfl_sync(kFull, g.pv, 0);
  } else {
    close_u32(jt, g, C);
  }
  // random(m) + successor jump (estimator.py:350-353)
  const double* cum = a.b.succ_cum + d.succ_off;
  const int32_t* nxt = a.b.succ_nxt + d.succ_off;
  const int ns = d.succ_len;
  uint32_t R = 0;
  for (int i = 0; i < W; ++i) {
    const int w = i * 32 + lane;
    const bool mem = w < n && ws.cur[w] == u;
    const unsigned bal = __ballot_sync(kFull, mem);
    if (mem) {
      const uint32_t r = R + __popc(bal & lt);
      const double uu = u53_double(pcg_out(pcg_jump(jt, g.s, g.inc, r + 1)));
      int idx = 0;
      while (idx < ns && __ldg(cum + idx) <= uu) ++idx;   // searchsorted(side="right")
      ws.cur[w] = int8_t(__ldg(nxt + idx));
      ws.tot[w] = dadd(ws.tot[w], ws.tmp[w]);
    }
    R += __popc(bal);
  }
  g.s = pcg_jump(jt, g.s, g.inc, m);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// K3: conditioned draw pools for the current unit (estimator.py:155-233)
// ---------------------------------------------------------------------------
__device__ bool condition(const EngineArgs& a, int gbase, int cur_unit, int obs_up,
                          const double* obs, const WarpState& ws, Pools& ovp,
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
  const CondDesc c = cd[ci];
  int ob[3];
  for (int t = 0; t < 3; ++t)
    ob[t] = c.ok[t] ? bucket_of(obs[t], c.lo[t], c.hi[t], c.k[t]) : -2;
  // which upstream variables condition which target (estimator.py:209-221)
  const bool iui = d.flags & F_IUI, iuo = d.flags & F_IUO;
  const bool ouo = d.flags & F_OUO, pup = d.flags & F_PUP;
  const PairRec* pr = reinterpret_cast<const PairRec*>(a.b.pairs) + c.pair_off;
  const unsigned lt = lanemask_lt();
  uint32_t nin = 0, nout = 0, npar = 0;
  for (int base = 0; base < c.pair_len; base += 32) {
    const int p = base + lane;
    bool kin = false, kout = false, kpar = false;
    PairRec rec;
    if (p < c.pair_len) {
      rec = pr[p];
      // a condition on an empty upstream distribution never matches
      kin = (iui || iuo) && (!iui || (ob[0] >= 0 && rec.bk[0] == ob[0])) &&
            (!iuo || (ob[1] >= 0 && rec.bk[1] == ob[1]));
      kout = ouo && ob[1] >= 0 && rec.bk[1] == ob[1];
      kpar = pup && ob[2] >= 0 && rec.bk[2] == ob[2];
    }
    const unsigned bi = __ballot_sync(kFull, kin), bo = __ballot_sync(kFull, kout);
    if (kin) ws.kin[nin + __popc(bi & lt)] = rec.in;
    if (kout) ws.kout[nout + __popc(bo & lt)] = rec.out;
    nin += __popc(bi);
    nout += __popc(bo);
    npar += __popc(__ballot_sync(kFull, kpar));
  }
  __syncwarp();
  const int capu = a.b.unit_capacity ? a.b.unit_capacity[gbase + cur_unit] : 1000;
  constexpr uint32_t kMin = 5;          // MIN_CONDITIONAL_SAMPLES (estimator.py:25)
  if ((iui || iuo) && nin >= kMin) {    // FIFO cap keeps the last `capacity` kept values
    const uint32_t keep = nin > uint32_t(capu) ? uint32_t(capu) : nin;
    ovp.A = ws.kin + (nin - keep);
    ovp.pa = int(keep);
    conditioned = true;
  }
  if (ouo && nout >= kMin) {
    const uint32_t keep = nout > uint32_t(capu) ? uint32_t(capu) : nout;
    ovp.B = ws.kout + (nout - keep);
    ovp.pb = int(keep);
    conditioned = true;
  }
  if (pup && npar >= kMin) conditioned = true;
  return true;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWarps * 32) mc_engine_kernel(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = a.n;
  const bool in_smem = n <= kSmemWalks;
  // per-warp shared block: counters, then (if small n) walk state
  const size_t per_warp_smem = size_t(a.counters) * 4 +
                               (in_smem ? size_t(kSmemWalks) * 19 : 0);
  unsigned char* sb = smem + per_warp_smem * wib;
  const int64_t gwarp = int64_t(blockIdx.x) * kWarps + wib;
  char* gs = a.scratch + size_t(gwarp) * a.scratch_per_warp;
  WarpState ws;
  ws.cnt = reinterpret_cast<uint32_t*>(sb);
  unsigned char* walk_base = in_smem ? sb + size_t(a.counters) * 4 : reinterpret_cast<unsigned char*>(gs);
  const int nw = in_smem ? kSmemWalks : n;
  ws.tot = reinterpret_cast<double*>(walk_base);
  ws.tmp = ws.tot + nw;
  ws.bkt = reinterpret_cast<uint16_t*>(ws.tmp + nw);
  ws.cur = reinterpret_cast<int8_t*>(ws.bkt + nw);
  char* k3 = gs + (in_smem ? 0 : size_t(n) * 19 + 16);
  k3 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(k3) + 15) & ~uintptr_t(15));
  ws.kin = reinterpret_cast<double*>(k3);
  ws.kout = ws.kin + a.max_pairs;

  const int64_t stride = int64_t(gridDim.x) * kWarps;
  const int W = (n + 31) >> 5;
  for (int64_t job = gwarp; job < a.n_jobs; job += stride) {
    const int gi = a.j.graph[job];
    const int gbase = a.b.graph_base[gi];
    const int u0 = a.j.unit[job];
    Stream g;
    pcg_seed(a.j.seed[job], g.s, g.inc);
    g.pend = false;
    g.pv = 0;
    // K3 conditioning of the current unit
    Pools ovp{nullptr, 0, nullptr, 0};
    bool conditioned = false;
    const int obs_up = a.j.obs_unit ? a.j.obs_unit[job] : -1;
    double obs[3] = {0.0, 0.0, 0.0};
    if (obs_up >= 0) {
      obs[0] = a.j.obs_val[3 * job];
      obs[1] = a.j.obs_val[3 * job + 1];
      obs[2] = a.j.obs_val[3 * job + 2];
    }
    const bool has_ov = condition(a, gbase, u0, obs_up, obs, ws, ovp, conditioned, lane);

    for (int i = 0; i < W; ++i) {
      const int w = i * 32 + lane;
      if (w < n) {
        ws.cur[w] = int8_t(u0);
        ws.tot[w] = 0.0;
      }
    }
    __syncwarp();
    for (int step = 0; step < a.cap; ++step) {
      unsigned occ = 0;
      for (int i = 0; i < W; ++i) {
        const int w = i * 32 + lane;
        if (w < n && ws.cur[w] >= 0) occ |= 1u << ws.cur[w];
      }
      occ = __reduce_or_sync(kFull, occ);
      if (!occ) break;
      while (occ) {
        const int u = __ffs(occ) - 1;
        occ &= occ - 1;
        visit_unit(a, gbase, u, ovp, has_ov, u0, ws, g, lane);
      }
    }
    // capped walks, samples, bucketing (distributions.py:79-105)
    int capped = 0;
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    for (int i = 0; i < W; ++i) {
      const int w = i * 32 + lane;
      if (w < n) {
        capped += ws.cur[w] >= 0;
        const double s = ws.tot[w];
        lo = fmin(lo, s);
        hi = fmax(hi, s);
        if (a.o.samples) a.o.samples[job * int64_t(a.o.samples_stride) + w] = s;
      }
    }
    capped = warp_sum(capped);
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(kFull, lo, o));
      hi = fmax(hi, __shfl_xor_sync(kFull, hi, o));
    }
    const int64_t row = a.o.slot ? a.o.slot[job] : job;
    int k = a.k_out;
    double width = 0.0;
    if (lo == hi) {
      k = 1;
    } else {
      width = __ddiv_rn(dsub(hi, lo), small_int_to_double(k));
    }
    for (int b = lane; b < k; b += 32) ws.cnt[b] = 0;
    __syncwarp();
    for (int i = 0; i < W; ++i) {
      const int w = i * 32 + lane;
      if (w < n) {
        int idx = 0;
        if (k > 1) {
          idx = __double2int_rz(__ddiv_rn(dsub(ws.tot[w], lo), width));
          idx = idx < k - 1 ? idx : k - 1;
        }
        atomicAdd(&ws.cnt[idx], 1u);
      }
    }
    __syncwarp();
    if (a.o.counts) {
      uint16_t* crow = a.o.counts + row * a.o.stride;
      for (int b = lane; b < a.o.stride; b += 32) crow[b] = b < k ? uint16_t(ws.cnt[b]) : 0;
    }
    if (lane == 0) {
      if (a.o.lo) a.o.lo[row] = lo;
      if (a.o.width) a.o.width[row] = width;
      if (a.o.nbins) a.o.nbins[row] = k;
      if (a.o.nsamp) a.o.nsamp[row] = n;
      if (a.o.capped) a.o.capped[job] = capped;
      if (a.o.flags) a.o.flags[job] = (conditioned ? 1 : 0) | (has_ov ? 2 : 0);
    }
    __syncwarp();
  }
}

}  // namespace pdg

using namespace pdg;

static size_t walk_scratch(int n) { return n <= kSmemWalks ? 0 : size_t(n) * 19 + 32; }

extern "C" size_t pdg_mc_scratch_bytes(int32_t n_samples, int32_t max_pairs, int32_t grid_warps) {
  const size_t per = (walk_scratch(n_samples) + size_t(max_pairs) * 16 + 64 + 255) & ~size_t(255);
  return per * size_t(grid_warps);
}

extern "C" int pdg_mc_grid_warps(void) { return sm_count() * 8 * kWarps; }

extern "C" int pdg_mc_remaining_demand(const pdg_graph_bank* bank, const pdg_mc_jobs* jobs,
                                       int64_t n_jobs, int32_t n_samples, int32_t visit_cap,
                                       int32_t bucket_count, int32_t max_unit_k,
                                       int32_t max_pairs, const pdg_mc_out* out,
                                       void* scratch, size_t scratch_bytes, void* stream) {
  if (!bank || !jobs || !out || n_jobs < 0 || n_samples < 1 || n_samples > (1 << 19) ||
      visit_cap < 0 || bucket_count < 1 || bucket_count > 1024 || max_unit_k > 1024 ||
      max_pairs < 0) {
    set_error("pdg_mc_remaining_demand: invalid arguments");
    return PDG_EINVAL;
  }
  if (out->counts && out->stride < bucket_count) {
    set_error("pdg_mc_remaining_demand: histogram stride < bucket_count");
    return PDG_EINVAL;
  }
  if (n_jobs == 0) return PDG_OK;
  const int grid_warps = pdg_mc_grid_warps();
  const size_t need = pdg_mc_scratch_bytes(n_samples, max_pairs, grid_warps);
  if (scratch_bytes < need || (need > 0 && !scratch)) {
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
  int c = bucket_count > max_unit_k ? bucket_count : max_unit_k;
  a.counters = (c + 3) & ~3;
  a.max_pairs = max_pairs;
  a.scratch = static_cast<char*>(scratch);
  a.scratch_per_warp = (walk_scratch(n_samples) + size_t(max_pairs) * 16 + 64 + 255) & ~size_t(255);
  const size_t smem = size_t(kWarps) * (size_t(a.counters) * 4 +
                                        (n_samples <= kSmemWalks ? size_t(kSmemWalks) * 19 : 0));
  cudaError_t e = cudaFuncSetAttribute(mc_engine_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(mc_engine_kernel)");
  int64_t blocks = (n_jobs + kWarps - 1) / kWarps;
  const int64_t capb = grid_warps / kWarps;
  if (blocks > capb) blocks = capb;
  mc_engine_kernel<<<unsigned(blocks), kWarps * 32, smem, (cudaStream_t)stream>>>(a);
  return launch_status("mc_engine_kernel");
}
