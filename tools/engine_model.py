"""Executable model of the GPU demand engine's random-stream arithmetic.

Design tool (not product code, not the oracle): it re-derives every random
draw of the reference Monte Carlo walk (estimator.py:305-362) by *position*
in numpy's PCG64 stream -- jump-ahead from a group base state instead of
sequential consumption -- which is exactly what the CUDA kernel
(paper_2506_14851_b200/csrc/engine.cu) does with one lane per walk.
tests/test_engine_model_cpu.py checks it against the oracle's samples.

numpy facts it relies on (verified against numpy 2.3 in that test):
* default_rng(seed): SeedSequence(seed).generate_state(4, uint64) ->
  PCG64 srandom(initstate = w0:w1, initseq = w2:w3).
* random(m): m words, double = (word >> 11) * 2^-53.
* choice(pool, m) with len(pool) = P > 1: m bounded draws, each Lemire on one
  32-bit half (low half first; a leftover high half is kept across calls).
  Rejection (leftover < (2^32 - P) % P) consumes extra halves.  P == 1
  consumes nothing.
"""

from __future__ import annotations

import numpy as np

M128 = (1 << 128) - 1
M64 = (1 << 64) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645

# ---- SeedSequence (numpy/random/bit_generator.pyx) -------------------------
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
M32 = 0xFFFFFFFF


def _words32(n: int) -> list[int]:
    if n == 0:
        return [0]
    out = []
    while n:
        out.append(n & M32)
        n >>= 32
    return out


def seed_state(seed: int) -> tuple[int, int]:
    """PCG64 (state, inc) for np.random.default_rng(seed), seed >= 0."""
    ent = _words32(seed)
    hc = INIT_A
    pool = []

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & M32
        hc = (hc * MULT_A) & M32
        v = (v * hc) & M32
        return v ^ (v >> 16)

    for i in range(4):
        pool.append(hashmix(ent[i] if i < len(ent) else 0))

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return r ^ (r >> 16)

    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    hb = INIT_B
    st = []
    for i in range(8):
        v = pool[i % 4] ^ hb
        hb = (hb * MULT_B) & M32
        v = (v * hb) & M32
        st.append(v ^ (v >> 16))
    w = [st[2 * i] | (st[2 * i + 1] << 32) for i in range(4)]
    initstate = (w[0] << 64) | w[1]
    initseq = (w[2] << 64) | w[3]
    inc = ((initseq << 1) | 1) & M128
    s = (0 * MULT + inc) & M128
    s = (s + initstate) & M128
    s = (s * MULT + inc) & M128
    return s, inc


def out64(s: int) -> int:
    hi, lo = s >> 64, s & M64
    x, r = hi ^ lo, hi >> 58
    return ((x >> r) | (x << ((64 - r) & 63))) & M64


# jump tables: state after j steps = A[j]*s + inc*G[j]
def jump_tables(jmax: int):
    A, G = [1], [0]
    for _ in range(jmax):
        A.append((A[-1] * MULT) & M128)
        G.append((G[-1] * MULT + 1) & M128)
    return A, G


class Stream:
    """Group-level view of the generator: base state after w words, plus the
    buffered high half (or None)."""

    def __init__(self, seed: int, tables):
        self.s, self.inc = seed_state(seed)
        self.pend = None
        self.A, self.G = tables

    def word(self, q: int) -> int:          # q-th fresh word from the base
        j = q + 1
        return out64((self.A[j] * self.s + self.inc * self.G[j]) & M128)

    def advance(self, words: int):
        self.s = (self.A[words] * self.s + self.inc * self.G[words]) & M128

    def half(self, R: int) -> int:          # R-th half of the current u32 stream
        if self.pend is not None:
            if R == 0:
                return self.pend
            R -= 1
        w = self.word(R >> 1)
        return (w >> 32) if (R & 1) else (w & M32)

    def close_u32(self, C: int):
        """C halves were drawn by the group (positions 0..C-1)."""
        if C == 0:
            return
        F = C - (1 if self.pend is not None else 0)
        if F & 1:
            self.pend = self.word((F - 1) >> 1) >> 32
        else:
            self.pend = None
        self.advance((F + 1) >> 1)

    def double(self, r: int) -> float:
        return (self.word(r) >> 11) * (1.0 / 9007199254740992.0)


class Rejected(Exception):
    pass


def lemire(h: int, P: int) -> int:
    m = h * P
    left = m & M32
    if left < P and left < ((1 << 32) - P) % P:
        raise Rejected
    return m >> 32


def walk(g, current, override, n, seed, cap, tables, prefill=1e4, decode=50.0):
    """Positional re-derivation of oracle.mc_remaining_demand (no rejection
    handling: raises Rejected, which the kernel resolves serially)."""
    from oracle import pdg_oracle as O
    order = sorted(g.units)
    pos = {u: i for i, u in enumerate(order)}
    units = [g.units[u] for u in order]
    st = Stream(seed, tables)
    cur = np.full(n, pos[current], dtype=np.int64)
    tot = np.zeros(n)
    for _ in range(cap):
        occ = sorted(set(int(c) for c in cur if c >= 0))
        if not occ:
            break
        for ui in occ:
            mem = np.flatnonzero(cur == ui)
            m = len(mem)
            u = units[ui]
            ov = override if order[ui] == current else None
            if not u.is_llm:
                dv = np.asarray(u.samples("duration"))
                P = len(dv)
                t = np.array([dv[lemire(st.half(r), P)] if P > 1 else dv[0] for r in range(m)])
                st.close_u32(m if P > 1 else 0)
            else:
                iv = np.asarray(ov.input_vals if ov else u.samples("input"))
                ovv = np.asarray(ov.output_vals if ov else u.samples("output"))
                Pi, Po = len(iv), len(ovv)
                c1 = m if Pi > 1 else 0
                ii = np.array([iv[lemire(st.half(r), Pi)] if Pi > 1 else iv[0] for r in range(m)])
                own = u.masks.get("output_own_input") and ov is None and u.records
                if own:
                    bins = u.binning("input")
                    pools: dict = {}
                    for rec in u.records:
                        pools.setdefault(bins.index_of(rec.input_len), []).append(rec.output_len)
                    key = np.array([bins.index_of(x) for x in ii])
                    oo = np.empty(m)
                    R = c1
                    for b in sorted(set(key.tolist())):
                        sel = np.flatnonzero(key == b)
                        pool = np.asarray(pools.get(b) or ovv)
                        P = len(pool)
                        for k, wk in enumerate(sel):
                            oo[wk] = pool[lemire(st.half(R + k), P)] if P > 1 else pool[0]
                        if P > 1:
                            R += len(sel)
                    st.close_u32(R)
                else:
                    oo = np.array([ovv[lemire(st.half(c1 + r), Po)] if Po > 1 else ovv[0]
                                   for r in range(m)])
                    st.close_u32(c1 + (m if Po > 1 else 0))
                t = ii / prefill + oo / decode
            tot[mem] += t
            succ = sorted(u.succ.items())
            cum = np.cumsum([p for _, p in succ])
            nxt = np.array([pos[s] for s, _ in succ] + [-1])
            uu = np.array([st.double(r) for r in range(m)])
            st.advance(m)
            cur[mem] = nxt[np.searchsorted(cum, uu, side="right")] if len(cum) else -1
    return tot, int((cur >= 0).sum())



def walk_units(g, current, override, n, seed, cap, tables, prefill=1e4, decode=50.0):
    """Model of the kernel's per-visit word decode (engine.cu visit_words):
    a unit visit's stream segment -- wb words of bounded-halves, then m
    uniforms -- is cut into contiguous word ranges, each decoded from the
    visit's base state by position.  The occupied set of the next step is
    tracked as a pending mask (arrivals after a unit's visit).  Own-input
    units are not modelled (returns None)."""
    order = sorted(g.units)
    pos = {u: i for i, u in enumerate(order)}
    units = [g.units[u] for u in order]
    s0, inc = seed_state(seed)
    A, G = tables
    st = {"base": s0, "pend": 0, "pv": 0}

    def word(q):
        j = q + 1
        return out64((A[j] * st["base"] + inc * G[j]) & M128)

    cur = np.full(n, pos[current], dtype=np.int64)
    tot = np.zeros(n)
    pending = {pos[current]}
    for _ in range(cap):
        occ = sorted(pending)
        assert occ == sorted(set(int(c) for c in cur if c >= 0))
        if not occ:
            break
        for ui in occ:
            mem = np.flatnonzero(cur == ui)
            pending.discard(ui)
            m = len(mem)
            u = units[ui]
            ov = override if order[ui] == current else None
            if u.is_llm:
                if u.masks.get("output_own_input") and ov is None and u.records:
                    return None
                pa = np.asarray(ov.input_vals if ov else u.samples("input"))
                pb = np.asarray(ov.output_vals if ov else u.samples("output"))
            else:
                pa = np.asarray(u.samples("duration"))
                pb = None
            mA = m if len(pa) > 1 else 0
            C = mA + (m if (u.is_llm and len(pb) > 1) else 0)
            pin = st["pend"]
            wb = (C - pin + 1) >> 1 if C else 0
            W = wb + m
            ia = np.zeros(m, dtype=np.int64)
            ib = np.zeros(m, dtype=np.int64)
            pend_hi = None
            for q in range(wb):
                wd = word(q)
                for t, h in enumerate((wd & M32, wd >> 32)):
                    r = 2 * q + pin + t
                    if r < mA:
                        ia[r] = lemire(h, len(pa))
                    elif r < C:
                        ib[r - mA] = lemire(h, len(pb))
                    elif r == C:
                        pend_hi = h
            if pin and C:
                if mA:
                    ia[0] = lemire(st["pv"], len(pa))
                else:
                    ib[0] = lemire(st["pv"], len(pb))
            t = pa[ia]
            if u.is_llm:
                t = t / prefill + pb[ib] / decode
            tot[mem] += t
            succ = sorted(u.succ.items())
            cum = np.cumsum([p for _, p in succ])
            nx = np.array([pos[s] for s, _ in succ] + [-1])
            uu = np.array([(word(wb + k) >> 11) * (1.0 / 9007199254740992.0) for k in range(m)])
            v = nx[np.searchsorted(cum, uu, side="right")] if len(cum) else np.full(m, -1)
            cur[mem] = v
            pending |= set(int(x) for x in v if x >= 0)
            st["base"] = (A[W] * st["base"] + inc * G[W]) & M128
            if C:
                st["pend"] = (pin + C) & 1
                if st["pend"]:
                    st["pv"] = pend_hi
    return tot, int((cur >= 0).sum())
