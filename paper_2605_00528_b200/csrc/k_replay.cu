// A7 epoch-synchronous replay (SURVEY §8.C.5 rules R1-R4) with the A5 key
// (eq:eviction ... eq:overlap, Alg. alg:ttl, eq:pressure) and the A6 capacity-bounded top-k.
//
// Work item = (policy, capacity, node).  Time is sequential inside an item and items are
// independent, so one CTA replays one item at a time (persistent CTAs pull items, largest
// capacity first).  The replay never scans the resident set S per eviction event.  Instead it
// keeps, per item, incremental indices whose cost per event is O(records + live units + victims):
//
//   res_pos[lid]  the position of the block's latest access if resident, else NONE.  A
//                 first-in-epoch record p of block b is a hit iff res_pos[b] != NONE (R2).
//   BELADY        key = (nu << 32) | lid.  Two hierarchical bitmaps (HB: bits, per-1024-bit
//                 counts c1, per-2^20-bit counts c2):
//                   pend over stream positions: bit q set iff q = next_use of a resident block
//                     (finite nu; distinct blocks have distinct next uses, so bit order = key order);
//                   dead over local ids: resident blocks with nu = INF (largest keys; lid order).
//                 The k largest keys = the top dead lids, then the top pending positions.  At
//                 its next access p the block's pending bit is exactly p (nu = p), so R2 clears
//                 bit p; R4 sets bit next_use[p] (or the dead bit) for the block's last record.
//   AEG           the key of block b is ((!prot << 63) | q << 32 | lid) where prot and q depend
//                 only on (t_last(b), owner(b)) at T_e.  Positions are grouped into units = maximal
//                 runs of one record group with one owner; a resident block's latest position
//                 lies in exactly one unit, and all blocks of a unit share (t_last, owner), hence
//                 (prot, q).  Per unit: cnt = resident non-in-flight blocks; `alive` = bitmap of
//                 latest positions of resident blocks.  Per eviction: normalisers tau_max /
//                 size_max over live units, per-unit key part kp = (!prot << 31) | q, a weighted
//                 radix select over units gives the pivot kp*, units above it are evicted whole,
//                 and the pivot units' blocks are ranked by lid (radix select) for the remainder.
//   EVICT_ALL     every live unit evicted whole.
//
// In-flight blocks (A ∩ S, not evictable at this boundary) are removed from the index in R2 and
// re-inserted at their last record of the epoch in R4, which also sets t_last / nu.  The victim
// hash is an order-independent sum (DESIGN.md R-hash), so parallel emission is deterministic.
#include <algorithm>

#include "block_select.cuh"

namespace saga {
namespace {

constexpr int RT = 512;
constexpr int RW = RT / 32;
constexpr uint32_t KIND_MIG = 0x80000000u;
constexpr uint32_t UMASK = 0x7FFFFFFFu;
constexpr int H1 = 4096;  // first-level key-part digit: [!prot:1 | q >> 10 : 11]

// hierarchical bitmap; storage is allocated in whole c2 blocks (2^20 bits)
struct HB {
  uint32_t* bits;  // [n2 * 32768] words
  uint32_t* c1;    // [n2 * 1024]  set bits per 1024-bit block
  uint32_t* c2;    // [n2]         set bits per 2^20-bit block
  uint32_t n2;
};

struct NodeArr {
  uint64_t N;
  uint32_t J, n_local, n_units, pad;
  const uint64_t* ev_pos;
  const uint32_t* ev_e;
  const uint32_t* ev_inv;
  const uint32_t* ev_act;
  const uint32_t* ev_unit;
  const uint32_t* ev_upd;
  const uint32_t* inv_s;
  const uint32_t* lidf;
  const uint32_t* nxt;
  const uint32_t* u_of;
  const uint32_t* u_pos;
  const int64_t* u_t;
  const uint32_t* u_own;
  const uint32_t* lid2gid;
  const uint32_t* upd_c;
};

struct ReplayArgs {
  TraceView v;
  const NodeArr* nodes;
  const uint32_t* caps;
  const uint32_t* items;  // packed (pi << 28) | (ci << 12) | node_list index, largest capacity first
  uint32_t n_items;
  const uint32_t* node_list;
  uint32_t pol[3];
  uint32_t n_caps;
  uint32_t n_nodes_total;
  int64_t* counters;
  float alpha, beta, gamma;
  uint32_t p_low, p_high;
  int64_t ttl_max;
  // per-CTA scratch (strides in elements)
  uint8_t* scratch;
  uint64_t cta_bytes;
  uint64_t o_res, o_bits, o_c1, o_c2, o_dbits, o_dc1, o_dc2, o_cnt, o_list0, o_list1, o_lkp, o_kbuf, o_sst;
  uint32_t* work;
  uint32_t* err;
};

struct Smem {
  BlockScratch<RT> b;
  uint32_t hist[H1];
  uint32_t res_j, res_rem, thr, item;
  uint32_t n_app, n_piv;
  uint32_t ilo, ihi;
};

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// arr[lo..hi) scanned from hi-1 downwards: j with sum(arr[j+1..hi)) < k <= sum(arr[j..hi)) and
// rem = k - sum(arr[j+1..hi)).  Requires 1 <= k <= sum(arr[lo..hi)).  Block-wide.
__device__ void find_level(const uint32_t* arr, uint32_t lo, uint32_t hi, uint32_t k, uint32_t& j, uint32_t& rem,
                           Smem& sm) {
  uint32_t carry = 0;
  for (uint32_t base = 0; base < hi - lo; base += RT) {
    const uint32_t t = base + threadIdx.x;
    const bool in = t < hi - lo;
    const uint32_t idx = hi - 1 - t;
    const uint32_t v = in ? arr[idx] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<RT>(v, &tot, sm.b.u32);
    if (in && carry + ex < k && k <= carry + ex + v) { sm.res_j = idx; sm.res_rem = k - carry - ex; }
    carry += tot;
    if (carry >= k) break;
  }
  __syncthreads();
  j = sm.res_j;
  rem = sm.res_rem;
}

__device__ __forceinline__ void hb_set(const HB& h, uint32_t i) {
  atomicOr(&h.bits[i >> 5], 1u << (i & 31));
  atomicAdd(&h.c1[i >> 10], 1u);
  atomicAdd(&h.c2[i >> 20], 1u);
}
__device__ __forceinline__ void hb_clear(const HB& h, uint32_t i) {
  atomicAnd(&h.bits[i >> 5], ~(1u << (i & 31)));
  atomicSub(&h.c1[i >> 10], 1u);
  atomicSub(&h.c2[i >> 20], 1u);
}
// warp-cooperative update (all lanes call): lanes with `act` set (or clear) bit i; the count
// updates of lanes that hit the same 1024-bit block are aggregated.
__device__ __forceinline__ void hb_update_warp(const HB& h, bool act, uint32_t i, bool set) {
  const uint32_t am = __ballot_sync(0xffffffffu, act);
  if (!act) return;
  const int lane = threadIdx.x & 31;
  if (set) atomicOr(&h.bits[i >> 5], 1u << (i & 31));
  else atomicAnd(&h.bits[i >> 5], ~(1u << (i & 31)));
  const uint32_t p1 = __match_any_sync(am, i >> 10);
  if (lane == 31 - __clz(p1)) {
    const uint32_t n = __popc(p1);
    atomicAdd(&h.c1[i >> 10], set ? n : (uint32_t)(-(int32_t)n));
    atomicAdd(&h.c2[i >> 20], set ? n : (uint32_t)(-(int32_t)n));
  }
}

// number of set bits (block-wide sum of c2)
__device__ uint32_t hb_total(const HB& h, Smem& sm) {
  uint32_t s = 0;
  for (uint32_t i = threadIdx.x; i < h.n2; i += RT) s += h.c2[i];
  return block_reduce<RT, uint32_t>(s, Add(), sm.b.u32);
}

// take (clear and emit) every set bit with index >= T, starting at c1 block j1 of c2 block j2
template <class Emit>
__device__ void hb_take_from(const HB& h, uint32_t j2, uint32_t j1, uint32_t T, Emit& emit) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t tw = T >> 5;
  for (uint32_t jb = j2; jb < h.n2; ++jb) {
    if (jb > j2 && h.c2[jb] == 0) continue;
    const uint32_t lo = (jb == j2) ? j1 : jb * 1024u, hi = jb * 1024u + 1024u;
    for (uint32_t i0 = lo + (uint32_t)wid * 32u; i0 < hi; i0 += RW * 32u) {
      const uint32_t ci = i0 + lane;
      const uint32_t cv = ci < hi ? h.c1[ci] : 0u;
      uint32_t nz = __ballot_sync(0xffffffffu, cv != 0);
      while (nz) {
        const int l = __ffs(nz) - 1;
        nz &= nz - 1;
        const uint32_t c1i = i0 + l;
        const uint32_t wi = c1i * 32u + lane;
        const uint32_t m = wi > tw ? 0xffffffffu : (wi == tw ? ~((1u << (T & 31)) - 1u) : 0u);
        const uint32_t wv = h.bits[wi];
        const uint32_t tk = wv & m;
        if (tk) {
          h.bits[wi] = wv & ~m;
          for (uint32_t x = tk; x; x &= x - 1) emit(wi * 32u + (uint32_t)(__ffs(x) - 1));
        }
        const uint32_t n = warp_sum(__popc(tk));
        if (lane == 0 && n) { h.c1[c1i] -= n; atomicSub(&h.c2[jb], n); }
      }
    }
  }
}

// take the k highest set bits (1 <= k <= total)
template <class Emit>
__device__ void hb_take_top(const HB& h, uint32_t k, Emit& emit, Smem& sm) {
  uint32_t j2, r2, j1, r1;
  find_level(h.c2, 0, h.n2, k, j2, r2, sm);
  find_level(h.c1, j2 * 1024u, j2 * 1024u + 1024u, r2, j1, r1, sm);
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    const uint32_t wi = j1 * 32u + (31u - lane);  // lane 0 = highest word of the block
    const uint32_t wv = h.bits[wi];
    const uint32_t c = __popc(wv);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (x - c < r1 && r1 <= x) {
      uint32_t need = r1 - (x - c), w2 = wv;
      int b = 31 - __clz(w2);
      while (--need) { w2 &= ~(1u << b); b = 31 - __clz(w2); }
      sm.thr = wi * 32u + (uint32_t)b;
    }
  }
  __syncthreads();
  const uint32_t T = sm.thr;
  hb_take_from(h, j2, j1, T, emit);
  __syncthreads();
}

template <class Emit>
__device__ void hb_take_all(const HB& h, Emit& emit) {
  hb_take_from(h, 0, 0, 0, emit);
  __syncthreads();
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (a[mid] < x) lo = mid + 1; else hi = mid; }
  return lo;
}

// owner state of a private session / shared prefix at the current boundary
__device__ __forceinline__ OwnerKeyIn owner_in(const TraceView& v, const uint32_t* sstate, uint32_t o, uint32_t act) {
  OwnerKeyIn r;
  if (o >= v.n_sessions) {
    const uint32_t t = o - v.n_sessions;
    const bool on = (act >> t) & 1u;
    r.shared = true; r.prot_shared = on; r.size = v.tlen[t]; r.P = on ? 1.0f : 0.0f;
    r.fin = false; r.t_call = 0; r.ttl_base = 0;
    return r;
  }
  const uint32_t c1 = sstate[o];
  const uint32_t c = c1 ? c1 - 1 : 0;
  r.shared = false; r.prot_shared = false;
  r.size = __ldg(&v.ci_size[c]);
  r.fin = __ldg(&v.ci_fin[c]) != 0;
  r.P = __ldg(&v.ci_P[c]);
  r.t_call = __ldg(&v.tend[c]);
  r.ttl_base = __ldg(&v.ttl[__ldg(&v.call_v[c])]);
  return r;
}

__device__ __forceinline__ uint32_t owner_size(const TraceView& v, const uint32_t* sstate, uint32_t o) {
  if (o >= v.n_sessions) return v.tlen[o - v.n_sessions];
  const uint32_t c1 = sstate[o];
  return __ldg(&v.ci_size[c1 ? c1 - 1 : 0]);
}

// per-thread victim bookkeeping
struct Vict {
  uint32_t* res_pos;
  unsigned long long hash;
  uint32_t n, np;
  uint64_t eh;  // e << 32
  __device__ __forceinline__ void operator()(uint32_t lid) {
    res_pos[lid] = NONE;
    hash += splitmix64(eh | lid);
    ++n;
  }
};

__global__ void __launch_bounds__(RT) k_replay(ReplayArgs a) {
  __shared__ Smem sm;
  __shared__ long long s_ctr[SAGA_NCOUNT];
  const TraceView& v = a.v;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* base = a.scratch + (uint64_t)blockIdx.x * a.cta_bytes;
  uint32_t* res_pos = reinterpret_cast<uint32_t*>(base + a.o_res);
  uint32_t* alive = reinterpret_cast<uint32_t*>(base + a.o_bits);   // AEG / EVICT_ALL (aliases pend.bits)
  uint32_t* cnt = reinterpret_cast<uint32_t*>(base + a.o_cnt);
  uint32_t* lists[2] = {reinterpret_cast<uint32_t*>(base + a.o_list0), reinterpret_cast<uint32_t*>(base + a.o_list1)};
  uint32_t* lkp = reinterpret_cast<uint32_t*>(base + a.o_lkp);
  uint64_t* kbuf = reinterpret_cast<uint64_t*>(base + a.o_kbuf);
  uint32_t* sstate = reinterpret_cast<uint32_t*>(base + a.o_sst);

  while (true) {
    if (threadIdx.x == 0) sm.item = atomicAdd(a.work, 1u);
    __syncthreads();
    const uint32_t it = sm.item;
    __syncthreads();
    if (it >= a.n_items) break;
    const uint32_t packed = a.items[it];
    const uint32_t pi = packed >> 28, ci = (packed >> 12) & 0xFFFFu, ni = packed & 0xFFFu;
    const uint32_t pol = a.pol[pi];
    const uint32_t C = a.caps[ci];
    const uint32_t w = a.node_list[ni];
    const NodeArr nd = a.nodes[w];
    const bool belady = pol == SAGA_POLICY_BELADY;
    const bool aeg = pol == SAGA_POLICY_AEG;
    const uint32_t n2N = (uint32_t)((nd.N + (1u << 20) - 1) >> 20) + 0u;
    const uint32_t n2L = (nd.n_local + (1u << 20) - 1) >> 20;
    HB pend{reinterpret_cast<uint32_t*>(base + a.o_bits), reinterpret_cast<uint32_t*>(base + a.o_c1),
            reinterpret_cast<uint32_t*>(base + a.o_c2), n2N > 0 ? n2N : 1u};
    HB dead{reinterpret_cast<uint32_t*>(base + a.o_dbits), reinterpret_cast<uint32_t*>(base + a.o_dc1),
            reinterpret_cast<uint32_t*>(base + a.o_dc2), n2L > 0 ? n2L : 1u};
    // ---- reset the item state ----
    {
      uint4 ones = make_uint4(NONE, NONE, NONE, NONE), zero = make_uint4(0, 0, 0, 0);
      uint4* r4 = reinterpret_cast<uint4*>(res_pos);
      for (uint32_t i = threadIdx.x; i < (nd.n_local + 3) / 4; i += RT) r4[i] = ones;
      const uint32_t nbw = pend.n2 * 32768u;
      uint4* b4 = reinterpret_cast<uint4*>(pend.bits);
      for (uint32_t i = threadIdx.x; i < nbw / 4; i += RT) b4[i] = zero;
      if (belady) {
        uint4* c4 = reinterpret_cast<uint4*>(pend.c1);
        for (uint32_t i = threadIdx.x; i < pend.n2 * 256u; i += RT) c4[i] = zero;
        for (uint32_t i = threadIdx.x; i < pend.n2; i += RT) pend.c2[i] = 0;
        uint4* d4 = reinterpret_cast<uint4*>(dead.bits);
        for (uint32_t i = threadIdx.x; i < dead.n2 * 8192u; i += RT) d4[i] = zero;
        uint4* dc4 = reinterpret_cast<uint4*>(dead.c1);
        for (uint32_t i = threadIdx.x; i < dead.n2 * 256u; i += RT) dc4[i] = zero;
        for (uint32_t i = threadIdx.x; i < dead.n2; i += RT) dead.c2[i] = 0;
      } else {
        for (uint32_t i = threadIdx.x; i < nd.n_units; i += RT) cnt[i] = 0;
      }
      if (aeg) for (uint32_t i = threadIdx.x; i < v.n_sessions; i += RT) sstate[i] = 0;
      if (threadIdx.x < SAGA_NCOUNT) s_ctr[threadIdx.x] = 0;
      __syncthreads();
    }
    uint32_t S = 0;       // |S| (uniform)
    uint32_t nL = 0;      // live unit list length (uniform)
    int cur = 0;          // active list buffer
    uint32_t ucur = 0;    // session-update cursor (uniform)
    long long c_hit = 0, c_miss = 0, c_mhit = 0, c_mmiss = 0, c_comp = 0, c_regen = 0, c_inv = 0;
    long long c_ev = 0, c_prot = 0, c_evev = 0, c_events = 0, c_peak = 0, infeasible = 0;
    unsigned long long hash = 0;
    uint32_t bad = 0;

    for (uint32_t j = 0; j < nd.J; ++j) {
      const uint32_t e = nd.ev_e[j];
      const int64_t Te = (int64_t)e * v.epoch_us;
      // ---- AEG session state at T_e: newest call c* with e(c*) <= e ----
      if (aeg && j + 1 < nd.J) {
        const uint32_t ue = nd.ev_upd[j];
        for (uint32_t i = ucur + threadIdx.x; i < ue; i += RT) {
          const uint32_t c = nd.upd_c[i];
          atomicMax(&sstate[v.call_sess[c]], c + 1);
        }
        ucur = ue;
      }
      // ---- R1: invalidate the blocks of sessions migrated away ----
      const uint32_t i0 = nd.ev_inv[j], i1 = nd.ev_inv[j + 1];
      for (uint32_t ii = i0; ii < i1; ++ii) {
        __syncthreads();
        if (threadIdx.x == 0) {
          const uint32_t s = nd.inv_s[ii];
          sm.ilo = lower_bound_u32(nd.lid2gid, nd.n_local, v.slo[s]);
          sm.ihi = lower_bound_u32(nd.lid2gid, nd.n_local, v.slo[s] + v.slen[s]);
        }
        __syncthreads();
        uint32_t nrm = 0;
        for (uint32_t l = sm.ilo + threadIdx.x; l < sm.ihi; l += RT) {
          const uint32_t p = res_pos[l];
          if (p == NONE) continue;
          res_pos[l] = NONE;
          ++nrm;
          if (belady) {
            const uint32_t q = nd.nxt[p];
            if (q == INF32) hb_clear(dead, l); else hb_clear(pend, q);
          } else {
            atomicAnd(&alive[p >> 5], ~(1u << (p & 31)));
            atomicSub(&cnt[nd.u_of[p] & UMASK], 1u);
          }
        }
        nrm = block_reduce<RT, uint32_t>(nrm, Add(), sm.b.u32);
        S -= nrm;
        c_inv += nrm;  // uniform
      }
      if (j + 1 == nd.J) break;  // sentinel: trailing invalidations only
      const uint64_t P0 = nd.ev_pos[j], P1 = nd.ev_pos[j + 1];
      if (P0 == P1) continue;    // only empty record groups (the oracle skips the epoch)
      __syncthreads();
      // ---- R2: |A|, new = |A \ S|; hits / misses; in-flight blocks leave the index ----
      uint32_t nA = 0, nnew = 0;
      uint32_t t_hit = 0, t_miss = 0, t_mhit = 0, t_mmiss = 0, t_comp = 0, t_regen = 0;
      for (uint64_t wb = (P0 & ~31ull) + (uint64_t)wid * 32u; wb < P1; wb += RT) {
        const uint64_t pb = wb + lane;
        const bool in = pb >= P0 && pb < P1;
        uint32_t lf = 0, uo = 0, lid = 0;
        bool first = false, resident = false;
        uint32_t rp = NONE;
        if (in) {
          lf = nd.lidf[pb];
          uo = nd.u_of[pb];
          lid = lf & LID_MASK;
          first = !(lf & LID_NFIE);
          const bool mig = (uo & KIND_MIG) != 0;
          if (first) {
            ++nA;
            rp = res_pos[lid];
            resident = rp != NONE;
            if (!resident) {
              ++nnew;
              if (mig) ++t_mmiss; else { ++t_miss; if (!(lf & LID_FTN)) ++t_regen; }
              if (lf & LID_FTN) ++t_comp;
            } else {
              if (mig) ++t_mhit; else ++t_hit;
            }
          } else {
            if (mig) ++t_mhit; else ++t_hit;
          }
        }
        if (belady) {
          hb_update_warp(pend, in && first && resident, (uint32_t)pb, false);
        } else if (in && first && resident) {
          atomicAnd(&alive[rp >> 5], ~(1u << (rp & 31)));
          atomicSub(&cnt[nd.u_of[rp] & UMASK], 1u);
        }
      }
      {
        const unsigned long long pk = block_reduce<RT, unsigned long long>(
            ((unsigned long long)nA << 32) | nnew, Add(), sm.b.u64);
        nA = (uint32_t)(pk >> 32);
        nnew = (uint32_t)pk;
      }
      if (nA > C) { infeasible = e; break; }
      c_hit += t_hit; c_miss += t_miss; c_mhit += t_mhit; c_mmiss += t_mmiss; c_comp += t_comp; c_regen += t_regen;
      const uint32_t inAS = nA - nnew;  // in-flight (resident) blocks
      const int64_t kk = (pol == SAGA_POLICY_EVICT_ALL) ? (int64_t)S - (int64_t)inAS
                                                        : (int64_t)S + (int64_t)nnew - (int64_t)C;
      // ---- R3: evict the k largest keys among cand = S \ A ----
      if (kk > 0) {
        const uint32_t k = (uint32_t)kk;
        Vict vc{res_pos, 0ull, 0u, 0u, (uint64_t)e << 32};
        if (belady) {
          const uint32_t nd_ = hb_total(dead, sm);
          auto emit_dead = [&](uint32_t lid) { vc(lid); };
          auto emit_pend = [&](uint32_t q) { vc(nd.lidf[q] & LID_MASK); };
          if (k <= nd_) {
            hb_take_top(dead, k, emit_dead, sm);
          } else {
            if (nd_ > 0) hb_take_all(dead, emit_dead);
            const uint32_t np_ = hb_total(pend, sm);
            if (k - nd_ <= np_) hb_take_top(pend, k - nd_, emit_pend, sm);
            else if (threadIdx.x == 0) bad = 1;
          }
        } else {
          const uint32_t* L = lists[cur];
          // unit eviction: all resident latest positions of unit u (warp-cooperative)
          auto evict_unit = [&](uint32_t u, bool prot) {
            const uint32_t pa = nd.u_pos[u], pe = nd.u_pos[u + 1];
            uint32_t taken = 0;
            for (uint32_t wi = (pa >> 5) + lane; wi <= ((pe - 1) >> 5); wi += 32) {
              uint32_t m = 0xffffffffu;
              if (wi == (pa >> 5)) m &= ~((1u << (pa & 31)) - 1u);
              if (wi == ((pe - 1) >> 5) && (pe & 31)) m &= (1u << (pe & 31)) - 1u;
              const uint32_t wv = alive[wi] & m;
              if (wv) {
                atomicAnd(&alive[wi], ~wv);
                for (uint32_t x = wv; x; x &= x - 1) vc(nd.lidf[wi * 32u + (uint32_t)(__ffs(x) - 1)] & LID_MASK);
                taken += __popc(wv);
              }
            }
            if (prot) vc.np += taken;
            taken = warp_sum(taken);
            if (lane == 0) cnt[u] -= taken;
          };
          if (!aeg) {  // EVICT_ALL: every candidate
            for (uint32_t i = wid; i < nL; i += RW) {
              const uint32_t u = L[i];
              if (cnt[u]) evict_unit(u, false);
            }
            __syncthreads();
          } else {
            // pass a: normalisers over cand (eq:recency tau_max, eq:size size_max)
            long long tau = 0;
            uint32_t smax = 1;
            for (uint32_t i = threadIdx.x; i < nL; i += RT) {
              const uint32_t u = L[i];
              if (!cnt[u]) continue;
              tau = max(tau, (long long)(Te - nd.u_t[u]));
              smax = max(smax, owner_size(v, sstate, nd.u_own[u]));
            }
            tau = block_reduce<RT, long long>(tau, Max(), sm.b.i64);
            smax = block_reduce<RT, uint32_t>(smax, Max(), sm.b.u32);
            KeyCtx x;
            x.Te = Te; x.tau = tau; x.smax = smax;
            x.den = (int64_t)(a.p_high - a.p_low) * C;
            x.num = min(x.den, max((int64_t)0, 1000 * (int64_t)S - (int64_t)a.p_low * C));
            x.ttl_max = a.ttl_max; x.alpha = a.alpha; x.beta = a.beta; x.gamma = a.gamma;
            const uint32_t act = nd.ev_act[j];
            // pass b: per-unit key part kp = (!prot << 31) | q, weighted histogram of the top digit
            for (uint32_t i = threadIdx.x; i < H1; i += RT) sm.hist[i] = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < nL; i += RT) {
              const uint32_t u = L[i];
              const uint32_t c = cnt[u];
              uint32_t kp = 0;
              if (c) {
                const OwnerKeyIn oi = owner_in(v, sstate, nd.u_own[u], act);
                const uint32_t q = quantize_q20(wa_lru_score(x, nd.u_t[u], oi.size, oi.P));
                kp = ((uint32_t)!ttl_protected(x, oi) << 31) | q;
                atomicAdd(&sm.hist[((kp >> 31) << 11) | (q >> 10)], c);
              }
              lkp[i] = kp;
            }
            __syncthreads();
            uint32_t d1, r1, d2, r2;
            find_level(sm.hist, 0, H1, k, d1, r1, sm);
            for (uint32_t i = threadIdx.x; i < 1024; i += RT) sm.hist[i] = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < nL; i += RT) {
              const uint32_t kp = lkp[i];
              if ((((kp >> 31) << 11) | ((kp & 0x1FFFFFu) >> 10)) != d1) continue;
              const uint32_t c = cnt[L[i]];
              if (c) atomicAdd(&sm.hist[kp & 1023u], c);
            }
            __syncthreads();
            find_level(sm.hist, 0, 1024, r1, d2, r2, sm);
            const uint32_t kps = ((d1 >> 11) << 31) | ((d1 & 2047u) << 10) | d2;
            const bool prot_piv = !(kps >> 31);
            const bool whole = sm.hist[d2] == r2;  // the pivot units are evicted whole
            if (threadIdx.x == 0) sm.n_piv = 0;
            __syncthreads();
            // pass c: units above the pivot are evicted whole; pivot units are gathered by lid
            for (uint32_t i = wid; i < nL; i += RW) {
              const uint32_t u = L[i];
              const uint32_t kp = lkp[i];
              if (!cnt[u] || kp < kps) continue;
              if (kp > kps || whole) { evict_unit(u, !(kp >> 31)); continue; }
              const uint32_t pa = nd.u_pos[u], pe = nd.u_pos[u + 1];
              for (uint32_t wb = (pa >> 5); wb <= ((pe - 1) >> 5); wb += 32) {
                const uint32_t wi = wb + lane;
                uint32_t wv = 0;
                if (wi <= ((pe - 1) >> 5)) {
                  uint32_t m = 0xffffffffu;
                  if (wi == (pa >> 5)) m &= ~((1u << (pa & 31)) - 1u);
                  if (wi == ((pe - 1) >> 5) && (pe & 31)) m &= (1u << (pe & 31)) - 1u;
                  wv = alive[wi] & m;
                }
                const uint32_t c = __popc(wv);
                uint32_t xs = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                  const uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
                  if (lane >= o) xs += y;
                }
                const uint32_t tot = __shfl_sync(0xffffffffu, xs, 31);
                uint32_t b0 = 0;
                if (lane == 31 && tot) b0 = atomicAdd(&sm.n_piv, tot);
                b0 = __shfl_sync(0xffffffffu, b0, 31) + xs - c;
                for (uint32_t y = wv; y; y &= y - 1) {
                  const uint32_t p = wi * 32u + (uint32_t)(__ffs(y) - 1);
                  kbuf[b0++] = ((uint64_t)(nd.lidf[p] & LID_MASK) << 32) | p;
                }
              }
            }
            __syncthreads();
            const uint32_t npv = sm.n_piv;
            if (!whole && npv) {
              const uint64_t T = radix_select<RT>(kbuf, npv, r2, sm.b);
              uint32_t tk = 0;
              for (uint32_t i = threadIdx.x; i < npv; i += RT) {
                const uint64_t kv = kbuf[i];
                if (kv < T) continue;
                const uint32_t p = (uint32_t)kv;
                atomicAnd(&alive[p >> 5], ~(1u << (p & 31)));
                atomicSub(&cnt[nd.u_of[p] & UMASK], 1u);
                vc((uint32_t)(kv >> 32));
                ++tk;
              }
              if (prot_piv) vc.np += tk;
            }
            __syncthreads();
          }
        }
        const uint32_t nv = block_reduce<RT, uint32_t>(vc.n, Add(), sm.b.u32);
        const uint32_t np = block_reduce<RT, uint32_t>(vc.np, Add(), sm.b.u32);
        hash += vc.hash;
        if (nv != k) bad = 1;
        S -= nv;
        c_ev += nv; c_prot += aeg ? np : 0; c_evev += 1;  // uniform
      }
      // ---- R4: the last record of each block in the epoch re-enters the index ----
      __syncthreads();
      if (threadIdx.x == 0) sm.n_app = 0;
      for (uint64_t wb = (P0 & ~31ull) + (uint64_t)wid * 32u; wb < P1; wb += RT) {
        const uint64_t pb = wb + lane;
        const bool in = pb >= P0 && pb < P1;
        uint32_t q = 0, lid = 0;
        bool last = false;
        if (in) {
          q = nd.nxt[pb];
          last = (uint64_t)q >= P1;  // INF included
          if (last) { lid = nd.lidf[pb] & LID_MASK; res_pos[lid] = (uint32_t)pb; }
        }
        if (belady) {
          if (last && q == INF32) hb_set(dead, lid);
          hb_update_warp(pend, last && q != INF32, q, true);
        } else {
          const uint32_t wv = __ballot_sync(0xffffffffu, last);
          if (lane == 0 && wv) atomicOr(&alive[wb >> 5], wv);
          const uint32_t u = in ? (nd.u_of[pb] & UMASK) : 0u;
          const uint32_t lm = __ballot_sync(0xffffffffu, last);
          if (last) {
            const uint32_t pr = __match_any_sync(lm, u);
            if (lane == 31 - __clz(pr)) atomicAdd(&cnt[u], (uint32_t)__popc(pr));
          }
        }
      }
      S += nnew;
      // ---- live unit list: keep units with cnt > 0, append this epoch's units ----
      if (!belady) {
        __syncthreads();
        const uint32_t* L = lists[cur];
        uint32_t* L2 = lists[cur ^ 1];
        const uint32_t U0 = nd.ev_unit[j], U1 = nd.ev_unit[j + 1];
        const uint32_t tot = nL + (U1 - U0);
        for (uint32_t i = threadIdx.x; i < ((tot + 31) & ~31u); i += RT) {
          uint32_t u = 0;
          bool keep = false;
          if (i < tot) {
            u = i < nL ? L[i] : U0 + (i - nL);
            keep = cnt[u] != 0;
          }
          const uint32_t km = __ballot_sync(0xffffffffu, keep);
          uint32_t b0 = 0;
          if (lane == 0 && km) b0 = atomicAdd(&sm.n_app, (uint32_t)__popc(km));
          b0 = __shfl_sync(0xffffffffu, b0, 0);
          if (keep) L2[b0 + __popc(km & ((1u << lane) - 1u))] = u;
        }
        __syncthreads();
        nL = sm.n_app;
        cur ^= 1;
      }
      c_peak = max(c_peak, (long long)S);
      c_events += 1;
    }
    // ---- counters ----
    __syncthreads();
    {
      unsigned long long* sc = reinterpret_cast<unsigned long long*>(s_ctr);
      atomicAdd(&sc[SAGA_C_HITS], (unsigned long long)c_hit);
      atomicAdd(&sc[SAGA_C_MISSES], (unsigned long long)c_miss);
      atomicAdd(&sc[SAGA_C_MIG_HITS], (unsigned long long)c_mhit);
      atomicAdd(&sc[SAGA_C_MIG_MISSES], (unsigned long long)c_mmiss);
      atomicAdd(&sc[SAGA_C_COMPULSORY], (unsigned long long)c_comp);
      atomicAdd(&sc[SAGA_C_REGEN_TOKENS], (unsigned long long)c_regen);
      atomicAdd(&sc[SAGA_C_VICTIM_HASH], hash);
    }
    if (bad) atomicOr(a.err, 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t* out = a.counters + (((uint64_t)pi * a.n_caps + ci) * a.n_nodes_total + w) * SAGA_NCOUNT;
      const long long rg = s_ctr[SAGA_C_REGEN_TOKENS];
      out[SAGA_C_ACCESSES] = s_ctr[SAGA_C_HITS] + s_ctr[SAGA_C_MISSES] + s_ctr[SAGA_C_MIG_HITS] + s_ctr[SAGA_C_MIG_MISSES];
      out[SAGA_C_HITS] = s_ctr[SAGA_C_HITS];
      out[SAGA_C_MISSES] = s_ctr[SAGA_C_MISSES];
      out[SAGA_C_MIG_HITS] = s_ctr[SAGA_C_MIG_HITS];
      out[SAGA_C_MIG_MISSES] = s_ctr[SAGA_C_MIG_MISSES];
      out[SAGA_C_COMPULSORY] = s_ctr[SAGA_C_COMPULSORY];
      out[SAGA_C_INVALIDATED] = c_inv;
      out[SAGA_C_EVICTIONS] = c_ev;
      out[SAGA_C_EVICT_PROTECTED] = c_prot;
      out[SAGA_C_EVICT_EVENTS] = c_evev;
      out[SAGA_C_REGEN_TOKENS] = rg * (long long)v.btok;
      out[SAGA_C_REGEN_US] = rg * ((long long)v.btok * 1000000 / (long long)v.prefill_tok_s);
      out[SAGA_C_VICTIM_HASH] = s_ctr[SAGA_C_VICTIM_HASH];
      out[SAGA_C_INFEASIBLE_EPOCH] = infeasible;
      out[SAGA_C_PEAK_RESIDENT] = c_peak;
      out[SAGA_C_EVENT_EPOCHS] = c_events;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// replay index of a node (built once): event positions, units, session-update ranges
// ------------------------------------------------------------------------------------------
__global__ void k_ev_pos(const uint64_t* g_pos, const uint32_t* ev_g, uint32_t J, uint64_t* ev_pos) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= J; j += gridDim.x * blockDim.x) ev_pos[j] = g_pos[ev_g[j]];
}

// unit heads: first position of a non-empty record group, or an owner change
__global__ void k_unit_head(const uint32_t* lidf, const uint32_t* lown, uint64_t N, uint32_t* head) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (uint64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || lown[lidf[p] & LID_MASK] != lown[lidf[p - 1] & LID_MASK]) ? 1u : 0u;
}
__global__ void k_group_head(const uint64_t* g_pos, uint32_t G, uint32_t* head) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x)
    if (g_pos[g] < g_pos[g + 1]) head[g_pos[g]] = 1u;
}
// hpos = exclusive scan of head: unit of p = hpos[p+1] - 1
__global__ void k_unit_fill(const uint32_t* head, const uint32_t* hpos, uint64_t N, const uint32_t* lidf,
                            const uint32_t* lown, const uint64_t* g_pos, uint32_t G, const int64_t* g_t,
                            const uint32_t* g_kind, uint32_t* u_pos, int64_t* u_t, uint32_t* u_own, uint32_t* u_kind) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (uint64_t)gridDim.x * blockDim.x) {
    if (!head[p]) continue;
    const uint32_t u = hpos[p];
    uint32_t lo = 0, hi = G;  // last group with g_pos[g] <= p
    while (lo + 1 < hi) { const uint32_t mid = (lo + hi) >> 1; if (g_pos[mid] <= p) lo = mid; else hi = mid; }
    u_pos[u] = (uint32_t)p;
    u_t[u] = g_t[lo];
    u_own[u] = lown[lidf[p] & LID_MASK];
    u_kind[u] = g_kind[lo];
  }
}
__global__ void k_unit_of(const uint32_t* hpos, uint64_t N, const uint32_t* u_kind, uint32_t* u_of) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = hpos[p + 1] - 1;
    u_of[p] = u | (u_kind[u] ? KIND_MIG : 0u);
  }
}
__global__ void k_ev_index(TraceView v, const uint64_t* ev_pos, const uint32_t* ev_e, uint32_t J, const uint32_t* hpos,
                           uint64_t N, uint32_t n_units, const uint32_t* upd_c, uint32_t n_upd, uint32_t* ev_unit,
                           uint32_t* ev_upd, uint32_t* u_pos, uint64_t* N_out_unused, uint32_t* max_ev_units) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= J; j += gridDim.x * blockDim.x) {
    const uint64_t p = ev_pos[j];
    ev_unit[j] = p < N ? hpos[p] : n_units;
    if (j < J) {
      const uint32_t e = ev_e[j];
      uint32_t lo = 0, hi = n_upd;  // #updates with e(c) <= e
      while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (v.ecall[upd_c[mid]] <= e) lo = mid + 1; else hi = mid; }
      ev_upd[j] = lo;
      const uint64_t p1 = ev_pos[j + 1];
      const uint32_t u1 = p1 < N ? hpos[p1] : n_units;
      atomicMax(max_ev_units, u1 - ev_unit[j]);
    }
    if (j == 0) u_pos[n_units] = (uint32_t)N;
  }
}

unsigned grid_for(uint64_t n, int threads = NTHREADS) {
  uint64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148u * 64u) g = 148u * 64u;
  return (unsigned)g;
}

saga_status build_replay_index(saga_trace* t, uint32_t w, cudaStream_t s) {
  NodeDev& nd = t->nodes[w];
  if (nd.rp_done) return SAGA_OK;
  const uint64_t N = nd.N;
  const uint32_t J = nd.J;
  uint32_t* head = nullptr;
  uint32_t* hpos = nullptr;
  uint32_t* u_kind = nullptr;
  uint32_t* dmax = nullptr;
  SAGA_CK(cudaMallocAsync((void**)&head, (N + 1) * 4, s));
  SAGA_CK(cudaMallocAsync((void**)&hpos, (N + 2) * 4, s));
  SAGA_CK(cudaMallocAsync((void**)&dmax, 4, s));
  SAGA_CK(cudaMemsetAsync(dmax, 0, 4, s));
  nd.ev_pos = dalloc<uint64_t>(t, size_t(J) + 1);
  nd.u_of = dalloc<uint32_t>(t, N);
  if (!nd.ev_pos || !nd.u_of) { set_error("out of device memory (replay index)"); return SAGA_ERR_OOM; }
  k_ev_pos<<<grid_for(size_t(J) + 1), NTHREADS, 0, s>>>(nd.g_pos, nd.ev_g, J, nd.ev_pos);
  count_launch();
  if (N > 0) {
    k_unit_head<<<grid_for(N), NTHREADS, 0, s>>>(nd.lidf, nd.lown, N, head);
    if (nd.G) k_group_head<<<grid_for(nd.G), NTHREADS, 0, s>>>(nd.g_pos, nd.G, head);
    count_launch(2);
  }
  SAGA_CK(scan_u32(t, head, hpos, N));
  uint32_t nu = 0;
  SAGA_CK(cudaMemcpyAsync(&nu, hpos + N, 4, cudaMemcpyDeviceToHost, s));
  SAGA_CK(cudaStreamSynchronize(s));
  nd.n_units = nu;
  // hpos[N] = n_units is read by k_unit_of as hpos[p + 1] for p = N - 1
  nd.u_pos = dalloc<uint32_t>(t, size_t(nu) + 1);
  nd.u_t = dalloc<int64_t>(t, nu);
  nd.u_own = dalloc<uint32_t>(t, nu);
  nd.ev_unit = dalloc<uint32_t>(t, size_t(J) + 1);
  nd.ev_upd = dalloc<uint32_t>(t, J);
  SAGA_CK(cudaMallocAsync((void**)&u_kind, (size_t(nu) + 1) * 4, s));
  if (!nd.u_pos || !nd.u_t || !nd.u_own || !nd.ev_unit || !nd.ev_upd) { set_error("out of device memory (replay index)"); return SAGA_ERR_OOM; }
  if (N > 0) {
    k_unit_fill<<<grid_for(N), NTHREADS, 0, s>>>(head, hpos, N, nd.lidf, nd.lown, nd.g_pos, nd.G, nd.g_t, nd.g_kind,
                                                 nd.u_pos, nd.u_t, nd.u_own, u_kind);
    k_unit_of<<<grid_for(N), NTHREADS, 0, s>>>(hpos, N, u_kind, nd.u_of);
    count_launch(2);
  }
  k_ev_index<<<grid_for(size_t(J) + 1), NTHREADS, 0, s>>>(t->v, nd.ev_pos, nd.ev_e, J, hpos, N, nu, nd.upd_c, nd.n_upd,
                                                          nd.ev_unit, nd.ev_upd, nd.u_pos, nullptr, dmax);
  count_launch();
  uint32_t hm = 0;
  SAGA_CK(cudaMemcpyAsync(&hm, dmax, 4, cudaMemcpyDeviceToHost, s));
  SAGA_CK_LAUNCH();
  SAGA_CK(cudaStreamSynchronize(s));
  nd.max_ev_units = hm;
  cudaFreeAsync(head, s);
  cudaFreeAsync(hpos, s);
  cudaFreeAsync(u_kind, s);
  cudaFreeAsync(dmax, s);
  nd.rp_done = true;
  return SAGA_OK;
}

}  // namespace

saga_status run_replay(saga_trace* t, const saga_replay_cfg* cfg, const uint32_t* caps, uint32_t n_caps,
                       const uint32_t* nodes, uint32_t n_owned, int64_t* counters, cudaStream_t s) {
  const TraceView& v = t->v;
  uint32_t pol[3], n_pol = 0;
  for (uint32_t p : {1u, 2u, 4u}) if (cfg->policy_mask & p) pol[n_pol++] = p;
  if (n_pol == 0 || n_caps == 0 || n_owned == 0) return SAGA_OK;
  if (n_caps > 0xFFFFu || n_owned > 0xFFFu) { set_error("saga_replay: at most 65535 capacities and 4095 nodes per call"); return SAGA_ERR_INVALID_ARG; }
  uint32_t cap_max = 0;
  for (uint32_t i = 0; i < n_caps; ++i) cap_max = std::max(cap_max, caps[i]);
  uint64_t max_local = 1, maxN = 1, max_units = 1;
  for (uint32_t i = 0; i < n_owned; ++i) {
    saga_status st = build_replay_index(t, nodes[i], s);
    if (st != SAGA_OK) return st;
    const NodeDev& nd = t->nodes[nodes[i]];
    max_local = std::max<uint64_t>(max_local, nd.n_local);
    maxN = std::max<uint64_t>(maxN, nd.N);
    max_units = std::max<uint64_t>(max_units, nd.n_units);
  }
  std::vector<NodeArr> hn(t->n_nodes);
  for (uint32_t w = 0; w < t->n_nodes; ++w) {
    const NodeDev& nd = t->nodes[w];
    NodeArr x{};
    x.N = nd.N; x.J = nd.J; x.n_local = nd.n_local; x.n_units = nd.n_units;
    x.ev_pos = nd.ev_pos; x.ev_e = nd.ev_e; x.ev_inv = nd.ev_inv; x.ev_act = nd.ev_act; x.ev_unit = nd.ev_unit;
    x.ev_upd = nd.ev_upd; x.inv_s = nd.inv_s; x.lidf = nd.lidf; x.nxt = nd.nxt; x.u_of = nd.u_of; x.u_pos = nd.u_pos;
    x.u_t = nd.u_t; x.u_own = nd.u_own; x.lid2gid = nd.lid2gid; x.upd_c = nd.upd_c;
    hn[w] = x;
  }
  // items, largest capacity first (the per-event cost grows with |S| <= C)
  std::vector<uint32_t> items;
  items.reserve(size_t(n_pol) * n_caps * n_owned);
  std::vector<uint32_t> corder(n_caps);
  for (uint32_t i = 0; i < n_caps; ++i) corder[i] = i;
  std::stable_sort(corder.begin(), corder.end(), [&](uint32_t x, uint32_t y) { return caps[x] > caps[y]; });
  for (uint32_t ci : corder)
    for (uint32_t pi = 0; pi < n_pol; ++pi)
      for (uint32_t ni = 0; ni < n_owned; ++ni) items.push_back((pi << 28) | (ci << 12) | ni);
  const uint32_t n_items = (uint32_t)items.size();
  // per-CTA scratch layout (all offsets 16-byte aligned)
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  const uint64_t n2N = std::max<uint64_t>(1, (maxN + (1u << 20) - 1) >> 20);
  const uint64_t n2L = std::max<uint64_t>(1, (max_local + (1u << 20) - 1) >> 20);
  ReplayArgs a{};
  uint64_t off = 0;
  a.o_res = off; off += al(max_local * 4 + 16);
  a.o_bits = off; off += al(n2N * 32768 * 4);
  a.o_c1 = off; off += al(n2N * 1024 * 4);
  a.o_c2 = off; off += al(n2N * 4);
  a.o_dbits = off; off += al(n2L * 32768 * 4);
  a.o_dc1 = off; off += al(n2L * 1024 * 4);
  a.o_dc2 = off; off += al(n2L * 4);
  a.o_cnt = off; off += al(max_units * 4);
  a.o_list0 = off; off += al(max_units * 4);
  a.o_list1 = off; off += al(max_units * 4);
  a.o_lkp = off; off += al(max_units * 4);
  a.o_kbuf = off; off += al(((uint64_t)cap_max + 1) * 8);
  a.o_sst = off; off += al((uint64_t)std::max(v.n_sessions, 1u) * 4);
  a.cta_bytes = off;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_replay, RT, 0);
  uint32_t grid = std::min<uint32_t>(n_items, (uint32_t)nsm * (uint32_t)std::max(occ, 1));
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const uint64_t budget = free_b > (4ull << 30) ? (free_b - (4ull << 30)) / 2 : free_b / 4;
  grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(grid, budget / std::max<uint64_t>(a.cta_bytes, 1)));
  NodeArr* d_nodes = nullptr;
  uint32_t *d_caps = nullptr, *d_list = nullptr, *d_items = nullptr, *work = nullptr;
  uint8_t* scratch = nullptr;
  SAGA_CK(cudaMallocAsync((void**)&d_nodes, sizeof(NodeArr) * t->n_nodes, s));
  SAGA_CK(cudaMallocAsync((void**)&d_caps, 4 * n_caps, s));
  SAGA_CK(cudaMallocAsync((void**)&d_list, 4 * n_owned, s));
  SAGA_CK(cudaMallocAsync((void**)&d_items, 4 * n_items, s));
  SAGA_CK(cudaMallocAsync((void**)&work, 8, s));
  if (cudaMallocAsync((void**)&scratch, a.cta_bytes * grid, s) != cudaSuccess) {
    set_error("out of device memory (replay scratch %llu bytes)", (unsigned long long)(a.cta_bytes * grid));
    return SAGA_ERR_OOM;
  }
  SAGA_CK(cudaMemcpyAsync(d_nodes, hn.data(), sizeof(NodeArr) * t->n_nodes, cudaMemcpyHostToDevice, s));
  SAGA_CK(cudaMemcpyAsync(d_caps, caps, 4 * n_caps, cudaMemcpyHostToDevice, s));
  SAGA_CK(cudaMemcpyAsync(d_list, nodes, 4 * n_owned, cudaMemcpyHostToDevice, s));
  SAGA_CK(cudaMemcpyAsync(d_items, items.data(), 4 * n_items, cudaMemcpyHostToDevice, s));
  SAGA_CK(cudaMemsetAsync(work, 0, 8, s));
  a.v = v;
  a.nodes = d_nodes; a.caps = d_caps; a.items = d_items; a.n_items = n_items; a.node_list = d_list;
  a.pol[0] = pol[0]; a.pol[1] = n_pol > 1 ? pol[1] : 0; a.pol[2] = n_pol > 2 ? pol[2] : 0;
  a.n_caps = n_caps; a.n_nodes_total = t->n_nodes; a.counters = counters;
  a.alpha = cfg->alpha; a.beta = cfg->beta; a.gamma = cfg->gamma;
  a.p_low = cfg->p_low_pm; a.p_high = cfg->p_high_pm; a.ttl_max = cfg->ttl_max_us;
  a.scratch = scratch; a.work = work; a.err = work + 1;
  prof_begin(SAGA_PROF_REPLAY, s);
  k_replay<<<grid, RT, 0, s>>>(a);
  prof_end(SAGA_PROF_REPLAY, s);
  count_launch();
  SAGA_CK_LAUNCH();
  uint32_t herr = 0;
  SAGA_CK(cudaMemcpyAsync(&herr, work + 1, 4, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(d_nodes, s); cudaFreeAsync(d_caps, s); cudaFreeAsync(d_list, s); cudaFreeAsync(d_items, s);
  cudaFreeAsync(scratch, s);
  cudaFreeAsync(work, s);
  SAGA_CK(cudaStreamSynchronize(s));
  if (herr) { set_error("saga_replay: internal selection check failed"); return SAGA_ERR_STATE; }
  return SAGA_OK;
}

}  // namespace saga
