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
  uint64_t o_res, o_bits, o_c1, o_dbits, o_dc1, o_cnt, o_list0, o_list1, o_lkp, o_kbuf, o_vl, o_sst;
  uint32_t n2N_max, n2L_max;   // c2 entries of the two bitmaps (dynamic shared memory)
  uint32_t dyn_c1;             // the c1 arrays are in dynamic shared memory too
  uint32_t dyn_words;          // dynamic shared memory size in 32-bit words
  unsigned long long* item_cyc;  // optional per-item SM cycles (SAGA_REPLAY_TRACE)
  uint32_t* work;
  uint32_t* err;
};

struct Smem {
  BlockScratch<RT> b;
  uint32_t hist[H1];
  uint32_t res_j, res_rem, thr, item;
  uint32_t hb_j2, hb_j1;
  uint32_t n_app, n_piv, n_vict;
  uint32_t ilo, ihi;
  uint32_t tot_dead, tot_pend;  // BELADY: set bits of the two hierarchical bitmaps
};

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// arr[lo..hi) scanned from hi-1 downwards: j with sum(arr[j+1..hi)) < k <= sum(arr[j..hi)) and
// rem = k - sum(arr[j+1..hi)).  Requires 1 <= k <= sum(arr[lo..hi)).  Block-wide; each thread
// takes IT consecutive entries per round, so up to RT*IT entries cost one collective.
template <int IT>
__device__ void find_level(const uint32_t* arr, uint32_t lo, uint32_t hi, uint32_t k, uint32_t& j, uint32_t& rem,
                           Smem& sm, Par& par) {
  uint32_t carry = 0;
  const uint32_t n = hi - lo;
  for (uint32_t base = 0; base < n; base += RT * IT) {
    uint32_t val[IT], sum = 0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const uint32_t t = base + threadIdx.x * IT + i;
      val[i] = t < n ? arr[hi - 1 - t] : 0u;
      sum += val[i];
    }
    uint32_t tot;
    const uint32_t ex = block_excl_scan<RT>(sum, &tot, sm.b, par);
    uint32_t c = carry + ex;
    if (c < k && k <= c + sum) {
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        if (c < k && k <= c + val[i]) { sm.res_j = hi - 1 - (base + threadIdx.x * IT + i); sm.res_rem = k - c; }
        c += val[i];
      }
    }
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

// Warp-collective (all lanes call): each lane appends idx(b) | tag for every set bit b of
// `bits` (bit b of word wi is index wi * 32 + b) to the victim list.
__device__ __forceinline__ void emit_bits(uint32_t* vlist, uint32_t* n_vict, uint32_t wi, uint32_t bits, uint32_t tag) {
  const int lane = threadIdx.x & 31;
  const uint32_t c = __popc(bits);
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
  if (tot == 0) return;
  uint32_t b0 = 0;
  if (lane == 31) b0 = atomicAdd(n_vict, tot);
  b0 = __shfl_sync(0xffffffffu, b0, 31) + x - c;
  for (uint32_t y = bits; y; y &= y - 1) vlist[b0++] = (wi * 32u + (uint32_t)(__ffs(y) - 1)) | tag;
}

// take (clear and list) every set bit with index >= T, starting at c1 block j1 of c2 block j2
__device__ void hb_take_from(const HB& h, uint32_t j2, uint32_t j1, uint32_t T, uint32_t* vlist, uint32_t* n_vict,
                             uint32_t tag) {
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
        if (tk) h.bits[wi] = wv & ~m;
        emit_bits(vlist, n_vict, wi, tk, tag);
        const uint32_t n = warp_sum(__popc(tk));
        if (lane == 0 && n) { h.c1[c1i] -= n; atomicSub(&h.c2[jb], n); }
      }
    }
  }
}

// take the k highest set bits (1 <= k <= total).  The threshold is found by warp 0 alone
// (c2 level, then the 1024 c1 entries of the pivot c2 block as 32 lanes x 32, then 32 words).
__device__ void hb_take_top(const HB& h, uint32_t k, uint32_t* vlist, uint32_t tag, Smem& sm) {
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    // c2 level
    uint32_t carry = 0, j2 = 0, r2 = 0;
    for (uint32_t base = 0; base < h.n2; base += 32) {
      const uint32_t idx = h.n2 - 1 - (base + lane);
      const uint32_t v = base + lane < h.n2 ? h.c2[idx] : 0u;
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      const uint32_t hit = __ballot_sync(0xffffffffu, carry + x - v < k && k <= carry + x);
      if (hit) {
        const int l = __ffs(hit) - 1;
        j2 = __shfl_sync(0xffffffffu, idx, l);
        r2 = k - __shfl_sync(0xffffffffu, carry + x - v, l);
        break;
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    // c1 level: lane l owns entries [top - 32 l - 31, top - 32 l] of block j2
    const uint32_t b0 = j2 * 1024u + 1024u - 32u * (lane + 1);
    const uint4* c4 = reinterpret_cast<const uint4*>(h.c1 + b0);
    uint32_t e[32], sum = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 t = c4[q];
      e[4 * q] = t.x; e[4 * q + 1] = t.y; e[4 * q + 2] = t.z; e[4 * q + 3] = t.w;
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) sum += e[q];
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    const uint32_t hit = __ballot_sync(0xffffffffu, x - sum < r2 && r2 <= x);
    const int L = __ffs(hit) - 1;
    uint32_t j1 = 0, r1 = 0;
    if ((int)lane == L) {
      uint32_t c = x - sum;
#pragma unroll
      for (int q = 31; q >= 0; --q) {
        if (c < r2 && r2 <= c + e[q]) { j1 = b0 + (uint32_t)q; r1 = r2 - c; }
        c += e[q];
      }
    }
    j1 = __shfl_sync(0xffffffffu, j1, L);
    r1 = __shfl_sync(0xffffffffu, r1, L);
    // word level
    const uint32_t wi = j1 * 32u + (31u - lane);  // lane 0 = highest word of the block
    const uint32_t wv = h.bits[wi];
    const uint32_t cw = __popc(wv);
    uint32_t xw = cw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xw, o);
      if (lane >= (uint32_t)o) xw += y;
    }
    if (xw - cw < r1 && r1 <= xw) {
      uint32_t need = r1 - (xw - cw), w2 = wv;
      int b = 31 - __clz(w2);
      while (--need) { w2 &= ~(1u << b); b = 31 - __clz(w2); }
      sm.thr = wi * 32u + (uint32_t)b;
      sm.hb_j2 = j2;
      sm.hb_j1 = j1;
    }
  }
  __syncthreads();
  hb_take_from(h, sm.hb_j2, sm.hb_j1, sm.thr, vlist, &sm.n_vict, tag);
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

constexpr uint32_t VT_LID = 0x80000000u;  // victim-list tag: the entry is a local id, else a position
constexpr int UNR = 4;                    // record chunks whose loads are issued together (R2 / R4)

__global__ void __launch_bounds__(RT) k_replay(ReplayArgs a) {
  __shared__ Smem sm;
  __shared__ long long s_ctr[SAGA_NCOUNT];
  extern __shared__ __align__(16) uint32_t dyn[];  // c2 (+ c1) counts / AEG unit counts
  Par par;
  const TraceView& v = a.v;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* base = a.scratch + (uint64_t)blockIdx.x * a.cta_bytes;
  uint32_t* res_pos = reinterpret_cast<uint32_t*>(base + a.o_res);
  uint32_t* alive = reinterpret_cast<uint32_t*>(base + a.o_bits);   // AEG / EVICT_ALL (aliases pend.bits)
  uint32_t* lists[2] = {reinterpret_cast<uint32_t*>(base + a.o_list0), reinterpret_cast<uint32_t*>(base + a.o_list1)};
  uint32_t* lkp = reinterpret_cast<uint32_t*>(base + a.o_lkp);
  uint64_t* kbuf = reinterpret_cast<uint64_t*>(base + a.o_kbuf);
  uint32_t* vlist = reinterpret_cast<uint32_t*>(base + a.o_vl);
  uint32_t* sstate = reinterpret_cast<uint32_t*>(base + a.o_sst);

  while (true) {
    if (threadIdx.x == 0) sm.item = atomicAdd(a.work, 1u);
    __syncthreads();
    const uint32_t it = sm.item;
    __syncthreads();
    if (it >= a.n_items) break;
    const long long t_start = clock64();
    const uint32_t packed = a.items[it];
    const uint32_t pi = packed >> 28, ci = (packed >> 12) & 0xFFFFu, ni = packed & 0xFFFu;
    const uint32_t pol = a.pol[pi];
    const uint32_t C = a.caps[ci];
    const uint32_t w = a.node_list[ni];
    const NodeArr nd = a.nodes[w];
    const bool belady = pol == SAGA_POLICY_BELADY;
    const bool aeg = pol == SAGA_POLICY_AEG;
    const uint32_t n2N = max(1u, (uint32_t)((nd.N + (1u << 20) - 1) >> 20));
    const uint32_t n2L = max(1u, (nd.n_local + (1u << 20) - 1) >> 20);
    // count arrays: c2 always in shared memory, c1 there too when it fits (a.dyn_c1)
    uint32_t* c2N = dyn;
    uint32_t* c2L = dyn + a.n2N_max;
    uint32_t* c1N = a.dyn_c1 ? dyn + ((a.n2N_max + a.n2L_max + 3u) & ~3u) : reinterpret_cast<uint32_t*>(base + a.o_c1);
    uint32_t* c1L = a.dyn_c1 ? c1N + a.n2N_max * 1024u : reinterpret_cast<uint32_t*>(base + a.o_dc1);
    HB pend{reinterpret_cast<uint32_t*>(base + a.o_bits), c1N, c2N, n2N};
    HB dead{reinterpret_cast<uint32_t*>(base + a.o_dbits), c1L, c2L, n2L};
    // AEG / EVICT_ALL unit counts: in shared memory when they fit
    uint32_t* cnt = (a.dyn_words >= nd.n_units) ? dyn : reinterpret_cast<uint32_t*>(base + a.o_cnt);
    // ---- reset the item state ----
    {
      const uint4 ones = make_uint4(NONE, NONE, NONE, NONE), zero = make_uint4(0, 0, 0, 0);
      uint4* r4 = reinterpret_cast<uint4*>(res_pos);
      for (uint32_t i = threadIdx.x; i < (nd.n_local + 3) / 4; i += RT) r4[i] = ones;
      uint4* b4 = reinterpret_cast<uint4*>(pend.bits);
      for (uint32_t i = threadIdx.x; i < n2N * 8192u; i += RT) b4[i] = zero;
      if (belady) {
        for (uint32_t i = threadIdx.x; i < n2N * 1024u; i += RT) c1N[i] = 0;
        for (uint32_t i = threadIdx.x; i < n2L * 1024u; i += RT) c1L[i] = 0;
        for (uint32_t i = threadIdx.x; i < a.n2N_max + a.n2L_max; i += RT) dyn[i] = 0;
        uint4* d4 = reinterpret_cast<uint4*>(dead.bits);
        for (uint32_t i = threadIdx.x; i < n2L * 8192u; i += RT) d4[i] = zero;
      } else {
        for (uint32_t i = threadIdx.x; i < nd.n_units; i += RT) cnt[i] = 0;
      }
      if (aeg) for (uint32_t i = threadIdx.x; i < v.n_sessions; i += RT) sstate[i] = 0;
      if (threadIdx.x < SAGA_NCOUNT) s_ctr[threadIdx.x] = 0;
      if (threadIdx.x == 0) { sm.tot_dead = 0; sm.tot_pend = 0; }
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
            if (q == INF32) { hb_clear(dead, l); atomicSub(&sm.tot_dead, 1u); }
            else { hb_clear(pend, q); atomicSub(&sm.tot_pend, 1u); }
          } else {
            atomicAnd(&alive[p >> 5], ~(1u << (p & 31)));
            atomicSub(&cnt[nd.u_of[p] & UMASK], 1u);
          }
        }
        nrm = block_reduce<RT, uint32_t>(nrm, Add(), sm.b, par);
        S -= nrm;
        c_inv += nrm;  // uniform
      }
      if (j + 1 == nd.J) break;  // sentinel: trailing invalidations only
      const uint64_t P0 = nd.ev_pos[j], P1 = nd.ev_pos[j + 1];
      if (P0 == P1) continue;    // only empty record groups (the oracle skips the epoch)
      __syncthreads();
      if (threadIdx.x == 0) sm.n_vict = 0;
      // ---- R2: |A|, new = |A \ S|; hits / misses; in-flight blocks leave the index ----
      uint32_t nA = 0, nnew = 0;
      uint32_t t_hit = 0, t_miss = 0, t_mhit = 0, t_mmiss = 0, t_comp = 0, t_regen = 0;
      for (uint64_t wb = (P0 & ~31ull) + (uint64_t)wid * 32u; wb < P1; wb += (uint64_t)RT * UNR) {
        uint32_t lf[UNR], uo[UNR], rp[UNR];
        bool in[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint64_t pb = wb + (uint64_t)u * RT + lane;
          in[u] = pb >= P0 && pb < P1;
          lf[u] = in[u] ? nd.lidf[pb] : 0u;
          uo[u] = in[u] ? nd.u_of[pb] : 0u;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) rp[u] = (in[u] && !(lf[u] & LID_NFIE)) ? res_pos[lf[u] & LID_MASK] : NONE;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const bool first = in[u] && !(lf[u] & LID_NFIE);
          const bool resident = first && rp[u] != NONE;
          const bool mig = (uo[u] & KIND_MIG) != 0;
          if (in[u]) {
            if (first && !resident) {
              ++nA; ++nnew;
              if (mig) ++t_mmiss; else { ++t_miss; if (!(lf[u] & LID_FTN)) ++t_regen; }
              if (lf[u] & LID_FTN) ++t_comp;
            } else {
              if (first) ++nA;
              if (mig) ++t_mhit; else ++t_hit;
            }
          }
          if (belady) {
            hb_update_warp(pend, resident, (uint32_t)(wb + (uint64_t)u * RT + lane), false);
          } else if (resident) {
            atomicAnd(&alive[rp[u] >> 5], ~(1u << (rp[u] & 31)));
            atomicSub(&cnt[nd.u_of[rp[u]] & UMASK], 1u);
          }
        }
      }
      {
        const unsigned long long pk = block_reduce<RT, unsigned long long>(
            ((unsigned long long)nA << 32) | nnew, Add(), sm.b, par);
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
        const uint64_t eh = (uint64_t)e << 32;
        unsigned long long hs = 0;
        uint32_t n_direct = 0, n_prot = 0;  // victims handled outside the list; protected victims
        if (belady) {
          // in-flight blocks left `pend` in R2 (their next use is this epoch)
          const uint32_t nd_ = sm.tot_dead, np_ = sm.tot_pend - inAS;
          if (k <= nd_) {
            hb_take_top(dead, k, vlist, VT_LID, sm);
          } else {
            if (nd_ > 0) hb_take_from(dead, 0, 0, 0, vlist, &sm.n_vict, VT_LID);
            if (k - nd_ <= np_) { __syncthreads(); hb_take_top(pend, k - nd_, vlist, 0u, sm); }
            else bad = 1;
          }
          if (threadIdx.x == 0) {
            sm.tot_dead = nd_ - min(k, nd_);
            sm.tot_pend = np_ - (k > nd_ ? k - nd_ : 0u);
          }
        } else {
          const uint32_t* L = lists[cur];
          // whole-unit eviction: list every resident latest position of unit u (warp-collective)
          auto evict_unit = [&](uint32_t u, bool prot) {
            const uint32_t pa = nd.u_pos[u], pe = nd.u_pos[u + 1];
            const uint32_t wlast = (pe - 1) >> 5;
            uint32_t taken = 0;
            for (uint32_t wb = pa >> 5; wb <= wlast; wb += 32) {
              const uint32_t wi = wb + lane;
              uint32_t wv = 0;
              if (wi <= wlast) {
                uint32_t m = 0xffffffffu;
                if (wi == (pa >> 5)) m &= ~((1u << (pa & 31)) - 1u);
                if (wi == wlast && (pe & 31)) m &= (1u << (pe & 31)) - 1u;
                wv = alive[wi] & m;
                if (wv) atomicAnd(&alive[wi], ~wv);
              }
              emit_bits(vlist, &sm.n_vict, wi, wv, 0u);
              taken += __popc(wv);
            }
            taken = warp_sum(taken);
            if (lane == 0) { cnt[u] -= taken; if (prot) n_prot += taken; }
          };
          if (!aeg) {  // EVICT_ALL: every candidate
            for (uint32_t i = wid; i < nL; i += RW) {
              const uint32_t u = L[i];
              if (cnt[u]) evict_unit(u, false);
            }
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
            tau = block_reduce<RT, long long>(tau, Max(), sm.b, par);
            smax = block_reduce<RT, uint32_t>(smax, Max(), sm.b, par);
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
            find_level<H1 / RT>(sm.hist, 0, H1, k, d1, r1, sm, par);
            for (uint32_t i = threadIdx.x; i < 1024; i += RT) sm.hist[i] = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < nL; i += RT) {
              const uint32_t kp = lkp[i];
              if ((((kp >> 31) << 11) | ((kp & 0x1FFFFFu) >> 10)) != d1) continue;
              const uint32_t c = cnt[L[i]];
              if (c) atomicAdd(&sm.hist[kp & 1023u], c);
            }
            __syncthreads();
            find_level<1024 / RT>(sm.hist, 0, 1024, r1, d2, r2, sm, par);
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
                for (uint32_t y = wv; y; y &= y - 1) kbuf[b0++] = wi * 32u + (uint32_t)(__ffs(y) - 1);
              }
            }
            __syncthreads();
            const uint32_t npv = sm.n_piv;
            if (!whole && npv) {
              // pivot keys differ only in lid: rank (lid << 32 | position) and keep the top r2
              for (uint32_t i = threadIdx.x; i < npv; i += RT) {
                const uint32_t p = (uint32_t)kbuf[i];
                kbuf[i] = ((uint64_t)(nd.lidf[p] & LID_MASK) << 32) | p;
              }
              __syncthreads();
              const uint64_t T = radix_select<RT>(kbuf, npv, r2, sm.b, par);
              uint32_t tk = 0;
              for (uint32_t i = threadIdx.x; i < npv; i += RT) {
                const uint64_t kv = kbuf[i];
                if (kv < T) continue;
                const uint32_t p = (uint32_t)kv, lid = (uint32_t)(kv >> 32);
                atomicAnd(&alive[p >> 5], ~(1u << (p & 31)));
                atomicSub(&cnt[nd.u_of[p] & UMASK], 1u);
                res_pos[lid] = NONE;
                hs += splitmix64(eh | lid);
                ++tk;
              }
              n_direct += tk;
              if (prot_piv) n_prot += tk;
            }
          }
        }
        __syncthreads();
        // listed victims: positions (block at that position) or local ids (VT_LID)
        const uint32_t nvl = sm.n_vict;
        for (uint32_t i = threadIdx.x; i < nvl; i += RT) {
          const uint32_t x = vlist[i];
          const uint32_t lid = (x & VT_LID) ? (x & ~VT_LID) : (nd.lidf[x] & LID_MASK);
          res_pos[lid] = NONE;
          hs += splitmix64(eh | lid);
        }
        const unsigned long long nvp = block_reduce<RT, unsigned long long>(
            ((unsigned long long)n_direct << 32) | n_prot, Add(), sm.b, par);
        const uint32_t nv = nvl + (uint32_t)(nvp >> 32), np = (uint32_t)nvp;
        hash += hs;
        if (nv != k) bad = 1;
        S -= nv;
        c_ev += nv; c_prot += aeg ? np : 0; c_evev += 1;  // uniform
      }
      // ---- R4: the last record of each block in the epoch re-enters the index ----
      __syncthreads();
      if (threadIdx.x == 0) {
        sm.n_app = 0;
        if (belady && kk <= 0) atomicSub(&sm.tot_pend, inAS);  // (R3 already accounted for it)
      }
      for (uint64_t wb = (P0 & ~31ull) + (uint64_t)wid * 32u; wb < P1; wb += (uint64_t)RT * UNR) {
        uint32_t q[UNR], lf[UNR], uo[UNR];
        bool last[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint64_t pb = wb + (uint64_t)u * RT + lane;
          const bool in = pb >= P0 && pb < P1;
          q[u] = in ? nd.nxt[pb] : 0u;
          lf[u] = in ? nd.lidf[pb] : 0u;
          uo[u] = (in && !belady) ? nd.u_of[pb] : 0u;
          last[u] = in && (uint64_t)q[u] >= P1;  // INF included
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint64_t pb = wb + (uint64_t)u * RT + lane;
          const uint32_t lid = lf[u] & LID_MASK;
          if (last[u]) res_pos[lid] = (uint32_t)pb;
          if (belady) {
            if (last[u] && q[u] == INF32) hb_set(dead, lid);
            hb_update_warp(pend, last[u] && q[u] != INF32, q[u], true);
            const uint32_t md = __ballot_sync(0xffffffffu, last[u] && q[u] == INF32);
            const uint32_t mp = __ballot_sync(0xffffffffu, last[u] && q[u] != INF32);
            if (lane == 0 && (md | mp)) { atomicAdd(&sm.tot_dead, __popc(md)); atomicAdd(&sm.tot_pend, __popc(mp)); }
          } else {
            const uint32_t wv = __ballot_sync(0xffffffffu, last[u]);
            if (lane == 0 && wv) atomicOr(&alive[(wb + (uint64_t)u * RT) >> 5], wv);
            const uint32_t un = uo[u] & UMASK;
            if (last[u]) {
              const uint32_t pr = __match_any_sync(wv, un);
              if (lane == 31 - __clz(pr)) atomicAdd(&cnt[un], (uint32_t)__popc(pr));
            }
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
      if (a.item_cyc) a.item_cyc[it] = (unsigned long long)(clock64() - t_start);
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
  SAGA_CK(ws_malloc((void**)&head, (N + 1) * 4, s));
  SAGA_CK(ws_malloc((void**)&hpos, (N + 2) * 4, s));
  SAGA_CK(ws_malloc((void**)&dmax, 4, s));
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
  SAGA_CK(ws_malloc((void**)&u_kind, (size_t(nu) + 1) * 4, s));
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
  ws_free(head, s);
  ws_free(hpos, s);
  ws_free(u_kind, s);
  ws_free(dmax, s);
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
  // per-CTA scratch layout (all offsets 256-byte aligned)
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  const uint64_t n2N = std::max<uint64_t>(1, (maxN + (1u << 20) - 1) >> 20);
  const uint64_t n2L = std::max<uint64_t>(1, (max_local + (1u << 20) - 1) >> 20);
  ReplayArgs a{};
  uint64_t off = 0;
  a.o_res = off; off += al(max_local * 4 + 16);
  a.o_bits = off; off += al(n2N * 32768 * 4);
  a.o_c1 = off; off += al(n2N * 1024 * 4);
  a.o_dbits = off; off += al(n2L * 32768 * 4);
  a.o_dc1 = off; off += al(n2L * 1024 * 4);
  a.o_cnt = off; off += al(max_units * 4);
  a.o_list0 = off; off += al(max_units * 4);
  a.o_list1 = off; off += al(max_units * 4);
  a.o_lkp = off; off += al(max_units * 4);
  a.o_kbuf = off; off += al(((uint64_t)cap_max + 1) * 8);
  a.o_vl = off; off += al(((uint64_t)cap_max + 1) * 4);
  a.o_sst = off; off += al((uint64_t)std::max(v.n_sessions, 1u) * 4);
  a.cta_bytes = off;
  // dynamic shared memory: the c2 counts always; the c1 counts (BELADY) and the unit counts
  // (AEG / EVICT_ALL; same region) when they fit
  const uint64_t dyn_max = 160ull * 1024;
  const uint64_t c2_bytes = ((n2N + n2L + 3) & ~3ull) * 4;
  const uint64_t c1_bytes = (n2N + n2L) * 1024 * 4;
  a.n2N_max = (uint32_t)n2N; a.n2L_max = (uint32_t)n2L;
  a.dyn_c1 = (c2_bytes + c1_bytes <= dyn_max) ? 1u : 0u;
  uint64_t dyn = std::max<uint64_t>(a.dyn_c1 ? c2_bytes + c1_bytes : c2_bytes, std::min<uint64_t>(max_units * 4, dyn_max));
  dyn = (dyn + 15) & ~15ull;
  a.dyn_words = (uint32_t)(dyn / 4);
  SAGA_CK(cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_replay, RT, (size_t)dyn);
  uint32_t grid = std::min<uint32_t>(n_items, (uint32_t)nsm * (uint32_t)std::max(occ, 1));
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const uint64_t budget = free_b > (4ull << 30) ? (free_b - (4ull << 30)) / 2 : free_b / 4;
  grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(grid, budget / std::max<uint64_t>(a.cta_bytes, 1)));
  const bool trace = getenv("SAGA_REPLAY_TRACE") != nullptr;
  NodeArr* d_nodes = nullptr;
  uint32_t *d_caps = nullptr, *d_list = nullptr, *d_items = nullptr, *work = nullptr;
  unsigned long long* d_cyc = nullptr;
  uint8_t* scratch = nullptr;
  SAGA_CK(ws_malloc((void**)&d_nodes, sizeof(NodeArr) * t->n_nodes, s));
  SAGA_CK(ws_malloc((void**)&d_caps, 4 * n_caps, s));
  SAGA_CK(ws_malloc((void**)&d_list, 4 * n_owned, s));
  SAGA_CK(ws_malloc((void**)&d_items, 4 * n_items, s));
  SAGA_CK(ws_malloc((void**)&work, 8, s));
  if (trace) SAGA_CK(ws_malloc((void**)&d_cyc, 8ull * n_items, s));
  if (ws_malloc((void**)&scratch, a.cta_bytes * grid, s) != cudaSuccess) {
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
  a.scratch = scratch; a.work = work; a.err = work + 1; a.item_cyc = d_cyc;
  prof_begin(SAGA_PROF_REPLAY, s);
  k_replay<<<grid, RT, dyn, s>>>(a);
  prof_end(SAGA_PROF_REPLAY, s);
  count_launch();
  SAGA_CK_LAUNCH();
  uint32_t herr = 0;
  SAGA_CK(cudaMemcpyAsync(&herr, work + 1, 4, cudaMemcpyDeviceToHost, s));
  std::vector<unsigned long long> cyc(trace ? n_items : 0);
  if (trace) SAGA_CK(cudaMemcpyAsync(cyc.data(), d_cyc, 8ull * n_items, cudaMemcpyDeviceToHost, s));
  ws_free(d_nodes, s); ws_free(d_caps, s); ws_free(d_list, s); ws_free(d_items, s);
  ws_free(scratch, s);
  ws_free(work, s);
  if (d_cyc) ws_free(d_cyc, s);
  SAGA_CK(cudaStreamSynchronize(s));
  if (trace) {
    fprintf(stderr, "[saga replay] grid %u x %d threads, dyn smem %llu B (c1 %s), %u items\n", grid, RT,
            (unsigned long long)dyn, a.dyn_c1 ? "smem" : "global", n_items);
    for (uint32_t i = 0; i < n_items; ++i) {
      const uint32_t pk = items[i];
      const uint32_t w = nodes[pk & 0xFFFu];
      fprintf(stderr, "[saga replay] item pol=%u cap=%u node=%u events=%u Mcycles=%.2f\n", pol[pk >> 28],
              caps[(pk >> 12) & 0xFFFFu], w, t->nodes[w].J, cyc[i] / 1e6);
    }
  }
  if (herr) { set_error("saga_replay: internal selection check failed"); return SAGA_ERR_STATE; }
  return SAGA_OK;
}

}  // namespace saga
