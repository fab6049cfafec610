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

// CTA shape (overridable at build time for occupancy experiments: SAGA_NVCC_EXTRA="-DSAGA_REPLAY_RT=256 ...")
#ifndef SAGA_REPLAY_RT
#define SAGA_REPLAY_RT 512
#endif
#ifndef SAGA_REPLAY_MINB
#define SAGA_REPLAY_MINB 1
#endif
#ifndef SAGA_REPLAY_PF
#define SAGA_REPLAY_PF 2048
#endif
#ifndef SAGA_REPLAY_DYN_KB
#define SAGA_REPLAY_DYN_KB 64
#endif
#ifndef SAGA_REPLAY_ENTRY
#define SAGA_REPLAY_ENTRY run_replay
#define SAGA_REPLAY_IS_WIDE 0
#endif
constexpr int RT = SAGA_REPLAY_RT;
constexpr int RW = RT / 32;
constexpr uint32_t KIND_MIG = 0x80000000u;  // u_of bit 31: the position is a MIG record
constexpr uint32_t U_SHARED = 0x40000000u;  // u_of bit 30: the block is a shared-prefix block
constexpr uint32_t KIND_PF = 0x20000000u;   // u_of bit 29: the position is a PREFETCH record
constexpr uint32_t UMASK = 0x1FFFFFFFu;
// first-level key-part digit: !prot * 1025 + (q >> 10), q <= 2^20 (2050 values, kp order)
constexpr int H1 = 2560;
__device__ __forceinline__ uint32_t kp_digit(uint32_t kp) { return (kp >> 31) * 1025u + ((kp & 0x1FFFFFu) >> 10); }

// hierarchical bitmap; storage is allocated in whole c2 blocks (2^20 bits)
struct HB {
  uint32_t* bits;  // [n2 * 32768] words
  uint32_t* c1;    // [n2 * 1024]  set bits per 1024-bit block
  uint32_t* c2;    // [n2]         set bits per 2^20-bit block
  uint32_t n2;
};

constexpr uint32_t LO_SHARED = 0x80000000u;  // local owner tag: shared prefix of type (lo & ~LO_SHARED)

// static description of a unit (maximal run of one record group with one owner)
struct __align__(8) UnitRec {
  int64_t t;        // t_last of its blocks: t_c of the CALL group, T_e of a MIG group
  uint32_t pa, pe;  // positions [pa, pe)
  uint32_t lo;      // local owner id (private session) or LO_SHARED | type
  uint32_t flags;   // U_MONO: local ids strictly increase with position inside the unit
};
constexpr uint32_t U_MONO = 1u;
// live-list entry: the unit record plus the per-event key part
struct __align__(16) ListRec {
  int64_t t;
  uint32_t u, pa, pe, lo, kp, flags;
};
// per-call inputs of the WA-LRU key of a private session whose newest call is c
struct __align__(8) CallKey {
  int64_t tend;     // tool start (Alg. 1 elapsed-time origin)
  float P;          // P_reuse (eq:reuse with eq:overlap), fp32 pinned
  uint32_t size;    // ceil(n_cur / block_tokens) (eq:size numerator)
  uint32_t ttl;     // ttl_base of the call's AEG node (<= 1e9)
  uint32_t fin;     // is_last || terminal
};

struct NodeArr {
  uint64_t N;
  uint32_t J, n_local, n_units, n_lo;
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
  const uint32_t* prv;
  const uint32_t* upu;
  const UnitRec* urec;
  const uint32_t* lid2gid;
  const uint32_t* upd_c;
  const uint32_t* upd_lo;
};

struct ReplayArgs {
  TraceView v;
  const NodeArr* nodes;
  const uint32_t* caps;
  const uint32_t* items;  // packed (pi << 28) | (ci << 12) | node_list index, largest capacity first
  uint32_t n_items;
  const uint32_t* node_list;
  uint32_t pol[5];
  uint32_t n_caps;
  uint32_t n_nodes_total;
  int64_t* counters;
  float alpha, beta, gamma;
  uint32_t p_low, p_high;
  int64_t ttl_max;
  // per-CTA scratch (strides in elements)
  uint8_t* scratch;
  uint64_t cta_bytes;
  const CallKey* callkey;
  uint64_t o_res, o_nres, o_bits, o_c1, o_dbits, o_dc1, o_cnt, o_list0, o_list1, o_kbuf, o_vl, o_vu, o_ocall;
  uint32_t n2N_max, n2L_max;   // c2 entries of the two bitmaps (dynamic shared memory)
  uint32_t n2R_max;            // c2 entries of the LRU bitmap (2N domain for LRU + Prefix)
  uint32_t dyn_c1;             // BELADY: the c1 arrays are in dynamic shared memory too
  uint32_t dyn_dbits_words;    // BELADY: dead bits in shared memory when n_local <= 32 * this
  uint32_t dyn_words;          // dynamic shared memory size in 32-bit words
  uint32_t ocall_smem;         // AEG: newest-call table (n_lo words) in shared memory
  unsigned long long* item_cyc;  // optional per-item SM cycles (SAGA_REPLAY_TRACE)
  unsigned long long* phase_cyc; // optional [item][8] per-phase cycles of thread 0
  unsigned long long* vlog;      // optional victim log ((epoch << 32) | lid), saga_replay_victims
  unsigned long long* vlog_n;    // entries written (may exceed vlog_cap: the caller sees the need)
  unsigned long long vlog_cap;
  uint32_t* work;
  uint32_t* err;
  uint32_t* dbg;  // [4] first failed invariant
};

struct Smem {
  BlockScratch<RT> b;
  uint32_t hist[H1];
  uint32_t hist2[1024];  // second-level digit histogram (cleared with hist, no extra barrier)
  uint32_t res_j, res_rem, thr, item;
  uint32_t hb_j2, hb_j1, hb_r1;
  uint32_t n_app, n_piv, n_vict, n_vu, n_pu, pu_i;
  uint32_t ilo, ihi;
  uint32_t tot_dead, tot_pend;  // BELADY: set bits of the two hierarchical bitmaps
  __align__(8) uint64_t pbar[2];  // TMA prefetch stages of per-position arrays
};

// Per-position arrays of an epoch (lidf, u_of, nxt, prv, upu) are staged in shared memory by TMA
// bulk copies one epoch ahead: PF positions per array and stage, two stages.
constexpr uint32_t PF = SAGA_REPLAY_PF;
constexpr uint32_t NPA = 5;
constexpr uint32_t PF_WORDS = 2 * NPA * PF;

// first failed invariant of the launch: [0] = line, [1..3] = values (host reports it)
__device__ __forceinline__ void dbg_fail(uint32_t* dbg, uint32_t line, uint32_t x, uint32_t y, uint32_t z) {
  if (atomicCAS(&dbg[0], 0u, line) == 0u) { dbg[1] = x; dbg[2] = y; dbg[3] = z; }
}

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
// Grouping lanes by target word for one atomic per word: positions and local ids come in runs,
// so usually every active lane hits the same word -- one shuffle and one vote detect that and a
// single atomic carries the whole warp; otherwise each lane issues its own atomic (atomics
// commute: the result is the same; MATCH.ANY, which the general grouping needs, costs more than
// the handful of separate atomics of the rare mixed warp).
#ifndef SAGA_REPLAY_MATCH_ANY
// Warp-collective (all lanes call): lanes with `act` set (or clear) bit `idx` of `bits`.
__device__ __forceinline__ void warp_bits(uint32_t* bits, bool act, uint32_t idx, bool set) {
  const uint32_t am = __ballot_sync(0xffffffffu, act);
  if (!am) return;
  const uint32_t w = idx >> 5;
  const uint32_t w0 = __shfl_sync(0xffffffffu, w, __ffs(am) - 1);
  if (__all_sync(0xffffffffu, !act || w == w0)) {
    const uint32_t m = __reduce_or_sync(0xffffffffu, act ? 1u << (idx & 31) : 0u);
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(am) - 1)) {
      if (set) atomicOr(&bits[w0], m);
      else atomicAnd(&bits[w0], ~m);
    }
  } else if (act) {
    if (set) atomicOr(&bits[w], 1u << (idx & 31));
    else atomicAnd(&bits[w], ~(1u << (idx & 31)));
  }
}
// Warp-collective: lanes with `act` add (or subtract) 1 to counts[key].
__device__ __forceinline__ void warp_count(uint32_t* counts, bool act, uint32_t key, bool add) {
  const uint32_t am = __ballot_sync(0xffffffffu, act);
  if (!am) return;
  const uint32_t k0 = __shfl_sync(0xffffffffu, key, __ffs(am) - 1);
  if (__all_sync(0xffffffffu, !act || key == k0)) {
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(am) - 1)) {
      const uint32_t n = __popc(am);
      atomicAdd(&counts[k0], add ? n : (uint32_t)(-(int32_t)n));
    }
  } else if (act) {
    atomicAdd(&counts[key], add ? 1u : 0xFFFFFFFFu);
  }
}
// warp-collective update of a hierarchical bitmap: bits, then the c1 / c2 counts
__device__ __forceinline__ void hb_update_warp(const HB& h, bool act, uint32_t i, bool set) {
  const uint32_t am = __ballot_sync(0xffffffffu, act);
  if (!am) return;
  warp_bits(h.bits, act, i, set);
  const uint32_t c0 = __shfl_sync(0xffffffffu, i >> 10, __ffs(am) - 1);
  const uint32_t d = set ? 1u : 0xFFFFFFFFu;
  if (__all_sync(0xffffffffu, !act || (i >> 10) == c0)) {
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(am) - 1)) {
      const uint32_t n = __popc(am);
      atomicAdd(&h.c1[c0], set ? n : (uint32_t)(-(int32_t)n));
      atomicAdd(&h.c2[c0 >> 10], set ? n : (uint32_t)(-(int32_t)n));
    }
  } else if (act) {
    atomicAdd(&h.c1[i >> 10], d);
    atomicAdd(&h.c2[i >> 20], d);
  }
}
#else
// Warp-collective (all lanes call): lanes with `act` set (or clear) bit `idx` of `bits`; one
// atomic per distinct word (lanes usually hit few words: positions and local ids come in runs).
__device__ __forceinline__ void warp_bits(uint32_t* bits, bool act, uint32_t idx, bool set) {
  const uint32_t am = __ballot_sync(0xffffffffu, act);
  if (!act) return;
  const uint32_t w = idx >> 5;
  const uint32_t peers = __match_any_sync(am, w);
  const uint32_t m = __reduce_or_sync(peers, 1u << (idx & 31));
  if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) {
    if (set) atomicOr(&bits[w], m);
    else atomicAnd(&bits[w], ~m);
  }
}
// Warp-collective: lanes with `act` add (or subtract) 1 to counts[key]; one atomic per distinct key.
__device__ __forceinline__ void warp_count(uint32_t* counts, bool act, uint32_t key, bool add) {
  const uint32_t am = __ballot_sync(0xffffffffu, act);
  if (!act) return;
  const uint32_t peers = __match_any_sync(am, key);
  if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) {
    const uint32_t n = __popc(peers);
    atomicAdd(&counts[key], add ? n : (uint32_t)(-(int32_t)n));
  }
}
// warp-collective update of a hierarchical bitmap: bits, then the c1 / c2 counts
__device__ __forceinline__ void hb_update_warp(const HB& h, bool act, uint32_t i, bool set) {
  const uint32_t am = __ballot_sync(0xffffffffu, act);
  if (!am) return;
  warp_bits(h.bits, act, i, set);
  if (!act) return;
  const uint32_t p1 = __match_any_sync(am, i >> 10);
  if ((threadIdx.x & 31) == (uint32_t)(__ffs(p1) - 1)) {
    const uint32_t n = __popc(p1);
    atomicAdd(&h.c1[i >> 10], set ? n : (uint32_t)(-(int32_t)n));
    atomicAdd(&h.c2[i >> 20], set ? n : (uint32_t)(-(int32_t)n));
  }
}

#endif

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

#ifndef SAGA_HB_BATCH
#define SAGA_HB_BATCH 4
#endif
constexpr int HB_BATCH = SAGA_HB_BATCH;
// take (clear and list) the r1 highest set bits of c1 block j1 (r1 = NONE: all of them) and every
// set bit above that block, starting in c2 block j2.  Block j1's cut is found here from the words
// the take loads anyway (a suffix count over the warp, lane 31 = highest word), so the threshold
// search above stops at the c1 level and saves one dependent global round trip.
__device__ void hb_take_from(const HB& h, uint32_t j2, uint32_t j1, uint32_t r1, uint32_t* vlist, uint32_t* n_vict,
                             uint32_t tag) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t jb = j2; jb < h.n2; ++jb) {
    if (jb > j2 && h.c2[jb] == 0) continue;
    const uint32_t lo = (jb == j2) ? j1 : jb * 1024u, hi = jb * 1024u + 1024u;
    for (uint32_t i0 = lo + (uint32_t)wid * 32u; i0 < hi; i0 += RW * 32u) {
      const uint32_t ci = i0 + lane;
      const uint32_t cv = ci < hi ? h.c1[ci] : 0u;
      uint32_t nz = __ballot_sync(0xffffffffu, cv != 0);
      while (nz) {  // up to HB_BATCH non-empty c1 blocks at a time: their word loads are issued together
        uint32_t c1i[HB_BATCH], wv[HB_BATCH];
        int nb = 0;
#pragma unroll
        for (int b = 0; b < HB_BATCH; ++b) {
          c1i[b] = NONE;
          if (nz) { c1i[b] = i0 + (uint32_t)(__ffs(nz) - 1); nz &= nz - 1; ++nb; }
        }
#pragma unroll
        for (int b = 0; b < HB_BATCH; ++b) wv[b] = c1i[b] != NONE ? h.bits[c1i[b] * 32u + lane] : 0u;
#pragma unroll
        for (int b = 0; b < HB_BATCH; ++b) {
          if (b >= nb) break;
          const uint32_t wi = c1i[b] * 32u + lane;
          uint32_t tk = wv[b];
          if (c1i[b] == j1 && r1 != NONE) {  // keep all but the r1 highest set bits of the block
            const uint32_t c = __popc(tk);
            uint32_t xs = c;  // inclusive suffix count from lane 31 down
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_down_sync(0xffffffffu, xs, o);
              if (lane + o < 32) xs += y;
            }
            const uint32_t above = xs - c;  // set bits in higher words of the block
            if (above >= r1) tk = 0;
            else if (above + c > r1)
              for (uint32_t z = above + c - r1; z > 0; --z) tk &= tk - 1;  // the lowest bits stay
          }
          if (tk) h.bits[wi] = wv[b] & ~tk;
          emit_bits(vlist, n_vict, wi, tk, tag);
          const uint32_t n = warp_sum(__popc(tk));
          if (lane == 0 && n) { h.c1[c1i[b]] -= n; atomicSub(&h.c2[jb], n); }
        }
      }
    }
  }
}

// take the k highest set bits (1 <= k <= total).  The cut is found by warp 0 alone at the count
// levels (c2, then the 1024 c1 entries of the pivot c2 block as 32 lanes x 32); hb_take_from
// places it inside the pivot c1 block from the words it loads.
// (SAGA_REPLAY_TRACE: ph / ph_t non-null -> the threshold search's cycles go to phase slot 2)
__device__ void hb_take_top(const HB& h, uint32_t k, uint32_t* vlist, uint32_t tag, Smem& sm, uint32_t* dbg,
                            long long* ph = nullptr, long long* ph_t = nullptr) {
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    if (lane == 0) sm.thr = NONE;
    // c2 level
    uint32_t carry = 0, j2 = NONE, r2 = 0;
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
    if (j2 == NONE) { if (lane == 0) dbg_fail(dbg, __LINE__, k, carry, h.n2); goto done; }
    {
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
    if (!hit) { if (lane == 0) dbg_fail(dbg, __LINE__, k, r2, j2); goto done; }
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
    if (lane == 0) { sm.thr = 1u; sm.hb_j2 = j2; sm.hb_j1 = j1; sm.hb_r1 = r1; }
    }
  done:;
  }
  __syncthreads();
  if (ph && threadIdx.x == 0) { const long long t = clock64(); ph[2] += t - *ph_t; *ph_t = t; }
  if (sm.thr != NONE) hb_take_from(h, sm.hb_j2, sm.hb_j1, sm.hb_r1, vlist, &sm.n_vict, tag);
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (a[mid] < x) lo = mid + 1; else hi = mid; }
  return lo;
}

// owner inputs of the WA-LRU key at the current boundary (lo = local owner id or shared type)
__device__ __forceinline__ OwnerKeyIn owner_in(const TraceView& v, const CallKey* ck, const uint32_t* ocall, uint32_t lo,
                                               uint32_t act) {
  OwnerKeyIn r;
  if (lo & LO_SHARED) {
    const uint32_t t = lo & ~LO_SHARED;
    const bool on = (act >> t) & 1u;
    r.shared = true; r.prot_shared = on; r.size = __ldg(&v.tlen[t]); r.P = on ? 1.0f : 0.0f;
    r.fin = false; r.t_call = 0; r.ttl_base = 0;
    return r;
  }
  const uint32_t c1 = ocall[lo];
  const CallKey k = ck[c1 ? c1 - 1 : 0];
  r.shared = false; r.prot_shared = false;
  r.size = k.size; r.fin = k.fin != 0; r.P = k.P; r.t_call = k.tend; r.ttl_base = (int64_t)k.ttl;
  return r;
}

__device__ __forceinline__ uint32_t owner_size(const TraceView& v, const CallKey* ck, const uint32_t* ocall, uint32_t lo) {
  if (lo & LO_SHARED) return __ldg(&v.tlen[lo & ~LO_SHARED]);
  const uint32_t c1 = ocall[lo];
  return ck[c1 ? c1 - 1 : 0].size;
}

// per-phase SM cycles of thread 0 (SAGA_REPLAY_TRACE): 0 updates+R1, 1 R2, 2 R3 normalisers,
// 3 R3 keys+pivot, 4 R3 evict, 5 victims, 6 R4, 7 live list (BELADY / LRU: 2 = threshold
// searches of the hierarchical bitmaps, 3 = taking every dead block)
#ifndef SAGA_TRACE_COUNT_PIVOT
#define PH(i)                                                   \
  do {                                                          \
    if (a.phase_cyc && threadIdx.x == 0) {                      \
      const long long _n = clock64();                           \
      ph[i] += _n - ph_t;                                       \
      ph_t = _n;                                                \
    }                                                           \
  } while (0)
#else  // (experiment: slots 0 / 5 / 6 count AEG eviction epochs by pivot path instead of cycles)
#define PH(i)                                                   \
  do {                                                          \
    if (a.phase_cyc && threadIdx.x == 0) {                      \
      const long long _n = clock64();                           \
      if ((i) != 0 && (i) != 5 && (i) != 6) ph[i] += _n - ph_t; \
      ph_t = _n;                                                \
    }                                                           \
  } while (0)
#endif

constexpr uint32_t VT_LID = 0x80000000u;  // victim-list tag: the entry is a local id, else a position
#ifndef SAGA_REPLAY_UNR
#define SAGA_REPLAY_UNR 2
#endif
constexpr int UNR = SAGA_REPLAY_UNR;      // record chunks whose loads are issued together (R2 / R4)

__device__ __forceinline__ uint32_t unit_mask(uint32_t wi, uint32_t pa, uint32_t pe) {
  uint32_t m = 0xffffffffu;
  if (wi == (pa >> 5)) m &= ~((1u << (pa & 31)) - 1u);
  if (wi == ((pe - 1) >> 5) && (pe & 31)) m &= (1u << (pe & 31)) - 1u;
  return m;
}

__device__ __forceinline__ void log_victim(const ReplayArgs& a, unsigned long long x) {
  const unsigned long long i = atomicAdd(a.vlog_n, 1ull);
  if (i < a.vlog_cap) a.vlog[i] = x;
}

__global__ void __launch_bounds__(RT, SAGA_REPLAY_MINB) k_replay(ReplayArgs a) {
  __shared__ Smem sm;
  __shared__ long long s_ctr[SAGA_NCOUNT];
  extern __shared__ __align__(16) uint32_t dyn_all[];
  uint32_t* const dyn = dyn_all + PF_WORDS;  // per-item count / table region (after the staging area)
  Par par;
  if (threadIdx.x == 0) { mbar_init(&sm.pbar[0], 1); mbar_init(&sm.pbar[1], 1); }
  __syncthreads();
  uint32_t pf_seq = 0;  // prefetches issued by this CTA (uniform); stage = seq & 1, parity = (seq >> 1) & 1
  const TraceView& v = a.v;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* base = a.scratch + (uint64_t)blockIdx.x * a.cta_bytes;
  uint32_t* res_pos = reinterpret_cast<uint32_t*>(base + a.o_res);
  uint32_t* alive = reinterpret_cast<uint32_t*>(base + a.o_bits);   // AEG / EVICT_ALL (aliases pend.bits)
  uint32_t* nres_a = reinterpret_cast<uint32_t*>(base + a.o_nres);  // AEG / EVICT_ALL next-use-resident bits
  uint32_t* vunits = reinterpret_cast<uint32_t*>(base + a.o_vu);    // AEG: list entries evicted this epoch
  ListRec* lists[2] = {reinterpret_cast<ListRec*>(base + a.o_list0), reinterpret_cast<ListRec*>(base + a.o_list1)};
  uint64_t* kbuf = reinterpret_cast<uint64_t*>(base + a.o_kbuf);
  uint32_t* vlist = reinterpret_cast<uint32_t*>(base + a.o_vl);
  const CallKey* ck = a.callkey;

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
    const bool lru = pol == SAGA_POLICY_LRU || pol == SAGA_POLICY_LRU_PREFIX;
    const bool pfx = pol == SAGA_POLICY_LRU_PREFIX;
    const bool units = !belady && !lru;  // AEG / EVICT_ALL keep units and the live list
    // LRU order: hierarchical bitmap over mirrored latest positions (oldest access = top bit);
    // LRU + Prefix puts private blocks in the upper half so they go before any shared block
    const uint64_t NM = pfx ? 2 * nd.N : nd.N;
    auto lru_idx = [&](uint32_t p, bool shared) -> uint32_t {
      return pfx && !shared ? (uint32_t)(2 * nd.N - 1 - p) : (uint32_t)(nd.N - 1 - p);
    };
    auto lru_pos = [&](uint32_t i) -> uint32_t {
      return (uint32_t)(i >= nd.N ? 2 * nd.N - 1 - i : nd.N - 1 - i);
    };
    const uint32_t n2N = max(1u, (uint32_t)((nd.N + (1u << 20) - 1) >> 20));
    const uint32_t n2L = max(1u, (nd.n_local + (1u << 20) - 1) >> 20);
    const uint32_t n1L = (nd.n_local + 1023u) >> 10;  // c1 blocks holding local ids
    // BELADY: c2 always in shared memory; c1 and the dead bits there too when they fit
    uint32_t* c2N = dyn;
    uint32_t* c2L = dyn + a.n2N_max;
    const uint32_t c1off = (max(a.n2N_max + a.n2L_max, a.n2R_max) + 3u) & ~3u;
    uint32_t* c1N = a.dyn_c1 ? dyn + c1off : reinterpret_cast<uint32_t*>(base + a.o_c1);
    uint32_t* c1L = a.dyn_c1 ? c1N + a.n2N_max * 1024u : reinterpret_cast<uint32_t*>(base + a.o_dc1);
    const uint32_t dboff = a.dyn_c1 ? c1off + (a.n2N_max + a.n2L_max) * 1024u : c1off;
    uint32_t* dbits = (n1L * 32u <= a.dyn_dbits_words) ? dyn + dboff : reinterpret_cast<uint32_t*>(base + a.o_dbits);
    HB pend{reinterpret_cast<uint32_t*>(base + a.o_bits), c1N, c2N, n2N};
    HB dead{dbits, c1L, c2L, n2L};
    const uint32_t n2R = max(1u, (uint32_t)((NM + (1u << 20) - 1) >> 20));
    HB rec{reinterpret_cast<uint32_t*>(base + a.o_bits), reinterpret_cast<uint32_t*>(base + a.o_c1), dyn, n2R};
    // AEG / EVICT_ALL: newest-call table, then the unit counts, in shared memory when they fit
    uint32_t* ocall = a.ocall_smem ? dyn : reinterpret_cast<uint32_t*>(base + a.o_ocall);
    const uint32_t cnt_off = a.ocall_smem ? ((nd.n_lo + 3u) & ~3u) : 0u;
    uint32_t* cnt = (cnt_off + nd.n_units <= a.dyn_words) ? dyn + cnt_off : reinterpret_cast<uint32_t*>(base + a.o_cnt);
    // ---- reset the item state ----
    {
      const uint4 ones = make_uint4(NONE, NONE, NONE, NONE), zero = make_uint4(0, 0, 0, 0);
      uint4* r4 = reinterpret_cast<uint4*>(res_pos);
      for (uint32_t i = threadIdx.x; i < (nd.n_local + 3) / 4; i += RT) r4[i] = ones;
      uint4* b4 = reinterpret_cast<uint4*>(pend.bits);
      // whole 1024-bit blocks: the threshold search reads all 32 words of a block
      for (uint32_t i = threadIdx.x; i < (uint32_t)((nd.N + 1023) / 1024) * 8u; i += RT) b4[i] = zero;
      if (lru) {
        for (uint32_t i = threadIdx.x; i < (uint32_t)((NM + 1023) / 1024) * 8u; i += RT) b4[i] = zero;
        for (uint32_t i = threadIdx.x; i < n2R * 1024u; i += RT) rec.c1[i] = 0;
        for (uint32_t i = threadIdx.x; i < n2R; i += RT) rec.c2[i] = 0;
        uint4* n4 = reinterpret_cast<uint4*>(nres_a);
        for (uint32_t i = threadIdx.x; i < (uint32_t)((nd.N + 1023) / 1024) * 8u; i += RT) n4[i] = zero;
      } else if (belady) {
        for (uint32_t i = threadIdx.x; i < n2N * 1024u; i += RT) c1N[i] = 0;
        for (uint32_t i = threadIdx.x; i < n2L * 1024u; i += RT) c1L[i] = 0;
        for (uint32_t i = threadIdx.x; i < a.n2N_max + a.n2L_max; i += RT) dyn[i] = 0;
        for (uint32_t i = threadIdx.x; i < n1L * 32u; i += RT) dbits[i] = 0;
      } else {
        uint4* n4 = reinterpret_cast<uint4*>(nres_a);
        for (uint32_t i = threadIdx.x; i < (uint32_t)((nd.N + 1023) / 1024) * 8u; i += RT) n4[i] = zero;
        for (uint32_t i = threadIdx.x; i < nd.n_units; i += RT) cnt[i] = 0;
        if (aeg) for (uint32_t i = threadIdx.x; i < nd.n_lo; i += RT) ocall[i] = 0;
      }
      if (threadIdx.x < SAGA_NCOUNT) s_ctr[threadIdx.x] = 0;
      if (threadIdx.x == 0) { sm.tot_dead = 0; sm.tot_pend = 0; }
      __syncthreads();
    }
    uint32_t S = 0;       // |S| (uniform)
    uint32_t nL = 0;      // live unit list length (uniform)
    int cur = 0;          // active list buffer
    uint32_t ucur = 0;    // session-update cursor (uniform)
    long long c_hit = 0, c_miss = 0, c_mhit = 0, c_mmiss = 0, c_comp = 0, c_compg = 0, c_regen = 0, c_inv = 0;
    long long c_phit = 0, c_pmiss = 0;
    long long c_ev = 0, c_prot = 0, c_evev = 0, c_peak = 0, infeasible = 0;
    unsigned long long hash = 0;
    uint32_t bad = 0;
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_t = clock64();
    const uint32_t npa = belady ? 3u : NPA;       // BELADY never reads prv / upu
    const uint32_t* pa_src[NPA] = {nd.lidf, nd.u_of, nd.nxt, nd.prv, nd.upu};
    // staged epoch: event pf_j in stage pf_seq & 1, covering positions [pf_b0, pf_b0 + pf_n)
    uint32_t pf_j = NONE, pf_n = 0;
    uint64_t pf_b0 = 0;
    auto issue = [&](uint32_t jj) {  // uniform; thread 0 issues the bulk copies of event jj
      const uint64_t q0 = nd.ev_pos[jj], q1 = nd.ev_pos[jj + 1];
      pf_j = jj;
      pf_b0 = q0 & ~3ull;
      pf_n = (uint32_t)min((unsigned long long)(((q1 - pf_b0) + 3) & ~3ull), (unsigned long long)PF);
      if (threadIdx.x == 0) {
        const uint32_t st = pf_seq & 1u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&sm.pbar[st])),
                     "r"(pf_n * 4u * npa) : "memory");
        for (uint32_t k2 = 0; k2 < npa; ++k2)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(dyn_all + (st * NPA + k2) * PF)), "l"(pa_src[k2] + pf_b0), "r"(pf_n * 4u),
                       "r"(smem_u32(&sm.pbar[st])) : "memory");
      }
      ++pf_seq;
    };
    auto await_pf = [&]() {  // all threads: the staged epoch has landed
      const uint32_t sq = pf_seq - 1u;
      mbar_wait(&sm.pbar[sq & 1u], (sq >> 1) & 1u);
    };

    for (uint32_t j = 0; j < nd.J; ++j) {
      const uint32_t e = nd.ev_e[j];
      const int64_t Te = (int64_t)e * v.epoch_us;
      // ---- AEG session state at T_e: newest call c* with e(c*) <= e ----
      if (aeg && j + 1 < nd.J) {
        const uint32_t ue = nd.ev_upd[j];
        for (uint32_t i = ucur + threadIdx.x; i < ue; i += RT) atomicMax(&ocall[nd.upd_lo[i]], nd.upd_c[i] + 1);
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
          } else if (lru) {  // migrated-away blocks are private
            hb_clear(rec, lru_idx(p, false));
            const uint32_t q = nd.nxt[p];
            if (q != INF32) atomicAnd(&nres_a[q >> 5], ~(1u << (q & 31)));
          } else {
            atomicAnd(&alive[p >> 5], ~(1u << (p & 31)));
            atomicSub(&cnt[nd.u_of[p] & UMASK], 1u);
            const uint32_t q = nd.nxt[p];
            if (q != INF32) atomicAnd(&nres_a[q >> 5], ~(1u << (q & 31)));
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
      // staged per-position arrays of this epoch (issued one epoch ahead), then stage the next one
      if (pf_j != j) {
        if (pf_j != NONE) await_pf();  // drain a stale stage before reusing the sequence
        issue(j);
      }
      await_pf();
      const uint32_t* stg = dyn_all + ((pf_seq - 1u) & 1u) * NPA * PF;
      const uint64_t sb0 = pf_b0;
      const uint32_t sn = pf_n;
      // (the other stage was last read two epochs ago, before this epoch's first barrier)
      if (j + 2 < nd.J && nd.ev_pos[j + 2] > nd.ev_pos[j + 1]) issue(j + 1);
      // position p's value of array k: staged when p - sb0 < sn, else from global memory
      auto P = [&](uint32_t k2, uint64_t p) -> uint32_t {
        const uint64_t o = p - sb0;
        return o < sn ? stg[k2 * PF + o] : pa_src[k2][p];
      };
      PH(0);
      // ---- R2: |A|, new = |A \ S|; hits / misses; in-flight blocks leave the index ----
      uint32_t nA = 0, nnew = 0;
      uint32_t t_hit = 0, t_miss = 0, t_mhit = 0, t_mmiss = 0, t_phit = 0, t_pmiss = 0, t_comp = 0, t_compg = 0,
               t_regen = 0;
      // A first-in-epoch record p is a hit iff bit p of the next-use-resident bitmap is set (the
      // resident block's next use is p); a warp's 32 positions are one aligned bitmap word.
      uint32_t* nres = belady ? pend.bits : nres_a;
      for (uint64_t wb = (P0 & ~31ull) + (uint64_t)wid * 32u; wb < P1; wb += (uint64_t)RT * UNR) {
        uint32_t lf[UNR], uo[UNR], pv[UNR], up[UNR], nw[UNR];
        bool in[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint64_t wbu = wb + (uint64_t)u * RT;
          const uint64_t pb = wbu + lane;
          in[u] = pb >= P0 && pb < P1;
          lf[u] = in[u] ? P(0, pb) : 0u;
          uo[u] = in[u] ? P(1, pb) : 0u;
          pv[u] = (in[u] && !belady) ? P(3, pb) : 0u;
          up[u] = (in[u] && units) ? P(4, pb) : 0u;
          nw[u] = wbu < P1 ? nres[wbu >> 5] : 0u;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint64_t wbu = wb + (uint64_t)u * RT;
          const bool first = in[u] && !(lf[u] & LID_NFIE);
          const bool resident = first && ((nw[u] >> lane) & 1u);
          const bool mig = (uo[u] & KIND_MIG) != 0;
          const bool pf = (uo[u] & KIND_PF) != 0;
          if (in[u]) {
            if (first && !resident) {
              ++nA; ++nnew;
              // CALL miss: compulsory only at the block's first touch in the whole trace, else a
              // re-prefill = regeneration ("tokens prefilled"), also after a reroute
              if (mig) ++t_mmiss;
              else if (pf) ++t_pmiss;
              else { ++t_miss; if (lf[u] & LID_FTG) ++t_compg; else ++t_regen; }
              if (lf[u] & LID_FTN) ++t_comp;
            } else {
              if (first) ++nA;
              if (mig) ++t_mhit; else if (pf) ++t_phit; else ++t_hit;
            }
          }
          // in-flight blocks leave the index until R4
          const uint32_t rm = __ballot_sync(0xffffffffu, resident);
          if (rm && lane == 0) {
            atomicAnd(&nres[wbu >> 5], ~rm);
            if (belady) { atomicSub(&pend.c1[wbu >> 10], (uint32_t)__popc(rm)); atomicSub(&pend.c2[wbu >> 20], (uint32_t)__popc(rm)); }
          }
          if (units) {
            warp_bits(alive, resident, pv[u], false);
            warp_count(cnt, resident, up[u], false);
          } else if (lru) {
            hb_update_warp(rec, resident, lru_idx(pv[u], (uo[u] & U_SHARED) != 0), false);
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
      c_hit += t_hit; c_miss += t_miss; c_mhit += t_mhit; c_mmiss += t_mmiss; c_comp += t_comp; c_compg += t_compg;
      c_regen += t_regen; c_phit += t_phit; c_pmiss += t_pmiss;
      const uint32_t inAS = nA - nnew;  // in-flight (resident) blocks
      const int64_t kk = (pol == SAGA_POLICY_EVICT_ALL) ? (int64_t)S - (int64_t)inAS
                                                        : (int64_t)S + (int64_t)nnew - (int64_t)C;
      PH(1);
      // ---- R3: evict the k largest keys among cand = S \ A ----
      if (kk > 0) {
        const uint32_t k = (uint32_t)kk;
        const uint64_t eh = (uint64_t)e << 32;
        unsigned long long hs = 0;
        uint32_t n_direct = 0, n_prot = 0;  // victims handled outside the list; protected victims
        if (belady) {
          // in-flight blocks left `pend` in R2 (their next use is this epoch)
          const uint32_t nd_ = sm.tot_dead, np_ = sm.tot_pend - inAS;
          if (threadIdx.x == 0 && sm.tot_pend < inAS) dbg_fail(a.dbg, __LINE__, sm.tot_pend, inAS, e);
          if (k <= nd_) {
            hb_take_top(dead, k, vlist, VT_LID, sm, a.dbg, a.phase_cyc ? ph : nullptr, &ph_t);
          } else {
            if (nd_ > 0) hb_take_from(dead, 0, 0, NONE, vlist, &sm.n_vict, VT_LID);
            __syncthreads();
            PH(3);  // (BELADY: slot 3 = taking every dead block)
            if (k - nd_ <= np_) hb_take_top(pend, k - nd_, vlist, 0u, sm, a.dbg, a.phase_cyc ? ph : nullptr, &ph_t);
            else { bad = 1; if (threadIdx.x == 0) dbg_fail(a.dbg, __LINE__, k, nd_, np_); }
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            sm.tot_dead = nd_ - min(k, nd_);
            sm.tot_pend = np_ - (k > nd_ ? k - nd_ : 0u);
          }
        } else if (lru) {
          // every resident non-in-flight block has one bit; k <= |cand| because |A| <= C
          hb_take_top(rec, k, vlist, 0u, sm, a.dbg, a.phase_cyc ? ph : nullptr, &ph_t);
        } else {
          ListRec* L = lists[cur];
          // whole-unit eviction: list every resident latest position of unit u (warp-collective)
          auto evict_unit = [&](uint32_t u, uint32_t pa, uint32_t pe, bool prot) {
            const uint32_t wlast = (pe - 1) >> 5;
            uint32_t taken = 0;
            for (uint32_t wb = pa >> 5; wb <= wlast; wb += 32) {
              const uint32_t wi = wb + lane;
              uint32_t wv = 0;
              if (wi <= wlast) {
                wv = alive[wi] & unit_mask(wi, pa, pe);
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
              const ListRec r = L[i];
              if (cnt[r.u]) evict_unit(r.u, r.pa, r.pe, false);
            }
          } else {
            // pass a: normalisers over cand (eq:recency tau_max, eq:size size_max)
            long long tau = 0;
            uint32_t smax = 1;
            for (uint32_t i = threadIdx.x; i < nL; i += RT) {
              const ListRec r = L[i];
              if (!cnt[r.u]) continue;
              if (cnt[r.u] > r.pe - r.pa) dbg_fail(a.dbg, __LINE__, r.u, cnt[r.u], r.pe - r.pa);
              tau = max(tau, (long long)(Te - r.t));
              smax = max(smax, owner_size(v, ck, ocall, r.lo));
            }
            // both digit histograms are cleared here: the barrier of block_max2 orders the clear
            // before pass b / b2 (their last readers were the previous epoch's find_level)
            for (uint32_t i = threadIdx.x; i < H1; i += RT) sm.hist[i] = 0;
            for (uint32_t i = threadIdx.x; i < 1024; i += RT) sm.hist2[i] = 0;
            block_max2<RT>(tau, smax, sm.b, par);  // eq:recency / eq:size normalisers, one barrier
            KeyCtx x;
            x.Te = Te; x.tau = tau; x.smax = smax;
            x.den = (int64_t)(a.p_high - a.p_low) * C;
            x.num = min(x.den, max((int64_t)0, 1000 * (int64_t)S - (int64_t)a.p_low * C));
            x.ttl_max = a.ttl_max; x.alpha = a.alpha; x.beta = a.beta; x.gamma = a.gamma;
            const uint32_t act = nd.ev_act[j];
            PH(2);
            // pass b: per-unit key part kp = (!prot << 31) | q, weighted histogram of the top digit
            for (uint32_t i = threadIdx.x; i < nL; i += RT) {
              const ListRec r = L[i];
              const uint32_t c = cnt[r.u];
              uint32_t kp = 0;
              if (c) {
                const OwnerKeyIn oi = owner_in(v, ck, ocall, r.lo, act);
                const uint32_t q = quantize_q20(wa_lru_score(x, r.t, oi.size, oi.P));
                kp = ((uint32_t)!ttl_protected(x, oi) << 31) | q;
                atomicAdd(&sm.hist[kp_digit(kp)], c);
              }
              L[i].kp = kp;
            }
            __syncthreads();
            uint32_t d1, r1, d2, r2;
            find_level<H1 / RT>(sm.hist, 0, H1, k, d1, r1, sm, par);
            for (uint32_t i = threadIdx.x; i < nL; i += RT) {
              const uint32_t kp = L[i].kp;
              if (kp_digit(kp) != d1) continue;
              const uint32_t c = cnt[L[i].u];
              if (c) atomicAdd(&sm.hist2[kp & 1023u], c);
            }
            __syncthreads();
            find_level<1024 / RT>(sm.hist2, 0, 1024, r1, d2, r2, sm, par);
            const uint32_t pb1 = d1 >= 1025u ? 1u : 0u;
            const uint32_t kps = (pb1 << 31) | ((d1 - pb1 * 1025u) << 10) | d2;
            const bool prot_piv = !(kps >> 31);
            const bool whole = sm.hist2[d2] == r2;  // the pivot units are evicted whole
            if (threadIdx.x == 0) { sm.n_piv = 0; sm.n_vu = 0; sm.n_pu = 0; }
            __syncthreads();
            PH(3);
            // pass c: list the entries with kp >= kp* (flat), then evict units above the pivot
            // whole and gather the blocks of the pivot units by lid (a warp per listed entry)
            for (uint32_t i = threadIdx.x; i < ((nL + 31) & ~31u); i += RT) {
              bool vic = false;
              if (i < nL) vic = L[i].kp >= kps && cnt[L[i].u] != 0;
              if (vic && L[i].kp == kps) { atomicAdd(&sm.n_pu, 1u); sm.pu_i = i; }
              const uint32_t vm = __ballot_sync(0xffffffffu, vic);
              uint32_t b0 = 0;
              if (lane == 0 && vm) b0 = atomicAdd(&sm.n_vu, (uint32_t)__popc(vm));
              b0 = __shfl_sync(0xffffffffu, b0, 0);
              if (vic) vunits[b0 + __popc(vm & ((1u << lane) - 1u))] = i;
            }
            __syncthreads();
#ifdef SAGA_TRACE_SPLIT4
            PH(7);  // (experiment: pass c's cycles into slot 7)
#endif
            const uint32_t nvu = sm.n_vu;
            // one pivot unit whose local ids increase with position: its r2 largest lids are its
            // r2 highest resident positions -- no ranking needed
            const bool mono_piv = !whole && sm.n_pu == 1 && (L[sm.pu_i].flags & U_MONO);
            for (uint32_t q = wid; q < nvu; q += RW) {
              const ListRec r = L[vunits[q]];
              if (r.kp > kps || whole) { evict_unit(r.u, r.pa, r.pe, !(r.kp >> 31)); continue; }
              if (mono_piv) {
                const uint32_t wfirst = r.pa >> 5, wlast = (r.pe - 1) >> 5;
                uint32_t need = r2;  // take from the top word down
                for (int64_t wb = (int64_t)wlast - 31; need > 0; wb -= 32) {
                  const int64_t wi = wb + lane;
                  const uint32_t wv = (wi >= (int64_t)wfirst && wi <= (int64_t)wlast)
                                          ? (alive[wi] & unit_mask((uint32_t)wi, r.pa, r.pe)) : 0u;
                  const uint32_t c = __popc(wv);
                  uint32_t xs = c;  // inclusive suffix sum from lane 31 down
#pragma unroll
                  for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_down_sync(0xffffffffu, xs, o);
                    if (lane + o < 32) xs += y;
                  }
                  const uint32_t above = xs - c;  // resident positions in higher words of the chunk
                  uint32_t tk = 0;
                  if (above < need) {
                    tk = wv;
                    const uint32_t keep = above + c > need ? above + c - need : 0u;  // lowest bits stay
                    for (uint32_t z = 0; z < keep; ++z) tk &= tk - 1;
                  }
                  if (tk) atomicAnd(&alive[wi], ~tk);
                  emit_bits(vlist, &sm.n_vict, (uint32_t)(wi > 0 ? wi : 0), tk, 0u);
                  const uint32_t tot = __shfl_sync(0xffffffffu, xs, 0);
                  need = tot >= need ? 0u : need - tot;
                  if (wb <= (int64_t)wfirst) break;
                }
                if (lane == 0) { cnt[r.u] -= r2; if (prot_piv) n_prot += r2; }
                continue;
              }
              const uint32_t wlast = (r.pe - 1) >> 5;
              for (uint32_t wb = (r.pa >> 5); wb <= wlast; wb += 32) {
                const uint32_t wi = wb + lane;
                const uint32_t wv = wi <= wlast ? (alive[wi] & unit_mask(wi, r.pa, r.pe)) : 0u;
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
                for (uint32_t y = wv; y; y &= y - 1) kbuf[b0++] = ((uint64_t)r.u << 32) | (wi * 32u + (uint32_t)(__ffs(y) - 1));
              }
            }
            __syncthreads();
            const uint32_t npv = sm.n_piv;
            if (threadIdx.x == 0 && npv > C) dbg_fail(a.dbg, __LINE__, npv, C, r2);
#ifdef SAGA_TRACE_COUNT_PIVOT
            if (threadIdx.x == 0) ph[whole ? 0 : (mono_piv ? 5 : 6)] += 1000000ll;
#endif
            if (!whole && !mono_piv && npv) {
              // pivot keys differ only in lid: rank (lid << 32 | slot) and keep the top r2
              uint32_t* pslot = vlist + k;  // (unit, position) of gathered slot i, after the list
              for (uint32_t i = threadIdx.x; i < npv; i += RT) {
                const uint64_t g = kbuf[i];
                const uint32_t p = (uint32_t)g;
                pslot[2 * i] = (uint32_t)(g >> 32);
                pslot[2 * i + 1] = p;
                kbuf[i] = ((uint64_t)(nd.lidf[p] & LID_MASK) << 32) | i;
              }
              __syncthreads();
              const uint64_t T = radix_select<RT>(kbuf, npv, r2, sm.b, par);
              uint32_t tk = 0;
              for (uint32_t i = threadIdx.x; i < npv; i += RT) {
                const uint64_t kv = kbuf[i];
                if (kv < T) continue;
                const uint32_t sl = (uint32_t)kv, lid = (uint32_t)(kv >> 32);
                const uint32_t u = pslot[2 * sl], p = pslot[2 * sl + 1];
                atomicAnd(&alive[p >> 5], ~(1u << (p & 31)));
                atomicSub(&cnt[u], 1u);
                const uint32_t qn = nd.nxt[p];
                if (qn != INF32) atomicAnd(&nres_a[qn >> 5], ~(1u << (qn & 31)));
                res_pos[lid] = NONE;
                hs += splitmix64(eh | lid);
                if (a.vlog) log_victim(a, eh | lid);
                ++tk;
              }
              n_direct += tk;
              if (prot_piv) n_prot += tk;
            }
          }
        }
        __syncthreads();
        PH(4);
        // listed victims: positions (block at that position) or local ids (VT_LID)
        const uint32_t nvl = sm.n_vict;
        if (threadIdx.x == 0 && nvl > k) dbg_fail(a.dbg, __LINE__, nvl, k, pol);
        for (uint32_t i = threadIdx.x; i < ((nvl + 31) & ~31u); i += RT) {
          const bool in = i < nvl;
          uint32_t x = in ? vlist[i] : 0u;
          if (lru && in) x = lru_pos(x);  // LRU lists bitmap indices of mirrored positions
          const uint32_t lid = (x & VT_LID) ? (x & ~VT_LID) : (in ? nd.lidf[x] & LID_MASK : 0u);
          if (!belady) {  // a victim's next use is no longer resident
            const uint32_t qn = in ? nd.nxt[x] : INF32;
            warp_bits(nres_a, qn != INF32, qn, false);
          }
          if (in) {
            res_pos[lid] = NONE;
            hs += splitmix64(eh | lid);
            if (a.vlog) log_victim(a, eh | lid);
          }
        }
        const unsigned long long nvp = block_reduce<RT, unsigned long long>(
            ((unsigned long long)n_direct << 32) | n_prot, Add(), sm.b, par);
        const uint32_t nv = nvl + (uint32_t)(nvp >> 32), np = (uint32_t)nvp;
        hash += hs;
        if (nv != k) { bad = 1; if (threadIdx.x == 0) dbg_fail(a.dbg, __LINE__, nv, k, pol); }
        S -= nv;
        c_ev += nv; c_prot += aeg ? np : 0; c_evev += 1;  // uniform
      }
      PH(5);
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
          q[u] = in ? P(2, pb) : 0u;
          lf[u] = in ? P(0, pb) : 0u;
          uo[u] = (in && !belady) ? P(1, pb) : 0u;
          last[u] = in && (uint64_t)q[u] >= P1;  // INF included
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint64_t pb = wb + (uint64_t)u * RT + lane;
          const uint32_t lid = lf[u] & LID_MASK;
          if (last[u]) res_pos[lid] = (uint32_t)pb;
          if (belady) {
            hb_update_warp(dead, last[u] && q[u] == INF32, lid, true);
            hb_update_warp(pend, last[u] && q[u] != INF32, q[u], true);
            const uint32_t md = __ballot_sync(0xffffffffu, last[u] && q[u] == INF32);
            const uint32_t mp = __ballot_sync(0xffffffffu, last[u] && q[u] != INF32);
            if (lane == 0 && (md | mp)) { atomicAdd(&sm.tot_dead, __popc(md)); atomicAdd(&sm.tot_pend, __popc(mp)); }
          } else if (lru) {
            hb_update_warp(rec, last[u], lru_idx((uint32_t)pb, (uo[u] & U_SHARED) != 0), true);
            warp_bits(nres_a, last[u] && q[u] != INF32, q[u], true);
          } else {
            const uint32_t wv = __ballot_sync(0xffffffffu, last[u]);
            if (lane == 0 && wv) atomicOr(&alive[(wb + (uint64_t)u * RT) >> 5], wv);
            const uint32_t un = uo[u] & UMASK;
            warp_bits(nres_a, last[u] && q[u] != INF32, q[u], true);
            warp_count(cnt, last[u], un, true);
          }
        }
      }
      S += nnew;
      PH(6);
      // ---- live unit list: append this epoch's units; every 16th epoch also drop the units
      // whose count reached 0 (until then the passes skip them: each one tests cnt first) ----
      if (units && (j & 15u) != 15u) {
        ListRec* L = lists[cur];
        const uint32_t U0 = nd.ev_unit[j], U1 = nd.ev_unit[j + 1];
        for (uint32_t i = threadIdx.x; i < U1 - U0; i += RT) {
          const UnitRec ur = nd.urec[U0 + i];
          ListRec r{};
          r.t = ur.t; r.u = U0 + i; r.pa = ur.pa; r.pe = ur.pe; r.lo = ur.lo; r.kp = 0; r.flags = ur.flags;
          L[nL + i] = r;
        }
        nL += U1 - U0;  // read again only after the next epoch's first barrier
      } else if (units) {
        __syncthreads();
        const ListRec* L = lists[cur];
        ListRec* L2 = lists[cur ^ 1];
        const uint32_t U0 = nd.ev_unit[j], U1 = nd.ev_unit[j + 1];
        const uint32_t tot = nL + (U1 - U0);
        for (uint32_t i = threadIdx.x; i < ((tot + 31) & ~31u); i += RT) {
          ListRec r{};
          bool keep = false;
          if (i < tot) {
            if (i < nL) {
              r = L[i];
            } else {
              const uint32_t u = U0 + (i - nL);
              const UnitRec ur = nd.urec[u];
              r.t = ur.t; r.u = u; r.pa = ur.pa; r.pe = ur.pe; r.lo = ur.lo; r.kp = 0; r.flags = ur.flags;
            }
            keep = cnt[r.u] != 0;
          }
          const uint32_t km = __ballot_sync(0xffffffffu, keep);
          uint32_t b0 = 0;
          if (lane == 0 && km) b0 = atomicAdd(&sm.n_app, (uint32_t)__popc(km));
          b0 = __shfl_sync(0xffffffffu, b0, 0);
          if (keep) L2[b0 + __popc(km & ((1u << lane) - 1u))] = r;
        }
        __syncthreads();
        nL = sm.n_app;
        cur ^= 1;
      }
      PH(7);
      c_peak = max(c_peak, (long long)S);
    }
    // ---- counters ----
    if (pf_j != NONE) await_pf();  // no bulk copy may target the staging area after the item
    __syncthreads();
    {
      unsigned long long* sc = reinterpret_cast<unsigned long long*>(s_ctr);
      atomicAdd(&sc[SAGA_C_HITS], (unsigned long long)c_hit);
      atomicAdd(&sc[SAGA_C_MISSES], (unsigned long long)c_miss);
      atomicAdd(&sc[SAGA_C_MIG_HITS], (unsigned long long)c_mhit);
      atomicAdd(&sc[SAGA_C_MIG_MISSES], (unsigned long long)c_mmiss);
      atomicAdd(&sc[SAGA_C_COMPULSORY_NODE], (unsigned long long)c_comp);
      atomicAdd(&sc[SAGA_C_COMPULSORY_GLOBAL], (unsigned long long)c_compg);
      atomicAdd(&sc[SAGA_C_REGEN_TOKENS], (unsigned long long)c_regen);
      atomicAdd(&sc[SAGA_C_VICTIM_HASH], hash);
      atomicAdd(&sc[SAGA_C_PF_HITS], (unsigned long long)c_phit);
      atomicAdd(&sc[SAGA_C_PF_MISSES], (unsigned long long)c_pmiss);
    }
    if (bad) atomicOr(a.err, 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t* out = a.counters + (((uint64_t)pi * a.n_caps + ci) * a.n_nodes_total + w) * SAGA_NCOUNT;
      const long long rg = s_ctr[SAGA_C_REGEN_TOKENS];
      out[SAGA_C_ACCESSES] = s_ctr[SAGA_C_HITS] + s_ctr[SAGA_C_MISSES] + s_ctr[SAGA_C_MIG_HITS] + s_ctr[SAGA_C_MIG_MISSES] +
                             s_ctr[SAGA_C_PF_HITS] + s_ctr[SAGA_C_PF_MISSES];
      out[SAGA_C_HITS] = s_ctr[SAGA_C_HITS];
      out[SAGA_C_MISSES] = s_ctr[SAGA_C_MISSES];
      out[SAGA_C_MIG_HITS] = s_ctr[SAGA_C_MIG_HITS];
      out[SAGA_C_MIG_MISSES] = s_ctr[SAGA_C_MIG_MISSES];
      out[SAGA_C_COMPULSORY_GLOBAL] = s_ctr[SAGA_C_COMPULSORY_GLOBAL];
      out[SAGA_C_COMPULSORY_NODE] = s_ctr[SAGA_C_COMPULSORY_NODE];
      out[SAGA_C_INVALIDATED] = c_inv;
      out[SAGA_C_EVICTIONS] = c_ev;
      out[SAGA_C_EVICT_PROTECTED] = c_prot;
      out[SAGA_C_EVICT_EVENTS] = c_evev;
      out[SAGA_C_REGEN_TOKENS] = rg * (long long)v.btok;
      out[SAGA_C_REGEN_US] = rg * ((long long)v.btok * 1000000 / (long long)v.prefill_tok_s);
      out[SAGA_C_VICTIM_HASH] = s_ctr[SAGA_C_VICTIM_HASH];
      out[SAGA_C_INFEASIBLE_EPOCH] = infeasible;
      out[SAGA_C_PEAK_RESIDENT] = c_peak;
      out[SAGA_C_PF_HITS] = s_ctr[SAGA_C_PF_HITS];
      out[SAGA_C_PF_MISSES] = s_ctr[SAGA_C_PF_MISSES];
      out[SAGA_C_RESERVED18] = 0;
      out[SAGA_C_RESERVED19] = 0;
      if (a.item_cyc) a.item_cyc[it] = (unsigned long long)(clock64() - t_start);
      if (a.phase_cyc)
        for (int i = 0; i < 8; ++i) a.phase_cyc[(uint64_t)it * 8 + i] = (unsigned long long)ph[i];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// replay index of a node (built once): event positions, units, local owners, update ranges
// ------------------------------------------------------------------------------------------
__global__ void k_call_key(TraceView v, CallKey* ck) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.n_calls; c += gridDim.x * blockDim.x) {
    CallKey k;
    k.tend = v.tend[c];
    k.P = v.ci_P[c];
    k.size = v.ci_size[c];
    k.ttl = (uint32_t)call_ttl_base(v, c);
    k.fin = v.ci_fin[c];
    ck[c] = k;
  }
}

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
// private owners present at the node -> dense local ids
__global__ void k_owner_flag(const uint32_t* lown, uint32_t n_local, uint32_t n_sessions, uint32_t* flag) {
  for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n_local; l += gridDim.x * blockDim.x) {
    const uint32_t o = lown[l];
    if (o < n_sessions) flag[o] = 1u;
  }
}
// hpos = exclusive scan of head: the unit of p is hpos[p+1] - 1
__global__ void k_unit_fill(const uint32_t* head, const uint32_t* hpos, uint64_t N, const uint32_t* lidf,
                            const uint32_t* lown, const uint64_t* g_pos, uint32_t G, const int64_t* g_t,
                            const uint32_t* g_kind, const uint32_t* s2lo, uint32_t n_sessions, uint32_t* u_pos,
                            UnitRec* urec, uint32_t* u_kind) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (uint64_t)gridDim.x * blockDim.x) {
    if (!head[p]) continue;
    const uint32_t u = hpos[p];
    uint32_t lo = 0, hi = G;  // last group with g_pos[g] <= p
    while (lo + 1 < hi) { const uint32_t mid = (lo + hi) >> 1; if (g_pos[mid] <= p) lo = mid; else hi = mid; }
    const uint32_t own = lown[lidf[p] & LID_MASK];
    u_pos[u] = (uint32_t)p;
    UnitRec r;
    r.t = g_t[lo];
    r.pa = (uint32_t)p;
    r.pe = 0;
    r.lo = own < n_sessions ? s2lo[own] : (LO_SHARED | (own - n_sessions));
    r.flags = U_MONO;
    urec[u] = r;
    u_kind[u] = g_kind[lo];
  }
}
// a unit loses U_MONO where a local id does not increase from one position to the next
__global__ void k_unit_mono(const uint32_t* lidf, const uint32_t* u_of, uint64_t N, UnitRec* urec) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p + 1 < N; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = u_of[p] & UMASK;
    if ((u_of[p + 1] & UMASK) == u && (lidf[p + 1] & LID_MASK) <= (lidf[p] & LID_MASK)) atomicAnd(&urec[u].flags, ~U_MONO);
  }
}
__global__ void k_unit_end(const uint32_t* u_pos, uint32_t n_units, uint64_t N, UnitRec* urec) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n_units; u += gridDim.x * blockDim.x)
    urec[u].pe = u + 1 < n_units ? u_pos[u + 1] : (uint32_t)N;
}
__global__ void k_unit_of(const uint32_t* hpos, uint64_t N, const uint32_t* u_kind, const UnitRec* urec,
                          uint32_t* u_of) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = hpos[p + 1] - 1;
    u_of[p] = u | (u_kind[u] == 1 ? KIND_MIG : 0u) | (u_kind[u] == 2 ? KIND_PF : 0u) |
              ((urec[u].lo & LO_SHARED) ? U_SHARED : 0u);
  }
}
__global__ void k_ev_index(TraceView v, const uint64_t* ev_pos, const uint32_t* ev_e, uint32_t J, const uint32_t* hpos,
                           uint64_t N, uint32_t n_units, const uint32_t* upd_c, uint32_t n_upd, const uint32_t* s2lo,
                           uint32_t* ev_unit, uint32_t* ev_upd, uint32_t* upd_lo) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= J; j += gridDim.x * blockDim.x) {
    const uint64_t p = ev_pos[j];
    ev_unit[j] = p < N ? hpos[p] : n_units;
    if (j < J) {
      const uint32_t e = ev_e[j];
      uint32_t lo = 0, hi = n_upd;  // #updates with e(c) <= e
      while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (v.ecall[upd_c[mid]] <= e) lo = mid + 1; else hi = mid; }
      ev_upd[j] = lo;
    }
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_upd; i += gridDim.x * blockDim.x)
    upd_lo[i] = s2lo[v.call_sess[upd_c[i]]];
}

// unit of the previous occurrence of the block at each position
__global__ void k_prev_unit(const uint32_t* prv, const uint32_t* u_of, uint64_t N, uint32_t* upu) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = prv[p];
    upu[p] = q != NONE ? (u_of[q] & UMASK) : 0u;
  }
}

unsigned grid_for(uint64_t n, int threads = NTHREADS) {
  uint64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148u * 64u) g = 148u * 64u;
  return (unsigned)g;
}

// The replay index of a node, in two phases so that the index of every node of a launch needs
// ONE host read of the sizes (each host sync waits for SMs the replays in flight may hold):
// phase A launches the unit-head scans and copies their totals to `cnt2` on the device; phase B,
// after the caller read them, sizes and fills the unit tables.
struct IndexScratch { uint32_t *head = nullptr, *hpos = nullptr, *sflag = nullptr, *s2lo = nullptr; };

saga_status replay_index_a(saga_trace* t, uint32_t w, cudaStream_t s, IndexScratch& x, uint32_t* cnt2) {
  NodeDev& nd = t->nodes[w];
  const TraceView& v = t->v;
  const uint64_t N = nd.N;
  const uint32_t J = nd.J;
  const uint32_t NS = std::max(v.n_sessions, 1u);
  SAGA_CK(ws_malloc((void**)&x.head, (N + 1) * 4, s));
  SAGA_CK(ws_malloc((void**)&x.hpos, (N + 2) * 4, s));
  SAGA_CK(ws_malloc((void**)&x.sflag, (size_t(NS) + 1) * 4, s));
  SAGA_CK(ws_malloc((void**)&x.s2lo, (size_t(NS) + 1) * 4, s));
  SAGA_CK(cudaMemsetAsync(x.sflag, 0, (size_t(NS) + 1) * 4, s));
  nd.ev_pos = dalloc<uint64_t>(t, size_t(J) + 1);
  nd.u_of = dalloc<uint32_t>(t, N);
  nd.upu = dalloc<uint32_t>(t, N);
  if (!nd.ev_pos || !nd.u_of || !nd.upu) { set_error("out of device memory (replay index)"); return SAGA_ERR_OOM; }
  // nd.prv (previous occurrence of each position's block) comes from the segmented scan of A4
  k_ev_pos<<<grid_for(size_t(J) + 1), NTHREADS, 0, s>>>(nd.g_pos, nd.ev_g, J, nd.ev_pos);
  count_launch();
  if (nd.n_local) {
    k_owner_flag<<<grid_for(nd.n_local), NTHREADS, 0, s>>>(nd.lown, nd.n_local, v.n_sessions, x.sflag);
    count_launch();
  }
  SAGA_CK(scan_u32(t, x.sflag, x.s2lo, NS));
  if (N > 0) {
    k_unit_head<<<grid_for(N), NTHREADS, 0, s>>>(nd.lidf, nd.lown, N, x.head);
    if (nd.G) k_group_head<<<grid_for(nd.G), NTHREADS, 0, s>>>(nd.g_pos, nd.G, x.head);
    count_launch(2);
  }
  SAGA_CK(scan_u32(t, x.head, x.hpos, N));
  SAGA_CK(cudaMemcpyAsync(cnt2, x.hpos + N, 4, cudaMemcpyDeviceToDevice, s));
  SAGA_CK(cudaMemcpyAsync(cnt2 + 1, x.s2lo + NS, 4, cudaMemcpyDeviceToDevice, s));
  return SAGA_OK;
}

saga_status replay_index_b(saga_trace* t, uint32_t w, cudaStream_t s, IndexScratch& x, const uint32_t* hv) {
  NodeDev& nd = t->nodes[w];
  const TraceView& v = t->v;
  const uint64_t N = nd.N;
  const uint32_t J = nd.J;
  uint32_t *u_kind = nullptr, *u_pos = nullptr;
  const uint32_t nu = hv[0];
  if (nu >= (1u << 29)) { set_error("node %u has %u units (limit 2^29)", w, nu); return SAGA_ERR_STATE; }
  nd.n_units = nu;
  nd.n_lo = hv[1];
  nd.urec = dalloc<UnitRec>(t, nu);
  nd.ev_unit = dalloc<uint32_t>(t, size_t(J) + 1);
  nd.ev_upd = dalloc<uint32_t>(t, J);
  nd.upd_lo = dalloc<uint32_t>(t, nd.n_upd);
  SAGA_CK(ws_malloc((void**)&u_kind, (size_t(nu) + 1) * 4, s));
  SAGA_CK(ws_malloc((void**)&u_pos, (size_t(nu) + 1) * 4, s));
  if (!nd.urec || !nd.ev_unit || !nd.ev_upd || !nd.upd_lo) { set_error("out of device memory (replay index)"); return SAGA_ERR_OOM; }
  if (N > 0) {
    UnitRec* ur = static_cast<UnitRec*>(nd.urec);
    k_unit_fill<<<grid_for(N), NTHREADS, 0, s>>>(x.head, x.hpos, N, nd.lidf, nd.lown, nd.g_pos, nd.G, nd.g_t, nd.g_kind,
                                                 x.s2lo, v.n_sessions, u_pos, ur, u_kind);
    k_unit_end<<<grid_for(nu), NTHREADS, 0, s>>>(u_pos, nu, N, ur);
    k_unit_of<<<grid_for(N), NTHREADS, 0, s>>>(x.hpos, N, u_kind, ur, nd.u_of);
    k_prev_unit<<<grid_for(N), NTHREADS, 0, s>>>(nd.prv, nd.u_of, N, nd.upu);
    k_unit_mono<<<grid_for(N), NTHREADS, 0, s>>>(nd.lidf, nd.u_of, N, ur);
    count_launch(5);
  }
  k_ev_index<<<grid_for(std::max<size_t>(size_t(J) + 1, nd.n_upd)), NTHREADS, 0, s>>>(
      v, nd.ev_pos, nd.ev_e, J, x.hpos, N, nu, nd.upd_c, nd.n_upd, x.s2lo, nd.ev_unit, nd.ev_upd, nd.upd_lo);
  count_launch();
  SAGA_CK_LAUNCH();
  ws_free(x.head, s);
  ws_free(x.hpos, s);
  ws_free(u_kind, s);
  ws_free(u_pos, s);
  ws_free(x.sflag, s);
  ws_free(x.s2lo, s);
  x = IndexScratch{};
  nd.rp_done = true;
  return SAGA_OK;
}

// the replay index of every listed node that lacks one: phase A for all, one host read, phase B
saga_status build_replay_indices(saga_trace* t, const uint32_t* nodes, uint32_t n, cudaStream_t s) {
  std::vector<uint32_t> todo;
  for (uint32_t i = 0; i < n; ++i)
    if (!t->nodes[nodes[i]].rp_done && std::find(todo.begin(), todo.end(), nodes[i]) == todo.end()) todo.push_back(nodes[i]);
  if (todo.empty()) return SAGA_OK;
  std::vector<IndexScratch> xs(todo.size());
  uint32_t* cnt = nullptr;
  SAGA_CK(ws_malloc((void**)&cnt, 8 * todo.size(), s));
  saga_status st = SAGA_OK;
  for (size_t i = 0; i < todo.size() && st == SAGA_OK; ++i) st = replay_index_a(t, todo[i], s, xs[i], cnt + 2 * i);
  std::vector<uint32_t> hv(2 * todo.size());
  if (st == SAGA_OK && d2h(hv.data(), cnt, 8 * todo.size(), s) != cudaSuccess) { set_error("replay index: %s", "d2h"); st = SAGA_ERR_CUDA; }
  for (size_t i = 0; i < todo.size() && st == SAGA_OK; ++i) st = replay_index_b(t, todo[i], s, xs[i], &hv[2 * i]);
  ws_free(cnt, s);
  return st;
}

}  // namespace

#if !SAGA_REPLAY_IS_WIDE
// k_replay_wide.cu: the same kernel at 256 threads x 2 CTAs per SM for launches of more items
// than SMs (DESIGN.md §6 "Replay occupancy")
saga_status run_replay_wide(saga_trace* t, const saga_replay_cfg* cfg, const uint32_t* caps, uint32_t n_caps,
                            const uint32_t* nodes, uint32_t n_owned, int64_t* counters, cudaStream_t s,
                            uint64_t* vlog, uint64_t vlog_cap, uint64_t* vlog_n);
#endif

saga_status SAGA_REPLAY_ENTRY(saga_trace* t, const saga_replay_cfg* cfg, const uint32_t* caps, uint32_t n_caps,
                       const uint32_t* nodes, uint32_t n_owned, int64_t* counters, cudaStream_t s,
                       uint64_t* vlog, uint64_t vlog_cap, uint64_t* vlog_n) {
  const TraceView& v = t->v;
  uint32_t pol[5], n_pol = 0;
  for (uint32_t p : {1u, 2u, 4u, 8u, 16u}) if (cfg->policy_mask & p) pol[n_pol++] = p;
  if (n_pol == 0 || n_caps == 0 || n_owned == 0) return SAGA_OK;
  if (n_caps > 0xFFFFu || n_owned > 0xFFFu) { set_error("saga_replay: at most 65535 capacities and 4095 nodes per call"); return SAGA_ERR_INVALID_ARG; }
  uint32_t cap_max = 0;
  for (uint32_t i = 0; i < n_caps; ++i) cap_max = std::max(cap_max, caps[i]);
  if (!t->callkey) {
    t->callkey = dalloc<CallKey>(t, v.n_calls);
    if (!t->callkey) { set_error("out of device memory (replay)"); return SAGA_ERR_OOM; }
    if (v.n_calls) {
      k_call_key<<<grid_for(v.n_calls), NTHREADS, 0, s>>>(v, static_cast<CallKey*>(t->callkey));
      count_launch();
    }
  }
  uint64_t max_local = 1, maxN = 1, max_units = 1, max_lo = 1;
  {
    const saga_status st = build_replay_indices(t, nodes, n_owned, s);
    if (st != SAGA_OK) return st;
  }
  for (uint32_t i = 0; i < n_owned; ++i) {
    const NodeDev& nd = t->nodes[nodes[i]];
    max_local = std::max<uint64_t>(max_local, nd.n_local);
    maxN = std::max<uint64_t>(maxN, nd.N);
    max_units = std::max<uint64_t>(max_units, nd.n_units);
    max_lo = std::max<uint64_t>(max_lo, nd.n_lo);
  }
  std::vector<NodeArr> hn(t->n_nodes);
  for (uint32_t w = 0; w < t->n_nodes; ++w) {
    const NodeDev& nd = t->nodes[w];
    NodeArr x{};
    x.N = nd.N; x.J = nd.J; x.n_local = nd.n_local; x.n_units = nd.n_units; x.n_lo = nd.n_lo;
    x.ev_pos = nd.ev_pos; x.ev_e = nd.ev_e; x.ev_inv = nd.ev_inv; x.ev_act = nd.ev_act; x.ev_unit = nd.ev_unit;
    x.ev_upd = nd.ev_upd; x.inv_s = nd.inv_s; x.lidf = nd.lidf; x.nxt = nd.nxt; x.u_of = nd.u_of;
    x.prv = nd.prv; x.upu = nd.upu;
    x.urec = static_cast<const UnitRec*>(nd.urec); x.lid2gid = nd.lid2gid; x.upd_c = nd.upd_c; x.upd_lo = nd.upd_lo;
    hn[w] = x;
  }
  // items, longest first: by policy (measured per-event cost: AEG > LRU + Prefix > LRU > EVICT_ALL
  // > BELADY), then largest capacity first (the per-event cost grows with |S| <= C).  Persistent
  // CTAs take items in this order, so the long items start first and the short ones fill the
  // tail (and a following launch on another stream can use the SMs the short ones free).
  std::vector<uint32_t> items;
  items.reserve(size_t(n_pol) * n_caps * n_owned);
  std::vector<uint32_t> corder(n_caps);
  for (uint32_t i = 0; i < n_caps; ++i) corder[i] = i;
  std::stable_sort(corder.begin(), corder.end(), [&](uint32_t x, uint32_t y) { return caps[x] > caps[y]; });
  std::vector<uint32_t> porder(n_pol);
  for (uint32_t i = 0; i < n_pol; ++i) porder[i] = i;
  auto prank = [](uint32_t p) {
    return p == SAGA_POLICY_AEG ? 0 : p == SAGA_POLICY_LRU_PREFIX ? 1 : p == SAGA_POLICY_LRU ? 2 : p == SAGA_POLICY_EVICT_ALL ? 3 : 4;
  };
  std::stable_sort(porder.begin(), porder.end(), [&](uint32_t x, uint32_t y) { return prank(pol[x]) < prank(pol[y]); });
  for (uint32_t pi : porder)
    for (uint32_t ci : corder)
      for (uint32_t ni = 0; ni < n_owned; ++ni) items.push_back((pi << 28) | (ci << 12) | ni);
  const uint32_t n_items = (uint32_t)items.size();
#if !SAGA_REPLAY_IS_WIDE
  {
    // one item per CTA at 512 threads is fastest while the items fit the SMs once; beyond that,
    // two 256-thread CTAs per SM overlap two items' barrier / latency chains (C4: -24 %).
    // SAGA_REPLAY_WIDE=1 / 0 forces either variant (parity tests run both).
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const char* f = getenv("SAGA_REPLAY_WIDE");
    const bool wide = f ? (f[0] == '1') : (n_items > (uint32_t)nsm);
    if (wide) return run_replay_wide(t, cfg, caps, n_caps, nodes, n_owned, counters, s, vlog, vlog_cap, vlog_n);
  }
#endif
  // per-CTA scratch layout (all offsets 256-byte aligned)
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  const uint64_t n2N = std::max<uint64_t>(1, (maxN + (1u << 20) - 1) >> 20);
  const uint64_t n2L = std::max<uint64_t>(1, (max_local + (1u << 20) - 1) >> 20);
  const bool any_pfx = (cfg->policy_mask & SAGA_POLICY_LRU_PREFIX) != 0;
  if (any_pfx && 2 * maxN >= (1ull << 31)) {
    set_error("saga_replay: LRU + Prefix needs node streams below 2^30 accesses");
    return SAGA_ERR_INVALID_ARG;
  }
  const uint64_t n2R = std::max<uint64_t>(1, ((any_pfx ? 2 * maxN : maxN) + (1u << 20) - 1) >> 20);
  const uint64_t n2B = std::max(n2N, n2R);  // the position bitmap serves BELADY, AEG and LRU
  ReplayArgs a{};
  uint64_t off = 0;
  a.o_res = off; off += al(max_local * 4 + 16);
  a.o_nres = off; off += al(n2N * 32768 * 4);
  a.o_bits = off; off += al(n2B * 32768 * 4);
  a.o_c1 = off; off += al(n2B * 1024 * 4);
  a.o_dbits = off; off += al(n2L * 32768 * 4);
  a.o_dc1 = off; off += al(n2L * 1024 * 4);
  a.o_cnt = off; off += al(max_units * 4);
  a.o_list0 = off; off += al(max_units * sizeof(ListRec));
  a.o_list1 = off; off += al(max_units * sizeof(ListRec));
  a.o_kbuf = off; off += al(((uint64_t)cap_max + 1) * 8);
  a.o_vl = off; off += al(((uint64_t)cap_max + 1) * 12);  // victim list + pivot (unit, position) pairs
  a.o_vu = off; off += al(max_units * 4);
  a.o_ocall = off; off += al(max_lo * 4);
  a.cta_bytes = off;
  // dynamic shared memory (one CTA per SM):
  //   BELADY: c2 counts of both bitmaps, then their c1 counts, then the dead bits, while they fit;
  //   AEG / EVICT_ALL: the newest-call table, then the unit counts, while they fit.
  // the rest of the 228 KB unified L1/shared array stays L1 cache, which the per-event loads need
  uint64_t dyn_max = (uint64_t)SAGA_REPLAY_DYN_KB * 1024;
  if (const char* e = getenv("SAGA_REPLAY_SMEM_KB")) dyn_max = std::max<uint64_t>(1, strtoull(e, nullptr, 10)) * 1024;
  dyn_max = std::min<uint64_t>(dyn_max, 200ull * 1024);
  const uint64_t c2_bytes = ((std::max(n2N + n2L, n2R) + 3) & ~3ull) * 4;
  const uint64_t c1_bytes = (n2N + n2L) * 1024 * 4;
  const uint64_t db_bytes = ((max_local + 1023) >> 10) * 32 * 4;
  a.n2N_max = (uint32_t)n2N; a.n2L_max = (uint32_t)n2L; a.n2R_max = (uint32_t)n2R;
  a.dyn_c1 = (c2_bytes + c1_bytes <= dyn_max) ? 1u : 0u;
  uint64_t dyn_b = a.dyn_c1 ? c2_bytes + c1_bytes : c2_bytes;
  if (dyn_b + db_bytes <= dyn_max) { a.dyn_dbits_words = (uint32_t)(db_bytes / 4); dyn_b += db_bytes; }
  else a.dyn_dbits_words = 0;
  const uint64_t oc_bytes = ((max_lo + 3) & ~3ull) * 4;
  a.ocall_smem = oc_bytes <= 64 * 1024 ? 1u : 0u;
  uint64_t dyn_a = (a.ocall_smem ? oc_bytes : 0) + max_units * 4;
  dyn_a = std::min<uint64_t>(dyn_a, dyn_max);
  uint64_t dyn = std::max<uint64_t>(std::max<uint64_t>(dyn_b, dyn_a), a.ocall_smem ? oc_bytes : 16);
  dyn = (dyn + 15) & ~15ull;
  a.dyn_words = (uint32_t)(dyn / 4);
  dyn += (uint64_t)PF_WORDS * 4;  // TMA staging area in front
  SAGA_CK(cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_replay, RT, (size_t)dyn);
  uint32_t grid = std::min<uint32_t>(n_items, (uint32_t)nsm * (uint32_t)std::max(occ, 1));
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  // idle blocks of the workspace cache are released by ws_malloc when the scratch needs them
  const uint64_t avail = (uint64_t)free_b + ws_idle_bytes();
  const uint64_t budget = avail > (4ull << 30) ? (avail - (4ull << 30)) / 10 * 8 : avail / 4;
  grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(grid, budget / std::max<uint64_t>(a.cta_bytes, 1)));
  const bool trace = getenv("SAGA_REPLAY_TRACE") != nullptr;
  NodeArr* d_nodes = nullptr;
  uint32_t *d_caps = nullptr, *d_list = nullptr, *d_items = nullptr, *work = nullptr;
  unsigned long long* d_cyc = nullptr;
  uint8_t* scratch = nullptr;
  // the launch's parameter arrays in one block, copied by one h2d (each copy syncs the stream)
  const size_t o_caps = (sizeof(NodeArr) * t->n_nodes + 15) & ~size_t(15);
  const size_t o_list = o_caps + ((4 * size_t(n_caps) + 15) & ~size_t(15));
  const size_t o_items = o_list + ((4 * size_t(n_owned) + 15) & ~size_t(15));
  const size_t par_bytes = o_items + 4 * size_t(n_items);
  uint8_t* d_par = nullptr;
  SAGA_CK(ws_malloc((void**)&d_par, par_bytes, s));
  d_nodes = reinterpret_cast<NodeArr*>(d_par);
  d_caps = reinterpret_cast<uint32_t*>(d_par + o_caps);
  d_list = reinterpret_cast<uint32_t*>(d_par + o_list);
  d_items = reinterpret_cast<uint32_t*>(d_par + o_items);
  SAGA_CK(ws_malloc((void**)&work, 32, s));
  if (!t->replay_status) {  // [0] error flag, [1..4] first failed invariant (checked by saga_replay_wait)
    t->replay_status = dalloc<uint32_t>(t, 8);
    if (!t->replay_status) { set_error("out of device memory (replay)"); return SAGA_ERR_OOM; }
    SAGA_CK(cudaMemsetAsync(t->replay_status, 0, 32, s));
  }
  if (trace) SAGA_CK(ws_malloc((void**)&d_cyc, 8ull * 9 * n_items, s));
  if (ws_malloc((void**)&scratch, a.cta_bytes * grid, s) != cudaSuccess) {
    set_error("out of device memory (replay scratch %llu bytes)", (unsigned long long)(a.cta_bytes * grid));
    return SAGA_ERR_OOM;
  }
  {
    std::vector<uint8_t> hp(par_bytes, 0);
    memcpy(hp.data(), hn.data(), sizeof(NodeArr) * t->n_nodes);
    memcpy(hp.data() + o_caps, caps, 4 * size_t(n_caps));
    memcpy(hp.data() + o_list, nodes, 4 * size_t(n_owned));
    memcpy(hp.data() + o_items, items.data(), 4 * size_t(n_items));
    SAGA_CK(h2d(d_par, hp.data(), par_bytes, s));
  }
  SAGA_CK(cudaMemsetAsync(work, 0, 32, s));
  a.v = v;
  a.nodes = d_nodes; a.caps = d_caps; a.items = d_items; a.n_items = n_items; a.node_list = d_list;
  for (uint32_t i = 0; i < 5; ++i) a.pol[i] = i < n_pol ? pol[i] : 0u;
  a.n_caps = n_caps; a.n_nodes_total = t->n_nodes; a.counters = counters;
  a.alpha = cfg->alpha; a.beta = cfg->beta; a.gamma = cfg->gamma;
  a.p_low = cfg->p_low_pm; a.p_high = cfg->p_high_pm; a.ttl_max = cfg->ttl_max_us;
  a.callkey = static_cast<const CallKey*>(t->callkey);
  a.scratch = scratch; a.work = work; a.err = t->replay_status; a.dbg = t->replay_status + 4; a.item_cyc = d_cyc;
  a.phase_cyc = d_cyc ? d_cyc + n_items : nullptr;
  a.vlog = reinterpret_cast<unsigned long long*>(vlog);
  a.vlog_n = reinterpret_cast<unsigned long long*>(vlog_n);
  a.vlog_cap = vlog_cap;
  // the kernel runs on the handle's lowest-priority stream, ordered after everything queued on s
  // and before anything queued on s later (scratch stays stream-ordered on s)
  cudaStream_t ks = s;
  if (s && !getenv("SAGA_REPLAY_SAME_STREAM")) {
    if (!t->replay_stream) {
      int least = 0, greatest = 0;
      SAGA_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      SAGA_CK(cudaStreamCreateWithPriority(&t->replay_stream, cudaStreamNonBlocking, least));
    }
    ks = t->replay_stream;
    cudaEvent_t ev;
    SAGA_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SAGA_CK(cudaEventRecord(ev, s));
    SAGA_CK(cudaStreamWaitEvent(ks, ev, 0));
    cudaEventDestroy(ev);
  }
  prof_begin(SAGA_PROF_REPLAY, ks);
  k_replay<<<grid, RT, dyn, ks>>>(a);
  prof_end(SAGA_PROF_REPLAY, ks);
  count_launch();
  SAGA_CK_LAUNCH();
  if (ks != s) {
    cudaEvent_t ev;
    SAGA_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SAGA_CK(cudaEventRecord(ev, ks));
    SAGA_CK(cudaStreamWaitEvent(s, ev, 0));
    cudaEventDestroy(ev);
  }
  // asynchronous: the scratch returns to the stream-ordered cache; the kernel's internal checks
  // land in t->replay_status and are reported by saga_replay_wait (or a synchronising call)
  std::vector<unsigned long long> cyc(trace ? 9ull * n_items : 0);
  if (trace) SAGA_CK(d2h(cyc.data(), d_cyc, 8ull * 9 * n_items, s));
  ws_free(d_par, s);
  ws_free(scratch, s);
  ws_free(work, s);
  if (d_cyc) ws_free(d_cyc, s);
  if (trace) {
    fprintf(stderr, "[saga replay] grid %u x %d threads, dyn smem %llu B (c1 %s, dead bits %s, ocall %s), %u items\n",
            grid, RT, (unsigned long long)dyn, a.dyn_c1 ? "smem" : "global", a.dyn_dbits_words ? "smem" : "global",
            a.ocall_smem ? "smem" : "global", n_items);
    for (uint32_t i = 0; i < n_items; ++i) {
      const uint32_t pk = items[i];
      const uint32_t w = nodes[pk & 0xFFFu];
      const unsigned long long* ph = &cyc[n_items + 8ull * i];
      fprintf(stderr, "[saga replay] item pol=%u cap=%u node=%u events=%u units=%u Mcycles=%.2f phases=%.1f,%.1f,%.1f,%.1f,%.1f,%.1f,%.1f,%.1f\n",
              pol[pk >> 28], caps[(pk >> 12) & 0xFFFFu], w, t->nodes[w].J, t->nodes[w].n_units, cyc[i] / 1e6,
              ph[0] / 1e6, ph[1] / 1e6, ph[2] / 1e6, ph[3] / 1e6, ph[4] / 1e6, ph[5] / 1e6, ph[6] / 1e6, ph[7] / 1e6);
    }
  }
  return SAGA_OK;
}

#if !SAGA_REPLAY_IS_WIDE
// the kernel's internal checks of every replay launched so far on the handle (syncs its stream)
saga_status replay_check(saga_trace* t) {
  if (!t->replay_status) return SAGA_OK;
  uint32_t hw[8] = {0};
  SAGA_CK(d2h(hw, t->replay_status, 32, t->stream));
  SAGA_CK(cudaStreamSynchronize(t->stream));
  if (hw[0] || hw[4]) {
    set_error("saga_replay: internal selection check failed (k_replay.cu:%u values %u %u %u)", hw[4], hw[5], hw[6], hw[7]);
    return SAGA_ERR_STATE;
  }
  return SAGA_OK;
}
#endif

}  // namespace saga
