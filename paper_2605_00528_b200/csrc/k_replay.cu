// A7 epoch-synchronous replay (rules R1-R4) with the A5 key and A6 top-k as
// device functions.  Work item = (policy, capacity, node); one CTA replays one item at a time
// (persistent CTAs pull items from an atomic counter) because time is sequential inside a
// replay while different items are independent.
//
// Per-CTA state lives in global memory (L2-resident: <= C slots of 24 B + a local-id -> slot
// map): the resident set S is a compact slot array (lid, t_last, nu, owner, stamp) and
// slot_of[lid] maps local ids to slots.  Per epoch:
//   R1  drop slots whose owner migrated away (compaction);
//   R2  |A| = #first-in-epoch records, new = those not resident; infeasible if |A| > C;
//   R3  k = |S| + new - C (EVICT_ALL: |S \ A|); stamp A n S; AEG: max-reduce tau_max and
//       size_max over cand = S \ A (eq:recency/eq:size normalisers), then fp32 keys; BELADY:
//       (nu << 32) | lid; radix-select the k largest keys (8-bit digits from the highest
//       differing bit, early exit when the pivot bucket is exactly consumed); evict; compact;
//   R4  first-in-epoch records hit iff resident, else insert; later records of the block in
//       the epoch hit; the last record of a block in the epoch writes t_last and nu.
#include "block_select.cuh"

namespace saga {
namespace {

constexpr int RT = 512;
constexpr int RW = RT / 32;
constexpr uint32_t VICTIM = 0xFFFFFFFFu;

struct NodeArr {
  uint64_t N;
  uint32_t J, n_local, n_upd, pad;
  const uint64_t* g_pos;
  const int64_t* g_t;
  const uint32_t* g_kind;
  const uint32_t* ev_e;
  const uint32_t* ev_g;
  const uint32_t* ev_inv;
  const uint32_t* ev_act;
  const uint32_t* inv_s;
  const uint32_t* lidf;
  const uint32_t* nxt;
  const uint32_t* lown;
  const uint32_t* upd_c;
};

struct ReplayArgs {
  TraceView v;
  const NodeArr* nodes;
  const uint32_t* caps;
  uint32_t n_caps;
  const uint32_t* node_list;
  uint32_t n_list;
  uint32_t pol[3];
  uint32_t n_pol;
  uint32_t n_nodes_total;
  int64_t* counters;
  float alpha, beta, gamma;
  uint32_t p_low, p_high;
  int64_t ttl_max;
  // per-CTA scratch
  uint32_t* slot_of;   // [cta][max_local]
  uint32_t* sl_lid;    // [cta][slot_cap]
  int64_t* sl_t;
  uint32_t* sl_nu;
  uint32_t* sl_own;
  uint32_t* sl_stamp;
  uint64_t* kbuf;      // [cta][slot_cap]
  uint32_t* kslot;
  uint32_t* sstate;    // [cta][n_sessions] 1 + newest call (0 = none)
  uint64_t max_local, slot_cap;
  uint32_t* work;      // work counter
  uint32_t* err;       // error flag
};

struct Scratch : BlockScratch<RT> {
  uint32_t S, nnew, u, u_end;
};

// owner state of a private session / shared prefix at the current boundary
__device__ __forceinline__ OwnerKeyIn owner_in(const ReplayArgs& a, const uint32_t* sstate, uint32_t o, uint32_t act) {
  OwnerKeyIn r;
  const TraceView& v = a.v;
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

// in-place stable compaction of the slot array keeping slots for which keep(slot) is true;
// updates slot_of for moved slots; returns the new size.  dst <= src always holds.
template <class Keep>
__device__ uint32_t compact_slots(uint32_t S, Keep keep, uint32_t* slot_of, uint32_t* sl_lid, int64_t* sl_t,
                                  uint32_t* sl_nu, uint32_t* sl_own, uint32_t* sl_stamp, Scratch& sm) {
  uint32_t run = 0;
  for (uint32_t b = 0; b < S; b += RT) {
    const uint32_t i = b + threadIdx.x;
    const bool in = i < S;
    uint32_t lid = 0, nu = 0, own = 0;
    int64_t tl = 0;
    bool k = false;
    if (in) {
      k = keep(i);
      if (k) { lid = sl_lid[i]; tl = sl_t[i]; nu = sl_nu[i]; own = sl_own[i]; }
    }
    uint32_t tot;
    const uint32_t ex = block_excl_scan<RT>(k ? 1u : 0u, &tot, sm.u32);  // has __syncthreads: reads done
    if (k) {
      const uint32_t d = run + ex;
      if (d != i) {
        sl_lid[d] = lid; sl_t[d] = tl; sl_nu[d] = nu; sl_own[d] = own; sl_stamp[d] = 0;
        slot_of[lid] = d;
      }
    }
    run += tot;
    __syncthreads();
  }
  return run;
}

__global__ void __launch_bounds__(RT) k_replay(ReplayArgs a) {
  __shared__ Scratch sm;
  __shared__ uint32_t s_item;
  __shared__ long long s_ctr[SAGA_NCOUNT];
  __shared__ unsigned long long s_hash;
  __shared__ uint32_t s_inv[32];
  const TraceView& v = a.v;
  const uint32_t cta = blockIdx.x;
  uint32_t* slot_of = a.slot_of + (uint64_t)cta * a.max_local;
  uint32_t* sl_lid = a.sl_lid + (uint64_t)cta * a.slot_cap;
  int64_t* sl_t = a.sl_t + (uint64_t)cta * a.slot_cap;
  uint32_t* sl_nu = a.sl_nu + (uint64_t)cta * a.slot_cap;
  uint32_t* sl_own = a.sl_own + (uint64_t)cta * a.slot_cap;
  uint32_t* sl_stamp = a.sl_stamp + (uint64_t)cta * a.slot_cap;
  uint64_t* kb = a.kbuf + (uint64_t)cta * a.slot_cap;
  uint32_t* ks = a.kslot + (uint64_t)cta * a.slot_cap;
  uint32_t* sstate = a.sstate + (uint64_t)cta * v.n_sessions;
  const uint32_t n_items = a.n_pol * a.n_caps * a.n_list;

  while (true) {
    if (threadIdx.x == 0) s_item = atomicAdd(a.work, 1u);
    __syncthreads();
    const uint32_t item = s_item;
    __syncthreads();
    if (item >= n_items) break;
    const uint32_t pi = item / (a.n_caps * a.n_list);
    const uint32_t ci = (item / a.n_list) % a.n_caps;
    const uint32_t ni = item % a.n_list;
    const uint32_t pol = a.pol[pi];
    const uint32_t C = a.caps[ci];
    const uint32_t w = a.node_list[ni];
    const NodeArr nd = a.nodes[w];
    if (threadIdx.x < SAGA_NCOUNT) s_ctr[threadIdx.x] = 0;
    if (threadIdx.x == 0) { s_hash = 0; sm.S = 0; sm.u = 0; }
    __syncthreads();
    uint32_t S = 0;          // |S| (uniform)
    uint32_t u = 0;          // session-update cursor (uniform)
    // per-thread counters
    long long c_hit = 0, c_miss = 0, c_mhit = 0, c_mmiss = 0, c_comp = 0, c_regen = 0;
    long long c_inv = 0, c_ev = 0, c_prot = 0, c_events = 0, c_evev = 0, c_peak = 0;
    long long infeasible = 0;
    unsigned long long hash = 0;
    for (uint32_t j = 0; j < nd.J; ++j) {
      const uint32_t e = nd.ev_e[j];
      const int64_t Te = (int64_t)e * v.epoch_us;
      // ---- session state at T_e (AEG): newest call c* with e(c*) <= e ----
      if (pol == SAGA_POLICY_AEG && j + 1 < nd.J) {
        if (threadIdx.x == 0) {
          uint32_t lo = u, hi = nd.n_upd;
          while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (v.ecall[nd.upd_c[mid]] <= e) lo = mid + 1; else hi = mid; }
          sm.u_end = lo;
        }
        __syncthreads();
        const uint32_t ue = sm.u_end;
        for (uint32_t i = u + threadIdx.x; i < ue; i += RT) {
          const uint32_t c = nd.upd_c[i];
          atomicMax(&sstate[v.call_sess[c]], c + 1);
        }
        u = ue;
        __syncthreads();
      }
      // ---- R1 invalidate sessions migrated away ----
      const uint32_t i0 = nd.ev_inv[j], i1 = nd.ev_inv[j + 1];
      if (i1 > i0 && S > 0) {
        uint32_t done = 0;
        while (done < i1 - i0) {
          const uint32_t m = min(32u, i1 - i0 - done);
          if (threadIdx.x < m) s_inv[threadIdx.x] = nd.inv_s[i0 + done + threadIdx.x];
          __syncthreads();
          uint32_t cnt = 0;
          const uint32_t S0 = S;
          auto keep = [&](uint32_t i) {
            const uint32_t o = sl_own[i];
            for (uint32_t q = 0; q < m; ++q) if (s_inv[q] == o) { slot_of[sl_lid[i]] = NONE; return false; }
            return true;
          };
          S = compact_slots(S, keep, slot_of, sl_lid, sl_t, sl_nu, sl_own, sl_stamp, sm);
          cnt = S0 - S;
          if (threadIdx.x == 0) c_inv += cnt;
          done += m;
          __syncthreads();
        }
      }
      if (j + 1 == nd.J) break;  // sentinel: trailing invalidations only
      const uint32_t g0 = nd.ev_g[j], g1 = nd.ev_g[j + 1];
      const uint64_t P0 = nd.g_pos[g0], P1 = nd.g_pos[g1];
      // ---- R2 need ----
      uint32_t nA = 0, nnew = 0;
      for (uint64_t p = P0 + threadIdx.x; p < P1; p += RT) {
        const uint32_t lf = nd.lidf[p];
        if (!(lf & LID_NFIE)) {
          ++nA;
          if (slot_of[lf & LID_MASK] == NONE) ++nnew;
        }
      }
      nA = block_reduce<RT, uint32_t>(nA, Add(), sm.u32);
      nnew = block_reduce<RT, uint32_t>(nnew, Add(), sm.u32);
      if (nA > C) { infeasible = e; break; }
      const int64_t kk = (pol == SAGA_POLICY_EVICT_ALL) ? (int64_t)S - (int64_t)(nA - nnew)
                                                        : (int64_t)S + (int64_t)nnew - (int64_t)C;
      // ---- R3 evict ----
      if (kk > 0) {
        const uint32_t stamp = j + 1;
        for (uint64_t p = P0 + threadIdx.x; p < P1; p += RT) {
          const uint32_t lf = nd.lidf[p];
          if (!(lf & LID_NFIE)) {
            const uint32_t sl = slot_of[lf & LID_MASK];
            if (sl != NONE) sl_stamp[sl] = stamp;
          }
        }
        __syncthreads();
        KeyCtx x;
        x.Te = Te; x.tau = 0; x.smax = 1;
        x.den = (int64_t)(a.p_high - a.p_low) * C;
        x.num = min(x.den, max((int64_t)0, 1000 * (int64_t)S - (int64_t)a.p_low * C));
        x.ttl_max = a.ttl_max; x.alpha = a.alpha; x.beta = a.beta; x.gamma = a.gamma;
        const uint32_t act = nd.ev_act[j];
        if (pol == SAGA_POLICY_AEG) {  // pass 1: normalisers over cand (eq:recency, eq:size)
          long long tau = 0;
          uint32_t smax = 1;
          for (uint32_t i = threadIdx.x; i < S; i += RT) {
            if (sl_stamp[i] == stamp) continue;
            tau = max(tau, (long long)(Te - sl_t[i]));
            const uint32_t o = sl_own[i];
            uint32_t sz;
            if (o >= v.n_sessions) sz = v.tlen[o - v.n_sessions];
            else sz = __ldg(&v.ci_size[sstate[o] - 1]);
            smax = max(smax, sz);
          }
          tau = block_reduce<RT, long long>(tau, Max(), sm.i64);
          smax = block_reduce<RT, uint32_t>(smax, Max(), sm.u32);
          x.tau = tau; x.smax = smax;
        }
        // pass 2: keys of cand compacted into kb / ks
        uint32_t ncand = 0;
        for (uint32_t b = 0; b < S; b += RT) {
          const uint32_t i = b + threadIdx.x;
          const bool c = i < S && sl_stamp[i] != stamp;
          uint64_t key = 0;
          if (c) {
            const uint32_t lid = sl_lid[i];
            if (pol == SAGA_POLICY_AEG) {
              const OwnerKeyIn oi = owner_in(a, sstate, sl_own[i], act);
              const float sc = wa_lru_score(x, sl_t[i], oi.size, oi.P);
              key = aeg_key(ttl_protected(x, oi), quantize_q20(sc), lid);
            } else if (pol == SAGA_POLICY_BELADY) {
              key = ((uint64_t)sl_nu[i] << 32) | lid;
            } else {
              key = lid;
            }
          }
          uint32_t tot;
          const uint32_t ex = block_excl_scan<RT>(c ? 1u : 0u, &tot, sm.u32);
          if (c) { kb[ncand + ex] = key; ks[ncand + ex] = i; }
          ncand += tot;
        }
        __syncthreads();
        const uint32_t kv = (uint32_t)(kk < (int64_t)ncand ? kk : (int64_t)ncand);
        uint64_t T = 0;
        if (pol != SAGA_POLICY_EVICT_ALL && kv < ncand) T = radix_select<RT>(kb, ncand, kv, sm);
        // pass 3: evict keys >= T
        uint32_t nv = 0, np = 0;
        unsigned long long hs = 0;
        for (uint32_t i = threadIdx.x; i < ncand; i += RT) {
          const uint64_t key = kb[i];
          if (key >= T) {
            const uint32_t sl = ks[i];
            const uint32_t lid = sl_lid[sl];
            sl_stamp[sl] = VICTIM;
            slot_of[lid] = NONE;
            hs += splitmix64(((uint64_t)e << 32) | lid);
            ++nv;
            if (pol == SAGA_POLICY_AEG && !(key >> 63)) ++np;
          }
        }
        nv = block_reduce<RT, uint32_t>(nv, Add(), sm.u32);
        np = block_reduce<RT, uint32_t>(np, Add(), sm.u32);
        hs = block_reduce<RT, unsigned long long>(hs, Add(), sm.u64);
        if (nv != kv || kv != (uint32_t)kk) { if (threadIdx.x == 0) atomicOr(a.err, 1u); }
        hash += hs;
        if (threadIdx.x == 0) { c_ev += nv; c_prot += np; c_evev += 1; }
        auto keep = [&](uint32_t i) { return sl_stamp[i] != VICTIM; };
        S = compact_slots(S, keep, slot_of, sl_lid, sl_t, sl_nu, sl_own, sl_stamp, sm);
      }
      // ---- R4 apply: phase a (hits / inserts), phase b (t_last / nu of the last record) ----
      if (threadIdx.x == 0) sm.nnew = 0;
      __syncthreads();
      for (uint32_t g = g0; g < g1; ++g) {
        const uint64_t q0 = nd.g_pos[g], q1 = nd.g_pos[g + 1];
        const bool mig = nd.g_kind[g] != 0;
        for (uint64_t p = q0 + threadIdx.x; p < q1; p += RT) {
          const uint32_t lf = nd.lidf[p];
          const uint32_t lid = lf & LID_MASK;
          bool hit = true;
          if (!(lf & LID_NFIE)) {
            if (slot_of[lid] == NONE) {
              hit = false;
              const uint32_t sl = S + atomicAdd(&sm.nnew, 1u);
              slot_of[lid] = sl;
              sl_lid[sl] = lid;
              sl_own[sl] = nd.lown[lid];
              sl_stamp[sl] = 0;
            }
          }
          if (hit) { if (mig) ++c_mhit; else ++c_hit; }
          else {
            if (mig) ++c_mmiss; else { ++c_miss; if (!(lf & LID_FTN)) ++c_regen; }
            if (lf & LID_FTN) ++c_comp;
          }
        }
      }
      __syncthreads();
      S += sm.nnew;
      for (uint32_t g = g0; g < g1; ++g) {
        const uint64_t q0 = nd.g_pos[g], q1 = nd.g_pos[g + 1];
        const int64_t tv = nd.g_t[g];
        for (uint64_t p = q0 + threadIdx.x; p < q1; p += RT) {
          const uint32_t nu = nd.nxt[p];
          if ((uint64_t)nu >= P1) {  // last record of the block in this epoch (INF included)
            const uint32_t sl = slot_of[nd.lidf[p] & LID_MASK];
            sl_t[sl] = tv;
            sl_nu[sl] = nu;
          }
        }
      }
      __syncthreads();
      c_peak = max(c_peak, (long long)S);
      c_events += 1;
    }
    // ---- counters ----
    const long long acc = block_reduce<RT, long long>(c_hit + c_miss + c_mhit + c_mmiss, Add(), sm.i64);
    const long long h1 = block_reduce<RT, long long>(c_hit, Add(), sm.i64);
    const long long m1 = block_reduce<RT, long long>(c_miss, Add(), sm.i64);
    const long long h2 = block_reduce<RT, long long>(c_mhit, Add(), sm.i64);
    const long long m2 = block_reduce<RT, long long>(c_mmiss, Add(), sm.i64);
    const long long cp = block_reduce<RT, long long>(c_comp, Add(), sm.i64);
    const long long rg = block_reduce<RT, long long>(c_regen, Add(), sm.i64);
    if (threadIdx.x == 0) {
      int64_t* out = a.counters + (((uint64_t)pi * a.n_caps + ci) * a.n_nodes_total + w) * SAGA_NCOUNT;
      out[SAGA_C_ACCESSES] = acc;
      out[SAGA_C_HITS] = h1;
      out[SAGA_C_MISSES] = m1;
      out[SAGA_C_MIG_HITS] = h2;
      out[SAGA_C_MIG_MISSES] = m2;
      out[SAGA_C_COMPULSORY] = cp;
      out[SAGA_C_INVALIDATED] = c_inv;
      out[SAGA_C_EVICTIONS] = c_ev;
      out[SAGA_C_EVICT_PROTECTED] = c_prot;
      out[SAGA_C_EVICT_EVENTS] = c_evev;
      out[SAGA_C_REGEN_TOKENS] = rg * (long long)v.btok;
      out[SAGA_C_REGEN_US] = rg * ((long long)v.btok * 1000000 / (long long)v.prefill_tok_s);
      out[SAGA_C_VICTIM_HASH] = (long long)hash;
      out[SAGA_C_INFEASIBLE_EPOCH] = infeasible;
      out[SAGA_C_PEAK_RESIDENT] = c_peak;
      out[SAGA_C_EVENT_EPOCHS] = c_events;
    }
    // ---- reset per-CTA state for the next item ----
    for (uint32_t i = threadIdx.x; i < S; i += RT) slot_of[sl_lid[i]] = NONE;
    if (pol == SAGA_POLICY_AEG)
      for (uint32_t i = threadIdx.x; i < u; i += RT) sstate[v.call_sess[nd.upd_c[i]]] = 0;
    __syncthreads();
  }
}

}  // namespace

saga_status run_replay(saga_trace* t, const saga_replay_cfg* cfg, const uint32_t* caps, uint32_t n_caps,
                       const uint32_t* nodes, uint32_t n_owned, int64_t* counters, cudaStream_t s) {
  const TraceView& v = t->v;
  uint32_t pol[3], n_pol = 0;
  for (uint32_t p : {1u, 2u, 4u}) if (cfg->policy_mask & p) pol[n_pol++] = p;
  if (n_pol == 0 || n_caps == 0 || n_owned == 0) return SAGA_OK;
  uint32_t cap_max = 0;
  for (uint32_t i = 0; i < n_caps; ++i) cap_max = std::max(cap_max, caps[i]);
  uint64_t max_local = 1;
  std::vector<NodeArr> hn(t->n_nodes);
  for (uint32_t i = 0; i < n_owned; ++i) {
    const NodeDev& nd = t->nodes[nodes[i]];
    max_local = std::max<uint64_t>(max_local, nd.n_local);
  }
  for (uint32_t w = 0; w < t->n_nodes; ++w) {
    const NodeDev& nd = t->nodes[w];
    NodeArr x{};
    x.N = nd.N; x.J = nd.J; x.n_local = nd.n_local; x.n_upd = nd.n_upd;
    x.g_pos = nd.g_pos; x.g_t = nd.g_t; x.g_kind = nd.g_kind; x.ev_e = nd.ev_e; x.ev_g = nd.ev_g;
    x.ev_inv = nd.ev_inv; x.ev_act = nd.ev_act; x.inv_s = nd.inv_s; x.lidf = nd.lidf; x.nxt = nd.nxt;
    x.lown = nd.lown; x.upd_c = nd.upd_c;
    hn[w] = x;
  }
  const uint32_t n_items = n_pol * n_caps * n_owned;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t grid = std::min<uint32_t>(n_items, (uint32_t)nsm * 2);
  const uint64_t slot_cap = (uint64_t)cap_max + 1;
  // scratch
  NodeArr* d_nodes = nullptr;
  uint32_t *d_caps = nullptr, *d_list = nullptr, *work = nullptr, *err = nullptr;
  uint32_t *slot_of = nullptr, *sl_lid = nullptr, *sl_nu = nullptr, *sl_own = nullptr, *sl_stamp = nullptr, *kslot = nullptr,
           *sstate = nullptr;
  int64_t* sl_t = nullptr;
  uint64_t* kbuf = nullptr;
  SAGA_CK(cudaMallocAsync((void**)&d_nodes, sizeof(NodeArr) * t->n_nodes, s));
  SAGA_CK(cudaMallocAsync((void**)&d_caps, 4 * n_caps, s));
  SAGA_CK(cudaMallocAsync((void**)&d_list, 4 * n_owned, s));
  SAGA_CK(cudaMallocAsync((void**)&work, 8, s));
  err = work + 1;
  SAGA_CK(cudaMallocAsync((void**)&slot_of, 4 * max_local * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&sl_lid, 4 * slot_cap * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&sl_t, 8 * slot_cap * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&sl_nu, 4 * slot_cap * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&sl_own, 4 * slot_cap * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&sl_stamp, 4 * slot_cap * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&kbuf, 8 * slot_cap * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&kslot, 4 * slot_cap * grid, s));
  SAGA_CK(cudaMallocAsync((void**)&sstate, 4 * (uint64_t)std::max(v.n_sessions, 1u) * grid, s));
  SAGA_CK(cudaMemcpyAsync(d_nodes, hn.data(), sizeof(NodeArr) * t->n_nodes, cudaMemcpyHostToDevice, s));
  SAGA_CK(cudaMemcpyAsync(d_caps, caps, 4 * n_caps, cudaMemcpyHostToDevice, s));
  SAGA_CK(cudaMemcpyAsync(d_list, nodes, 4 * n_owned, cudaMemcpyHostToDevice, s));
  SAGA_CK(cudaMemsetAsync(work, 0, 8, s));
  SAGA_CK(cudaMemsetAsync(slot_of, 0xFF, 4 * max_local * grid, s));
  SAGA_CK(cudaMemsetAsync(sstate, 0, 4 * (uint64_t)std::max(v.n_sessions, 1u) * grid, s));
  ReplayArgs a{};
  a.v = v;
  a.nodes = d_nodes; a.caps = d_caps; a.n_caps = n_caps; a.node_list = d_list; a.n_list = n_owned;
  a.pol[0] = pol[0]; a.pol[1] = n_pol > 1 ? pol[1] : 0; a.pol[2] = n_pol > 2 ? pol[2] : 0; a.n_pol = n_pol;
  a.n_nodes_total = t->n_nodes; a.counters = counters;
  a.alpha = cfg->alpha; a.beta = cfg->beta; a.gamma = cfg->gamma;
  a.p_low = cfg->p_low_pm; a.p_high = cfg->p_high_pm; a.ttl_max = cfg->ttl_max_us;
  a.slot_of = slot_of; a.sl_lid = sl_lid; a.sl_t = sl_t; a.sl_nu = sl_nu; a.sl_own = sl_own; a.sl_stamp = sl_stamp;
  a.kbuf = kbuf; a.kslot = kslot; a.sstate = sstate; a.max_local = max_local; a.slot_cap = slot_cap;
  a.work = work; a.err = err;
  prof_begin(SAGA_PROF_REPLAY, s);
  k_replay<<<grid, RT, 0, s>>>(a);
  prof_end(SAGA_PROF_REPLAY, s);
  count_launch();
  SAGA_CK_LAUNCH();
  uint32_t herr = 0;
  SAGA_CK(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(d_nodes, s); cudaFreeAsync(d_caps, s); cudaFreeAsync(d_list, s);
  cudaFreeAsync(slot_of, s); cudaFreeAsync(sl_lid, s); cudaFreeAsync(sl_t, s); cudaFreeAsync(sl_nu, s);
  cudaFreeAsync(sl_own, s); cudaFreeAsync(sl_stamp, s); cudaFreeAsync(kbuf, s); cudaFreeAsync(kslot, s);
  cudaFreeAsync(sstate, s);
  cudaFreeAsync(work, s);
  SAGA_CK(cudaStreamSynchronize(s));
  if (herr) { set_error("saga_replay: internal selection check failed"); return SAGA_ERR_STATE; }
  return SAGA_OK;
}

}  // namespace saga
