// A2 placement on the device: epoch-synchronous session routing (eq:routing) and
// randomised work stealing with the AND trigger and anti-thrash safeguards (P:748-758, P:361,
// P:766).  Rules P1-P6 of DESIGN.md §4.2.
//
// The method is sequential in time (every boundary depends on the previous one), so this is a
// single warp: lane w owns cache node w (n_nodes <= 32).  Queues live in shared memory
// (per-node FIFO arrays of (call | started, remaining us)); per-session state in global memory.
// Epochs in which nothing can happen but service (no admission, every queued call already in
// service so no victim can exist) are advanced in closed form, so the loop visits only
// admission epochs and epochs with waiting calls.
#include "saga_internal.cuh"

namespace saga {
namespace {

constexpr uint32_t STARTED = 1u << 31;
constexpr uint32_t CMASK = STARTED - 1;
constexpr uint64_t PHI = 0x9E3779B97F4A7C15ull;

struct PlaceArgs {
  TraceView v;
  uint32_t kappa, theta_pm, rmax_pm, qcap;
  int64_t t_idle_us;
  uint64_t seed;
  uint8_t* node_of;
  Mig* migs;
  uint32_t mig_cap;
  ActRec* act;
  uint32_t act_cap;
  uint32_t* out_n;               // [0] n_mig, [1] n_act, [2] error (1 queue overflow, 2 log overflow)
  unsigned long long* out_stats; // [0] steals, [1] reroutes
  volatile int32_t* aff;
  volatile int32_t* last_c;
  volatile uint8_t* moved;
  volatile uint8_t* fin;
};

__device__ __forceinline__ int64_t warp_min64(int64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = min(x, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)x, o));
  return x;
}

__global__ void __launch_bounds__(32, 1) k_place(PlaceArgs a) {
  extern __shared__ uint32_t smem[];
  const uint32_t W = a.v.n_nodes, lane = threadIdx.x, K = a.kappa, Q = a.qcap;
  const int64_t E = a.v.epoch_us;
  uint32_t* qc = smem + lane * Q;                       // call | STARTED
  uint32_t* qr = smem + W * Q + lane * Q;               // remaining work (us)
  __shared__ int32_t cnt[32][32];                       // sessions with aff = w, !fin, by type
  __shared__ int32_t act_tot[32];
  __shared__ uint32_t xfer_c[64], xfer_r[64];
  __shared__ uint32_t xfer_n, n_mig, n_act, errf;
  __shared__ unsigned long long steals, reroutes;
  for (int i = lane; i < 32 * 32; i += 32) (&cnt[0][0])[i] = 0;
  act_tot[lane] = 0;
  if (lane == 0) { n_mig = 0; n_act = 0; errf = 0; steals = 0; reroutes = 0; xfer_n = 0; }
  __syncwarp();
  const bool act_lane = lane < W;
  uint32_t len = 0;
  int64_t L = 0, idle = 0;
  const TraceView& v = a.v;
  uint32_t next = 0;
  uint64_t e = 1;

  auto recompute_L = [&]() {
    int64_t s = 0;
    for (uint32_t i = 0; i < len; ++i) s += min((int64_t)qr[i], E);
    L = s;
  };
  // oldest pending (never served) call of a session that is not `moved` and has no call in
  // service in this queue (DESIGN.md R-steal)
  auto find_stealable = [&]() -> int32_t {
    for (uint32_t i = 0; i < len; ++i) {
      uint32_t x = qc[i];
      if (x & STARTED) continue;
      uint32_t s = v.call_sess[x & CMASK];
      if (a.moved[s]) continue;
      bool busy = false;
      for (uint32_t j = 0; j < len; ++j)
        if ((qc[j] & STARTED) && v.call_sess[qc[j] & CMASK] == s) { busy = true; break; }
      if (!busy) return (int32_t)s;
    }
    return -1;
  };

  while (true) {
    bool any = __ballot_sync(0xffffffffu, act_lane && len > 0) != 0;
    if (next >= v.n_calls && !any) break;
    const int64_t Te = (int64_t)e * E;
    bool got = false;
    // ---------------- P1 service: the first kappa calls progress by one epoch ----------------
    if (act_lane) {
      int64_t served = 0;
      uint32_t k = 0;
      for (uint32_t i = 0; i < len; ++i) {
        uint32_t x = qc[i], r = qr[i];
        if (i < K) {
          uint32_t d = (uint32_t)min((int64_t)r, E);
          r -= d;
          served += d;
          x |= STARTED;
          if (r == 0) { a.moved[v.call_sess[x & CMASK]] = 0; continue; }
        }
        qc[k] = x; qr[k] = r; ++k;
      }
      len = k;
      idle = served == 0 ? idle + 1 : 0;
      recompute_L();
    }
    __syncwarp();
    // ---------------- P2 steal: idle thief AND load-ratio guard (P:361, P:766(a)) ----------------
    uint32_t thieves = __ballot_sync(0xffffffffu, act_lane && idle * E >= a.t_idle_us);
    bool unst = false;
    if (act_lane) for (uint32_t i = 0; i < len; ++i) if (!(qc[i] & STARTED)) { unst = true; break; }
    if (thieves && __ballot_sync(0xffffffffu, unst)) {
      while (thieves) {
        const uint32_t th = __ffs(thieves) - 1;
        thieves &= thieves - 1;
        int64_t Lmin = warp_min64(act_lane ? L : INT64_MAX);
        int32_t cand = -1;
        if (act_lane && lane != th && 1000 * L > (int64_t)a.rmax_pm * Lmin) cand = find_stealable();
        uint32_t O = __ballot_sync(0xffffffffu, cand >= 0);
        if (!O) continue;
        uint64_t r = splitmix64(a.seed ^ (e * PHI) ^ (uint64_t)th) % (uint64_t)__popc(O);
        uint32_t vv = 0, cntb = 0;
        for (uint32_t m = O; m; m &= m - 1) { if (cntb == r) { vv = __ffs(m) - 1; break; } ++cntb; }
        const int32_t s = __shfl_sync(0xffffffffu, cand, vv);
        if (lane == vv) {
          uint32_t k = 0, m = 0;
          for (uint32_t i = 0; i < len; ++i) {
            uint32_t x = qc[i];
            if (v.call_sess[x & CMASK] == (uint32_t)s) {
              if (m < 64) { xfer_c[m] = x; xfer_r[m] = qr[i]; }
              ++m;
            } else { qc[k] = x; qr[k] = qr[i]; ++k; }
          }
          if (m > 64) atomicOr(&errf, 4u);
          len = k;
          xfer_n = m;
          recompute_L();
        }
        __syncwarp();
        if (lane == th) {
          uint32_t m = min(xfer_n, 64u);
          for (uint32_t i = 0; i < m; ++i) {
            if (len >= Q) { atomicOr(&errf, 1u); break; }
            qc[len] = xfer_c[i]; qr[len] = xfer_r[i]; ++len;
          }
          recompute_L();
          idle = 0;
          got = true;
        }
        if (lane == 0) {
          uint32_t ty = v.styp[s];
          if (!a.fin[s]) {  // s is counted at its current affinity node
            const int32_t ao = a.aff[s];
            cnt[ao][ty]--; act_tot[ao]--; cnt[th][ty]++; act_tot[th]++;
          }
          a.aff[s] = (int32_t)th;
          a.moved[s] = 1;
          if (n_mig < a.mig_cap) a.migs[n_mig] = Mig{(uint32_t)e, (uint32_t)s, vv, th};
          else errf |= 2u;
          ++n_mig;
          ++steals;
        }
        __syncwarp();
      }
    }
    // ---------------- P3 route the calls admitted at T_e (eq:routing) ----------------
    while (next < v.n_calls && v.ecall[next] == e) {
      const uint32_t c = next + lane;
      const bool valid = c < v.n_calls && v.ecall[c] == e;
      const uint32_t nb = __popc(__ballot_sync(0xffffffffu, valid));
      uint32_t s = 0, vc = 0, ty = 0, newt = 0, prompt = 0, outt = 0;
      bool lastc = false, termc = false;
      int64_t tendc = 0, ttlc = 0;
      int32_t aff = -1, lc = -1;
      bool fin = false, term_lv = true;
      int64_t tend_lv = 0, ttl_lv = 0;
      if (valid) {
        s = v.call_sess[c]; vc = v.call_v[c]; ty = v.styp[s];
        newt = v.call_new[c]; prompt = v.call_prompt[c]; outt = v.call_out[c];
        lastc = v.call_last[c]; termc = v.term[vc]; tendc = v.tend[c]; ttlc = v.ttl[vc];
        aff = a.aff[s]; lc = a.last_c[s]; fin = a.fin[s];
        if (lc >= 0) { uint32_t lv = v.call_v[lc]; term_lv = v.term[lv]; tend_lv = v.tend[lc]; ttl_lv = v.ttl[lv]; }
      }
      const uint32_t same = __match_any_sync(0xffffffffu, valid ? s : 0xFFFFFFFFu);
      for (uint32_t i = 0; i < nb; ++i) {
        // lane i's view of its session state
        const int32_t ws = __shfl_sync(0xffffffffu, aff, i);
        bool cached_i = (aff >= 0) && !term_lv && (Te - tend_lv <= ttl_lv);   // Alg. 1 with m = 0
        const bool cached = __shfl_sync(0xffffffffu, cached_i, i);
        int64_t Lws = __shfl_sync(0xffffffffu, (long long)L, ws >= 0 ? ws : 0);
        uint32_t w;
        if (cached && 1000 * Lws < (int64_t)a.theta_pm * (int64_t)K * E) {
          w = (uint32_t)ws;
        } else {  // argmin load; ties -> fewer active sessions -> lowest id
          int64_t kL = act_lane ? L : INT64_MAX;
          int32_t kA = act_lane ? act_tot[lane] : INT32_MAX;
          uint32_t kW = lane;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            int64_t oL = __shfl_xor_sync(0xffffffffu, (long long)kL, o);
            int32_t oA = __shfl_xor_sync(0xffffffffu, kA, o);
            uint32_t oW = __shfl_xor_sync(0xffffffffu, kW, o);
            if (oL < kL || (oL == kL && (oA < kA || (oA == kA && oW < kW)))) { kL = oL; kA = oA; kW = oW; }
          }
          w = kW;
        }
        const uint32_t ci = __shfl_sync(0xffffffffu, c, i);
        const uint32_t si = __shfl_sync(0xffffffffu, s, i);
        const uint32_t tyi = __shfl_sync(0xffffffffu, ty, i);
        const bool fin_old = __shfl_sync(0xffffffffu, fin, i);
        const bool f_new = __shfl_sync(0xffffffffu, (int)(lastc || termc), i);
        const uint32_t pf = __shfl_sync(0xffffffffu, (cached && (int32_t)w == ws) ? newt : prompt, i);
        const uint32_t oi = __shfl_sync(0xffffffffu, outt, i);
        const int64_t omega = ceil_div64((int64_t)pf * 1000000, v.prefill_tok_s) +
                              ceil_div64((int64_t)oi * 1000000, v.decode_tok_s);
        if (lane == w) {
          if (len >= Q) atomicOr(&errf, 1u);
          else { qc[len] = ci; qr[len] = (uint32_t)omega; ++len; L += min(omega, E); }
          got = true;
        }
        if (lane == 0) {
          if (ws >= 0 && w != (uint32_t)ws) ++reroutes;
          if (ws >= 0 && !fin_old) { cnt[ws][tyi]--; act_tot[ws]--; }
          if (!f_new) { cnt[w][tyi]++; act_tot[w]++; }
        }
        if (lane == i) a.node_of[ci] = (uint8_t)w;
        // forward the post-call state to later lanes of the same session in this batch
        const uint32_t vci = __shfl_sync(0xffffffffu, vc, i);
        const int64_t tendi = __shfl_sync(0xffffffffu, (long long)tendc, i);
        const int64_t ttli = __shfl_sync(0xffffffffu, (long long)ttlc, i);
        const bool termi = __shfl_sync(0xffffffffu, (int)termc, i);
        if (valid && (lane == i || (lane > i && si == s && ((same >> i) & 1u)))) {
          aff = (int32_t)w; lc = (int32_t)ci; fin = f_new;
          term_lv = termi; tend_lv = tendi; ttl_lv = ttli;
        }
        (void)vci;
        __syncwarp();
      }
      // the last lane of each session in the batch publishes the session state
      const uint32_t later = same & ~((2u << lane) - 1u);
      if (valid && later == 0) { a.aff[s] = aff; a.last_c[s] = lc; a.fin[s] = fin; }
      __syncwarp();
      next += nb;
    }
    // ---------------- act(w, a) log for nodes that received records at this boundary ----------------
    const uint32_t gm = __ballot_sync(0xffffffffu, act_lane && got);
    if (gm) {
      uint32_t mask = 0;
      if (act_lane) for (uint32_t t2 = 0; t2 < v.n_types; ++t2) if (cnt[lane][t2] > 0) mask |= 1u << t2;
      uint32_t base = n_act;
      if (got) {
        uint32_t pos = base + __popc(gm & ((1u << lane) - 1u));
        if (pos < a.act_cap) a.act[pos] = ActRec{(uint32_t)e, lane, mask, 0u};
        else atomicOr(&errf, 2u);
      }
      __syncwarp();
      if (lane == 0) n_act = base + __popc(gm);
      __syncwarp();
    }
    if (errf & 1u) break;
    // ---------------- closed-form advance over service-only epochs ----------------
    const bool all_fit = __ballot_sync(0xffffffffu, act_lane && len > K) == 0;
    if (all_fit) {
      uint64_t e_adm = next < v.n_calls ? (uint64_t)v.ecall[next] : UINT64_MAX;
      uint64_t k;
      if (e_adm == UINT64_MAX) {
        int64_t mx = 0;
        if (act_lane) for (uint32_t i = 0; i < len; ++i) mx = max(mx, (int64_t)qr[i]);
        mx = -warp_min64(-mx);
        k = (uint64_t)ceil_div64(mx, E);
      } else {
        k = e_adm - 1 - e;
      }
      if (k > 0 && act_lane) {
        const int64_t budget = (int64_t)k * E;
        int64_t mx = 0;
        uint32_t kk = 0;
        for (uint32_t i = 0; i < len; ++i) {
          int64_t r = qr[i];
          mx = max(mx, r);
          if (r <= budget) { a.moved[v.call_sess[qc[i] & CMASK]] = 0; continue; }
          qc[kk] = qc[i] | STARTED; qr[kk] = (uint32_t)(r - budget); ++kk;
        }
        if (len == 0) idle += (int64_t)k;
        else {
          uint64_t m = (uint64_t)ceil_div64(mx, E);
          idle = m >= k ? 0 : (int64_t)(k - m);
        }
        len = kk;
        recompute_L();
      }
      e += k;
    }
    __syncwarp();
    ++e;
  }
  if (lane == 0) {
    a.out_n[0] = n_mig;
    a.out_n[1] = n_act;
    a.out_n[2] = errf;
    a.out_stats[0] = steals;
    a.out_stats[1] = reroutes;
  }
}

}  // namespace

saga_status run_placement(saga_trace* t) {
  const TraceView& v = t->v;
  const uint32_t W = v.n_nodes;
  size_t max_smem = 200 * 1024;
  uint32_t qcap = (uint32_t)(max_smem / (8ull * W));
  if (qcap > 65536) qcap = 65536;
  size_t smem = size_t(qcap) * W * 8;
  uint32_t mig_cap = v.n_calls + v.n_sessions + 64;
  uint32_t act_cap = v.n_calls + mig_cap + 64;
  t->node_of = dalloc<uint8_t>(t, v.n_calls);
  t->migs = dalloc<Mig>(t, mig_cap);
  t->act = dalloc<ActRec>(t, act_cap);
  uint32_t* out_n = dalloc<uint32_t>(t, 4);
  unsigned long long* out_stats = dalloc<unsigned long long>(t, 2);
  int32_t* aff = dalloc<int32_t>(t, v.n_sessions);
  int32_t* lastc = dalloc<int32_t>(t, v.n_sessions);
  uint8_t* moved = dalloc<uint8_t>(t, v.n_sessions);
  uint8_t* fin = dalloc<uint8_t>(t, v.n_sessions);
  if (!t->node_of || !t->migs || !t->act || !out_n || !out_stats || !aff || !lastc || !moved || !fin) {
    set_error("saga_load_trace: out of device memory (placement)");
    return SAGA_ERR_OOM;
  }
  SAGA_CK(cudaMemsetAsync(aff, 0xFF, size_t(v.n_sessions) * 4, t->stream));
  SAGA_CK(cudaMemsetAsync(lastc, 0xFF, size_t(v.n_sessions) * 4, t->stream));
  SAGA_CK(cudaMemsetAsync(moved, 0, v.n_sessions, t->stream));
  SAGA_CK(cudaMemsetAsync(fin, 0, v.n_sessions, t->stream));
  SAGA_CK(cudaMemsetAsync(out_n, 0, 16, t->stream));
  PlaceArgs a{};
  a.v = v;
  a.kappa = t->pcfg.kappa; a.theta_pm = t->pcfg.theta_pm; a.rmax_pm = t->pcfg.rmax_pm; a.qcap = qcap;
  a.t_idle_us = t->pcfg.t_idle_us; a.seed = t->pcfg.seed;
  a.node_of = t->node_of; a.migs = t->migs; a.mig_cap = mig_cap; a.act = t->act; a.act_cap = act_cap;
  a.out_n = out_n; a.out_stats = out_stats; a.aff = aff; a.last_c = lastc; a.moved = moved; a.fin = fin;
  SAGA_CK(cudaFuncSetAttribute(k_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prof_begin(SAGA_PROF_PLACE, t->stream);
  k_place<<<1, 32, smem, t->stream>>>(a);
  prof_end(SAGA_PROF_PLACE, t->stream);
  count_launch();
  SAGA_CK_LAUNCH();
  uint32_t hn[4];
  unsigned long long hs[2];
  SAGA_CK(cudaMemcpyAsync(hn, out_n, 16, cudaMemcpyDeviceToHost, t->stream));
  SAGA_CK(cudaMemcpyAsync(hs, out_stats, 16, cudaMemcpyDeviceToHost, t->stream));
  SAGA_CK(cudaStreamSynchronize(t->stream));
  if (hn[2]) {
    set_error("saga_load_trace: placement limit exceeded (%s); queue capacity %u calls per node",
              (hn[2] & 1u) ? "node queue overflow" : ((hn[2] & 4u) ? "steal transfer > 64 calls" : "log overflow"),
              qcap);
    return SAGA_ERR_STATE;
  }
  t->n_mig = hn[0];
  t->n_act = hn[1];
  t->n_steals = (int64_t)hs[0];
  t->n_reroutes = (int64_t)hs[1];
  return SAGA_OK;
}

}  // namespace saga
