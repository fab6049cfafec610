// A2 placement on the device: epoch-synchronous session routing (eq:routing) and
// randomised work stealing with the AND trigger and anti-thrash safeguards (P:748-758, P:361,
// P:766).  Rules P1-P6 of DESIGN.md §4.2.
//
// The method is sequential in time (every boundary depends on the previous one), so this is a
// single warp: lane w owns cache node w (n_nodes <= 32).  Its cost is the latency of one
// boundary, so the kernel is built around keeping that latency short:
//   * per-call inputs are packed by a parallel pre-pass into one 32-byte record (session, e(c),
//     work if routed to a cached affinity / elsewhere, type and flags, ttl, tool start);
//   * per-session routing state is one 16-byte record (affinity, fin, terminal/ttl/tool start of
//     the session's last call), held in shared memory when the session table fits;
//   * the records of the next 32 calls (and their sessions) are loaded while the current boundary
//     is still being processed, so a boundary normally waits on no global-memory round trip;
//   * queues are per-node FIFO arrays in shared memory; epochs in which nothing can happen but
//     service (no admission, every queued call in service) are advanced in closed form.
#include "saga_internal.cuh"

namespace saga {
namespace {

constexpr uint32_t STARTED = 1u << 31;
constexpr uint32_t CMASK = STARTED - 1;
constexpr uint64_t PHI = 0x9E3779B97F4A7C15ull;
constexpr uint32_t F_FNEW = 1u << 16;  // is_last || terminal(v): the session finishes with this call
constexpr uint32_t F_TERM = 1u << 17;  // terminal(v)

struct __align__(16) CallRec {
  uint32_t s, e, om_cached, om_full;  // work (us) if routed to its cached affinity / elsewhere
  uint32_t tyf;                       // session type | F_FNEW | F_TERM
  uint32_t ttl;                       // ttl_base of the call's AEG node (<= 1e9, validated)
  int64_t tend;                       // tool start t_c + prefill(new) + decode(out)
};
constexpr uint32_t S_FIN = 1u << 30;   // session finished (no affinity count)
constexpr uint32_t S_TERM = 1u << 31;  // the last call's AEG node is terminal
struct __align__(16) SessRec {
  int32_t aff;     // affinity node or -1
  uint32_t ttlf;   // ttl_base of the last call's node (< 2^30) | S_FIN | S_TERM
  int64_t tend_lv; // tool start of the last call
};

struct PlaceArgs {
  TraceView v;
  const CallRec* rec;
  uint32_t kappa, theta_pm, rmax_pm, qcap;
  int64_t t_idle_us;
  uint64_t seed;
  uint8_t* node_of;
  Mig* migs;
  uint32_t mig_cap;
  ActRec* act;
  uint32_t act_cap;
  uint32_t* out_n;               // [0] n_mig, [1] n_act, [2] error (1 queue overflow, 2 log overflow, 4 transfer)
  unsigned long long* out_stats; // [0] steals, [1] reroutes
  SessRec* sess_g;               // session table in global memory (when it does not fit in smem)
  uint8_t* moved_g;
};

__global__ void k_call_rec(TraceView v, CallRec* rec) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.n_calls; c += gridDim.x * blockDim.x) {
    const uint32_t s = v.call_sess[c], vc = v.call_v[c];
    const int64_t dec = ceil_div64((int64_t)v.call_out[c] * 1000000, v.decode_tok_s);
    CallRec r;
    r.s = s;
    r.e = v.ecall[c];
    r.om_cached = (uint32_t)(ceil_div64((int64_t)v.call_new[c] * 1000000, v.prefill_tok_s) + dec);
    r.om_full = (uint32_t)(ceil_div64((int64_t)v.call_prompt[c] * 1000000, v.prefill_tok_s) + dec);
    const bool term = v.term[vc] != 0;
    r.tyf = (uint32_t)v.styp[s] | ((v.call_last[c] || term) ? F_FNEW : 0u) | (term ? F_TERM : 0u);
    r.ttl = (uint32_t)call_ttl_base(v, c);  // per-call override or the node's value
    r.tend = v.tend[c];
    rec[c] = r;
  }
}

__device__ __forceinline__ int64_t warp_min64(int64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = min(x, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)x, o));
  return x;
}

// Per-node queue (lane w owns node w), an exact reformulation of the FIFO with kappa servers:
//   S  calls in service (the FIFO's first min(len, kappa) entries; every one progresses by
//      min(r, E) each epoch), kept sorted by a finish threshold F = r + V where V is the node's
//      virtual time (+E per epoch), so an epoch costs O(1 + completions) instead of O(len);
//   W  waiting calls (never served) in FIFO order with their full work r.
// L = sum over the queue of min(r, E) = sum_S min(F - V, E) + LW, with LW = sum_W min(r, E).
template <bool SS>
__global__ void __launch_bounds__(32, 1) k_place(PlaceArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t W = a.v.n_nodes, lane = threadIdx.x, K = a.kappa, Q = a.qcap;
  const int64_t E = a.v.epoch_us;
  const TraceView& v = a.v;
  const uint32_t NS = v.n_sessions, NC = v.n_calls;
  SessRec* sess = SS ? reinterpret_cast<SessRec*>(smem_raw) : a.sess_g;
  uint8_t* moved = SS ? smem_raw + (size_t)NS * sizeof(SessRec) : a.moved_g;
  size_t off = SS ? (((size_t)NS * (sizeof(SessRec) + 1) + 15) & ~(size_t)15) : 0;
  int64_t* sF = reinterpret_cast<int64_t*>(smem_raw + off) + (size_t)lane * K;     // S: finish thresholds
  off += (size_t)W * K * 8;
  uint32_t* sS = reinterpret_cast<uint32_t*>(smem_raw + off) + (size_t)lane * K;   // S: sessions
  off += (size_t)W * K * 4;
  uint32_t* wS = reinterpret_cast<uint32_t*>(smem_raw + off) + (size_t)lane * Q;   // W: sessions (ring)
  off += (size_t)W * Q * 4;
  uint32_t* wR = reinterpret_cast<uint32_t*>(smem_raw + off) + (size_t)lane * Q;   // W: work (us)
  __shared__ int32_t cnt[32][32];                       // sessions with aff = w, !fin, by type
  // call records streamed ahead by TMA bulk copies: chunk j (calls [256 j, 256 j + 256)) lives
  // in buffer j & 1; chunk j + 1 is requested when chunk j is first touched
  constexpr uint32_t CH = 256;
  __shared__ __align__(16) CallRec ring[2][CH];
  __shared__ __align__(8) uint64_t rbar[2];
  __shared__ uint32_t xfer_s[64], xfer_r[64];
  __shared__ uint32_t xfer_n, n_mig, n_act, errf;
  __shared__ unsigned long long steals, reroutes;
  for (int i = lane; i < 32 * 32; i += 32) (&cnt[0][0])[i] = 0;
  if (SS) {
    const SessRec init{-1, 0u, 0ll};
    for (uint32_t i = lane; i < NS; i += 32) { sess[i] = init; moved[i] = 0; }
  }
  if (lane == 0) { n_mig = 0; n_act = 0; errf = 0; steals = 0; reroutes = 0; xfer_n = 0; }
  const uint32_t n_chunks = (NC + CH - 1) / CH;
  auto fetch = [&](uint32_t j) {  // lane 0
    const uint32_t n = min(CH, NC - j * CH);
    tma_load_1d(&ring[j & 1][0], a.rec + (size_t)j * CH, n * (uint32_t)sizeof(CallRec), &rbar[j & 1]);
  };
  if (lane == 0) {
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    if (n_chunks > 0) fetch(0);
    if (n_chunks > 1) fetch(1);
  }
  __syncwarp();
  uint32_t have = n_chunks > 1 ? 2u : n_chunks;  // chunks requested so far
  uint32_t ready = 0;                            // chunks known complete
  // make calls [c0, c0 + 32) readable: wait for their chunks, request the chunk after them
  auto ensure = [&](uint32_t c0) {
    const uint32_t jl = min((c0 + 31) / CH, n_chunks ? n_chunks - 1 : 0);
    // chunk h reuses the buffer of chunk h - 2, free once no call below chunk h - 1 is needed
    while (have < n_chunks && have <= jl + 1 && have - 2 < c0 / CH) {
      if (lane == 0) fetch(have);
      ++have;
    }
    __syncwarp();
    while (ready <= jl && ready < n_chunks) {
      mbar_wait(&rbar[ready & 1], (ready >> 1) & 1u);
      ++ready;
    }
  };
  const bool act_lane = lane < W;
  uint32_t nS = 0, nW = 0, wh = 0, sh = 0;  // |S|, |W|, ring heads of W and S (S is a ring of K)
  int64_t V = 0, LW = 0, L = 0, idle = 0;
  uint32_t next = 0;
  uint64_t e = 1;

  // prefetched inputs of calls next .. next + 31 (lane i holds call next + i)
  CallRec pre;
  SessRec ps;
  auto load_pre = [&]() {
    ensure(next);
    const uint32_t c = next + lane;
    if (c < NC) pre = ring[(c / CH) & 1][c % CH];
    else { pre.e = 0xFFFFFFFFu; pre.s = 0; }
  };
  auto load_ps = [&]() {
    if (next + lane < NC) ps = sess[pre.s];
  };
  load_pre();
  load_ps();

  auto w_at = [&](uint32_t i) { uint32_t j = wh + i; return j >= Q ? j - Q : j; };
  auto s_at = [&](uint32_t i) { uint32_t j = sh + i; return j >= K ? j - K : j; };
  // insert a call into S keeping F ascending (new calls usually land at the tail)
  auto s_insert = [&](uint32_t sid, int64_t F) {
    uint32_t i = nS;
    while (i > 0) {
      const uint32_t jp = s_at(i - 1);
      if (sF[jp] <= F) break;
      const uint32_t j = s_at(i);
      sF[j] = sF[jp]; sS[j] = sS[jp];
      --i;
    }
    const uint32_t j = s_at(i);
    sF[j] = F; sS[j] = sid; ++nS;
  };
  // move waiting calls into service while a server is free (FIFO order)
  auto admit = [&]() {
    while (nS < K && nW > 0) {
      const uint32_t j = w_at(0);
      const int64_t r = wR[j];
      LW -= min(r, E);
      s_insert(wS[j], V + r);
      wh = w_at(1); --nW;
    }
  };
  // drop the calls of S whose threshold is reached (a prefix); returns the work they had left
  auto complete = [&](int64_t Vnew, int64_t Vold, int64_t& served) -> uint32_t {
    uint32_t m = 0;
    while (nS > 0) {
      const uint32_t j = s_at(0);
      if (sF[j] > Vnew) break;
      served += sF[j] - Vold;
      moved[sS[j]] = 0;
      sh = s_at(1); --nS; ++m;
    }
    return m;
  };
  auto load_of = [&]() {
    int64_t l = LW;
    uint32_t i = 0;
    for (; i < nS; ++i) {
      const int64_t r = sF[s_at(i)] - V;
      if (r >= E) break;
      l += r;
    }
    l += (int64_t)(nS - i) * E;
    return l;
  };
  // oldest waiting call of a session that is not `moved` and has no call in service here
  auto find_stealable = [&]() -> int32_t {
    for (uint32_t i = 0; i < nW; ++i) {
      const uint32_t s = wS[w_at(i)];
      if (moved[s]) continue;
      bool busy = false;
      for (uint32_t j = 0; j < nS; ++j) if (sS[s_at(j)] == s) { busy = true; break; }
      if (!busy) return (int32_t)s;
    }
    return -1;
  };

  while (true) {
    const bool any = __ballot_sync(0xffffffffu, act_lane && (nS + nW) > 0) != 0;
    if (next >= NC && !any) break;
    const int64_t Te = (int64_t)e * E;
    bool got = false;
    // ---------------- P1 service: the first kappa calls progress by one epoch ----------------
    if (act_lane) {
      admit();
      int64_t served = 0;
      const uint32_t m = complete(V + E, V, served);
      served += (int64_t)nS * E;  // every remaining call in service progressed by E
      (void)m;
      V += E;
      idle = served == 0 ? idle + 1 : 0;
      L = load_of();
    }
    __syncwarp();
    // ---------------- P2 steal: idle thief AND load-ratio guard (P:361, P:766(a)) ----------------
    uint32_t thieves = __ballot_sync(0xffffffffu, act_lane && idle * E >= a.t_idle_us);
    if (thieves && __ballot_sync(0xffffffffu, act_lane && nW > 0)) {
      bool stole = false;
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
        for (uint32_t mm = O; mm; mm &= mm - 1) { if (cntb == r) { vv = __ffs(mm) - 1; break; } ++cntb; }
        const int32_t s = __shfl_sync(0xffffffffu, cand, vv);
        if (lane == vv) {  // every call of s here is waiting: move them, order kept
          uint32_t kk = 0, m = 0;
          for (uint32_t i = 0; i < nW; ++i) {
            const uint32_t j = w_at(i);
            const uint32_t x = wS[j], rr = wR[j];
            if (x == (uint32_t)s) {
              if (m < 64) { xfer_s[m] = x; xfer_r[m] = rr; }
              ++m;
              LW -= min((int64_t)rr, E);
            } else {
              const uint32_t jd = w_at(kk);
              wS[jd] = x; wR[jd] = rr; ++kk;
            }
          }
          if (m > 64) atomicOr(&errf, 4u);
          nW = kk;
          xfer_n = m;
          L = load_of();
        }
        __syncwarp();
        if (lane == th) {
          const uint32_t m = min(xfer_n, 64u);
          for (uint32_t i = 0; i < m; ++i) {
            if (nW >= Q) { atomicOr(&errf, 1u); break; }
            const uint32_t j = w_at(nW);
            wS[j] = xfer_s[i]; wR[j] = xfer_r[i]; ++nW;
            LW += min((int64_t)xfer_r[i], E);
          }
          L = load_of();
          idle = 0;
          got = true;
        }
        if (lane == 0) {
          SessRec sr = sess[s];
          const uint32_t ty = v.styp[s];
          if (!(sr.ttlf & S_FIN)) {  // s is counted at its current affinity node
            const int32_t ao = sr.aff;
            cnt[ao][ty]--; cnt[th][ty]++;
          }
          sr.aff = (int32_t)th;
          sess[s] = sr;
          moved[s] = 1;
          if (n_mig < a.mig_cap) a.migs[n_mig] = Mig{(uint32_t)e, (uint32_t)s, vv, th};
          else errf |= 2u;
          ++n_mig;
          ++steals;
        }
        stole = true;
        __syncwarp();
      }
      if (stole) load_ps();  // affinities of prefetched sessions may have changed
    }
    // ---------------- P3 route the calls admitted at T_e (eq:routing) ----------------
    while (next < NC && __shfl_sync(0xffffffffu, pre.e, 0) == (uint32_t)e) {
      const uint32_t c = next + lane;
      const bool valid = c < NC && pre.e == (uint32_t)e;
      const uint32_t nb = __popc(__ballot_sync(0xffffffffu, valid));
      const uint32_t s = pre.s, ty = pre.tyf & 0xFFFFu;
      const bool f_new_l = (pre.tyf & F_FNEW) != 0;
      int32_t aff = valid ? ps.aff : -1;
      bool fin = valid && (ps.ttlf & S_FIN);
      bool term_lv = !valid || (ps.ttlf & S_TERM);
      int64_t tend_lv = ps.tend_lv, ttl_lv = ps.ttlf & (S_FIN - 1u);
      const uint32_t same = __match_any_sync(0xffffffffu, valid ? s : 0xFFFFFFFFu);
      for (uint32_t i = 0; i < nb; ++i) {
        // lane i's view of its session state
        const int32_t ws = __shfl_sync(0xffffffffu, aff, i);
        const bool cached_i = (aff >= 0) && !term_lv && (Te - tend_lv <= ttl_lv);   // Alg. 1 with m = 0
        const bool cached = __shfl_sync(0xffffffffu, cached_i, i);
        const int64_t Lws = __shfl_sync(0xffffffffu, (long long)L, ws >= 0 ? ws : 0);
        uint32_t w;
        if (cached && 1000 * Lws < (int64_t)a.theta_pm * (int64_t)K * E) {
          w = (uint32_t)ws;
        } else {  // argmin load; ties -> lowest worker id
          int64_t kL = act_lane ? L : INT64_MAX;
          uint32_t kW = lane;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            int64_t oL = __shfl_xor_sync(0xffffffffu, (long long)kL, o);
            uint32_t oW = __shfl_xor_sync(0xffffffffu, kW, o);
            if (oL < kL || (oL == kL && oW < kW)) { kL = oL; kW = oW; }
          }
          w = kW;
        }
        const bool use_cached = cached && (int32_t)w == ws;
        const uint32_t omega = __shfl_sync(0xffffffffu, use_cached ? pre.om_cached : pre.om_full, i);
        const uint32_t tyi = __shfl_sync(0xffffffffu, ty, i);
        const uint32_t si = __shfl_sync(0xffffffffu, s, i);
        const bool fin_old = __shfl_sync(0xffffffffu, fin, i);
        const bool f_new = __shfl_sync(0xffffffffu, f_new_l, i);
        if (lane == w) {
          if (nW >= Q) atomicOr(&errf, 1u);
          else {
            const uint32_t j = w_at(nW);
            wS[j] = si; wR[j] = omega; ++nW;
            LW += min((int64_t)omega, E);
            L += min((int64_t)omega, E);
          }
          got = true;
        }
        if (lane == 0) {
          if (ws >= 0 && w != (uint32_t)ws) ++reroutes;
          if (ws >= 0 && !fin_old) cnt[ws][tyi]--;
          if (!f_new) cnt[w][tyi]++;
        }
        if (lane == i) a.node_of[c] = (uint8_t)w;
        // forward the post-call state to later lanes of the same session in this batch
        const int64_t tendi = __shfl_sync(0xffffffffu, (long long)pre.tend, i);
        const uint32_t ttli = __shfl_sync(0xffffffffu, pre.ttl, i);
        const bool termi = __shfl_sync(0xffffffffu, (int)((pre.tyf & F_TERM) != 0), i);
        if (valid && (lane == i || (lane > i && ((same >> i) & 1u)))) {
          aff = (int32_t)w; fin = f_new;
          term_lv = termi; tend_lv = tendi; ttl_lv = ttli;
        }
        __syncwarp();
      }
      // the last lane of each session in the batch publishes the session state
      const uint32_t later = same & ~((2u << lane) - 1u);
      if (valid && later == 0) {
        SessRec r{aff, (uint32_t)ttl_lv | (fin ? S_FIN : 0u) | (term_lv ? S_TERM : 0u), tend_lv};
        sess[s] = r;
      }
      __syncwarp();
      next += nb;
      load_pre();
      __syncwarp();
      load_ps();
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
    const bool all_fit = __ballot_sync(0xffffffffu, act_lane && nS + nW > K) == 0;
    if (all_fit) {
      const uint32_t e_next = __shfl_sync(0xffffffffu, pre.e, 0);
      if (act_lane) admit();  // everything fits: every queued call is served each epoch
      uint64_t k;
      if (next >= NC) {
        int64_t mx = (act_lane && nS) ? sF[s_at(nS - 1)] - V : 0;
        mx = -warp_min64(-mx);
        k = (uint64_t)ceil_div64(mx, E);
      } else {
        k = (uint64_t)e_next - 1 - e;
      }
      if (k > 0 && act_lane) {
        const int64_t mx = nS ? sF[s_at(nS - 1)] - V : 0;  // < 2^32 (work is u32 us)
        const bool empty = nS + nW == 0;
        int64_t served = 0;
        complete(V + (int64_t)k * E, V, served);
        if (empty) idle += (int64_t)k;
        else {
          const uint32_t mx32 = (uint32_t)mx, E32 = (uint32_t)E;  // 0 <= mx < 2^32
          const uint64_t m = mx32 / E32 + (mx32 % E32 != 0u);
          idle = m >= k ? 0 : (int64_t)(k - m);
        }
        V += (int64_t)k * E;
        L = load_of();
      }
      e += k;
    }
    __syncwarp();
    ++e;
  }
  while (ready < have) {  // no bulk copy may still target this CTA's shared memory at exit
    mbar_wait(&rbar[ready & 1], (ready >> 1) & 1u);
    ++ready;
  }
  if (lane == 0) {
    a.out_n[0] = n_mig;
    a.out_n[1] = n_act;
    a.out_n[2] = errf;
    a.out_stats[0] = steals;
    a.out_stats[1] = reroutes;
  }
}

__global__ void k_sess_init(SessRec* s, uint8_t* moved, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    s[i] = SessRec{-1, 0u, 0ll};
    moved[i] = 0;
  }
}

unsigned grid_for(uint64_t n, int threads = NTHREADS) {
  uint64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148u * 64u) g = 148u * 64u;
  return (unsigned)g;
}

}  // namespace

saga_status run_placement(saga_trace* t) {
  const TraceView& v = t->v;
  const uint32_t W = v.n_nodes;
  const size_t max_smem = 200 * 1024;
  const uint32_t K = t->pcfg.kappa;
  if (K > 256) { set_error("saga_load_trace: kappa > 256 is not supported"); return SAGA_ERR_INVALID_ARG; }
  const size_t sess_bytes = ((size_t)v.n_sessions * (sizeof(SessRec) + 1) + 15) & ~(size_t)15;
  const size_t srv_bytes = (size_t)W * K * 12;  // S: finish thresholds + sessions
  // sessions in shared memory if that still leaves >= 256 waiting slots per node
  const bool ss = sess_bytes + srv_bytes + 256ull * 8 * W <= max_smem;
  if (srv_bytes + 64ull * 8 * W > max_smem) { set_error("saga_load_trace: kappa x nodes too large"); return SAGA_ERR_INVALID_ARG; }
  uint32_t qcap = (uint32_t)((max_smem - (ss ? sess_bytes : 0) - srv_bytes) / (8ull * W));
  if (qcap > 65536) qcap = 65536;
  const size_t smem = (ss ? sess_bytes : 0) + srv_bytes + size_t(qcap) * W * 8;
  uint32_t mig_cap = v.n_calls + v.n_sessions + 64;
  uint32_t act_cap = v.n_calls + mig_cap + 64;
  t->node_of = dalloc<uint8_t>(t, v.n_calls);
  t->migs = dalloc<Mig>(t, mig_cap);
  t->act = dalloc<ActRec>(t, act_cap);
  uint32_t* out_n = dalloc<uint32_t>(t, 4);
  unsigned long long* out_stats = dalloc<unsigned long long>(t, 2);
  CallRec* rec = dalloc<CallRec>(t, v.n_calls);
  SessRec* sess = ss ? nullptr : dalloc<SessRec>(t, v.n_sessions);
  uint8_t* moved = ss ? nullptr : dalloc<uint8_t>(t, v.n_sessions);
  if (!t->node_of || !t->migs || !t->act || !out_n || !out_stats || !rec || (!ss && (!sess || !moved))) {
    set_error("saga_load_trace: out of device memory (placement)");
    return SAGA_ERR_OOM;
  }
  SAGA_CK(cudaMemsetAsync(out_n, 0, 16, t->stream));
  PlaceArgs a{};
  a.v = v;
  a.rec = rec;
  a.kappa = t->pcfg.kappa; a.theta_pm = t->pcfg.theta_pm; a.rmax_pm = t->pcfg.rmax_pm; a.qcap = qcap;
  a.t_idle_us = t->pcfg.t_idle_us; a.seed = t->pcfg.seed;
  a.node_of = t->node_of; a.migs = t->migs; a.mig_cap = mig_cap; a.act = t->act; a.act_cap = act_cap;
  a.out_n = out_n; a.out_stats = out_stats; a.sess_g = sess; a.moved_g = moved;
  prof_begin(SAGA_PROF_PLACE, t->stream);
  if (v.n_calls) k_call_rec<<<grid_for(v.n_calls), NTHREADS, 0, t->stream>>>(v, rec);
  count_launch();
  if (ss) {
    SAGA_CK(cudaFuncSetAttribute(k_place<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_place<true><<<1, 32, smem, t->stream>>>(a);
  } else {
    k_sess_init<<<grid_for(v.n_sessions), NTHREADS, 0, t->stream>>>(sess, moved, v.n_sessions);
    count_launch();
    SAGA_CK(cudaFuncSetAttribute(k_place<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_place<false><<<1, 32, smem, t->stream>>>(a);
  }
  prof_end(SAGA_PROF_PLACE, t->stream);
  count_launch();
  SAGA_CK_LAUNCH();
  uint32_t hn[4];
  unsigned long long hs[2];
  SAGA_CK(d2h(hn, out_n, 16, t->stream));
  SAGA_CK(d2h(hs, out_stats, 16, t->stream));
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
