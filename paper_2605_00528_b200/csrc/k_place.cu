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
  // S lives in slots [sh, sh + nS) of a 2K-slot array (compacted to slot 0 when the tail is full)
  int64_t* sF = reinterpret_cast<int64_t*>(smem_raw + off) + (size_t)lane * 2 * K;  // S: finish thresholds
  off += (size_t)W * 2 * K * 8;
  uint32_t* sS = reinterpret_cast<uint32_t*>(smem_raw + off) + (size_t)lane * 2 * K;  // S: sessions
  off += (size_t)W * 2 * K * 4;
  uint32_t* wS = reinterpret_cast<uint32_t*>(smem_raw + off) + (size_t)lane * Q;   // W: sessions (ring)
  off += (size_t)W * Q * 4;
  uint32_t* wR = reinterpret_cast<uint32_t*>(smem_raw + off) + (size_t)lane * Q;   // W: work (us)
  __shared__ int32_t cnt[32][32];                       // sessions with aff = w, !fin, by type
  __shared__ uint32_t amask[32];                        // bit t of node w: cnt[w][t] > 0 (the act mask)
  __shared__ __align__(16) SessRec b_st[32];            // P3 batch: post-state of call next + i
  // call records streamed ahead by TMA bulk copies: chunk j (calls [256 j, 256 j + 256)) lives
  // in buffer j & 1; chunk j + 1 is requested when chunk j is first touched
  constexpr uint32_t CH = 256;
  __shared__ __align__(16) CallRec ring[2][CH];
  __shared__ __align__(8) uint64_t rbar[2];
  __shared__ uint32_t xfer_s[64], xfer_r[64];
  __shared__ uint32_t xfer_n, n_mig, n_act, errf;
  __shared__ unsigned long long steals, reroutes;
  for (int i = lane; i < 32 * 32; i += 32) (&cnt[0][0])[i] = 0;
  amask[lane] = 0;
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
  uint32_t nS = 0, nW = 0, wh = 0, sh = 0;  // |S|, |W|, ring head of W, first slot of S
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
  // insert a call into S keeping F ascending (new calls usually land at the tail)
  auto s_insert = [&](uint32_t sid, int64_t F) {
    if (sh + nS == 2 * K) {  // tail full: move S down to slot 0 (sh >= K, so at most once per K completions)
      for (uint32_t i = 0; i < nS; ++i) { sF[i] = sF[sh + i]; sS[i] = sS[sh + i]; }
      sh = 0;
    }
    uint32_t i = sh + nS;
    while (i > sh && sF[i - 1] > F) { sF[i] = sF[i - 1]; sS[i] = sS[i - 1]; --i; }
    sF[i] = F; sS[i] = sid; ++nS;
  };
  // move waiting calls into service while a server is free (FIFO order)
  auto admit = [&]() {
    while (nS < K && nW > 0) {
      const int64_t r = wR[wh];
      LW -= min(r, E);
      s_insert(wS[wh], V + r);
      wh = w_at(1); --nW;
    }
  };
  // drop the calls of S whose threshold is reached (a prefix)
  auto complete = [&](int64_t Vnew) {
    while (nS > 0 && sF[sh] <= Vnew) { moved[sS[sh]] = 0; ++sh; --nS; }
  };
  // load(w) = sum over the queue of min(rem, E): calls of S with F - V < E form a prefix
  auto load_of = [&]() {
    int64_t l = LW + (int64_t)nS * E;
    for (uint32_t j = sh; j < sh + nS; ++j) {
      const int64_t r = sF[j] - V;
      if (r >= E) break;
      l -= E - r;
    }
    return l;
  };
  // oldest waiting call of a session that is not `moved` and has no call in service here
  auto find_stealable = [&]() -> int32_t {
    for (uint32_t i = 0; i < nW; ++i) {
      const uint32_t s = wS[w_at(i)];
      if (moved[s]) continue;
      bool busy = false;
      for (uint32_t j = sh; j < sh + nS; ++j) if (sS[j] == s) { busy = true; break; }
      if (!busy) return (int32_t)s;
    }
    return -1;
  };

  bool p1_done = false;  // P1 of epoch e was applied by the previous closed-form advance
  while (true) {
    const int64_t Te = (int64_t)e * E;
    bool got = false;
    // ---------------- P1 service: the first kappa calls progress by one epoch ----------------
    if (!p1_done) {
      if (next >= NC && __ballot_sync(0xffffffffu, act_lane && (nS + nW) > 0) == 0) break;
      if (act_lane) {
        admit();
        idle = nS == 0 ? idle + 1 : 0;  // every call in service progresses by min(r, E) > 0
        complete(V + E);
        V += E;
        L = load_of();
      }
      __syncwarp();
    }
    p1_done = false;
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
            const int32_t xa = --cnt[sr.aff][ty], xt = ++cnt[th][ty];
            amask[sr.aff] = xa > 0 ? (amask[sr.aff] | (1u << ty)) : (amask[sr.aff] & ~(1u << ty));
            amask[th] = xt > 0 ? (amask[th] | (1u << ty)) : (amask[th] & ~(1u << ty));
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
    // One batch = the calls among next .. next + 31 admitted at T_e (a prefix; lane i holds call
    // next + i).  Each lane first evaluates cached(w*, s) for its own call from the prefetched
    // session state; the calls are then routed in order, every lane following call i uniformly
    // (one shuffle of lane i's packed view, the stay test, a two-step redux argmin).  A call whose
    // session already had a call earlier in the batch reads that call's post-state from b_st.
    // The affinity counts (and act-mask bits), reroute count and session records are updated per
    // batch, in parallel, after the routing.
    while (next < NC && __shfl_sync(0xffffffffu, pre.e, 0) == (uint32_t)e) {
      const bool valid = next + lane < NC && pre.e == (uint32_t)e;
      const uint32_t nb = __popc(__ballot_sync(0xffffffffu, valid));
      const uint32_t same = __match_any_sync(0xffffffffu, valid ? pre.s : 0xFFFFFFFFu);
      const uint32_t earlier = same & ((1u << lane) - 1u);
      const bool has_later = (same & ~((2u << lane) - 1u)) != 0;
      const int64_t cap_theta = (int64_t)a.theta_pm * (int64_t)K * E;
      auto is_cached = [&](const SessRec& st) {  // Alg. 1 with m = 0 at the affinity node
        return st.aff >= 0 && !(st.ttlf & S_TERM) && (Te - st.tend_lv <= (int64_t)(st.ttlf & (S_FIN - 1u)));
      };
      const uint32_t info = (ps.aff >= 0 ? (uint32_t)ps.aff : 0xFFu) | ((uint32_t)is_cached(ps) << 8) |
                            ((ps.ttlf & S_FIN) ? 1u << 9 : 0u) | (earlier ? 1u << 10 : 0u) |
                            (has_later ? 1u << 11 : 0u) | ((earlier ? 31u - __clz(earlier) : 0u) << 12);
      uint32_t my_w = 0;
      int32_t my_ws = -1;
      bool my_fin = false;
      for (uint32_t i = 0; i < nb; ++i) {
        const uint32_t inf = __shfl_sync(0xffffffffu, info, i);
        int32_t ws;
        bool cached, fin_old;
        if (inf & (1u << 10)) {  // post-state of the latest earlier call of the session
          const SessRec st = b_st[(inf >> 12) & 31u];
          ws = st.aff; cached = is_cached(st); fin_old = (st.ttlf & S_FIN) != 0;
        } else {
          ws = (inf & 0xFFu) == 0xFFu ? -1 : (int32_t)(inf & 0xFFu);
          cached = (inf >> 8) & 1u; fin_old = (inf >> 9) & 1u;
        }
        bool stay = false;
        if (cached) stay = 1000 * (int64_t)__shfl_sync(0xffffffffu, (long long)L, ws) < cap_theta;
        uint32_t w;
        if (stay) {
          w = (uint32_t)ws;
        } else {  // argmin load, ties -> lowest worker id: min of (L << 5 | w), 0 <= L < 2^58
          const uint64_t key = act_lane ? ((uint64_t)L << 5) | lane : ~0ull;
          const uint32_t hi = (uint32_t)(key >> 32);
          const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
          w = __reduce_min_sync(0xffffffffu, hi == mh ? (uint32_t)key : 0xFFFFFFFFu) & 31u;
        }
        const uint32_t c = next + i;
        const CallRec& r = ring[(c / CH) & 1][c % CH];
        if (lane == w) {
          const uint4 q = *reinterpret_cast<const uint4*>(&r);  // s, e, om_cached, om_full
          const uint32_t omega = (cached && (int32_t)w == ws) ? q.z : q.w;
          if (nW >= Q) atomicOr(&errf, 1u);
          else {
            const uint32_t j = w_at(nW);
            wS[j] = q.x; wR[j] = omega; ++nW;
            LW += min((int64_t)omega, E);
            L += min((int64_t)omega, E);
          }
          got = true;
        }
        if (lane == i) { my_w = w; my_ws = ws; my_fin = fin_old; }
        if (inf & (1u << 11)) {  // a later call of the session in this batch reads the post-state
          if (lane == 0) {
            const uint32_t tyf = r.tyf;
            b_st[i] = SessRec{(int32_t)w, r.ttl | ((tyf & F_FNEW) ? S_FIN : 0u) | ((tyf & F_TERM) ? S_TERM : 0u), r.tend};
          }
          __syncwarp();
        }
      }
      const uint32_t ty = pre.tyf & 0xFFFFu;
      const bool f_new = (pre.tyf & F_FNEW) != 0;
      const bool dec = valid && my_ws >= 0 && !my_fin, inc = valid && !f_new;
      if (dec) atomicSub(&cnt[my_ws][ty], 1);
      if (inc) atomicAdd(&cnt[my_w][ty], 1);
      const uint32_t rr = __popc(__ballot_sync(0xffffffffu, valid && my_ws >= 0 && my_w != (uint32_t)my_ws));
      if (lane == 0) reroutes += rr;
      if (valid) {
        a.node_of[next + lane] = (uint8_t)my_w;
        // the last call of each session in the batch publishes the session state
        if (!has_later)
          sess[pre.s] = SessRec{(int32_t)my_w, pre.ttl | (f_new ? S_FIN : 0u) | ((pre.tyf & F_TERM) ? S_TERM : 0u), pre.tend};
      }
      __syncwarp();
      // act-mask bits of the (node, type) counts this batch touched: every lane sees the final count
      if (dec) { if (cnt[my_ws][ty] > 0) atomicOr(&amask[my_ws], 1u << ty); else atomicAnd(&amask[my_ws], ~(1u << ty)); }
      if (inc) { if (cnt[my_w][ty] > 0) atomicOr(&amask[my_w], 1u << ty); else atomicAnd(&amask[my_w], ~(1u << ty)); }
      __syncwarp();
      next += nb;
      load_pre();
      __syncwarp();
      load_ps();
    }
    // ---------------- act(w, a) log for nodes that received records at this boundary ----------------
    // mask(w) = amask[w], kept up to date with the counts (bit t: cnt[w][t] > 0)
    const uint32_t gm = __ballot_sync(0xffffffffu, act_lane && got);
    if (gm) {
      const uint32_t base = n_act;
      if (got) {
        const uint32_t pos = base + __popc(gm & ((1u << lane) - 1u));
        if (pos < a.act_cap) a.act[pos] = ActRec{(uint32_t)e, lane, amask[lane], 0u};
        else atomicOr(&errf, 2u);
      }
      __syncwarp();
      if (lane == 0) n_act = base + __popc(gm);
      __syncwarp();
    }
    if (errf & 1u) break;
    // ---------------- closed-form advance over service-only epochs ----------------
    // When every queue fits its kappa servers, nothing happens before the next admission epoch
    // but service: jump there in one step, including that epoch's P1.
    if (__ballot_sync(0xffffffffu, act_lane && nS + nW > K) == 0) {
      if (next >= NC) break;  // no arrival, no waiting call to steal: only service remains
      const uint64_t e_next = __shfl_sync(0xffffffffu, pre.e, 0);
      const uint64_t k = e_next - e;  // >= 1 epochs of service (the last one is e_next's P1)
      if (act_lane) {
        admit();  // everything fits: every queued call is served each epoch
        if (nS == 0) {
          idle += (int64_t)k;
        } else {
          // m = ceil(mx / E) epochs with service (mx = the largest remaining work, 0 < mx < 2^32);
          // the last of the k epochs is served iff m >= k, i.e. mx > (k - 1) E
          const int64_t mx = sF[sh + nS - 1] - V;
          if (mx > (int64_t)(k - 1) * E) {
            idle = 0;
          } else {
            const uint32_t mx32 = (uint32_t)mx, E32 = (uint32_t)E;
            idle = (int64_t)k - (int64_t)(mx32 / E32 + (mx32 % E32 != 0u));
          }
        }
        complete(V + (int64_t)k * E);
        V += (int64_t)k * E;
        L = load_of();
      }
      __syncwarp();
      e = e_next;
      p1_done = true;
      continue;
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
  const size_t srv_bytes = (size_t)W * 2 * K * 12;  // S: finish thresholds + sessions (2K slots)
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
