// ============================================================================================
// SAGA hot-path CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// Plain, slow, sequential C++17 implementation of what the B200 path computes, written from
// PAPER.md (arXiv 2605.00528) and the readings listed in DESIGN.md "Readings".  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load this
// library.  It shares no code, header, table or helper with paper_2605_00528_b200/ (the CUDA
// path); the two only see the same seeded inputs produced by gen/.
//
// Sections (each cites the passage it follows):
//   validate()      trace format checks (AEG Def. P:526-534)
//   place()         session routing eq:routing, work stealing (P:748-758, P:361,
//                   P:766) -- SURVEY §8.C.2 rules P1-P6.            parity unpinned beyond the
//                   SPEC S:309-311 / S:319-321 examples and the P6 invariants
//   expand()        per-node access streams sigma -- SURVEY §8.C.3
//   next_use()      Belady next use by its plain definition: reverse scan with a
//                   hash map; local ids by sort-unique; first touches by forward scans
//   sweep_range()   W_lo / W_hi by direct counting
//   aeg_key()       WA-LRU eq:eviction, eq:recency/eq:size, eq:reuse
//                   (P:673-678), eq:overlap linear form, Alg. alg:ttl,
//                   eq:pressure -- fp32 in the pinned order of DESIGN.md; also fp64
//   replay()        epoch-synchronous replay R1-R4 for AEG, BELADY, EVICT_ALL and
//                   the baselines of Table tab:competitive: LRU and LRU + Prefix
//                   (DESIGN.md R-lru: recency = the block's latest position in the node stream)
//   min_misses()    exact per-access Belady MIN without bypass
// ============================================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

extern "C" {
struct ODesc {
  uint32_t n_calls, n_sessions, n_types, n_aeg_nodes, n_edges, n_ranges, n_blocks, n_nodes, block_tokens;
  const int64_t* call_t_us;
  const uint32_t* call_session;
  const uint32_t* call_aeg_node;
  const uint32_t* call_prompt_tokens;
  const uint32_t* call_output_tokens;
  const uint32_t* call_new_tokens;
  const uint8_t* call_is_last;
  const uint32_t* call_range_off;
  const uint32_t* range_block_lo;
  const uint32_t* range_len;
  const uint16_t* session_type;
  const uint32_t* session_block_lo;
  const uint32_t* session_block_len;
  const uint32_t* aeg_edge_off;
  const uint32_t* edge_dst;
  const float* edge_p;
  const uint32_t* edge_shared_q16;
  const int64_t* node_ttl_base_us;
  const uint32_t* node_obs_tokens;
  const uint8_t* node_terminal;
  const uint32_t* type_shared_lo;
  const uint32_t* type_shared_len;
  const int64_t* call_ttl_base_us;   // optional per-call overrides (NULL = node values)
  const uint32_t* call_obs_tokens;
};
struct OPlace {
  int64_t epoch_us;
  uint32_t kappa, prefill_tok_s, decode_tok_s, theta_pm, rmax_pm;
  int64_t t_idle_us;
  uint64_t seed;
};
struct OReplay {
  uint32_t policy;  // 1 AEG, 2 BELADY, 4 EVICT_ALL, 8 LRU, 16 LRU + Prefix (one policy per call)
  float alpha, beta, gamma;
  uint32_t p_low_pm, p_high_pm;
  int64_t ttl_max_us;
};
}

namespace {

const uint32_t INF = 0xFFFFFFFFu;
enum { POL_AEG = 1, POL_BELADY = 2, POL_EVICT_ALL = 4, POL_LRU = 8, POL_LRU_PREFIX = 16 };
// counter slots
// (SURVEY §8.C.7's list; its reserved slot holds the peak resident count)
enum {
  C_ACCESSES, C_HITS, C_MISSES, C_COMPULSORY_GLOBAL, C_COMPULSORY_NODE, C_MIG_HITS, C_MIG_MISSES,
  C_INVALIDATED, C_EVICTIONS, C_EVICT_PROTECTED, C_EVICT_EVENTS, C_REGEN_TOKENS, C_REGEN_US, C_VICTIM_HASH,
  C_INFEASIBLE_EPOCH, C_PEAK_RESIDENT, C_PF_HITS, C_PF_MISSES, C_RES18, C_RES19, C_N
};
enum { K_CALL = 0, K_MIG = 1, K_PF = 2 };   // record kinds of a node stream

// public-domain splitmix64 finaliser (Steele/Lea/Flood; constants of SURVEY §8.C.2 P5)
uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <class T>
std::vector<T> cp(const T* p, size_t n) {
  return p ? std::vector<T>(p, p + n) : std::vector<T>(n);
}

struct Group {           // one MIG, PREFETCH or CALL record group in a node stream
  uint64_t pos0, len;
  int kind;              // K_CALL, K_MIG, K_PF
  int64_t tval;          // t_last written by its records: t_c (CALL) or T_e (MIG, PREFETCH)
  uint32_t call;         // call whose ranges the records are
  uint64_t lim;          // at most this many of the call's blocks (the predicted prefix of a PREFETCH)
};
struct Event {           // one event epoch of a node
  uint32_t e;
  std::vector<Group> groups;
  std::vector<uint32_t> inv;  // sessions migrated away from this node at e (ascending)
  uint32_t act;               // act(w, a) bitmask over agent types at T_e (after P3)
  bool has_act = false;
};
struct NodeData {
  std::vector<uint32_t> block;   // global block id per position
  std::vector<Event> ev;
  std::vector<uint32_t> ev_of_pos;  // event index of each position
  // next-use products
  bool nu_done = false;
  std::vector<uint32_t> next_use, local_id, uniq;
  std::vector<uint8_t> ftn, fie;
  uint32_t w_lo = 0, w_hi = 0;
};

struct Oracle {
  // ---- trace (deep copy) ----
  uint32_t n_calls, n_sessions, n_types, n_aeg, n_edges, n_ranges, n_blocks, n_nodes, btok;
  std::vector<int64_t> t;
  std::vector<uint32_t> sess, vnode, prompt, outt, newt, roff, rlo, rlen, slo, slen, eoff, edst, eq16, obs, tlo, tlen;
  std::vector<uint8_t> last, term;
  std::vector<uint16_t> styp;
  std::vector<float> ep;
  std::vector<int64_t> ttl;
  std::vector<int64_t> cttl;          // optional per-call TTL base (empty = node values)
  std::vector<uint32_t> cobs;         // optional per-call expected observation length
  // TTL base / expected observation length of call c (per-call override, else its node's value)
  int64_t ttl_of(uint32_t c) const { return cttl.empty() ? ttl[vnode[c]] : cttl[c]; }
  uint32_t obs_of(uint32_t c) const { return cobs.empty() ? obs[vnode[c]] : cobs[c]; }
  OPlace pc;
  // ---- derived ----
  std::vector<uint32_t> owner;        // owner[b]: session id, or n_sessions + type for shared prefix
  std::vector<uint32_t> first_call;   // first call (global (t, s) order) whose ranges touch block b
  std::vector<uint32_t> pf_e, pf_len; // per call: PREFETCH epoch (0 = none) and prefix blocks
  std::vector<uint32_t> ecall;        // admission epoch e(c) = floor(t_c / E) + 1
  std::vector<std::vector<uint32_t>> scalls;  // calls of each session in order
  std::vector<uint8_t> node_of;
  struct Mig { uint32_t e, s, v, t; };
  std::vector<Mig> migs;
  int64_t n_steals = 0, n_reroutes = 0;
  std::map<std::pair<uint32_t, uint32_t>, uint32_t> act_log;  // (e, w) -> mask
  std::vector<NodeData> nodes;
  uint32_t node_mask = 0;             // nodes whose streams expand() builds (0 = all)
  int err = 0;

  int validate() {
    if (n_nodes < 1 || n_nodes > 32) return 1;
    if (n_types < 1 || n_types > 32) return 2;
    if (btok == 0) return 3;
    if (roff.size() != n_calls + 1 || roff[0] != 0 || roff[n_calls] != n_ranges) return 4;
    for (uint32_t c = 0; c < n_calls; ++c) {
      if (t[c] < 0 || t[c] > (int64_t(1) << 50)) return 5;
      if (c > 0 && !(t[c - 1] < t[c] || (t[c - 1] == t[c] && sess[c - 1] < sess[c]))) return 6;
      if (sess[c] >= n_sessions || vnode[c] >= n_aeg) return 7;
      if (prompt[c] < 1 || newt[c] > prompt[c]) return 8;
      if (roff[c + 1] <= roff[c]) return 9;   // every call touches >= 1 range
      int64_t work = (int64_t(prompt[c]) * 1000000 + pc.prefill_tok_s - 1) / pc.prefill_tok_s +
                     (int64_t(outt[c]) * 1000000 + pc.decode_tok_s - 1) / pc.decode_tok_s;
      if (work >= (int64_t(1) << 32)) return 23;   // a call's work must fit 32 bits
    }
    std::vector<std::pair<uint64_t, uint64_t>> spans;
    for (uint32_t a = 0; a < n_types; ++a) {
      if (uint64_t(tlo[a]) + tlen[a] > n_blocks) return 10;
      if (tlen[a]) spans.push_back({tlo[a], uint64_t(tlo[a]) + tlen[a]});
    }
    for (uint32_t s = 0; s < n_sessions; ++s) {
      if (styp[s] >= n_types) return 11;
      if (uint64_t(slo[s]) + slen[s] > n_blocks) return 12;
      if (slen[s]) spans.push_back({slo[s], uint64_t(slo[s]) + slen[s]});
    }
    std::sort(spans.begin(), spans.end());
    for (size_t i = 1; i < spans.size(); ++i)
      if (spans[i].first < spans[i - 1].second) return 13;  // spans must be disjoint
    for (uint32_t c = 0; c < n_calls; ++c)
      for (uint32_t r = roff[c]; r < roff[c + 1]; ++r) {
        uint64_t lo = rlo[r], hi = uint64_t(rlo[r]) + rlen[r];
        if (rlen[r] == 0 || hi > n_blocks) return 14;
        uint32_t s = sess[c], a = styp[s];
        bool in_priv = lo >= slo[s] && hi <= uint64_t(slo[s]) + slen[s];
        bool in_shared = lo >= tlo[a] && hi <= uint64_t(tlo[a]) + tlen[a];
        if (!in_priv && !in_shared) return 15;
      }
    if (eoff.size() != n_aeg + 1 || eoff[0] != 0 || eoff[n_aeg] != n_edges) return 16;
    for (uint32_t v = 0; v < n_aeg; ++v) {
      if (eoff[v + 1] < eoff[v]) return 17;
      double sum = 0;
      for (uint32_t e = eoff[v]; e < eoff[v + 1]; ++e) {
        if (edst[e] >= n_aeg) return 18;
        if (!(ep[e] >= 0.0f && ep[e] <= 1.0f)) return 19;
        if (eq16[e] > 65536) return 20;
        sum += ep[e];
      }
      if (sum > 1.0 + 1e-6) return 21;
      if (ttl[v] < 0 || ttl[v] > 1000000000) return 22;
    }
    for (int64_t x : cttl)
      if (x < 0 || x > 1000000000) return 22;
    return 0;
  }

  // ------------------------------------------------------------------------------------------
  // A2 placement: rules P1-P6, eq:routing, stealing
  // ------------------------------------------------------------------------------------------
  struct QE { uint32_t c; int64_t rem; bool started; };

  static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
  // tool-start time of call c in the open-loop timeline: t_c + prefill(new_c) + decode(out_c) (§8.C.1)
  int64_t t_end(uint32_t c) const {
    return t[c] + ceil_div(int64_t(newt[c]) * 1000000, pc.prefill_tok_s) +
           ceil_div(int64_t(outt[c]) * 1000000, pc.decode_tok_s);
  }

  // Speculative prefetch (§4.3; DESIGN.md R-prefetch): when call c finishes
  // inference and its tool starts (t_end(c)), predict the successor u = argmax_u' P(v_c -> u')
  // (ties: lowest node id) and prefetch the prefix it shares -- the first floor(n_sh / btok)
  // blocks of c's block list, n_sh = n_cur * shared_q16(v_c -> u) >> 16 (eq:overlap) -- at the
  // node that served c, at the first boundary after the tool start, e_pf = t_end(c) / E + 1.
  // Emitted only while the session is still in that tool call (its next call is admitted after
  // e_pf) and when e_pf > e(c); never for finished sessions (is_last or a terminal node).
  void plan_prefetch() {
    pf_e.assign(n_calls, 0);
    pf_len.assign(n_calls, 0);
    for (uint32_t c = 0; c < n_calls; ++c) {
      const uint32_t v = vnode[c];
      if (last[c] || term[v] || eoff[v + 1] == eoff[v]) continue;
      uint32_t best = eoff[v];
      for (uint32_t k = eoff[v] + 1; k < eoff[v + 1]; ++k)
        if (ep[k] > ep[best] || (ep[k] == ep[best] && edst[k] < edst[best])) best = k;
      const uint64_t ncur = uint64_t(prompt[c]) + outt[c];
      const uint64_t nsh = (ncur * uint64_t(eq16[best])) >> 16;
      uint64_t blocks = 0;
      for (uint32_t r = roff[c]; r < roff[c + 1]; ++r) blocks += rlen[r];
      const uint64_t len = std::min<uint64_t>(blocks, nsh / btok);
      const uint32_t e = uint32_t(t_end(c) / pc.epoch_us + 1);
      if (len == 0 || e <= ecall[c]) continue;
      const auto& cl = scalls[sess[c]];
      const auto it = std::upper_bound(cl.begin(), cl.end(), c);
      if (it != cl.end() && ecall[*it] <= e) continue;   // the next step is back by then
      pf_e[c] = e;
      pf_len[c] = uint32_t(len);
    }
  }

  void place() {
    const int64_t E = pc.epoch_us;
    const uint32_t K = pc.kappa;          // concurrent requests per node (continuous batching)
    const uint32_t W = n_nodes;
    std::vector<std::deque<QE>> Q(W);
    std::vector<int64_t> idle(W, 0);
    std::vector<int32_t> aff(n_sessions, -1);
    std::vector<int64_t> last_c(n_sessions, -1);
    std::vector<uint8_t> moved(n_sessions, 0), fin(n_sessions, 0);
    std::vector<std::vector<int32_t>> cnt(W, std::vector<int32_t>(n_types, 0));  // aff = w and !fin
    node_of.assign(n_calls, 0);
    uint32_t next = 0;
    // load(w): work committed for the next epoch, sum over queued calls of min(rem, E), against a
    // capacity of kappa*E (reading "load")
    auto load = [&](uint32_t w) {
      int64_t L = 0;
      for (auto& q : Q[w]) L += std::min(q.rem, E);
      return L;
    };
    for (uint64_t e = 1;; ++e) {
      bool any = false;
      for (uint32_t w = 0; w < W; ++w) any |= !Q[w].empty();
      if (next >= n_calls && !any) break;
      const int64_t Te = int64_t(e) * E;
      std::vector<uint8_t> got(W, 0);  // node received records (CALL or MIG) at this boundary
      // P1 service: the first kappa queued calls each progress by one epoch of wall time
      for (uint32_t w = 0; w < W; ++w) {
        int64_t served = 0;
        uint32_t n = 0;
        for (auto it = Q[w].begin(); it != Q[w].end() && n < K; ++n) {
          int64_t x = std::min(E, it->rem);
          it->rem -= x; served += x; it->started = true;
          if (it->rem == 0) { moved[sess[it->c]] = 0; it = Q[w].erase(it); }
          else ++it;
        }
        idle[w] = (served == 0) ? idle[w] + 1 : 0;
      }
      // P2 steal: trigger = idle thief AND load-ratio guard (P:361, P:766(a))
      for (uint32_t th = 0; th < W; ++th) {
        if (!(idle[th] * E >= pc.t_idle_us)) continue;
        int64_t Lmin = load(0);
        for (uint32_t w = 1; w < W; ++w) Lmin = std::min(Lmin, load(w));
        std::vector<uint32_t> O;
        for (uint32_t w = 0; w < W; ++w) {
          if (w == th) continue;
          if (!(1000 * load(w) > int64_t(pc.rmax_pm) * Lmin)) continue;
          if (stealable_session(Q[w], moved) >= 0) O.push_back(w);
        }
        if (O.empty()) continue;
        uint64_t r = splitmix64(pc.seed ^ (e * 0x9E3779B97F4A7C15ull) ^ uint64_t(th));
        uint32_t v = O[r % O.size()];
        int32_t s = stealable_session(Q[v], moved);
        std::deque<QE> keep;
        for (auto& q : Q[v]) {
          if (int32_t(sess[q.c]) == s) Q[th].push_back(q);
          else keep.push_back(q);
        }
        Q[v].swap(keep);
        if (!fin[s]) { cnt[aff[s]][styp[s]]--; cnt[th][styp[s]]++; }   // s counted at its affinity node
        aff[s] = int32_t(th); moved[s] = 1; idle[th] = 0;
        migs.push_back({uint32_t(e), uint32_t(s), v, th});
        got[th] = 1;
        n_steals++;
      }
      // P3 route every call admitted at T_e, in (t, s) order (eq:routing)
      while (next < n_calls && ecall[next] == e) {
        uint32_t c = next++;
        uint32_t s = sess[c];
        int32_t ws = aff[s];
        bool cached = false;
        if (ws >= 0) {
          uint32_t lv = vnode[last_c[s]];
          cached = !term[lv] && (Te - t_end(uint32_t(last_c[s])) <= ttl_of(uint32_t(last_c[s])));   // Alg. 1 with m = 0
        }
        uint32_t w;
        if (cached && 1000 * load(uint32_t(ws)) < int64_t(pc.theta_pm) * K * E) {
          w = uint32_t(ws);
        } else {  // argmin load, ties -> lowest worker id
          w = 0;
          for (uint32_t x = 1; x < W; ++x)
            if (load(x) < load(w)) w = x;
        }
        int64_t pf = (cached && int32_t(w) == ws) ? newt[c] : prompt[c];
        int64_t omega = ceil_div(pf * 1000000, pc.prefill_tok_s) + ceil_div(int64_t(outt[c]) * 1000000, pc.decode_tok_s);
        Q[w].push_back({c, omega, false});
        if (ws >= 0 && int32_t(w) != ws) n_reroutes++;
        if (ws >= 0 && !fin[s]) cnt[ws][styp[s]]--;
        bool f = last[c] || term[vnode[c]];
        if (!f) cnt[w][styp[s]]++;
        fin[s] = f;
        aff[s] = int32_t(w); last_c[s] = c;
        node_of[c] = uint8_t(w);
        got[w] = 1;
      }
      for (uint32_t w = 0; w < W; ++w)
        if (got[w]) {
          uint32_t m = 0;
          for (uint32_t a = 0; a < n_types; ++a) if (cnt[w][a] > 0) m |= 1u << a;
          act_log[{uint32_t(e), w}] = m;
        }
    }
  }

  // session of the oldest pending (never served) queue entry whose session is not flagged moved
  // and has no call already in service in this queue (reading "oldest pending session")
  int32_t stealable_session(const std::deque<QE>& q, const std::vector<uint8_t>& moved) const {
    for (auto& x : q) {
      if (x.started) continue;
      int32_t s = int32_t(sess[x.c]);
      if (moved[s]) continue;
      bool busy = false;
      for (auto& y : q) if (y.started && sess[y.c] == uint32_t(s)) { busy = true; break; }
      if (busy) continue;
      return s;
    }
    return -1;
  }

  // ------------------------------------------------------------------------------------------
  // A3 per-node streams: per epoch, MIG records (ascending s) then CALL records
  // ------------------------------------------------------------------------------------------
  void expand() {
    nodes.assign(n_nodes, NodeData());
    std::vector<std::map<uint32_t, Event>> evs(n_nodes);
    auto ev_at = [&](uint32_t w, uint32_t e) -> Event& {
      Event& x = evs[w][e];
      x.e = e;
      return x;
    };
    // MIG records and invalidations
    std::vector<std::pair<uint32_t, uint32_t>> mig_order;  // for ascending-s order within (w,e)
    std::vector<Mig> ms = migs;
    std::sort(ms.begin(), ms.end(), [](const Mig& a, const Mig& b) {
      return a.e != b.e ? a.e < b.e : (a.t != b.t ? a.t < b.t : a.s < b.s);
    });
    for (auto& m : ms) {
      // newest call of s admitted before T_e (e(c) < e)
      const auto& cl = scalls[m.s];
      int64_t cm = -1;
      for (uint32_t c : cl) if (ecall[c] < m.e) cm = c;
      Event& x = ev_at(m.t, m.e);
      x.groups.push_back({0, 0, K_MIG, int64_t(m.e) * pc.epoch_us, uint32_t(cm), UINT64_MAX});
      ev_at(m.v, m.e).inv.push_back(m.s);
    }
    for (uint32_t c = 0; c < n_calls; ++c) {   // PREFETCH groups (§4.3; DESIGN.md R-prefetch)
      if (pf_e.empty() || pf_e[c] == 0) continue;
      Event& x = ev_at(node_of[c], pf_e[c]);
      x.groups.push_back({0, 0, K_PF, int64_t(pf_e[c]) * pc.epoch_us, c, pf_len[c]});
    }
    for (uint32_t c = 0; c < n_calls; ++c) {
      Event& x = ev_at(node_of[c], ecall[c]);
      x.groups.push_back({0, 0, K_CALL, t[c], c, UINT64_MAX});
    }
    for (uint32_t w = 0; w < n_nodes; ++w) {
      NodeData& nd = nodes[w];
      if (node_mask && !((node_mask >> w) & 1u)) continue;   // stream not requested (left empty)
      for (auto& kv : evs[w]) {
        Event x = kv.second;
        std::sort(x.inv.begin(), x.inv.end());
        // per epoch: MIG records (ascending session), then PREFETCH (call order), then CALL (call order)
        auto rank_of = [](int kind) { return kind == K_MIG ? 0 : (kind == K_PF ? 1 : 2); };
        std::stable_sort(x.groups.begin(), x.groups.end(), [&](const Group& a, const Group& b) {
          if (a.kind != b.kind) return rank_of(a.kind) < rank_of(b.kind);
          if (a.kind == K_MIG) return sess[a.call] < sess[b.call];
          return false;   // PREFETCH / CALL groups were pushed in call order
        });
        uint32_t evi = uint32_t(nd.ev.size());
        for (auto& g : x.groups) {
          g.pos0 = nd.block.size();
          for (uint32_t r = roff[g.call]; r < roff[g.call + 1]; ++r)
            for (uint32_t i = 0; i < rlen[r]; ++i) {
              if (nd.block.size() - g.pos0 >= g.lim) break;
              nd.block.push_back(rlo[r] + i);
              nd.ev_of_pos.push_back(evi);
            }
          g.len = nd.block.size() - g.pos0;
        }
        auto it = act_log.find({x.e, w});
        if (it != act_log.end()) { x.act = it->second; x.has_act = true; }
        nd.ev.push_back(x);
      }
    }
  }

  // ------------------------------------------------------------------------------------------
  // A4 next use and derived quantities by their plain definitions
  // ------------------------------------------------------------------------------------------
  void next_use(uint32_t w) {
    NodeData& nd = nodes[w];
    if (nd.nu_done) return;
    const size_t N = nd.block.size();
    nd.next_use.assign(N, INF);
    std::unordered_map<uint32_t, uint32_t> later;
    later.reserve(N / 4 + 16);
    for (size_t i = N; i-- > 0;) {  // next_use[p] = min{q > p : block(q) = block(p)}
      auto it = later.find(nd.block[i]);
      nd.next_use[i] = (it == later.end()) ? INF : it->second;
      later[nd.block[i]] = uint32_t(i);
    }
    nd.uniq = nd.block;
    std::sort(nd.uniq.begin(), nd.uniq.end());
    nd.uniq.erase(std::unique(nd.uniq.begin(), nd.uniq.end()), nd.uniq.end());
    nd.local_id.resize(N);
    for (size_t i = 0; i < N; ++i)
      nd.local_id[i] = uint32_t(std::lower_bound(nd.uniq.begin(), nd.uniq.end(), nd.block[i]) - nd.uniq.begin());
    nd.ftn.assign(N, 0);
    {
      std::unordered_set<uint32_t> seen;
      for (size_t i = 0; i < N; ++i) nd.ftn[i] = seen.insert(nd.block[i]).second ? 1 : 0;
    }
    nd.fie.assign(N, 0);
    // W_lo: max distinct blocks among one epoch's records; W_hi: max live blocks over an epoch
    std::vector<int64_t> live(nd.ev.size() + 1, 0);
    std::vector<uint64_t> first(nd.uniq.size(), UINT64_MAX), lastp(nd.uniq.size(), 0);
    for (size_t i = 0; i < N; ++i) {
      uint32_t l = nd.local_id[i];
      if (first[l] == UINT64_MAX) first[l] = i;
      lastp[l] = i;
    }
    for (size_t l = 0; l < nd.uniq.size(); ++l) {
      live[nd.ev_of_pos[first[l]]] += 1;       // live in every record epoch from the one holding
      live[nd.ev_of_pos[lastp[l]] + 1] -= 1;   // its first access to the one holding its last
    }
    int64_t run = 0;
    uint32_t wlo = 0, whi = 0;
    for (size_t j = 0; j < nd.ev.size(); ++j) {
      run += live[j];
      uint64_t p0 = UINT64_MAX, p1 = 0;
      for (auto& g : nd.ev[j].groups) if (g.len) { p0 = std::min(p0, g.pos0); p1 = std::max(p1, g.pos0 + g.len); }
      if (p0 == UINT64_MAX) continue;  // invalidation-only epoch: no records
      std::unordered_set<uint32_t> d;
      for (uint64_t p = p0; p < p1; ++p) nd.fie[p] = d.insert(nd.block[p]).second ? 1 : 0;
      wlo = std::max<uint32_t>(wlo, uint32_t(d.size()));
      whi = std::max<uint32_t>(whi, uint32_t(run));
    }
    nd.w_lo = wlo;
    nd.w_hi = whi;
    nd.nu_done = true;
  }

  // newest call c* of session s with e(c*) <= e (SURVEY §8.C.6 "Session state at T_e")
  int64_t cstar(uint32_t s, uint32_t e) const {
    const auto& cl = scalls[s];   // the session's calls in (t, s) order, so e(c) is non-decreasing
    auto it = std::upper_bound(cl.begin(), cl.end(), e, [&](uint32_t ee, uint32_t c) { return ee < ecall[c]; });
    return it == cl.begin() ? -1 : int64_t(*(it - 1));   // last call with e(c) <= e
  }

  // ------------------------------------------------------------------------------------------
  // A5 WA-LRU score and key of one candidate block (fp32, pinned op order, no contraction)
  // ------------------------------------------------------------------------------------------
  struct KeyIn { uint32_t lid; int64_t t_last; uint32_t nu; };
  struct Ctx {   // per eviction event
    uint32_t e; int64_t Te; int64_t tau; uint32_t smax; int64_t den, num; uint32_t act;
  };

  // per-owner state: size(s) (eq:size), fin, P_reuse (eq:reuse + eq:overlap), prot inputs
  struct OwnerState { bool shared; uint32_t size; bool fin; float P; double P64; int64_t t_call, ttl_base; bool act; };

  OwnerState owner_state(uint32_t o, uint32_t e, uint32_t act) const {
    OwnerState st{};
    if (o >= n_sessions) {
      uint32_t a = o - n_sessions;
      st.shared = true;
      st.size = tlen[a];
      st.act = (act >> a) & 1u;
      st.P = st.act ? 1.0f : 0.0f;
      st.P64 = st.act ? 1.0 : 0.0;
      return st;
    }
    int64_t c = cstar(o, e);
    st.shared = false;
    uint64_t ncur = uint64_t(prompt[c]) + outt[c];                 // n_cur = prompt + output (§8.C.1)
    st.size = uint32_t((ncur + btok - 1) / btok);                    // size(s) in blocks
    uint32_t v = vnode[c];
    st.fin = last[c] || term[v];
    st.t_call = t_end(uint32_t(c));          // tool start of c* (Alg. 1 elapsed time)
    st.ttl_base = ttl_of(uint32_t(c));
    float P = 0.0f;
    double P64 = 0.0;
    if (!st.fin)
      P = reuse(&ep[eoff[v]], &eq16[eoff[v]], eoff[v + 1] - eoff[v], ncur, obs_of(uint32_t(c)), &P64);
    st.P = P;
    st.P64 = P64;
    return st;
  }

  // eq:reuse  P_reuse(s) = sum_u P(v->u) * overlap(s, u) over the out-edges of v in
  // CSR order, with eq:overlap's linear form n_sh / (n_cur + n_obs) per edge (DESIGN.md
  // R-overlap), clamped to 1 (R-clamp); fp32 in this order, plus the fp64 value
  static float reuse(const float* p, const uint32_t* q16, uint32_t n_edges, uint64_t ncur, uint64_t nobs, double* P64) {
    float P = 0.0f;
    double D = 0.0;
    for (uint32_t k = 0; k < n_edges; ++k) {
      uint64_t nsh = (ncur * uint64_t(q16[k])) >> 16;              // per-branch shared prefix
      uint64_t den = ncur + nobs;
      float ov = den == 0 ? 1.0f : float(int64_t(nsh)) / float(int64_t(den));   // n_cur/(n_cur+n_obs)
      double ov64 = den == 0 ? 1.0 : double(nsh) / double(den);
      P = P + p[k] * ov;
      D = D + double(p[k]) * ov64;
    }
    if (P64) *P64 = std::fmin(D, 1.0);
    return std::fmin(P, 1.0f);
  }

  // per-event context of the key: T_e, and the exact-integer memory pressure m = num / den of
  // eq:pressure at occupancy occ = |S| after R1 and capacity C; the normalisers
  // tau_max / size_max start at 0 / 1 and are maxed over the candidates by the caller (R-norm)
  static Ctx make_ctx(const OReplay& cfg, uint32_t e, int64_t Te, int64_t occ, uint32_t C, uint32_t act) {
    Ctx x{};
    x.e = e; x.Te = Te; x.tau = 0; x.smax = 1;
    x.den = int64_t(cfg.p_high_pm - cfg.p_low_pm) * C;
    x.num = std::min<int64_t>(x.den, std::max<int64_t>(0, 1000 * occ - int64_t(cfg.p_low_pm) * C));
    x.act = act;
    return x;
  }

  static void score(const OReplay& cfg, const Ctx& x, const OwnerState& st, const KeyIn& b,
                    float* s32, double* s64, uint32_t* q) {
    int64_t d = x.Te - b.t_last;
    float R = x.tau > 0 ? std::fmin(1.0f, float(d) / float(x.tau)) : 0.0f;          // eq:recency
    float S = float(int64_t(st.size)) / float(int64_t(x.smax));                        // eq:size
    float sc = ((cfg.alpha * R) + (cfg.beta * (1.0f - st.P))) + (cfg.gamma * S);      // eq:eviction
    double R64 = x.tau > 0 ? std::fmin(1.0, double(d) / double(x.tau)) : 0.0;
    double S64 = double(st.size) / double(x.smax);
    *s32 = sc;
    *s64 = (double(cfg.alpha) * R64 + double(cfg.beta) * (1.0 - st.P64)) + double(cfg.gamma) * S64;
    float f = std::floor(sc * 1048576.0f);
    int64_t qi = int64_t(f);
    if (qi < 0) qi = 0;
    if (qi > 1048576) qi = 1048576;
    *q = uint32_t(qi);
  }

  // Alg. alg:ttl with eq:pressure as exact integers (reading R-TTL)
  static bool prot(const OReplay& cfg, const Ctx& x, const OwnerState& st) {
    if (st.shared) return st.act;
    if (st.fin) return false;
    int64_t el = x.Te - st.t_call;
    if (!(el < cfg.ttl_max_us)) return false;
    // el < ttl_base * (1 - m/2) with m = num/den, multiplied out (128-bit: no overflow for any
    // capacity / ttl the ABI accepts)
    return (__int128)2 * x.den * el < (__int128)st.ttl_base * (2 * x.den - x.num);
  }

  // ------------------------------------------------------------------------------------------
  // A7 epoch-synchronous replay R1-R4 with A5 keys and A6 top-k
  // ------------------------------------------------------------------------------------------
  void replay(const OReplay& cfg, uint32_t w, uint32_t C, int64_t* ctr, std::vector<uint32_t>* vlog,
              std::vector<uint32_t>* vlog_e = nullptr) {
    next_use(w);
    const NodeData& nd = nodes[w];
    const uint32_t nl = uint32_t(nd.uniq.size());
    std::vector<uint8_t> res(nl, 0);
    std::vector<int64_t> tl(nl, 0);
    std::vector<uint32_t> nu(nl, INF);
    std::vector<uint32_t> lp(nl, 0);  // latest position of each block in the node stream (LRU)
    std::set<uint32_t> S;
    for (int i = 0; i < C_N; ++i) ctr[i] = 0;
    uint64_t hash = 0;
    for (size_t j = 0; j < nd.ev.size(); ++j) {
      const Event& ev = nd.ev[j];
      const uint32_t e = ev.e;
      const int64_t Te = int64_t(e) * pc.epoch_us;
      // R1 invalidate blocks of sessions migrated away at e
      for (uint32_t s : ev.inv)
        for (auto it = S.begin(); it != S.end();) {
          if (owner[nd.uniq[*it]] == s) { res[*it] = 0; it = S.erase(it); ctr[C_INVALIDATED]++; }
          else ++it;
        }
      bool any = false;
      for (auto& g : ev.groups) any |= g.len > 0;
      if (!any) continue;
      // R2 need
      std::set<uint32_t> A;
      for (auto& g : ev.groups) for (uint64_t p = g.pos0; p < g.pos0 + g.len; ++p) A.insert(nd.local_id[p]);
      int64_t nnew = 0, inA_S = 0;
      for (uint32_t b : A) { if (res[b]) inA_S++; else nnew++; }
      if (int64_t(A.size()) > int64_t(C)) { ctr[C_INFEASIBLE_EPOCH] = e; break; }
      int64_t k = (cfg.policy == POL_EVICT_ALL) ? int64_t(S.size()) - inA_S : int64_t(S.size()) + nnew - int64_t(C);
      // R3 evict the k largest keys among cand = S \ A
      if (k > 0) {
        std::vector<uint32_t> cand;
        for (uint32_t b : S) if (!A.count(b)) cand.push_back(b);
        std::vector<std::pair<uint64_t, uint32_t>> keys;  // (key, lid)
        if (cfg.policy == POL_AEG) {
          Ctx x = make_ctx(cfg, e, Te, int64_t(S.size()), C, ev.act);
          std::vector<OwnerState> sts;
          std::unordered_map<uint32_t, OwnerState> memo;   // owner_state is a function of (owner, e, act)
          for (uint32_t b : cand) {
            x.tau = std::max(x.tau, Te - tl[b]);                       // tau_max over candidates
            const uint32_t ow = owner[nd.uniq[b]];
            auto mi = memo.find(ow);
            if (mi == memo.end()) mi = memo.emplace(ow, owner_state(ow, e, ev.act)).first;
            sts.push_back(mi->second);
            x.smax = std::max(x.smax, sts.back().size);                 // size_max over candidates
          }
          for (size_t i = 0; i < cand.size(); ++i) {
            float s32; double s64; uint32_t q;
            KeyIn kin{cand[i], tl[cand[i]], nu[cand[i]]};
            score(cfg, x, sts[i], kin, &s32, &s64, &q);
            bool pr = prot(cfg, x, sts[i]);
            keys.push_back({(uint64_t(!pr) << 63) | (uint64_t(q) << 32) | cand[i], cand[i]});
          }
        } else if (cfg.policy == POL_BELADY) {
          for (uint32_t b : cand) keys.push_back({(uint64_t(nu[b]) << 32) | b, b});
        } else if (cfg.policy == POL_LRU || cfg.policy == POL_LRU_PREFIX) {
          // least recently used first: the smallest latest position has the largest key;
          // LRU + Prefix keeps shared-prefix blocks until no private block is left (vLLM's
          // prefix caching, the "LRU + Prefix" row of tab:competitive)
          for (uint32_t b : cand) {
            uint64_t key = (uint64_t(0xFFFFFFFFu - lp[b]) << 32) | b;
            if (cfg.policy == POL_LRU_PREFIX) {
              const bool priv = owner[nd.uniq[b]] < n_sessions;
              key = (uint64_t(priv) << 63) | (uint64_t(0x7FFFFFFFu - lp[b]) << 32) | b;
            }
            keys.push_back({key, b});
          }
        } else {
          for (uint32_t b : cand) keys.push_back({uint64_t(b), b});
        }
        // top-k by full descending sort (plain definition of the k largest unique keys)
        std::sort(keys.begin(), keys.end(), [](const std::pair<uint64_t, uint32_t>& a,
                                               const std::pair<uint64_t, uint32_t>& b) { return a.first > b.first; });
        for (int64_t i = 0; i < k; ++i) {
          uint32_t b = keys[i].second;
          S.erase(b); res[b] = 0;
          if (cfg.policy == POL_AEG && !(keys[i].first >> 63)) ctr[C_EVICT_PROTECTED]++;
          hash += splitmix64((uint64_t(e) << 32) | b);
          if (vlog) vlog->push_back(b);
          if (vlog_e) vlog_e->push_back(uint32_t(e));
        }
        ctr[C_EVICTIONS] += k;
        ctr[C_EVICT_EVENTS] += 1;
      }
      // R4 apply the records in stream order
      for (auto& g : ev.groups)
        for (uint64_t p = g.pos0; p < g.pos0 + g.len; ++p) {
          uint32_t b = nd.local_id[p];
          ctr[C_ACCESSES]++;
          if (res[b]) {
            ctr[g.kind == K_CALL ? C_HITS : (g.kind == K_MIG ? C_MIG_HITS : C_PF_HITS)]++;
          } else {
            res[b] = 1; S.insert(b);
            if (g.kind == K_PF) {
              ctr[C_PF_MISSES]++;   // the block is loaded ahead of the predicted next step
            } else if (g.kind == K_CALL) {
              ctr[C_MISSES]++;
              // "tokens prefilled": a CALL miss is unavoidable only at the block's first
              // touch in the whole trace; a re-prefill elsewhere (reroute) is regeneration
              if (first_call[nd.block[p]] == g.call) ctr[C_COMPULSORY_GLOBAL]++;
              else { ctr[C_REGEN_TOKENS] += btok; ctr[C_REGEN_US] += int64_t(btok) * 1000000 / pc.prefill_tok_s; }
            } else {
              ctr[C_MIG_MISSES]++;
            }
            if (nd.ftn[p]) ctr[C_COMPULSORY_NODE]++;
          }
          tl[b] = g.tval;
          nu[b] = nd.next_use[p];
          lp[b] = uint32_t(p);
        }
      ctr[C_PEAK_RESIDENT] = std::max<int64_t>(ctr[C_PEAK_RESIDENT], int64_t(S.size()));
    }
    ctr[C_VICTIM_HASH] = int64_t(hash);
  }

  // exact per-access Belady MIN without bypass on the whole node stream
  int64_t min_misses(uint32_t w, uint32_t C) {
    next_use(w);
    const NodeData& nd = nodes[w];
    std::set<std::pair<uint32_t, uint32_t>> heap;  // (next use, lid) of residents
    std::unordered_map<uint32_t, uint32_t> cur;    // lid -> its next use
    int64_t miss = 0;
    for (size_t p = 0; p < nd.block.size(); ++p) {
      uint32_t b = nd.local_id[p];
      auto it = cur.find(b);
      if (it != cur.end()) {
        heap.erase({it->second, b});
      } else {
        ++miss;
        if (cur.size() == C) {
          auto far = std::prev(heap.end());
          cur.erase(far->second);
          heap.erase(far);
        }
      }
      cur[b] = nd.next_use[p];
      heap.insert({nd.next_use[p], b});
    }
    return miss;
  }
};

Oracle* build(const ODesc* d, const OPlace* p, uint32_t node_mask, uint32_t flags, int* err) {
  Oracle* o = new Oracle();
  o->node_mask = node_mask;
  o->n_calls = d->n_calls; o->n_sessions = d->n_sessions; o->n_types = d->n_types; o->n_aeg = d->n_aeg_nodes;
  o->n_edges = d->n_edges; o->n_ranges = d->n_ranges; o->n_blocks = d->n_blocks; o->n_nodes = d->n_nodes;
  o->btok = d->block_tokens;
  o->t = cp(d->call_t_us, d->n_calls); o->sess = cp(d->call_session, d->n_calls);
  o->vnode = cp(d->call_aeg_node, d->n_calls); o->prompt = cp(d->call_prompt_tokens, d->n_calls);
  o->outt = cp(d->call_output_tokens, d->n_calls); o->newt = cp(d->call_new_tokens, d->n_calls);
  o->last = cp(d->call_is_last, d->n_calls); o->roff = cp(d->call_range_off, size_t(d->n_calls) + 1);
  o->rlo = cp(d->range_block_lo, d->n_ranges); o->rlen = cp(d->range_len, d->n_ranges);
  o->styp = cp(d->session_type, d->n_sessions); o->slo = cp(d->session_block_lo, d->n_sessions);
  o->slen = cp(d->session_block_len, d->n_sessions); o->eoff = cp(d->aeg_edge_off, size_t(d->n_aeg_nodes) + 1);
  o->edst = cp(d->edge_dst, d->n_edges); o->ep = cp(d->edge_p, d->n_edges); o->eq16 = cp(d->edge_shared_q16, d->n_edges);
  o->ttl = cp(d->node_ttl_base_us, d->n_aeg_nodes); o->obs = cp(d->node_obs_tokens, d->n_aeg_nodes);
  o->term = cp(d->node_terminal, d->n_aeg_nodes); o->tlo = cp(d->type_shared_lo, d->n_types);
  o->tlen = cp(d->type_shared_len, d->n_types);
  if (d->call_ttl_base_us) o->cttl = cp(d->call_ttl_base_us, d->n_calls);
  if (d->call_obs_tokens) o->cobs = cp(d->call_obs_tokens, d->n_calls);
  o->pc = *p;
  if (p->epoch_us <= 0 || p->kappa == 0 || p->prefill_tok_s == 0 || p->decode_tok_s == 0) { *err = 100; delete o; return nullptr; }
  int v = o->validate();
  if (v) { *err = v; delete o; return nullptr; }
  o->owner.assign(o->n_blocks, 0xFFFFFFFFu);
  for (uint32_t a = 0; a < o->n_types; ++a)
    for (uint32_t i = 0; i < o->tlen[a]; ++i) o->owner[o->tlo[a] + i] = o->n_sessions + a;
  for (uint32_t s = 0; s < o->n_sessions; ++s)
    for (uint32_t i = 0; i < o->slen[s]; ++i) o->owner[o->slo[s] + i] = s;
  // first_touch_global: walk the calls in (t, s) order; a block's first toucher
  // is the call that finds it untouched
  o->first_call.assign(o->n_blocks, 0xFFFFFFFFu);
  for (uint32_t c = 0; c < o->n_calls; ++c)
    for (uint32_t r = o->roff[c]; r < o->roff[c + 1]; ++r)
      for (uint32_t i = 0; i < o->rlen[r]; ++i)
        if (o->first_call[o->rlo[r] + i] == 0xFFFFFFFFu) o->first_call[o->rlo[r] + i] = c;
  o->ecall.resize(o->n_calls);
  o->scalls.assign(o->n_sessions, {});
  for (uint32_t c = 0; c < o->n_calls; ++c) {
    o->ecall[c] = uint32_t(o->t[c] / p->epoch_us + 1);   // admitted at the next 100 ms boundary
    o->scalls[o->sess[c]].push_back(c);
  }
  o->place();
  if (flags & 2u) o->plan_prefetch();   // SAGA_LOAD_PREFETCH
  o->expand();
  *err = 0;
  return o;
}

}  // namespace

// ============================================================================================
// C entry points (ctypes)
// ============================================================================================
extern "C" {

void* oracle_new(const ODesc* d, const OPlace* p, int* err) { return build(d, p, 0, 0, err); }
// as oracle_new, but only the streams of the nodes in node_mask are expanded (large traces);
// flags 2 = PREFETCH records (SAGA_LOAD_PREFETCH)
void* oracle_new_nodes(const ODesc* d, const OPlace* p, uint32_t node_mask, uint32_t flags, int* err) {
  return build(d, p, node_mask, flags, err);
}
// per call: PREFETCH epoch (0 = none) and prefix blocks (after oracle_new_nodes with flags 2)
void oracle_prefetch(void* h, uint32_t* e_out, uint32_t* len_out) {
  Oracle* o = static_cast<Oracle*>(h);
  for (uint32_t c = 0; c < o->n_calls; ++c) {
    e_out[c] = o->pf_e.empty() ? 0 : o->pf_e[c];
    len_out[c] = o->pf_len.empty() ? 0 : o->pf_len[c];
  }
}
void oracle_free(void* h) { delete static_cast<Oracle*>(h); }

void oracle_placement(void* h, uint8_t* node_out, int64_t* stats /*[steals, reroutes, n_mig]*/) {
  Oracle* o = static_cast<Oracle*>(h);
  if (node_out) std::memcpy(node_out, o->node_of.data(), o->n_calls);
  stats[0] = o->n_steals; stats[1] = o->n_reroutes; stats[2] = int64_t(o->migs.size());
}
void oracle_migrations(void* h, uint32_t* out /*[n_mig*4]: e, s, from, to*/) {
  Oracle* o = static_cast<Oracle*>(h);
  for (size_t i = 0; i < o->migs.size(); ++i) {
    out[4 * i] = o->migs[i].e; out[4 * i + 1] = o->migs[i].s; out[4 * i + 2] = o->migs[i].v; out[4 * i + 3] = o->migs[i].t;
  }
}
uint64_t oracle_n_act(void* h) { return static_cast<Oracle*>(h)->act_log.size(); }
void oracle_act(void* h, uint32_t* out /*[n*3]: e, w, mask*/) {
  Oracle* o = static_cast<Oracle*>(h);
  size_t i = 0;
  for (auto& kv : o->act_log) { out[3 * i] = kv.first.first; out[3 * i + 1] = kv.first.second; out[3 * i + 2] = kv.second; ++i; }
}
uint64_t oracle_stream_len(void* h, uint32_t w) { return static_cast<Oracle*>(h)->nodes[w].block.size(); }
uint64_t oracle_n_events(void* h, uint32_t w) { return static_cast<Oracle*>(h)->nodes[w].ev.size(); }
uint64_t oracle_n_groups(void* h, uint32_t w) {
  uint64_t n = 0;
  for (auto& e : static_cast<Oracle*>(h)->nodes[w].ev) n += e.groups.size();
  return n;
}
uint64_t oracle_n_inv(void* h, uint32_t w) {
  uint64_t n = 0;
  for (auto& e : static_cast<Oracle*>(h)->nodes[w].ev) n += e.inv.size();
  return n;
}
void oracle_stream(void* h, uint32_t w, uint32_t* block, uint32_t* ev /*[n_ev*4]: e, n_groups, n_inv, act*/,
                   int64_t* grp /*[n_groups*4]: pos0, len, kind, tval*/, uint32_t* inv) {
  Oracle* o = static_cast<Oracle*>(h);
  const NodeData& nd = o->nodes[w];
  if (block) std::memcpy(block, nd.block.data(), nd.block.size() * 4);
  size_t gi = 0, ii = 0;
  for (size_t j = 0; j < nd.ev.size(); ++j) {
    const Event& x = nd.ev[j];
    if (ev) { ev[4 * j] = x.e; ev[4 * j + 1] = uint32_t(x.groups.size()); ev[4 * j + 2] = uint32_t(x.inv.size()); ev[4 * j + 3] = x.act; }
    for (auto& g : x.groups) {
      if (grp) { grp[4 * gi] = int64_t(g.pos0); grp[4 * gi + 1] = int64_t(g.len); grp[4 * gi + 2] = g.kind; grp[4 * gi + 3] = g.tval; }
      ++gi;
    }
    for (uint32_t s : x.inv) { if (inv) inv[ii] = s; ++ii; }
  }
}
uint32_t oracle_n_local(void* h, uint32_t w) {
  Oracle* o = static_cast<Oracle*>(h);
  o->next_use(w);
  return uint32_t(o->nodes[w].uniq.size());
}
void oracle_next_use(void* h, uint32_t w, uint32_t* next_use, uint32_t* local_id, uint8_t* ftn, uint8_t* fie) {
  Oracle* o = static_cast<Oracle*>(h);
  o->next_use(w);
  const NodeData& nd = o->nodes[w];
  size_t N = nd.block.size();
  if (next_use) std::memcpy(next_use, nd.next_use.data(), N * 4);
  if (local_id) std::memcpy(local_id, nd.local_id.data(), N * 4);
  if (ftn) std::memcpy(ftn, nd.ftn.data(), N);
  if (fie) std::memcpy(fie, nd.fie.data(), N);
}
void oracle_lid_owner(void* h, uint32_t w, uint32_t* out) {
  Oracle* o = static_cast<Oracle*>(h);
  o->next_use(w);
  const NodeData& nd = o->nodes[w];
  for (size_t l = 0; l < nd.uniq.size(); ++l) out[l] = o->owner[nd.uniq[l]];
}
void oracle_sweep_range(void* h, uint32_t w, uint32_t* wlo, uint32_t* whi) {
  Oracle* o = static_cast<Oracle*>(h);
  o->next_use(w);
  *wlo = o->nodes[w].w_lo;
  *whi = o->nodes[w].w_hi;
}
// One replay; counters[16]; optional victim log (lids in emission order per event).
uint64_t oracle_replay(void* h, const OReplay* cfg, uint32_t w, uint32_t cap, int64_t* counters,
                       uint32_t* vlog, uint64_t vlog_cap) {
  Oracle* o = static_cast<Oracle*>(h);
  std::vector<uint32_t> log;
  o->replay(*cfg, w, cap, counters, vlog ? &log : nullptr);
  if (vlog) std::memcpy(vlog, log.data(), std::min<uint64_t>(log.size(), vlog_cap) * 4);
  return log.size();
}
// Victim log with epochs: out[i] = (epoch << 32) | local id, in eviction order; returns the count.
uint64_t oracle_replay_log(void* h, const OReplay* cfg, uint32_t w, uint32_t cap, int64_t* counters, uint64_t* out,
                           uint64_t out_cap) {
  Oracle* o = static_cast<Oracle*>(h);
  std::vector<uint32_t> lid, ep;
  o->replay(*cfg, w, cap, counters, &lid, &ep);
  for (uint64_t i = 0; i < std::min<uint64_t>(lid.size(), out_cap); ++i) out[i] = (uint64_t(ep[i]) << 32) | lid[i];
  return lid.size();
}
// Many replays over a std::thread pool: out[pol_idx][cap_idx][node][16] for policies in mask order
// (AEG, BELADY, EVICT_ALL), nodes listed in `nodes` (others left untouched).
void oracle_replay_many(void* h, const OReplay* cfg, uint32_t policy_mask, const uint32_t* caps, uint32_t n_caps,
                        const uint32_t* nodes_, uint32_t n_nodes_, int64_t* out, int nthreads) {
  Oracle* o = static_cast<Oracle*>(h);
  std::vector<uint32_t> pols;
  for (uint32_t p : {1u, 2u, 4u, 8u, 16u}) if (policy_mask & p) pols.push_back(p);
  // next use per node first (parallel over nodes)
  {
    std::atomic<uint32_t> it{0};
    std::vector<std::thread> th;
    for (int i = 0; i < std::max(1, nthreads); ++i)
      th.emplace_back([&] { for (uint32_t j; (j = it++) < n_nodes_;) o->next_use(nodes_[j]); });
    for (auto& x : th) x.join();
  }
  struct Task { uint32_t pi, ci, w; };
  std::vector<Task> tasks;
  for (uint32_t pi = 0; pi < pols.size(); ++pi)
    for (uint32_t ci = 0; ci < n_caps; ++ci)
      for (uint32_t j = 0; j < n_nodes_; ++j) tasks.push_back({pi, ci, nodes_[j]});
  std::atomic<size_t> it{0};
  std::vector<std::thread> th;
  for (int i = 0; i < std::max(1, nthreads); ++i)
    th.emplace_back([&] {
      for (size_t j; (j = it++) < tasks.size();) {
        const Task& tk = tasks[j];
        OReplay c = *cfg;
        c.policy = pols[tk.pi];
        int64_t* dst = out + ((size_t(tk.pi) * n_caps + tk.ci) * o->n_nodes + tk.w) * C_N;
        o->replay(c, tk.w, caps[tk.ci], dst, nullptr);
      }
    });
  for (auto& x : th) x.join();
}
int64_t oracle_min_misses(void* h, uint32_t w, uint32_t cap) { return static_cast<Oracle*>(h)->min_misses(w, cap); }

// Keys of an explicit candidate batch at node w, boundary e (standalone saga_aeg_score parity).
// occ = |S|, cap = C, act = act(w, .) mask.  policy AEG or BELADY.  score32/score64 nullable.
void oracle_keys(void* h, const OReplay* cfg, uint32_t w, uint32_t e, uint32_t occ, uint32_t cap, uint32_t act,
                 const uint32_t* lid, const int64_t* t_last, const uint32_t* nu, uint64_t n,
                 uint64_t* key, float* score32, double* score64) {
  Oracle* o = static_cast<Oracle*>(h);
  o->next_use(w);
  const NodeData& nd = o->nodes[w];
  if (cfg->policy == POL_BELADY) {
    for (uint64_t i = 0; i < n; ++i) key[i] = (uint64_t(nu[i]) << 32) | lid[i];
    return;
  }
  Oracle::Ctx x = Oracle::make_ctx(*cfg, e, int64_t(e) * o->pc.epoch_us, int64_t(occ), cap, act);
  std::vector<Oracle::OwnerState> sts(n);
  for (uint64_t i = 0; i < n; ++i) {
    x.tau = std::max(x.tau, x.Te - t_last[i]);
    sts[i] = o->owner_state(o->owner[nd.uniq[lid[i]]], e, act);
    x.smax = std::max(x.smax, sts[i].size);
  }
  for (uint64_t i = 0; i < n; ++i) {
    float s32; double s64; uint32_t q;
    Oracle::KeyIn kin{lid[i], t_last[i], nu[i]};
    Oracle::score(*cfg, x, sts[i], kin, &s32, &s64, &q);
    bool pr = Oracle::prot(*cfg, x, sts[i]);
    key[i] = (uint64_t(!pr) << 63) | (uint64_t(q) << 32) | lid[i];
    if (score32) score32[i] = s32;
    if (score64) score64[i] = s64;
  }
}

// Scalar entry points for the pins of SPEC's worked examples.  Each one is a thin caller of the
// function replay() uses: score() (eq:eviction / eq:recency / eq:size), reuse() (eq:reuse +
// eq:overlap) and prot() with make_ctx() (Alg. alg:ttl + eq:pressure).
// score of a private, unfinished candidate: idle d of tau_max, size of size_max, P_reuse P
float oracle_score32(float alpha, float beta, float gamma, int64_t d, int64_t tau, uint32_t size, uint32_t smax,
                     float P, uint32_t* q) {
  OReplay cfg{POL_AEG, alpha, beta, gamma, 700, 900, 300000000};
  Oracle::Ctx x = Oracle::make_ctx(cfg, 1, d, 0, 1, 0);   // T_e = d with t_last = 0
  x.tau = tau;
  x.smax = smax;
  Oracle::OwnerState st{};
  st.size = size;
  st.P = P;
  st.P64 = P;
  Oracle::KeyIn b{0, 0, 0};
  float s32; double s64; uint32_t qq;
  Oracle::score(cfg, x, st, b, &s32, &s64, &qq);
  if (q) *q = qq;
  return s32;
}
float oracle_reuse32(const float* p, const uint32_t* q16, uint32_t n_edges, uint32_t ncur, uint32_t nobs) {
  return Oracle::reuse(p, q16, n_edges, ncur, nobs, nullptr);
}
// protected?  el = T_e - t_call (a private, unfinished owner); 1 if the TTL (scaled by 1 - m/2) covers el
int oracle_ttl_protect(int64_t el, int64_t ttl_base, int64_t ttl_max, uint32_t occ, uint32_t cap,
                       uint32_t low_pm, uint32_t high_pm) {
  OReplay cfg{POL_AEG, 0.3f, 0.5f, 0.2f, low_pm, high_pm, ttl_max};
  Oracle::Ctx x = Oracle::make_ctx(cfg, 1, el, int64_t(occ), cap, 0);   // t_call = 0
  Oracle::OwnerState st{};
  st.t_call = 0;
  st.ttl_base = ttl_base;
  return Oracle::prot(cfg, x, st) ? 1 : 0;
}
uint64_t oracle_splitmix64(uint64_t x) { return splitmix64(x); }
}
