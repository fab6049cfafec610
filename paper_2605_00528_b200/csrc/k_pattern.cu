// F3: pattern-based AEG inference (saga_pattern_infer; §3.3 tier (b), tab:pattern
// P:1065-1085; readings R-pattern in DESIGN.md §3).
//
// Three launches over the session-ordered call list (sc_off / sc_call, built by A1), one warp
// per session (no per-call session / role gathers; the successor label comes by shuffle):
//   k_pat_count  each position i of a training session emits one transition x -> y (the next
//                call's label, or y = L for a completed session's final call) into a segmented
//                histogram [type][x][y], in shared memory when it fits (warp-aggregated with
//                __match_any_sync: one atomic per distinct bin per warp), flushed with one
//                global 64-bit atomic per non-zero bin per CTA;
//   k_pat_pred   one thread per (type, x): total, the retained successors (1000 c >= theta t),
//                the argmax among them (smallest y on ties), fp32 c / t of retained edges;
//   k_pat_eval   each position of a held-out session: transitions / predicted / correct per type.
// Algorithmic bytes per pass (DESIGN.md §6 F3): per session role 1 + type 2 + sc_off 4; per call
// of the pass's sessions sc_call 4 (coalesced) + label 4 (gathered) + call_is_last 1 at the end.
#include "saga_internal.cuh"

namespace saga {
namespace {

constexpr int PT = 256;
constexpr uint32_t PAT_NONE = 0xFFFFFFFFu;
constexpr uint32_t SMEM_BINS = 12288;  // 48 KB of u32 bins

struct PatArgs {
  TraceView v;
  const uint32_t* label;
  const uint8_t* role;
  uint32_t L;         // labels; successor L = "task ended"
  uint32_t bins;      // n_types * L * (L + 1)
  uint32_t theta_pm, min_tasks;
  unsigned long long* counts;
  uint32_t* tasks;
  uint32_t* pred;
  float* prob;
  unsigned long long* eval;
  uint32_t* err;      // [0] flag, [1] first offending call
};

__device__ __forceinline__ void bad_label(const PatArgs& a, uint32_t c) {
  if (atomicOr(&a.err[0], 1u) == 0u) a.err[1] = c;
}

// One warp per session of the wanted role (warp-uniform loop): lane l holds position i0 + l of
// the session's call list; the successor label comes from lane l + 1 (lane 31 reads it), or is
// L ("task ended") at a completed session's final call.  Returns via f(lane's bin or PAT_NONE, y).
template <class F>
__device__ __forceinline__ void for_each_transition(const PatArgs& a, uint8_t want, F&& f) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nw = gridDim.x * (PT / 32);
  for (uint32_t s = (blockIdx.x * PT + threadIdx.x) >> 5; s < a.v.n_sessions; s += nw) {
    if (a.role[s] != want) continue;
    const uint32_t b = a.v.sc_off[s], e = a.v.sc_off[s + 1];
    const uint32_t typ = a.v.styp[s];
    for (uint32_t i0 = b; i0 < e; i0 += 32) {
      const uint32_t i = i0 + lane;
      uint32_t c = 0, x = PAT_NONE;
      if (i < e) { c = a.v.sc_call[i]; x = a.label[c]; }
      uint32_t xn = __shfl_down_sync(0xffffffffu, x, 1);
      if (lane == 31 && i + 1 < e) xn = a.label[a.v.sc_call[i + 1]];
      uint32_t x_ok = PAT_NONE, y = PAT_NONE;
      if (i < e) {
        if (x >= a.L) {
          bad_label(a, c);
        } else {
          y = i + 1 < e ? xn : (a.v.call_last[c] ? a.L : PAT_NONE);
          if (y != PAT_NONE && y <= a.L) x_ok = x;  // a bad next label is reported by its own lane
          else y = PAT_NONE;
        }
      }
      f(typ, x_ok, y);
    }
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(PT) k_pat_count(PatArgs a) {
  extern __shared__ uint32_t hist[];
  __shared__ uint32_t s_tasks[32];
  if (SMEM)
    for (uint32_t b = threadIdx.x; b < a.bins; b += PT) hist[b] = 0;
  if (threadIdx.x < 32) s_tasks[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t L1 = a.L + 1;
  for_each_transition(a, 1, [&](uint32_t typ, uint32_t x, uint32_t y) {
    const uint32_t bin = x != PAT_NONE ? (typ * a.L + x) * L1 + y : PAT_NONE;
    if (SMEM) {
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (bin != PAT_NONE && (int)(threadIdx.x & 31u) == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
    } else if (bin != PAT_NONE) {
      atomicAdd(&a.counts[bin], 1ull);
    }
    if (bin != PAT_NONE && y == a.L) atomicAdd(&s_tasks[typ], 1u);
  });
  __syncthreads();
  if (SMEM)
    for (uint32_t b = threadIdx.x; b < a.bins; b += PT)
      if (hist[b]) atomicAdd(&a.counts[b], (unsigned long long)hist[b]);
  if (threadIdx.x < a.v.n_types && s_tasks[threadIdx.x]) atomicAdd(&a.tasks[threadIdx.x], s_tasks[threadIdx.x]);
}

__global__ void __launch_bounds__(PT) k_pat_pred(PatArgs a) {
  const uint32_t r = blockIdx.x * PT + threadIdx.x;  // (type, x) row
  if (r >= a.v.n_types * a.L) return;
  const uint32_t L1 = a.L + 1;
  const unsigned long long* row = a.counts + (uint64_t)r * L1;
  unsigned long long tot = 0;
  for (uint32_t y = 0; y < L1; ++y) tot += row[y];
  const bool ready = a.tasks[r / a.L] >= a.min_tasks;
  uint32_t best = PAT_NONE;
  unsigned long long bc = 0;
  for (uint32_t y = 0; y < L1; ++y) {
    const unsigned long long c = row[y];
    const bool keep = ready && tot > 0 && c > 0 && 1000ull * c >= (unsigned long long)a.theta_pm * tot;
    if (keep && (best == PAT_NONE || c > bc)) { best = y; bc = c; }
    if (a.prob) a.prob[(uint64_t)r * L1 + y] = keep ? __fdiv_rn((float)c, (float)tot) : 0.0f;
  }
  a.pred[r] = best;
}

__global__ void __launch_bounds__(PT) k_pat_eval(PatArgs a) {
  __shared__ unsigned long long s_ev[32 * 3];
  for (uint32_t b = threadIdx.x; b < 32 * 3; b += PT) s_ev[b] = 0;
  __syncthreads();
  for_each_transition(a, 2, [&](uint32_t typ, uint32_t x, uint32_t y) {
    uint32_t got = 0;  // bit 0 transition, 1 predicted, 2 correct (typ is warp-uniform)
    if (x != PAT_NONE) {
      const uint32_t p = a.pred[typ * a.L + x];
      got = 1u | (p != PAT_NONE ? 2u : 0u) | (p == y ? 4u : 0u);
    }
    const uint32_t nt = __popc(__ballot_sync(0xffffffffu, got & 1u));
    const uint32_t np = __popc(__ballot_sync(0xffffffffu, (got >> 1) & 1u));
    const uint32_t nc = __popc(__ballot_sync(0xffffffffu, (got >> 2) & 1u));
    if ((threadIdx.x & 31u) == 0 && nt) {
      atomicAdd(&s_ev[typ * 3 + 0], (unsigned long long)nt);
      if (np) atomicAdd(&s_ev[typ * 3 + 1], (unsigned long long)np);
      if (nc) atomicAdd(&s_ev[typ * 3 + 2], (unsigned long long)nc);
    }
  });
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < a.v.n_types * 3; b += PT)
    if (s_ev[b]) atomicAdd(&a.eval[(b / 3) * 4 + (b % 3)], s_ev[b]);
}

}  // namespace

saga_status run_pattern(const saga_trace* t, const uint32_t* label, uint32_t L, const uint8_t* role, uint32_t theta_pm,
                        uint32_t min_tasks, uint64_t* counts, uint32_t* tasks, uint32_t* pred, float* prob,
                        uint64_t* eval, cudaStream_t s) {
  const TraceView& v = t->v;
  PatArgs a{};
  a.v = v;
  a.label = label; a.role = role; a.L = L;
  a.bins = v.n_types * L * (L + 1);
  a.theta_pm = theta_pm; a.min_tasks = min_tasks;
  a.counts = reinterpret_cast<unsigned long long*>(counts);
  a.tasks = tasks; a.pred = pred; a.prob = prob;
  a.eval = reinterpret_cast<unsigned long long*>(eval);
  uint32_t* err = nullptr;
  SAGA_CK(ws_malloc((void**)&err, 8, s));
  a.err = err;
  SAGA_CK(cudaMemsetAsync(err, 0, 8, s));
  SAGA_CK(cudaMemsetAsync(counts, 0, (size_t)a.bins * 8, s));
  SAGA_CK(cudaMemsetAsync(tasks, 0, (size_t)v.n_types * 4, s));
  if (eval) SAGA_CK(cudaMemsetAsync(eval, 0, (size_t)v.n_types * 32, s));
  // one warp per session, at most one wave of resident CTAs (8 per SM)
  const uint64_t want = ((uint64_t)v.n_sessions * 32 + PT - 1) / PT;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, 148ull * 8ull));
  prof_begin(SAGA_PROF_PATTERN, s);
  if (a.bins <= SMEM_BINS) k_pat_count<true><<<grid, PT, a.bins * 4, s>>>(a);
  else k_pat_count<false><<<grid, PT, 0, s>>>(a);
  k_pat_pred<<<(v.n_types * L + PT - 1) / PT, PT, 0, s>>>(a);
  count_launch(2);
  if (eval) {
    k_pat_eval<<<grid, PT, 0, s>>>(a);
    count_launch();
  }
  prof_end(SAGA_PROF_PATTERN, s);
  SAGA_CK_LAUNCH();
  uint32_t he[2] = {0, 0};
  SAGA_CK(d2h(he, err, 8, s));
  ws_free(err, s);
  if (he[0]) {
    set_error("saga_pattern_infer: call_label[%u] >= n_labels (%u)", he[1], L);
    return SAGA_ERR_INVALID_ARG;
  }
  return SAGA_OK;
}

}  // namespace saga
