// F4 (online statistics): per-call TTL base and expected observation length from the tool
// history the trace itself reveals (saga_tool_stats; Alg. 1 line 2 "ttl_base <- Percentile(H_t,
// p)"; "tool-type-specific distributions maintained via exponential moving
// averages"; readings R-online in DESIGN.md §3).
//
//   k_samples    one thread per session-list position: call d with successor d' gives a sample of
//                tool label[d] completed at t(d'): latency t(d') - t_end(d) (clamped to
//                [0, 2^32 - 1]) and observation new_tokens[d'], stored at index d';
//   sort         stable onesweep of (tool, d') -> per tool, samples in completion order;
//   k_gather     sample time / latency / observation in that order (coalesced windows);
//   k_stats      one warp per call c: 32-ary search for k = samples of its tool completed by
//                t_end(c); nearest-rank percentile of the last `window` latencies by a bitwise
//                warp select (32 rounds of compare + warp sum); the truncated EMA in fp64
//                (no contraction, fixed order) by lane 0.
#include <mutex>

#include "saga_internal.cuh"

namespace saga {
namespace {

constexpr int ST = 256;
constexpr uint32_t MAXW = 1024;   // window limit: 32 latencies per lane
constexpr uint32_t MAXTERMS = 256;

struct StatArgs {
  TraceView v;
  const uint32_t* label;
  uint32_t L, p_pm, window, min_samples, terms;
  uint32_t* tool_of;     // [n_calls] tool of the sample completed at call d', L if none
  uint32_t* lat_of;      // [n_calls]
  const uint32_t* sv;    // sorted sample call indices d'
  const uint32_t* off;   // [L + 2] per-tool segment offsets in sv
  int64_t* s_t;          // [n_samples] completion time, in sorted order
  uint32_t* s_lat;
  uint32_t* s_obs;
  int64_t* ttl_out;
  uint32_t* obs_out;
  uint32_t* err;
};

__global__ void __launch_bounds__(ST) k_samples(StatArgs a) {
  const TraceView& v = a.v;
  for (uint32_t i = blockIdx.x * ST + threadIdx.x; i < v.n_calls; i += gridDim.x * ST) {
    const uint32_t d2 = v.sc_call[i];
    const uint32_t x2 = a.label[d2];
    if (x2 >= a.L && atomicOr(&a.err[0], 1u) == 0u) a.err[1] = d2;
    // i is d2's position; its predecessor d sits at i - 1 when that is the same session
    const uint32_t s = v.call_sess[d2];
    uint32_t tool = a.L, lat = 0;
    if (i > v.sc_off[s]) {
      const uint32_t d = v.sc_call[i - 1];
      const uint32_t x = a.label[d];
      if (x < a.L) {
        tool = x;
        const int64_t l = v.call_t[d2] - v.tend[d];
        lat = l < 0 ? 0u : (l > 0xFFFFFFFFll ? 0xFFFFFFFFu : (uint32_t)l);
      }
    }
    a.tool_of[d2] = tool;
    a.lat_of[d2] = lat;
  }
}

__global__ void __launch_bounds__(ST) k_gather(StatArgs a, uint32_t n) {
  for (uint32_t j = blockIdx.x * ST + threadIdx.x; j < n; j += gridDim.x * ST) {
    const uint32_t d2 = a.sv[j];
    a.s_t[j] = a.v.call_t[d2];
    a.s_lat[j] = a.lat_of[d2];
    a.s_obs[j] = a.v.call_new[d2];
  }
}

// off[x] = first index of the sorted tool keys >= x, x = 0..L+1 (keys are 0..L)
__global__ void k_offsets(const uint32_t* sk, uint32_t n, uint32_t L, uint32_t* off) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x > L + 1) return;
  uint32_t lo = 0, hi = n;
  while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (sk[mid] < x) lo = mid + 1; else hi = mid; }
  off[x] = lo;
}

// fp64 weights of the truncated EMA, built by repeated multiplication (host, same as the oracle)
__constant__ double c_w[MAXTERMS];     // 0.2 * 0.8^i
__constant__ double c_p[MAXTERMS + 1]; // 0.8^i

__global__ void __launch_bounds__(ST) k_stats(StatArgs a) {
  const TraceView& v = a.v;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nw = gridDim.x * (ST / 32);
  for (uint32_t c = (blockIdx.x * ST + threadIdx.x) >> 5; c < v.n_calls; c += nw) {
    const uint32_t x = a.label[c];
    if (x >= a.L) continue;  // reported by k_samples
    const uint32_t lo = a.off[x], hi = a.off[x + 1];
    const int64_t T = v.tend[c];  // decision at the tool start of c
    // u = first j in [lo, hi) with s_t[j] > T (s_t ascending in the segment): 32-ary search with
    // the invariant u in [b, e]; 33 intervals per round, then one round of 32 direct probes
    uint32_t b = lo, e = hi;
    while (e - b > 32) {
      const uint32_t len = e - b;
      const uint32_t p = b + (uint32_t)(((uint64_t)(lane + 1) * len) / 33u);  // strictly increasing, < e
      const uint32_t m = __ballot_sync(0xffffffffu, a.s_t[p] <= T);           // a prefix of the lanes
      const uint32_t nle = __popc(m);
      const uint32_t pb = __shfl_sync(0xffffffffu, p, nle > 0 ? nle - 1 : 0);
      const uint32_t pe = __shfl_sync(0xffffffffu, p, nle < 32 ? nle : 31);
      if (nle > 0) b = pb + 1;
      if (nle < 32) e = pe;
    }
    b += __popc(__ballot_sync(0xffffffffu, b + lane < e && a.s_t[b + lane] <= T));
    const uint32_t u = b;
    const uint32_t k = u - lo;  // samples of tool x completed by T
    // TTL base: nearest-rank percentile of the last min(k, window) latencies
    const uint32_t n = min(k, a.window);
    int64_t ttl = v.ttl[v.call_v[c]];  // cold start: the node's static TTL base
    if (n >= a.min_samples && n > 0) {
      const uint32_t nq = (n + 31u) / 32u;
      const uint32_t w0 = u - n;
      uint32_t val[MAXW / 32];
#pragma unroll
      for (uint32_t q = 0; q < MAXW / 32; ++q) {
        const uint32_t j = q * 32u + lane;
        val[q] = (q < nq && j < n) ? a.s_lat[w0 + j] : 0xFFFFFFFFu;
      }
      const uint32_t r = (uint32_t)(((uint64_t)a.p_pm * n + 999u) / 1000u);  // 1-indexed rank
      // r-th smallest = the largest t with #{x < t} < r (padding lanes hold 2^32 - 1 and are
      // excluded from the count by j < n)
      uint32_t ans = 0;
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t cand = ans | (1u << bit);
        uint32_t cnt = 0;
#pragma unroll
        for (uint32_t q = 0; q < MAXW / 32; ++q)
          if (q < nq) cnt += (q * 32u + lane < n && val[q] < cand) ? 1u : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (cnt < r) ans = cand;
      }
      ttl = min((int64_t)ans, (int64_t)1000000000);
    }
    if (lane == 0) {
      a.ttl_out[c] = ttl;
      // EMA (alpha = 0.2) from the node prior n0, truncated to the last `terms` samples
      const uint32_t m = min(k, a.terms);
      double acc = k <= a.terms ? __dmul_rn(c_p[k], (double)v.obs[v.call_v[c]]) : 0.0;
      for (int i = (int)m - 1; i >= 0; --i) acc = __dadd_rn(acc, __dmul_rn(c_w[i], (double)a.s_obs[u - 1 - (uint32_t)i]));
      const double rd = floor(__dadd_rn(acc, 0.5));
      a.obs_out[c] = rd >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)rd;
    }
  }
}

}  // namespace

saga_status run_tool_stats(const saga_trace* tc, const uint32_t* label, uint32_t L, uint32_t p_pm, uint32_t window,
                           uint32_t min_samples, uint32_t terms, int64_t* ttl_out, uint32_t* obs_out, cudaStream_t s) {
  saga_trace* t = const_cast<saga_trace*>(tc);  // workspace only
  const TraceView& v = t->v;
  const uint32_t n = v.n_calls;
  if (n == 0) return SAGA_OK;
  {
    // weights: the same fp64 products as the oracle (repeated multiplication), once per device
    static std::mutex mu;
    static uint64_t done_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (dev >= 64 || !((done_mask >> dev) & 1ull)) {
      double w[MAXTERMS], p[MAXTERMS + 1];
      p[0] = 1.0;
      for (uint32_t i = 0; i < MAXTERMS; ++i) p[i + 1] = p[i] * 0.8;
      w[0] = 0.2;
      for (uint32_t i = 1; i < MAXTERMS; ++i) w[i] = w[i - 1] * 0.8;
      SAGA_CK(cudaMemcpyToSymbol(c_w, w, sizeof(w)));
      SAGA_CK(cudaMemcpyToSymbol(c_p, p, sizeof(p)));
      if (dev < 64) done_mask |= 1ull << dev;
    }
  }
  StatArgs a{};
  a.v = v; a.label = label; a.L = L; a.p_pm = p_pm; a.window = window; a.min_samples = min_samples; a.terms = terms;
  a.ttl_out = ttl_out; a.obs_out = obs_out;
  uint32_t *err = nullptr, *tool_of = nullptr, *lat_of = nullptr, *sk = nullptr, *sv = nullptr, *off = nullptr,
           *s_lat = nullptr, *s_obs = nullptr;
  int64_t* s_t = nullptr;
  SAGA_CK(ws_malloc((void**)&err, 8, s));
  SAGA_CK(ws_malloc((void**)&tool_of, 4ull * n, s));
  SAGA_CK(ws_malloc((void**)&lat_of, 4ull * n, s));
  SAGA_CK(ws_malloc((void**)&sk, 4ull * n, s));
  SAGA_CK(ws_malloc((void**)&sv, 4ull * n, s));
  SAGA_CK(ws_malloc((void**)&off, 4ull * (L + 2), s));
  SAGA_CK(cudaMemsetAsync(err, 0, 8, s));
  a.err = err; a.tool_of = tool_of; a.lat_of = lat_of;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)n + ST - 1) / ST, 148ull * 16ull));
  prof_begin(SAGA_PROF_PATTERN, s);
  k_samples<<<grid, ST, 0, s>>>(a);
  count_launch();
  SAGA_CK_LAUNCH();
  uint32_t kb = 1;
  while ((1u << kb) <= L) ++kb;  // keys 0..L
  SAGA_CK(onesweep_sort_pairs(t, tool_of, n, kb, sk, sv, s));  // stable: completion order within a tool
  k_offsets<<<(L + 2 + 63) / 64, 64, 0, s>>>(sk, n, L, off);
  SAGA_CK(ws_malloc((void**)&s_t, 8ull * n, s));
  SAGA_CK(ws_malloc((void**)&s_lat, 4ull * n, s));
  SAGA_CK(ws_malloc((void**)&s_obs, 4ull * n, s));
  a.sv = sv; a.off = off; a.s_t = s_t; a.s_lat = s_lat; a.s_obs = s_obs;
  k_gather<<<grid, ST, 0, s>>>(a, n);
  const unsigned wgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)n * 32 + ST - 1) / ST, 148ull * 8ull));
  k_stats<<<wgrid, ST, 0, s>>>(a);
  count_launch(3);
  prof_end(SAGA_PROF_PATTERN, s);
  SAGA_CK_LAUNCH();
  uint32_t he[2] = {0, 0};
  SAGA_CK(d2h(he, err, 8, s));
  for (void* q : {(void*)err, (void*)tool_of, (void*)lat_of, (void*)sk, (void*)sv, (void*)off, (void*)s_t, (void*)s_lat,
                  (void*)s_obs})
    ws_free(q, s);
  if (he[0]) {
    set_error("saga_tool_stats: call_label[%u] >= n_labels (%u)", he[1], L);
    return SAGA_ERR_INVALID_ARG;
  }
  return SAGA_OK;
}

}  // namespace saga
