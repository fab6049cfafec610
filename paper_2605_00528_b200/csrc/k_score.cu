// A5 / A6 in bulk (saga_aeg_score, saga_evict_select): the same key and selection device code
// as the replay, over caller-provided candidate batches (one CTA per segment).
//
// Score: pass 1 max-reduces tau_max = max(T_e - t_last) and size_max over the segment
// (eq:recency / eq:size normalisers); pass 2 evaluates eq:eviction in fp32 with the
// pinned op order, quantises q = floor(score * 2^20) and the Alg. 1 / eq:pressure protection
// bit, and writes key = (!prot << 63) | (q << 32) | lid.  A segment's candidate rows are read
// twice; with one 1024-thread CTA per SM the second read hits L2 (<= 512 KB per segment).
// Session state c*(s, e) = newest call of s admitted at or before e (binary search; each lane
// caches its last owner because candidates arrive in runs of one session's blocks).
//
// Select: radix select of the k largest keys (block_select.cuh), then the k winners are
// bitonic-sorted in descending order in a global scratch area and their segment-relative
// indices written out.
#include "block_select.cuh"

namespace saga {
namespace {

constexpr int ST = 1024;

struct ScoreNode { const uint32_t* lown; uint32_t n_local; };

struct ScoreArgs {
  TraceView v;
  const ScoreNode* nodes;
  saga_score_batch b;
  float alpha, beta, gamma;
  uint32_t p_low, p_high;
  int64_t ttl_max;
  float* score;
  uint64_t* key;
};

__device__ __forceinline__ uint32_t cstar(const TraceView& v, uint32_t s, uint32_t e) {
  uint32_t lo = v.sc_off[s], hi = v.sc_off[s + 1];
  const uint32_t base = lo;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(&v.ecall[__ldg(&v.sc_call[mid])]) <= e) lo = mid + 1; else hi = mid;
  }
  return lo > base ? __ldg(&v.sc_call[lo - 1]) : 0u;
}

__device__ __forceinline__ OwnerKeyIn owner_at(const TraceView& v, uint32_t o, uint32_t e, uint32_t act) {
  OwnerKeyIn r;
  if (o >= v.n_sessions) {
    const uint32_t t = o - v.n_sessions;
    const bool on = (act >> t) & 1u;
    r.shared = true; r.prot_shared = on; r.size = __ldg(&v.tlen[t]); r.P = on ? 1.0f : 0.0f;
    r.fin = false; r.t_call = 0; r.ttl_base = 0;
    return r;
  }
  const uint32_t c = cstar(v, o, e);
  r.shared = false; r.prot_shared = false;
  r.size = __ldg(&v.ci_size[c]);
  r.fin = __ldg(&v.ci_fin[c]) != 0;
  r.P = __ldg(&v.ci_P[c]);
  r.t_call = __ldg(&v.tend[c]);
  r.ttl_base = __ldg(&v.ttl[__ldg(&v.call_v[c])]);
  return r;
}

__global__ void __launch_bounds__(ST) k_score(ScoreArgs a) {
  __shared__ BlockScratch<ST> sm;
  Par par;
  const TraceView& v = a.v;
  for (uint32_t sg = blockIdx.x; sg < a.b.n_seg; sg += gridDim.x) {
    const uint64_t c0 = a.b.seg_off[sg], c1 = a.b.seg_off[sg + 1];
    const uint32_t w = a.b.seg_node[sg];
    const uint32_t e = a.b.seg_epoch[sg];
    const int64_t Te = (int64_t)e * v.epoch_us;
    if (a.b.policy == SAGA_POLICY_BELADY) {
      for (uint64_t i = c0 + threadIdx.x; i < c1; i += ST)
        a.key[i] = ((uint64_t)__ldcs(&a.b.cand_nu[i]) << 32) | __ldcs(&a.b.cand_lid[i]);
      continue;
    }
    const uint32_t* lown = a.nodes[w].lown;
    const uint32_t act = a.b.seg_act[sg];
    const uint32_t C = a.b.seg_cap[sg], occ = a.b.seg_occ[sg];
    // pass 1: normalisers
    long long tau = 0;
    uint32_t smax = 1;
    uint32_t last_o = NONE, last_sz = 0;
    for (uint64_t i = c0 + threadIdx.x; i < c1; i += ST) {
      tau = max(tau, (long long)(Te - a.b.cand_t_last[i]));
      const uint32_t o = __ldg(&lown[a.b.cand_lid[i]]);
      if (o != last_o) {
        last_o = o;
        last_sz = o >= v.n_sessions ? __ldg(&v.tlen[o - v.n_sessions]) : __ldg(&v.ci_size[cstar(v, o, e)]);
      }
      smax = max(smax, last_sz);
    }
    tau = block_reduce<ST, long long>(tau, Max(), sm, par);
    smax = block_reduce<ST, uint32_t>(smax, Max(), sm, par);
    KeyCtx x;
    x.Te = Te; x.tau = tau; x.smax = smax;
    x.den = (int64_t)(a.p_high - a.p_low) * C;
    x.num = min(x.den, max((int64_t)0, 1000 * (int64_t)occ - (int64_t)a.p_low * C));
    x.ttl_max = a.ttl_max; x.alpha = a.alpha; x.beta = a.beta; x.gamma = a.gamma;
    // pass 2: keys
    last_o = NONE;
    OwnerKeyIn oi{};
    for (uint64_t i = c0 + threadIdx.x; i < c1; i += ST) {
      const uint32_t lid = __ldcs(&a.b.cand_lid[i]);
      const int64_t tl = __ldcs(&a.b.cand_t_last[i]);
      const uint32_t o = __ldg(&lown[lid]);
      if (o != last_o) { last_o = o; oi = owner_at(v, o, e, act); }
      const float sc = wa_lru_score(x, tl, oi.size, oi.P);
      __stcs(&a.key[i], aeg_key(ttl_protected(x, oi), quantize_q20(sc), lid));
      if (a.score) __stcs(&a.score[i], sc);
    }
    __syncthreads();
  }
}

// ---------------- bulk select ----------------
constexpr int SLT = 1024;

__device__ void bitonic_desc(uint64_t* k, uint32_t* idx, uint32_t n_pow2) {
  for (uint32_t size = 2; size <= n_pow2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < n_pow2; i += SLT) {
        const uint32_t jn = i ^ stride;
        if (jn > i) {
          const bool desc = (i & size) == 0;  // descending overall
          const uint64_t a = k[i], b = k[jn];
          const uint32_t ia = idx[i], ib = idx[jn];
          // order: larger key first; equal keys (only padding) by smaller index first
          const bool a_gt_b = a > b || (a == b && ia < ib);
          const bool b_gt_a = b > a || (a == b && ib < ia);
          if (desc ? b_gt_a : a_gt_b) {
            k[i] = b; k[jn] = a;
            const uint32_t t = idx[i]; idx[i] = idx[jn]; idx[jn] = t;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(SLT) k_select(const uint64_t* __restrict__ key, const uint64_t* __restrict__ seg_off,
                                                const uint32_t* __restrict__ kreq, uint32_t n_seg,
                                                const uint64_t* __restrict__ out_off, uint32_t* __restrict__ victim,
                                                uint64_t* scratch_k, uint32_t* scratch_i, uint64_t scratch_per_cta) {
  __shared__ BlockScratch<SLT> sm;
  __shared__ uint32_t s_cnt;
  Par par;
  uint64_t* sk = scratch_k + (uint64_t)blockIdx.x * scratch_per_cta;
  uint32_t* si = scratch_i + (uint64_t)blockIdx.x * scratch_per_cta;
  for (uint32_t sg = blockIdx.x; sg < n_seg; sg += gridDim.x) {
    const uint64_t c0 = seg_off[sg], c1 = seg_off[sg + 1];
    const uint32_t n = (uint32_t)(c1 - c0);
    uint32_t k = kreq[sg];
    if (k > n) k = n;
    if (k == 0) continue;
    const uint64_t* kb = key + c0;
    const uint64_t T = (k < n) ? radix_select<SLT>(kb, n, k, sm, par) : 0ull;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    uint32_t np2 = 1;
    while (np2 < k) np2 <<= 1;
    for (uint32_t i = threadIdx.x; i < n; i += SLT) {
      const uint64_t x = kb[i];
      if (x >= T) {
        const uint32_t p = atomicAdd(&s_cnt, 1u);
        sk[p] = x;
        si[p] = i;
      }
    }
    __syncthreads();
    for (uint32_t i = k + threadIdx.x; i < np2; i += SLT) { sk[i] = 0; si[i] = 0xFFFFFFFFu; }  // padding sorts last
    __syncthreads();
    bitonic_desc(sk, si, np2);
    const uint64_t o = out_off[sg];
    for (uint32_t i = threadIdx.x; i < k; i += SLT) victim[o + i] = si[i];
    __syncthreads();
  }
}

unsigned nsm_count() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return (unsigned)nsm;
}

}  // namespace

saga_status run_score(const saga_trace* t, const saga_score_batch* b, const saga_replay_cfg* cfg, float* score,
                      uint64_t* key, cudaStream_t s) {
  if (b->n_seg == 0) return SAGA_OK;
  std::vector<ScoreNode> hn(t->n_nodes);
  for (uint32_t w = 0; w < t->n_nodes; ++w) { hn[w].lown = t->nodes[w].lown; hn[w].n_local = t->nodes[w].n_local; }
  ScoreNode* dn = nullptr;
  SAGA_CK(ws_malloc((void**)&dn, sizeof(ScoreNode) * t->n_nodes, s));
  SAGA_CK(cudaMemcpyAsync(dn, hn.data(), sizeof(ScoreNode) * t->n_nodes, cudaMemcpyHostToDevice, s));
  ScoreArgs a{};
  a.v = t->v; a.nodes = dn; a.b = *b;
  a.alpha = cfg->alpha; a.beta = cfg->beta; a.gamma = cfg->gamma;
  a.p_low = cfg->p_low_pm; a.p_high = cfg->p_high_pm; a.ttl_max = cfg->ttl_max_us;
  a.score = score; a.key = key;
  const unsigned grid = std::min<unsigned>(b->n_seg, nsm_count());
  prof_begin(SAGA_PROF_SCORE, s);
  k_score<<<grid, ST, 0, s>>>(a);
  prof_end(SAGA_PROF_SCORE, s);
  count_launch();
  SAGA_CK_LAUNCH();
  ws_free(dn, s);
  return SAGA_OK;
}

saga_status run_select(const uint64_t* key, const uint64_t* seg_off, const uint32_t* k, uint32_t n_seg,
                       const uint64_t* out_off, uint32_t* victim, cudaStream_t s) {
  if (n_seg == 0) return SAGA_OK;
  // scratch: per CTA the largest power of two >= the largest segment (sizes read back once)
  std::vector<uint64_t> off(size_t(n_seg) + 1);
  SAGA_CK(cudaMemcpyAsync(off.data(), seg_off, 8 * (size_t(n_seg) + 1), cudaMemcpyDeviceToHost, s));
  SAGA_CK(cudaStreamSynchronize(s));
  uint64_t mx = 1;
  for (uint32_t i = 0; i < n_seg; ++i) mx = std::max<uint64_t>(mx, off[i + 1] - off[i]);
  uint64_t np2 = 1;
  while (np2 < mx) np2 <<= 1;
  const unsigned grid = std::min<unsigned>(n_seg, nsm_count());
  uint64_t* sk = nullptr;
  uint32_t* si = nullptr;
  SAGA_CK(ws_malloc((void**)&sk, 8 * np2 * grid, s));
  SAGA_CK(ws_malloc((void**)&si, 4 * np2 * grid, s));
  prof_begin(SAGA_PROF_SELECT, s);
  k_select<<<grid, SLT, 0, s>>>(key, seg_off, k, n_seg, out_off, victim, sk, si, np2);
  prof_end(SAGA_PROF_SELECT, s);
  count_launch();
  SAGA_CK_LAUNCH();
  ws_free(sk, s);
  ws_free(si, s);
  return SAGA_OK;
}

}  // namespace saga
