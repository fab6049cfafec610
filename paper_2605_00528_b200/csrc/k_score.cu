// A5 / A6 in bulk (saga_aeg_score, saga_evict_select): the same key and selection device code
// as the replay, over caller-provided candidate batches.
//
// Score (AEG): one CTA per segment.  Pass 1 max-reduces the eq:recency / eq:size normalisers
// tau_max = max(T_e - t_last) and size_max over the segment; pass 2 evaluates
// eq:eviction in fp32 with the pinned op order, quantises q = floor(score * 2^20) and the Alg. 1 /
// eq:pressure protection bit, and writes key = (!prot << 63) | (q << 32) | lid.  The second read
// of a segment's rows hits L2 (one 1024-thread CTA per SM keeps <= 148 x 384 KB in flight).
// (A 4-CTA-cluster variant that staged the rows in shared memory and combined the normalisers
// over DSMEM measured 0.44 ms vs 0.34 ms: cluster barriers dominated its stalls.)
// Session state c*(s, e) = newest call of s admitted at or before e (binary search; each lane
// caches its last owner because candidates arrive in runs of one session's blocks).
// Score (BELADY): key = (nu << 32) | lid, a flat 128-bit streaming pass.
//
// Select: radix select of the k largest keys (block_select.cuh), then the k winners are
// bitonic-sorted in descending order in a global scratch area and their segment-relative
// indices written out.  (A 4-CTA-cluster variant staging the keys in shared memory measured
// 0.32 ms vs 0.17 ms: cluster-barrier waits were half of its stall samples.)
#include "block_select.cuh"

namespace saga {
namespace {

constexpr int ST = 1024;
constexpr int SW = ST / 32;  // warps per CTA
constexpr int SU = 4;        // 32-candidate chunks whose loads are issued together

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
    if (__ldg(&v.sc_e[mid]) <= e) lo = mid + 1; else hi = mid;
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
  r.ttl_base = call_ttl_base(v, c);
  return r;
}

// owner reference of a candidate, resolved once in pass 1: the session's current call c*, or
// CREF_SHARED | type for a shared-prefix block
constexpr uint32_t CREF_SHARED = 0x80000000u;
constexpr uint32_t SC_STAGE = 32768;  // candidates per segment whose owner reference is kept in shared memory

__device__ __forceinline__ OwnerKeyIn owner_of_ref(const TraceView& v, uint32_t ref, uint32_t act) {
  OwnerKeyIn r;
  if (ref & CREF_SHARED) {
    const uint32_t t = ref & ~CREF_SHARED;
    const bool on = (act >> t) & 1u;
    r.shared = true; r.prot_shared = on; r.size = __ldg(&v.tlen[t]); r.P = on ? 1.0f : 0.0f;
    r.fin = false; r.t_call = 0; r.ttl_base = 0;
    return r;
  }
  const uint32_t c = ref;  // independent loads: one round trip per run of one session's blocks
  r.shared = false; r.prot_shared = false;
  r.size = __ldg(&v.ci_size[c]);
  r.fin = __ldg(&v.ci_fin[c]) != 0;
  r.P = __ldg(&v.ci_P[c]);
  r.t_call = __ldg(&v.tend[c]);
  r.ttl_base = call_ttl_base(v, c);
  return r;
}

__global__ void __launch_bounds__(ST) k_score(ScoreArgs a) {
  __shared__ BlockScratch<ST> sm;
  extern __shared__ uint32_t s_cref[];  // [SC_STAGE] owner reference per candidate of the segment
  Par par;
  const TraceView& v = a.v;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t sg = blockIdx.x; sg < a.b.n_seg; sg += gridDim.x) {
    const uint64_t c0 = a.b.seg_off[sg], c1 = a.b.seg_off[sg + 1];
    const uint32_t w = a.b.seg_node[sg];
    const uint32_t e = a.b.seg_epoch[sg];
    const int64_t Te = (int64_t)e * v.epoch_us;
    if (a.b.policy == SAGA_POLICY_BELADY) {
      for (uint64_t i = c0 + threadIdx.x; i < c1; i += ST)
        __stcs(&a.key[i], ((uint64_t)__ldcs(&a.b.cand_nu[i]) << 32) | __ldcs(&a.b.cand_lid[i]));
      continue;
    }
    const uint32_t* lown = a.nodes[w].lown;
    const uint32_t act = a.b.seg_act[sg];
    const uint32_t C = a.b.seg_cap[sg], occ = a.b.seg_occ[sg];
    // Each warp owns a contiguous slab of the segment and walks it 32 consecutive candidates at
    // a time (coalesced), so the owner (a run of one session's blocks) rarely changes within a
    // lane's sequence and its state is looked up once per run.
    const uint64_t n = c1 - c0;
    const uint64_t slab = ((n + SW - 1) / SW + 31) & ~31ull;
    const uint64_t w0 = c0 + (uint64_t)wid * slab, w1 = min(c1, w0 + slab);
    // pass 1: normalisers (eq:recency tau_max, eq:size size_max); each candidate's owner
    // reference (c* or the shared type) is kept for pass 2 when the segment fits
    const bool stage = n <= SC_STAGE;
    long long tau = 0;
    uint32_t smax = 1;
    uint32_t last_o = NONE, last_sz = 0, last_ref = 0;
    for (uint64_t b = w0; b < w1; b += 32 * SU) {
      uint32_t lid[SU];
      int64_t tl[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const uint64_t i = b + (uint64_t)u * 32 + lane;
        lid[u] = i < w1 ? __ldcs(&a.b.cand_lid[i]) : NONE;
        tl[u] = i < w1 ? a.b.cand_t_last[i] : Te;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        if (lid[u] == NONE) continue;
        tau = max(tau, (long long)(Te - tl[u]));
        const uint32_t o = __ldg(&lown[lid[u]]);
        if (o != last_o) {
          last_o = o;
          if (o >= v.n_sessions) {
            last_ref = CREF_SHARED | (o - v.n_sessions);
            last_sz = __ldg(&v.tlen[o - v.n_sessions]);
          } else {
            last_ref = cstar(v, o, e);
            last_sz = __ldg(&v.ci_size[last_ref]);
          }
        }
        if (stage) s_cref[b + (uint64_t)u * 32 + lane - c0] = last_ref;
        smax = max(smax, last_sz);
      }
    }
    tau = block_reduce<ST, long long>(tau, Max(), sm, par);
    smax = block_reduce<ST, uint32_t>(smax, Max(), sm, par);
    KeyCtx x;
    x.Te = Te; x.tau = tau; x.smax = smax;
    x.den = (int64_t)(a.p_high - a.p_low) * C;
    x.num = min(x.den, max((int64_t)0, 1000 * (int64_t)occ - (int64_t)a.p_low * C));
    x.ttl_max = a.ttl_max; x.alpha = a.alpha; x.beta = a.beta; x.gamma = a.gamma;
    // pass 2: keys (the slab re-read hits L2; owner references from shared memory)
    last_o = NONE;
    last_ref = NONE;
    OwnerKeyIn oi{};
    for (uint64_t b = w0; b < w1; b += 32 * SU) {
      uint32_t lid[SU];
      int64_t tl[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const uint64_t i = b + (uint64_t)u * 32 + lane;
        lid[u] = i < w1 ? __ldcs(&a.b.cand_lid[i]) : NONE;
        tl[u] = i < w1 ? __ldcs(&a.b.cand_t_last[i]) : 0;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        if (lid[u] == NONE) continue;
        const uint64_t i = b + (uint64_t)u * 32 + lane;
        if (stage) {
          const uint32_t ref = s_cref[i - c0];
          if (ref != last_ref) { last_ref = ref; oi = owner_of_ref(v, ref, act); }
        } else {
          const uint32_t o = __ldg(&lown[lid[u]]);
          if (o != last_o) { last_o = o; oi = owner_at(v, o, e, act); }
        }
        const float sc = wa_lru_score(x, tl[u], oi.size, oi.P);
        __stcs(&a.key[i], aeg_key(ttl_protected(x, oi), quantize_q20(sc), lid[u]));
        if (a.score) __stcs(&a.score[i], sc);
      }
    }
    __syncthreads();
  }
}


// BELADY keys (nu << 32) | lid over the whole candidate array: segments do not matter
__global__ void __launch_bounds__(256) k_key_belady(const uint32_t* __restrict__ lid, const uint32_t* __restrict__ nu,
                                                    const uint64_t* __restrict__ seg_off, uint32_t n_seg, bool vec,
                                                    uint64_t* __restrict__ key) {
  const uint64_t n = seg_off[n_seg], n0 = seg_off[0];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (vec) {  // 16-byte aligned: 4 candidates per thread and iteration
    const uint64_t nq = (n - n0) / 4;
    const uint4* l4 = reinterpret_cast<const uint4*>(lid + n0);
    const uint4* u4 = reinterpret_cast<const uint4*>(nu + n0);
    ulonglong2* k2 = reinterpret_cast<ulonglong2*>(key + n0);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += stride) {
      const uint4 a = __ldcs(l4 + i), b = __ldcs(u4 + i);
      __stcs(k2 + 2 * i, make_ulonglong2(((unsigned long long)b.x << 32) | a.x, ((unsigned long long)b.y << 32) | a.y));
      __stcs(k2 + 2 * i + 1, make_ulonglong2(((unsigned long long)b.z << 32) | a.z, ((unsigned long long)b.w << 32) | a.w));
    }
    for (uint64_t i = n0 + nq * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      key[i] = ((uint64_t)nu[i] << 32) | lid[i];
  } else {
    for (uint64_t i = n0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      __stcs(&key[i], ((uint64_t)__ldcs(&nu[i]) << 32) | __ldcs(&lid[i]));
  }
}

// ---------------- bulk select ----------------
constexpr int SLT = 512;  // several segments per SM: a segment's passes are latency-bound

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

constexpr uint32_t KMAX = 2048;  // winners and pivot bucket held in shared memory
constexpr int SEL_U = 8;         // keys per thread whose loads are issued together

// One CTA per segment.  pass 1: OR / AND of the keys (the one HBM read); pass 2: histogram of the
// 11 bits below the highest differing bit; pass 3: keys in digits above the pivot digit are
// winners, keys in the pivot digit are gathered; both lists live in shared memory, the pivot list
// is sorted to take the remaining winners and the winners are sorted.  Passes 2-3 re-read L2.
// Segments whose winners or pivot bucket exceed KMAX take the general path (radix select + a
// bitonic sort in global scratch).
__global__ void __launch_bounds__(SLT) k_select(const uint64_t* __restrict__ key, const uint64_t* __restrict__ seg_off,
                                                const uint32_t* __restrict__ kreq, uint32_t n_seg,
                                                const uint64_t* __restrict__ out_off, uint32_t* __restrict__ victim,
                                                uint64_t* scratch_k, uint32_t* scratch_i, uint64_t scratch_per_cta) {
  __shared__ BlockScratch<SLT> sm;
  __shared__ uint32_t hist[2048];
  extern __shared__ __align__(16) uint64_t sel_dyn[];  // winners / pivot lists (96 KB)
  uint64_t* wk = sel_dyn;
  uint64_t* pk = wk + KMAX;
  uint32_t* wix = reinterpret_cast<uint32_t*>(pk + KMAX);
  uint32_t* pix = wix + KMAX;
  __shared__ uint32_t s_cnt, s_np, s_d, s_above;
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
    const uint64_t o = out_off[sg];
    bool fast = false;
    if (k < n && k <= KMAX) {
      // pass 1
      unsigned long long orv = 0, anv = ~0ull;
      for (uint32_t b = threadIdx.x; b < n; b += SLT * SEL_U) {
        uint64_t x[SEL_U];
#pragma unroll
        for (int u = 0; u < SEL_U; ++u) x[u] = b + u * SLT < n ? __ldcg(&kb[b + u * SLT]) : 0ull;
#pragma unroll
        for (int u = 0; u < SEL_U; ++u) if (b + u * SLT < n) { orv |= x[u]; anv &= x[u]; }
      }
      orv = block_reduce<SLT, unsigned long long>(orv, Or(), sm, par);
      anv = block_reduce<SLT, unsigned long long>(anv, And(), sm, par);
      const unsigned long long diff = orv ^ anv;  // != 0: keys are unique and n > k >= 1
      const int top = 63 - __clzll(diff);
      const int width = min(11, top + 1);
      const int shift = top + 1 - width;
      const uint32_t dm = (1u << width) - 1u;
      // pass 2
      for (uint32_t i = threadIdx.x; i < 2048; i += SLT) hist[i] = 0;
      __syncthreads();
      for (uint32_t b = threadIdx.x; b < n; b += SLT * SEL_U) {
        uint64_t x[SEL_U];
#pragma unroll
        for (int u = 0; u < SEL_U; ++u) x[u] = b + u * SLT < n ? __ldcg(&kb[b + u * SLT]) : 0ull;
#pragma unroll
        for (int u = 0; u < SEL_U; ++u)
          if (b + u * SLT < n) atomicAdd(&hist[(uint32_t)(x[u] >> shift) & dm], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {  // pivot digit: the k-th largest key lies in it
        const int lane = threadIdx.x;
        uint32_t sum = 0;
        for (int q = 0; q < 64; ++q) sum += hist[2047 - (lane * 64 + q)];
        uint32_t x = sum;
#pragma unroll
        for (int of = 1; of < 32; of <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, of);
          if (lane >= of) x += y;
        }
        uint32_t c = x - sum;
        if (c < k && k <= x) {
          for (int q = 0; q < 64; ++q) {
            const uint32_t h = hist[2047 - (lane * 64 + q)];
            if (c < k && k <= c + h) { s_d = 2047u - (lane * 64u + q); s_above = c; }
            c += h;
          }
        }
      }
      __syncthreads();
      const uint32_t d = s_d, A = s_above, B = hist[d];
      fast = A <= KMAX && B <= KMAX;
      if (fast) {
        if (threadIdx.x == 0) { s_cnt = 0; s_np = 0; }
        __syncthreads();
        // pass 3
        for (uint32_t b = threadIdx.x; b < n; b += SLT * SEL_U) {
          uint64_t x[SEL_U];
#pragma unroll
          for (int u = 0; u < SEL_U; ++u) x[u] = b + u * SLT < n ? __ldcg(&kb[b + u * SLT]) : 0ull;
#pragma unroll
          for (int u = 0; u < SEL_U; ++u) {
            const uint32_t i = b + u * SLT;
            if (i >= n) continue;
            const uint32_t dg = (uint32_t)(x[u] >> shift) & dm;
            if (dg > d) { const uint32_t p = atomicAdd(&s_cnt, 1u); wk[p] = x[u]; wix[p] = i; }
            else if (dg == d) { const uint32_t p = atomicAdd(&s_np, 1u); pk[p] = x[u]; pix[p] = i; }
          }
        }
        __syncthreads();
        // Rank the candidates: every winner (digit above the pivot digit) outranks every pivot-digit
        // key, so a winner's rank is its rank among the winners and a pivot key's is A plus its
        // rank in the pivot digit.  Keys are unique: rank < k selects the k largest, in order.
        for (uint32_t i = threadIdx.x; i < A + B; i += SLT) {
          uint32_t r = 0;
          if (i < A) {
            const uint64_t x = wk[i];
            for (uint32_t j = 0; j < A; ++j) r += wk[j] > x;
            victim[o + r] = wix[i];
          } else {
            const uint64_t x = pk[i - A];
            r = A;
            for (uint32_t j = 0; j < B; ++j) r += pk[j] > x;
            if (r < k) victim[o + r] = pix[i - A];
          }
        }
        __syncthreads();
      }
    }
    if (fast) continue;
    // general path
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
  SAGA_CK(h2d(dn, hn.data(), sizeof(ScoreNode) * t->n_nodes, s));
  ScoreArgs a{};
  a.v = t->v; a.nodes = dn; a.b = *b;
  a.alpha = cfg->alpha; a.beta = cfg->beta; a.gamma = cfg->gamma;
  a.p_low = cfg->p_low_pm; a.p_high = cfg->p_high_pm; a.ttl_max = cfg->ttl_max_us;
  a.score = score; a.key = key;
  prof_begin(SAGA_PROF_SCORE, s);
  if (b->policy == SAGA_POLICY_BELADY) {
    const bool vec = ((uintptr_t)b->cand_lid % 16 == 0) && ((uintptr_t)b->cand_nu % 16 == 0) && ((uintptr_t)key % 16 == 0);
    k_key_belady<<<nsm_count() * 8, 256, 0, s>>>(b->cand_lid, b->cand_nu, b->seg_off, b->n_seg, vec, key);
  } else {
    const size_t dyn = (size_t)SC_STAGE * 4;
    SAGA_CK(cudaFuncSetAttribute(k_score, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    k_score<<<std::min<unsigned>(b->n_seg, nsm_count()), ST, dyn, s>>>(a);
  }
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
  SAGA_CK(d2h(off.data(), seg_off, 8 * (size_t(n_seg) + 1), s));
  SAGA_CK(cudaStreamSynchronize(s));
  uint64_t mx = 1;
  for (uint32_t i = 0; i < n_seg; ++i) mx = std::max<uint64_t>(mx, off[i + 1] - off[i]);
  uint64_t np2 = 1;
  while (np2 < mx) np2 <<= 1;
  const size_t dyn = (size_t)KMAX * (8 + 8 + 4 + 4);
  SAGA_CK(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_select, SLT, dyn);
  const unsigned grid = std::min<unsigned>(n_seg, nsm_count() * (unsigned)std::max(occ, 1));
  uint64_t* sk = nullptr;
  uint32_t* si = nullptr;
  SAGA_CK(ws_malloc((void**)&sk, 8 * np2 * grid, s));
  SAGA_CK(ws_malloc((void**)&si, 4 * np2 * grid, s));
  prof_begin(SAGA_PROF_SELECT, s);
  k_select<<<grid, SLT, dyn, s>>>(key, seg_off, k, n_seg, out_off, victim, sk, si, np2);
  prof_end(SAGA_PROF_SELECT, s);
  count_launch();
  SAGA_CK_LAUNCH();
  ws_free(sk, s);
  ws_free(si, s);
  return SAGA_OK;
}

}  // namespace saga
