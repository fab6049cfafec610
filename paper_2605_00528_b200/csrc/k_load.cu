// A1: ingest + validate the columnar trace and derive per-call / per-block tables.
//   * validation rules of include/saga.h (AEG Def. P:526-534; S:22-28 invariants)
//   * owner[b]: session for private spans, n_sessions + type for shared prefixes
//   * e(c) = floor(t_c / E) + 1 (admission at the next 100 ms boundary, P:361 / DESIGN.md R-adm)
//   * t_end(c) = t_c + prefill(new_c) + decode(out_c): tool start in the open-loop timeline
//   * per-call AEG reuse probability P_reuse = sum_u P(v->u) * overlap(s,u) (eq:reuse P:674,
//     eq:overlap linear form P:685) in fp32 with pinned order, size(s) and fin(s)
#include "saga_internal.cuh"

namespace saga {
namespace {

enum : uint32_t {
  V_CALL_ORDER = 1u << 0, V_CALL_RANGE = 1u << 1, V_CALL_IDS = 1u << 2, V_TOKENS = 1u << 3, V_RANGE = 1u << 4,
  V_SPAN = 1u << 5, V_OVERLAP = 1u << 6, V_AEG = 1u << 7, V_PROB = 1u << 8, V_TTL = 1u << 9, V_WORK = 1u << 10,
  V_TIME = 1u << 11, V_TYPE = 1u << 12
};

struct VErr { uint32_t flags; uint32_t first; };

__device__ __forceinline__ void fail(VErr* e, uint32_t bit, uint32_t idx) {
  atomicOr(&e->flags, bit);
  atomicMin(&e->first, idx);
}

__global__ void k_validate_calls(TraceView v, VErr* err) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.n_calls; c += gridDim.x * blockDim.x) {
    int64_t t = v.call_t[c];
    uint32_t s = v.call_sess[c];
    if (t < 0 || t > (int64_t(1) << 50)) fail(err, V_TIME, c);
    if (c > 0) {
      int64_t tp = v.call_t[c - 1];
      uint32_t sp = v.call_sess[c - 1];
      if (!(tp < t || (tp == t && sp < s))) fail(err, V_CALL_ORDER, c);
    }
    if (s >= v.n_sessions || v.call_v[c] >= v.n_aeg) { fail(err, V_CALL_IDS, c); continue; }
    if (v.cttl && (v.cttl[c] < 0 || v.cttl[c] > 1000000000ll)) fail(err, V_TTL, c);
    uint32_t pr = v.call_prompt[c];
    if (pr < 1 || v.call_new[c] > pr) fail(err, V_TOKENS, c);
    int64_t work = ceil_div64(int64_t(pr) * 1000000, v.prefill_tok_s) +
                   ceil_div64(int64_t(v.call_out[c]) * 1000000, v.decode_tok_s);
    if (work >= (int64_t(1) << 32)) fail(err, V_WORK, c);
    uint32_t r0 = v.roff[c], r1 = v.roff[c + 1];
    if (r1 <= r0 || r1 > v.n_ranges) { fail(err, V_CALL_RANGE, c); continue; }  // >= 1 range per call
    uint32_t ty = v.styp[s];
    if (ty >= v.n_types) { fail(err, V_TYPE, c); continue; }
    uint64_t plo = v.slo[s], phi = plo + v.slen[s], tlo = v.tlo[ty], thi = tlo + v.tlen[ty];
    for (uint32_t r = r0; r < r1; ++r) {
      uint64_t lo = v.rlo[r], hi = lo + v.rlen[r];
      if (v.rlen[r] == 0 || hi > v.n_blocks) { fail(err, V_RANGE, c); break; }
      bool ok = (lo >= plo && hi <= phi) || (lo >= tlo && hi <= thi);
      if (!ok) { fail(err, V_RANGE, c); break; }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (v.roff[0] != 0 || v.roff[v.n_calls] != v.n_ranges) fail(err, V_CALL_RANGE, 0);
  }
}

__global__ void k_validate_aeg(TraceView v, VErr* err) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < v.n_aeg; x += gridDim.x * blockDim.x) {
    uint32_t e0 = v.eoff[x], e1 = v.eoff[x + 1];
    if (e1 < e0 || e1 > v.n_edges) { fail(err, V_AEG, x); continue; }
    double sum = 0.0;
    for (uint32_t e = e0; e < e1; ++e) {
      float p = v.ep[e];
      if (v.edst[e] >= v.n_aeg || v.eq16[e] > 65536u) fail(err, V_AEG, x);
      if (!(p >= 0.0f && p <= 1.0f)) fail(err, V_PROB, x);
      sum += (double)p;
    }
    if (sum > 1.0 + 1e-6) fail(err, V_PROB, x);
    if (v.ttl[x] < 0 || v.ttl[x] > 1000000000ll) fail(err, V_TTL, x);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (v.eoff[0] != 0 || v.eoff[v.n_aeg] != v.n_edges)) fail(err, V_AEG, 0);
}

// owner[] by span fill; a second writer of a block means two spans overlap
__global__ void k_fill_owner(TraceView v, uint32_t* owner, VErr* err) {
  const uint32_t n_spans = v.n_sessions + v.n_types;
  const int lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_spans; i += (gridDim.x * blockDim.x) >> 5) {
    uint64_t lo, len;
    uint32_t id;
    if (i < v.n_sessions) {
      lo = v.slo[i]; len = v.slen[i]; id = i;
      if (v.styp[i] >= v.n_types) { if (lane == 0) fail(err, V_TYPE, i); continue; }
    } else {
      uint32_t a = i - v.n_sessions;
      lo = v.tlo[a]; len = v.tlen[a]; id = i;
    }
    if (lo + len > v.n_blocks) { if (lane == 0) fail(err, V_SPAN, i); continue; }
    for (uint64_t b = lane; b < len; b += 32) {
      uint32_t old = atomicCAS(&owner[lo + b], NONE, id);
      if (old != NONE) { fail(err, V_OVERLAP, i); break; }
    }
  }
}

__global__ void k_call_derived(TraceView v, uint32_t* ecall, int64_t* tend, uint64_t* rsum, float* ci_P,
                               uint32_t* ci_size, uint8_t* ci_fin, uint32_t* sess_cnt) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.n_calls; c += gridDim.x * blockDim.x) {
    int64_t t = v.call_t[c];
    ecall[c] = (uint32_t)(t / v.epoch_us + 1);
    tend[c] = t + ceil_div64(int64_t(v.call_new[c]) * 1000000, v.prefill_tok_s) +
              ceil_div64(int64_t(v.call_out[c]) * 1000000, v.decode_tok_s);
    uint64_t s = 0;
    for (uint32_t r = v.roff[c]; r < v.roff[c + 1]; ++r) s += v.rlen[r];
    rsum[c] = s;
    uint32_t x = v.call_v[c];
    uint64_t ncur = uint64_t(v.call_prompt[c]) + v.call_out[c];   // n_cur after the call
    ci_size[c] = (uint32_t)((ncur + v.btok - 1) / v.btok);
    bool fin = v.call_last[c] || v.term[x];
    ci_fin[c] = fin;
    float P = 0.0f;
    if (!fin) {
      for (uint32_t e = v.eoff[x]; e < v.eoff[x + 1]; ++e) {
        uint64_t nsh = (ncur * uint64_t(v.eq16[e])) >> 16;
        uint64_t den = ncur + call_obs(v, c);
        float ov = den == 0 ? 1.0f : __fdiv_rn(__ll2float_rn((long long)nsh), __ll2float_rn((long long)den));
        P = __fadd_rn(P, __fmul_rn(v.ep[e], ov));
      }
      P = fminf(P, 1.0f);
    }
    ci_P[c] = P;
    atomicAdd(&sess_cnt[v.call_sess[c]], 1u);
  }
}

// first_touch_global: the smallest call index (= earliest in (t, s) order) whose ranges touch the
// block; one warp per call, one atomicMin per accessed block (deterministic)
__global__ void k_first_call(TraceView v, uint32_t* fcall) {
  const int lane = threadIdx.x & 31;
  for (uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < v.n_calls; c += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t r = v.roff[c]; r < v.roff[c + 1]; ++r) {
      const uint32_t lo = v.rlo[r], n = v.rlen[r];
      for (uint32_t i = lane; i < n; i += 32) atomicMin(&fcall[lo + i], c);
    }
}

__global__ void k_sess_scatter(TraceView v, const uint32_t* sc_off, uint32_t* fill, uint32_t* sc_call) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.n_calls; c += gridDim.x * blockDim.x) {
    uint32_t s = v.call_sess[c];
    uint32_t k = atomicAdd(&fill[s], 1u);
    sc_call[sc_off[s] + k] = c;
  }
}

__global__ void k_sc_e(TraceView v, const uint32_t* ecall, const uint32_t* sc_call, uint32_t* sc_e) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < v.n_calls; i += gridDim.x * blockDim.x)
    sc_e[i] = ecall[sc_call[i]];
}

__global__ void k_sess_sort(TraceView v, const uint32_t* sc_off, uint32_t* sc_call) {
  // insertion sort of each session's (short) call list into call order
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < v.n_sessions; s += gridDim.x * blockDim.x) {
    uint32_t a = sc_off[s], b = sc_off[s + 1];
    for (uint32_t i = a + 1; i < b; ++i) {
      uint32_t x = sc_call[i];
      uint32_t j = i;
      while (j > a && sc_call[j - 1] > x) { sc_call[j] = sc_call[j - 1]; --j; }
      sc_call[j] = x;
    }
  }
}

// F4 speculative prefetch plan (§4.3; saga.h SAGA_LOAD_PREFETCH): per call
// the boundary at which its predicted successor's prefix is prefetched (0 = none) and its length
__global__ void k_prefetch_plan(TraceView v, uint32_t* pf_e, uint32_t* pf_len) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.n_calls; c += gridDim.x * blockDim.x) {
    uint32_t e_out = 0, len_out = 0;
    const uint32_t x = v.call_v[c];
    const uint32_t k0 = v.eoff[x], k1 = v.eoff[x + 1];
    if (!v.call_last[c] && !v.term[x] && k1 > k0) {
      uint32_t best = k0;  // argmax P(v -> u), ties -> lowest u
      for (uint32_t k = k0 + 1; k < k1; ++k)
        if (v.ep[k] > v.ep[best] || (v.ep[k] == v.ep[best] && v.edst[k] < v.edst[best])) best = k;
      const uint64_t ncur = uint64_t(v.call_prompt[c]) + v.call_out[c];
      const uint64_t nsh = (ncur * uint64_t(v.eq16[best])) >> 16;
      const uint64_t len = min((uint64_t)v.rsum[c], nsh / v.btok);
      const uint32_t e = (uint32_t)(v.tend[c] / v.epoch_us + 1);
      if (len > 0 && e > v.ecall[c]) {
        // the session's next call (call lists are ascending): it must arrive after the prefetch
        const uint32_t s = v.call_sess[c];
        uint32_t lo = v.sc_off[s], hi = v.sc_off[s + 1];
        while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (v.sc_call[mid] <= c) lo = mid + 1; else hi = mid; }
        if (lo == v.sc_off[s + 1] || v.ecall[v.sc_call[lo]] > e) { e_out = e; len_out = (uint32_t)len; }
      }
    }
    pf_e[c] = e_out;
    pf_len[c] = len_out;
  }
}

unsigned grid_for(uint64_t n, int threads = NTHREADS) {
  uint64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148u * 32u) g = 148u * 32u;
  return (unsigned)g;
}

const char* rule_name(uint32_t flags) {
  if (flags & V_CALL_ORDER) return "calls must be strictly increasing in (t, session)";
  if (flags & V_TIME) return "call time outside [0, 2^50]";
  if (flags & V_CALL_IDS) return "call session or AEG node out of range";
  if (flags & V_TOKENS) return "prompt >= 1 and new <= prompt required";
  if (flags & V_WORK) return "call work (prefill + decode us) must be < 2^32";
  if (flags & V_CALL_RANGE) return "call_range_off is not a CSR over n_ranges with >= 1 range per call";
  if (flags & V_RANGE) return "range empty, out of bounds, or outside its session/type span";
  if (flags & V_TYPE) return "session_type >= n_types";
  if (flags & V_SPAN) return "span outside [0, n_blocks)";
  if (flags & V_OVERLAP) return "session / shared spans overlap";
  if (flags & V_AEG) return "AEG CSR or edge endpoint invalid";
  if (flags & V_PROB) return "edge probability outside [0,1] or out-mass > 1";
  if (flags & V_TTL) return "node_ttl_base_us outside [0, 1e9]";
  return "unknown";
}

template <class T>
saga_status upload(saga_trace* t, const T* src, size_t n, const T** dst, bool required) {
  if (n == 0) { *dst = dalloc<T>(t, 1); return *dst ? SAGA_OK : SAGA_ERR_OOM; }
  if (!src) {
    if (required) { set_error("saga_load_trace: a required array pointer is NULL"); return SAGA_ERR_INVALID_ARG; }
  }
  T* p = dalloc<T>(t, n);
  if (!p) { set_error("saga_load_trace: out of device memory"); return SAGA_ERR_OOM; }
  SAGA_CK(cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyDefault, t->stream));  // host or device (UVA)
  *dst = p;
  return SAGA_OK;
}

}  // namespace

saga_status load_validate_and_derive(saga_trace* t, const saga_trace_desc* d) {
  ProfScope prof(SAGA_PROF_LOAD, t->stream);
  TraceView& v = t->v;
  v.n_calls = d->n_calls; v.n_sessions = d->n_sessions; v.n_types = d->n_types; v.n_aeg = d->n_aeg_nodes;
  v.n_edges = d->n_edges; v.n_ranges = d->n_ranges; v.n_blocks = d->n_blocks; v.n_nodes = d->n_nodes;
  v.btok = d->block_tokens;
  v.epoch_us = t->pcfg.epoch_us; v.prefill_tok_s = t->pcfg.prefill_tok_s; v.decode_tok_s = t->pcfg.decode_tok_s;
  if (d->n_nodes < 1 || d->n_nodes > 32) { set_error("saga_load_trace: n_nodes must be in [1, 32]"); return SAGA_ERR_TRACE; }
  if (d->n_types < 1 || d->n_types > 32) { set_error("saga_load_trace: n_types must be in [1, 32]"); return SAGA_ERR_TRACE; }
  if (d->block_tokens < 1) { set_error("saga_load_trace: block_tokens must be >= 1"); return SAGA_ERR_TRACE; }
  saga_status st;
#define UP(field, n, dst) if ((st = upload(t, d->field, (n), &v.dst, true)) != SAGA_OK) return st
  UP(call_t_us, d->n_calls, call_t);
  UP(call_session, d->n_calls, call_sess);
  UP(call_aeg_node, d->n_calls, call_v);
  UP(call_prompt_tokens, d->n_calls, call_prompt);
  UP(call_output_tokens, d->n_calls, call_out);
  UP(call_new_tokens, d->n_calls, call_new);
  UP(call_is_last, d->n_calls, call_last);
  UP(call_range_off, size_t(d->n_calls) + 1, roff);
  UP(range_block_lo, d->n_ranges, rlo);
  UP(range_len, d->n_ranges, rlen);
  UP(session_type, d->n_sessions, styp);
  UP(session_block_lo, d->n_sessions, slo);
  UP(session_block_len, d->n_sessions, slen);
  UP(aeg_edge_off, size_t(d->n_aeg_nodes) + 1, eoff);
  UP(edge_dst, d->n_edges, edst);
  UP(edge_p, d->n_edges, ep);
  UP(edge_shared_q16, d->n_edges, eq16);
  UP(node_ttl_base_us, d->n_aeg_nodes, ttl);
  UP(node_obs_tokens, d->n_aeg_nodes, obs);
  UP(node_terminal, d->n_aeg_nodes, term);
  UP(type_shared_lo, d->n_types, tlo);
  UP(type_shared_len, d->n_types, tlen);
#undef UP
  if (d->call_ttl_base_us && (st = upload(t, d->call_ttl_base_us, d->n_calls, &v.cttl, true)) != SAGA_OK) return st;
  if (d->call_obs_tokens && (st = upload(t, d->call_obs_tokens, d->n_calls, &v.cobs, true)) != SAGA_OK) return st;
  VErr* err = dalloc<VErr>(t, 1);
  uint32_t* owner = dalloc<uint32_t>(t, d->n_blocks);
  if (!err || !owner) { set_error("saga_load_trace: out of device memory"); return SAGA_ERR_OOM; }
  VErr init{0u, 0xFFFFFFFFu};
  SAGA_CK(h2d(err, &init, sizeof(VErr), t->stream));
  SAGA_CK(cudaMemsetAsync(owner, 0xFF, size_t(d->n_blocks) * 4, t->stream));
  k_validate_calls<<<grid_for(d->n_calls), NTHREADS, 0, t->stream>>>(v, err);
  k_validate_aeg<<<grid_for(d->n_aeg_nodes), NTHREADS, 0, t->stream>>>(v, err);
  k_fill_owner<<<grid_for(uint64_t(d->n_sessions + d->n_types) * 32), NTHREADS, 0, t->stream>>>(v, owner, err);
  count_launch(3);
  SAGA_CK_LAUNCH();
  VErr h{};
  SAGA_CK(d2h(&h, err, sizeof(VErr), t->stream));
  SAGA_CK(cudaStreamSynchronize(t->stream));
  if (h.flags) {
    set_error("saga_load_trace: invalid trace: %s (first offending index %u)", rule_name(h.flags), h.first);
    return SAGA_ERR_TRACE;
  }
  v.owner = owner;
  uint32_t* fcall = dalloc<uint32_t>(t, d->n_blocks);
  if (!fcall) { set_error("saga_load_trace: out of device memory"); return SAGA_ERR_OOM; }
  SAGA_CK(cudaMemsetAsync(fcall, 0xFF, size_t(d->n_blocks) * 4, t->stream));
  if (d->n_calls) {
    k_first_call<<<grid_for(uint64_t(d->n_calls) * 32), NTHREADS, 0, t->stream>>>(v, fcall);
    count_launch();
  }
  v.fcall = fcall;
  // derived per-call tables
  uint32_t* ecall = dalloc<uint32_t>(t, d->n_calls);
  int64_t* tend = dalloc<int64_t>(t, d->n_calls);
  uint64_t* rsum = dalloc<uint64_t>(t, d->n_calls);
  float* ciP = dalloc<float>(t, d->n_calls);
  uint32_t* cisz = dalloc<uint32_t>(t, d->n_calls);
  uint8_t* cifin = dalloc<uint8_t>(t, d->n_calls);
  uint32_t* scnt = dalloc<uint32_t>(t, size_t(d->n_sessions) + 1);
  uint32_t* scoff = dalloc<uint32_t>(t, size_t(d->n_sessions) + 1);
  uint32_t* sccall = dalloc<uint32_t>(t, d->n_calls);
  uint32_t* fill = dalloc<uint32_t>(t, d->n_sessions);
  if (!ecall || !tend || !rsum || !ciP || !cisz || !cifin || !scnt || !scoff || !sccall || !fill) {
    set_error("saga_load_trace: out of device memory");
    return SAGA_ERR_OOM;
  }
  SAGA_CK(cudaMemsetAsync(scnt, 0, (size_t(d->n_sessions) + 1) * 4, t->stream));
  SAGA_CK(cudaMemsetAsync(fill, 0, size_t(d->n_sessions) * 4, t->stream));
  k_call_derived<<<grid_for(d->n_calls), NTHREADS, 0, t->stream>>>(v, ecall, tend, rsum, ciP, cisz, cifin, scnt);
  count_launch();
  SAGA_CK_LAUNCH();
  SAGA_CK(scan_u32(t, scnt, scoff, d->n_sessions));
  k_sess_scatter<<<grid_for(d->n_calls), NTHREADS, 0, t->stream>>>(v, scoff, fill, sccall);
  k_sess_sort<<<grid_for(d->n_sessions), NTHREADS, 0, t->stream>>>(v, scoff, sccall);
  uint32_t* sce = dalloc<uint32_t>(t, d->n_calls);
  if (!sce) { set_error("saga_load_trace: out of device memory"); return SAGA_ERR_OOM; }
  k_sc_e<<<grid_for(d->n_calls), NTHREADS, 0, t->stream>>>(v, ecall, sccall, sce);
  count_launch(3);
  SAGA_CK_LAUNCH();
  v.ecall = ecall; v.tend = tend; v.rsum = rsum; v.ci_P = ciP; v.ci_size = cisz; v.ci_fin = cifin;
  v.sc_off = scoff; v.sc_call = sccall; v.sc_e = sce;
  return SAGA_OK;
}

saga_status run_prefetch_plan(saga_trace* t) {
  TraceView& v = t->v;
  uint32_t* pe = dalloc<uint32_t>(t, v.n_calls);
  uint32_t* pl = dalloc<uint32_t>(t, v.n_calls);
  if (!pe || !pl) { set_error("saga_load_trace: out of device memory (prefetch plan)"); return SAGA_ERR_OOM; }
  if (v.n_calls) {
    k_prefetch_plan<<<grid_for(v.n_calls), NTHREADS, 0, t->stream>>>(v, pe, pl);
    count_launch();
    SAGA_CK_LAUNCH();
  }
  v.pf_e = pe;
  v.pf_len = pl;
  return SAGA_OK;
}

}  // namespace saga
