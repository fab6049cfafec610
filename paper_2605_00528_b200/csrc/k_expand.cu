// A3 per-node access streams (the sigma of P:881-885 replayed in P:905).  For node w and each
// epoch e in increasing order:
//   MIG records: for each migration (e, s, v -> w) the block set of s's newest call admitted
//                before T_e (the session's KV moved in by the steal), ascending s;
//   CALL records: the ranges of every call placed at w with e(c) = e, in (t, s) order.
// Invalidations (e, s, w -> t) are attached to the first record epoch >= e of node w, plus a
// trailing sentinel event (DESIGN.md R-inv: equivalent to applying them at e because nothing
// happens at w in between).
#include "saga_internal.cuh"

namespace saga {
namespace {

unsigned grid_for(uint64_t n, int threads = NTHREADS) {
  uint64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148u * 64u) g = 148u * 64u;
  return (unsigned)g;
}

__global__ void k_flag_node(const uint8_t* node_of, uint32_t n, uint32_t w, uint32_t* flag) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) flag[c] = node_of[c] == w;
}
__global__ void k_scatter_flag(const uint32_t* flag, const uint32_t* pos, uint32_t n, uint32_t* out) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    if (flag[c]) out[pos[c]] = c;
}
__global__ void k_flag_mig(const Mig* m, uint32_t n, uint32_t w, uint32_t* fthief, uint32_t* fvict) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    fthief[i] = m[i].t == w;
    fvict[i] = m[i].v == w;
  }
}
__global__ void k_scatter_mig(const Mig* m, const uint32_t* flag, const uint32_t* pos, uint32_t n, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (flag[i]) out[pos[i]] = i;
}

// newest call of session s admitted strictly before epoch e (binary search in call order)
__device__ uint32_t newest_before(const TraceView& v, uint32_t s, uint32_t e) {
  uint32_t lo = v.sc_off[s], hi = v.sc_off[s + 1];
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (v.sc_e[mid] < e) lo = mid + 1; else hi = mid;
  }
  return lo > v.sc_off[s] ? v.sc_call[lo - 1] : NONE;
}

// merge CALL groups (node's calls in call order), MIG groups (by epoch) and PREFETCH groups (by
// epoch, call order within one) -> group arrays; per epoch MIG, then PREFETCH, then CALL
__device__ __forceinline__ uint32_t count_le(const uint32_t* list, uint32_t n, const uint32_t* key_of, uint32_t e,
                                             bool strict) {
  uint32_t lo = 0, hi = n;  // #entries with key < e (strict) or <= e
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t k = key_of[list[mid]];
    if (strict ? k < e : k <= e) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__global__ void k_groups(TraceView v, const uint32_t* clist, uint32_t nC, const Mig* migs, const uint32_t* mlist,
                         uint32_t nM, const uint32_t* mig_e, const uint32_t* plist, uint32_t nP, uint32_t* g_call,
                         uint32_t* g_kind, uint32_t* g_e, int64_t* g_t, uint64_t* g_len,
                         unsigned long long* max_len) {
  const uint32_t n = nC + nM + nP;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t dst, call, kind, e;
    int64_t tv;
    uint64_t len;
    if (i < nC) {
      call = clist[i];
      e = v.ecall[call];
      dst = i + count_le(mlist, nM, mig_e, e, false) + (nP ? count_le(plist, nP, v.pf_e, e, false) : 0u);
      kind = 0;
      tv = v.call_t[call];
      len = v.rsum[call];
    } else if (i < nC + nM) {
      const uint32_t m = i - nC;
      const Mig g = migs[mlist[m]];
      e = g.e;
      dst = m + count_le(clist, nC, v.ecall, e, true) + (nP ? count_le(plist, nP, v.pf_e, e, true) : 0u);
      call = newest_before(v, g.s, e);
      kind = 1;
      tv = (int64_t)e * v.epoch_us;
      len = call == NONE ? 0 : v.rsum[call];
    } else {
      const uint32_t p = i - nC - nM;
      call = plist[p];
      e = v.pf_e[call];
      dst = p + count_le(mlist, nM, mig_e, e, false) + count_le(clist, nC, v.ecall, e, true);
      kind = 2;
      tv = (int64_t)e * v.epoch_us;
      len = v.pf_len[call];
    }
    g_call[dst] = call;
    g_kind[dst] = kind;
    g_e[dst] = e;
    g_t[dst] = tv;
    g_len[dst] = len;
    atomicMax(max_len, (unsigned long long)len);  // largest single-call block set (SAGA_ERR_CAPACITY)
  }
}
// epoch of each migration (key table for the merge ranks)
__global__ void k_mig_e(const Mig* m, uint32_t n, uint32_t* e) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) e[i] = m[i].e;
}
// PREFETCH candidates of node w (in call order) and their sort keys
__global__ void k_flag_pf(const uint8_t* node_of, const uint32_t* pf_e, uint32_t n, uint32_t w, uint32_t* flag) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    flag[c] = node_of[c] == w && pf_e[c] != 0;
}
__global__ void k_pf_keys(const uint32_t* list, uint32_t n, const uint32_t* pf_e, uint32_t* key) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) key[i] = pf_e[list[i]];
}
__global__ void k_gather_u32(const uint32_t* src, const uint32_t* idx, uint32_t n, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}

__global__ void k_ev_head(const uint32_t* g_e, uint32_t G, uint32_t* head) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < G; i += gridDim.x * blockDim.x)
    head[i] = (i == 0 || g_e[i] != g_e[i - 1]) ? 1u : 0u;
}

__global__ void k_ev_fill(const uint32_t* g_e, const uint32_t* head, const uint32_t* hpos, uint32_t G, uint32_t* ev_e,
                          uint32_t* ev_g) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < G; i += gridDim.x * blockDim.x)
    if (head[i]) { ev_e[hpos[i]] = g_e[i]; ev_g[hpos[i]] = i; }
}

// sentinel event + invalidation attachment + act lookup
__global__ void k_ev_finish(uint32_t J, uint32_t G, uint32_t w, uint32_t* ev_e, uint32_t* ev_g, const Mig* migs,
                            const uint32_t* ilist, uint32_t nI, uint32_t* inv_s, uint32_t* inv_e, uint32_t* ev_inv,
                            const ActRec* act, uint32_t n_act, uint32_t* ev_act) {
  const uint32_t Jr = J - 1;  // record events
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= J; j += gridDim.x * blockDim.x) {
    if (j == Jr) { ev_e[j] = 0xFFFFFFFFu; ev_g[j] = G; ev_act[j] = 0; }
    if (j == J) { ev_g[j] = G; ev_inv[j] = nI; continue; }
    if (j == 0) ev_inv[0] = 0;
    else {
      uint32_t ep = ev_e[j - 1];  // #inv with epoch <= e_{j-1}
      if (j - 1 == Jr) ep = 0xFFFFFFFFu;
      uint32_t lo = 0, hi = nI;
      while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (migs[ilist[mid]].e <= ep) lo = mid + 1; else hi = mid; }
      ev_inv[j] = lo;
    }
    if (j < Jr) {
      const uint32_t e = ev_e[j];
      uint32_t lo = 0, hi = n_act;  // first act record >= (e, w)
      while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        const ActRec a = act[mid];
        if (a.e < e || (a.e == e && a.w < w)) lo = mid + 1; else hi = mid;
      }
      ev_act[j] = (lo < n_act && act[lo].e == e && act[lo].w == w) ? act[lo].mask : 0u;
    }
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nI; i += gridDim.x * blockDim.x) {
    inv_s[i] = migs[ilist[i]].s;
    inv_e[i] = migs[ilist[i]].e;
  }
}

// one warp per group: write the global block ids of the group's ranges at its positions (a
// PREFETCH group: its first g_len blocks) and mark the CALL records that are their block's first
// touch in the whole trace (ftg bitmap)
__global__ void k_fill_stream(TraceView v, const uint32_t* g_call, const uint32_t* g_kind, const uint64_t* g_pos,
                              uint32_t G, uint32_t* block, uint32_t* ftg) {
  const int lane = threadIdx.x & 31;
  for (uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < G; g += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t c = g_call[g];
    if (c == NONE) continue;
    const bool call_rec = g_kind[g] == 0;
    uint64_t p = g_pos[g];
    const uint64_t pe = g_pos[g + 1];
    for (uint32_t r = v.roff[c]; r < v.roff[c + 1] && p < pe; ++r) {
      const uint32_t lo = v.rlo[r], n = (uint32_t)min((uint64_t)v.rlen[r], pe - p);
      for (uint32_t i = lane; i < n; i += 32) {
        block[p + i] = lo + i;
        if (call_rec && v.fcall[lo + i] == c) atomicOr(&ftg[(p + i) >> 5], 1u << ((p + i) & 31));
      }
      p += n;
    }
  }
}

}  // namespace

saga_status run_expand(saga_trace* t, uint32_t w) {
  ProfScope prof(SAGA_PROF_EXPAND, t->stream);
  const TraceView& v = t->v;
  NodeDev& nd = t->nodes[w];
  cudaStream_t s = t->stream;
  const uint32_t nc = v.n_calls, nm = t->n_mig;
  // per-node CALL list (stable compaction of node_of == w)
  uint32_t* flag = dalloc<uint32_t>(t, nc);
  uint32_t* pos = dalloc<uint32_t>(t, size_t(nc) + 1);
  uint32_t* clist = dalloc<uint32_t>(t, nc);
  uint32_t* ft = dalloc<uint32_t>(t, size_t(nm) + 1);
  uint32_t* fv = dalloc<uint32_t>(t, size_t(nm) + 1);
  uint32_t* pt = dalloc<uint32_t>(t, size_t(nm) + 1);
  uint32_t* pv = dalloc<uint32_t>(t, size_t(nm) + 1);
  uint32_t* mlist = dalloc<uint32_t>(t, size_t(nm) + 1);
  uint32_t* ilist = dalloc<uint32_t>(t, size_t(nm) + 1);
  if (!flag || !pos || !clist || !ft || !fv || !pt || !pv || !mlist || !ilist) { set_error("out of device memory (expand)"); return SAGA_ERR_OOM; }
  k_flag_node<<<grid_for(nc), NTHREADS, 0, s>>>(t->node_of, nc, w, flag);
  count_launch();
  SAGA_CK(scan_u32(t, flag, pos, nc));
  k_scatter_flag<<<grid_for(nc), NTHREADS, 0, s>>>(flag, pos, nc, clist);
  count_launch();
  uint32_t nC = 0, nM = 0, nI = 0, nP = 0;
  uint32_t* mig_e = dalloc<uint32_t>(t, size_t(nm) + 1);
  uint32_t* plist = nullptr;
  if (!mig_e) { set_error("out of device memory (expand)"); return SAGA_ERR_OOM; }
  if (nm > 0) {
    k_mig_e<<<grid_for(nm), NTHREADS, 0, s>>>(t->migs, nm, mig_e);
    count_launch();
  }
  if (v.pf_e && nc > 0) {  // PREFETCH groups of this node, stably sorted by their boundary
    uint32_t* pflag = dalloc<uint32_t>(t, nc);
    uint32_t* ppos = dalloc<uint32_t>(t, size_t(nc) + 1);
    uint32_t* pl0 = dalloc<uint32_t>(t, nc);
    if (!pflag || !ppos || !pl0) { set_error("out of device memory (expand)"); return SAGA_ERR_OOM; }
    k_flag_pf<<<grid_for(nc), NTHREADS, 0, s>>>(t->node_of, v.pf_e, nc, w, pflag);
    count_launch();
    SAGA_CK(scan_u32(t, pflag, ppos, nc));
    k_scatter_flag<<<grid_for(nc), NTHREADS, 0, s>>>(pflag, ppos, nc, pl0);
    count_launch();
    SAGA_CK(d2h(&nP, ppos + nc, 4, s));
    if (nP > 0) {
      uint32_t* key = dalloc<uint32_t>(t, nP);
      uint32_t* skey = dalloc<uint32_t>(t, nP);
      uint32_t* perm = dalloc<uint32_t>(t, nP);
      plist = dalloc<uint32_t>(t, nP);
      if (!key || !skey || !perm || !plist) { set_error("out of device memory (expand)"); return SAGA_ERR_OOM; }
      k_pf_keys<<<grid_for(nP), NTHREADS, 0, s>>>(pl0, nP, v.pf_e, key);
      count_launch();
      SAGA_CK(onesweep_sort_pairs(t, key, nP, 32, skey, perm, s));  // stable: call order within a boundary
      k_gather_u32<<<grid_for(nP), NTHREADS, 0, s>>>(pl0, perm, nP, plist);
      count_launch();
    }
  }
  if (nm > 0) {
    k_flag_mig<<<grid_for(nm), NTHREADS, 0, s>>>(t->migs, nm, w, ft, fv);
    count_launch();
    SAGA_CK(scan_u32(t, ft, pt, nm));
    SAGA_CK(scan_u32(t, fv, pv, nm));
    k_scatter_mig<<<grid_for(nm), NTHREADS, 0, s>>>(t->migs, ft, pt, nm, mlist);
    k_scatter_mig<<<grid_for(nm), NTHREADS, 0, s>>>(t->migs, fv, pv, nm, ilist);
    count_launch(2);
    SAGA_CK(d2h(&nM, pt + nm, 4, s));
    SAGA_CK(d2h(&nI, pv + nm, 4, s));
  }
  SAGA_CK_LAUNCH();
  SAGA_CK(d2h(&nC, pos + nc, 4, s));
  SAGA_CK(cudaStreamSynchronize(s));
  const uint32_t G = nC + nM + nP;
  nd.G = G;
  nd.n_inv = nI;
  nd.g_call = dalloc<uint32_t>(t, G);
  nd.g_kind = dalloc<uint32_t>(t, G);
  nd.g_e = dalloc<uint32_t>(t, G);
  nd.g_t = dalloc<int64_t>(t, G);
  uint64_t* g_len = dalloc<uint64_t>(t, G);
  nd.g_pos = dalloc<uint64_t>(t, size_t(G) + 1);
  uint32_t* head = dalloc<uint32_t>(t, G);
  uint32_t* hpos = dalloc<uint32_t>(t, size_t(G) + 1);
  unsigned long long* gmax = dalloc<unsigned long long>(t, 1);
  if (!gmax) { set_error("out of device memory (expand)"); return SAGA_ERR_OOM; }
  SAGA_CK(cudaMemsetAsync(gmax, 0, 8, s));
  if (!nd.g_call || !nd.g_kind || !nd.g_e || !nd.g_t || !g_len || !nd.g_pos || !head || !hpos) {
    set_error("out of device memory (expand)");
    return SAGA_ERR_OOM;
  }
  if (G > 0) {
    k_groups<<<grid_for(G), NTHREADS, 0, s>>>(v, clist, nC, t->migs, mlist, nM, mig_e, plist, nP, nd.g_call, nd.g_kind,
                                              nd.g_e, nd.g_t, g_len, gmax);
    k_ev_head<<<grid_for(G), NTHREADS, 0, s>>>(nd.g_e, G, head);
    count_launch(2);
  }
  SAGA_CK(scan_u64(t, g_len, nd.g_pos, G));
  SAGA_CK(scan_u32(t, head, hpos, G));
  uint32_t Jr = 0;
  uint64_t N = 0;
  SAGA_CK_LAUNCH();
  SAGA_CK(d2h(&Jr, hpos + G, 4, s));
  SAGA_CK(d2h(&N, nd.g_pos + G, 8, s));
  unsigned long long gm = 0;
  SAGA_CK(d2h(&gm, gmax, 8, s));
  nd.max_group = gm;
  SAGA_CK(cudaStreamSynchronize(s));
  if (N >= (1ull << 31)) { set_error("node %u stream has %llu accesses (limit 2^31)", w, (unsigned long long)N); return SAGA_ERR_STATE; }
  nd.N = N;
  nd.J = Jr + 1;
  nd.ev_e = dalloc<uint32_t>(t, nd.J);
  nd.ev_g = dalloc<uint32_t>(t, size_t(nd.J) + 1);
  nd.ev_inv = dalloc<uint32_t>(t, size_t(nd.J) + 1);
  nd.ev_act = dalloc<uint32_t>(t, nd.J);
  nd.inv_s = dalloc<uint32_t>(t, nI);
  nd.inv_e = dalloc<uint32_t>(t, nI);
  nd.block = dalloc<uint32_t>(t, N);
  nd.ftg = dalloc<uint32_t>(t, N / 32 + 1);
  if (!nd.ev_e || !nd.ev_g || !nd.ev_inv || !nd.ev_act || !nd.inv_s || !nd.inv_e || !nd.block || !nd.ftg) {
    set_error("out of device memory (expand)");
    return SAGA_ERR_OOM;
  }
  if (G > 0) {
    k_ev_fill<<<grid_for(G), NTHREADS, 0, s>>>(nd.g_e, head, hpos, G, nd.ev_e, nd.ev_g);
    count_launch();
  }
  k_ev_finish<<<grid_for(size_t(nd.J) + 1 + nI), NTHREADS, 0, s>>>(nd.J, G, w, nd.ev_e, nd.ev_g, t->migs, ilist, nI,
                                                                  nd.inv_s, nd.inv_e, nd.ev_inv, t->act, t->n_act,
                                                                  nd.ev_act);
  count_launch();
  SAGA_CK(cudaMemsetAsync(nd.ftg, 0, (N / 32 + 1) * 4, s));
  if (G > 0) {
    k_fill_stream<<<grid_for(uint64_t(G) * 32), NTHREADS, 0, s>>>(v, nd.g_call, nd.g_kind, nd.g_pos, G, nd.block, nd.ftg);
    count_launch();
  }
  SAGA_CK_LAUNCH();
  return SAGA_OK;
}

}  // namespace saga
