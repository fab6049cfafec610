// A4 part 2: Belady next use and derived per-position quantities.
//
// k_segscan (sorted order): head flags mark the first occurrence of each block id in the sorted
//   (block, position) sequence; a single-pass decoupled look-back scan of the head count gives
//   the dense local id; the neighbour in sorted order gives next_use; heads are the node's first
//   touches.  Results are scattered to stream order.
// k_epoch_stats (stream order): the last record of a block in its epoch has next_use >= epoch
//   end, so per epoch distinct = #{p : nxt[p] >= end} (-> W_lo); records whose block repeats
//   later in the same epoch mark that later record "not first in epoch"; per-epoch counts of
//   first touches and last touches give the live-block count W_hi by a prefix scan.
#include "saga_internal.cuh"

namespace saga {
namespace {

constexpr int SS_T = 256;
constexpr int SS_ITEMS = 8;
constexpr int SS_TILE = SS_T * SS_ITEMS;
constexpr unsigned long long F_AGG = 1ull << 62;
constexpr unsigned long long F_INC = 2ull << 62;
constexpr unsigned long long V_MASK = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(SS_T) k_segscan(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ sval,
                                                  uint64_t n, const uint32_t* __restrict__ owner,
                                                  uint32_t* __restrict__ nxt, uint32_t* __restrict__ lidf,
                                                  uint32_t* __restrict__ lown, uint32_t* __restrict__ l2g,
                                                  unsigned long long* status,
                                                  uint32_t* tile_counter, uint32_t* n_local_out) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t wsum[SS_T / 32];
  __shared__ unsigned long long s_prefix;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * SS_TILE + (uint64_t)threadIdx.x * SS_ITEMS;
  uint32_t k[SS_ITEMS + 1], v[SS_ITEMS];
  uint32_t prevk = 0;
#pragma unroll
  for (int i = 0; i < SS_ITEMS; ++i) {
    const uint64_t j = base + i;
    k[i] = j < n ? skey[j] : 0xFFFFFFFFu;
    v[i] = j < n ? sval[j] : 0u;
  }
  k[SS_ITEMS] = (base + SS_ITEMS < n) ? skey[base + SS_ITEMS] : 0xFFFFFFFFu;
  prevk = (base > 0 && base - 1 < n) ? skey[base - 1] : 0xFFFFFFFFu;
  uint32_t heads = 0;
#pragma unroll
  for (int i = 0; i < SS_ITEMS; ++i) {
    const uint64_t j = base + i;
    const uint32_t pk = i == 0 ? prevk : k[i - 1];
    if (j < n && (j == 0 || pk != k[i])) ++heads;
  }
  // block exclusive scan of head counts
  uint32_t x = heads;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  for (int w = 0; w < SS_T / 32; ++w) { if (w < wid) wpre += wsum[w]; tot += wsum[w]; }
  const uint32_t texcl = wpre + x - heads;
  // decoupled look-back on the tile total, 32 predecessors per step (lane l reads tile t2 - l)
  if (wid == 0) {
    unsigned long long* my = status + tile;
    unsigned long long ex = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed64(my, F_INC | tot);
    } else {
      if (lane == 0) st_relaxed64(my, F_AGG | tot);
      int64_t t2 = (int64_t)tile - 1;
      while (true) {
        const int64_t idx = t2 - lane;
        unsigned long long s = F_INC;  // before tile 0: an inclusive zero
        if (idx >= 0) { do { s = ld_relaxed64(status + idx); } while ((s & (F_AGG | F_INC)) == 0); }
        const uint32_t inc = __ballot_sync(0xffffffffu, (s & F_INC) != 0);
        const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest inclusive predecessor, else all 32
        unsigned long long v = lane <= stop ? (s & V_MASK) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        ex += v;
        if (inc) break;
        t2 -= 32;
      }
      if (lane == 0) st_relaxed64(my, F_INC | (ex + tot));
    }
    if (lane == 0) s_prefix = ex;
  }
  __syncthreads();
  uint32_t lid = (uint32_t)(s_prefix + texcl);  // number of heads before this thread's first item
#pragma unroll
  for (int i = 0; i < SS_ITEMS; ++i) {
    const uint64_t j = base + i;
    if (j >= n) break;
    const uint32_t pk = i == 0 ? prevk : k[i - 1];
    const bool head = (j == 0 || pk != k[i]);
    if (head) ++lid;
    const uint32_t l = lid - 1;
    const bool has_next = (j + 1 < n) && k[i + 1] == k[i];
    const uint32_t pos = v[i];
    uint32_t nv;
    if (i + 1 < SS_ITEMS) nv = v[i + 1];
    else nv = has_next ? sval[j + 1] : 0u;
    nxt[pos] = has_next ? nv : INF32;
    lidf[pos] = l | (head ? LID_FTN : 0u);
    if (head) { lown[l] = owner[k[i]]; l2g[l] = k[i]; }
    if (j == n - 1) *n_local_out = l + 1;
  }
}

// per-event record ranges: ev_pos[j] = first position of event j (J+1 entries)
__global__ void k_ev_pos(const uint64_t* g_pos, const uint32_t* ev_g, uint32_t J, uint64_t* ev_pos) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= J; j += gridDim.x * blockDim.x) ev_pos[j] = g_pos[ev_g[j]];
}

// stream order: NFIE marks, per-event distinct / first-touch / last-touch counts
__global__ void __launch_bounds__(SS_T) k_epoch_stats(const uint32_t* __restrict__ nxt, uint32_t* lidf,
                                                      const uint32_t* __restrict__ ftg, uint64_t n,
                                                      const uint64_t* __restrict__ ev_pos, uint32_t J,
                                                      uint32_t* cnt_dist, uint32_t* cnt_first, uint32_t* cnt_last) {
  __shared__ uint32_t s_j0;
  const uint64_t t0 = (uint64_t)blockIdx.x * SS_T * SS_ITEMS;
  if (threadIdx.x == 0) {  // event containing the tile's first position: last j with ev_pos[j] <= t0
    uint32_t lo = 0, hi = J;
    while (lo + 1 < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (ev_pos[mid] <= t0) lo = mid; else hi = mid;
    }
    s_j0 = lo;
  }
  __syncthreads();
  const uint64_t p0 = ((uint64_t)blockIdx.x * SS_T + threadIdx.x) * SS_ITEMS;
  if (p0 >= n) return;
  uint32_t j = s_j0;  // a tile spans few events: walk forward to the one containing p0
  while (ev_pos[j + 1] <= p0) ++j;
  uint64_t end = ev_pos[j + 1];
  uint32_t cd = 0, cf = 0, cl = 0;
  for (int i = 0; i < SS_ITEMS; ++i) {
    const uint64_t p = p0 + i;
    if (p >= n) break;
    while (p >= end) {  // flush and move to the next event
      if (cd) atomicAdd(&cnt_dist[j], cd);
      if (cf) atomicAdd(&cnt_first[j], cf);
      if (cl) atomicAdd(&cnt_last[j], cl);
      cd = cf = cl = 0;
      ++j;
      end = ev_pos[j + 1];
    }
    const uint32_t q = nxt[p];
    if (q == INF32) ++cl;
    if ((uint64_t)q >= end) ++cd;                 // last record of its block in this epoch
    else atomicOr(&lidf[q], LID_NFIE);            // the block repeats later in the same epoch
    if (lidf[p] & LID_FTN) ++cf;
    if ((ftg[p >> 5] >> (p & 31)) & 1u) atomicOr(&lidf[p], LID_FTG);   // global first touch (rare)
  }
  if (cd) atomicAdd(&cnt_dist[j], cd);
  if (cf) atomicAdd(&cnt_first[j], cf);
  if (cl) atomicAdd(&cnt_last[j], cl);
}

// W_lo = max distinct; W_hi = max_j (sum_{i<=j} first_i - sum_{i<j} last_i)   (one CTA)
constexpr int SW_T = 1024;
__global__ void k_sweep(const uint32_t* cnt_dist, const uint32_t* cnt_first, const uint32_t* cnt_last, uint32_t Jr,
                        uint32_t* out /*[2]*/) {
  __shared__ long long s_carry_f, s_carry_l;
  __shared__ uint32_t s_lo, s_hi;
  __shared__ long long wf[SW_T / 32], wl[SW_T / 32];
  if (threadIdx.x == 0) { s_carry_f = 0; s_carry_l = 0; s_lo = 0; s_hi = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t b = 0; b < Jr; b += SW_T) {
    const uint32_t j = b + threadIdx.x;
    long long f = j < Jr ? cnt_first[j] : 0, l = j < Jr ? cnt_last[j] : 0;
    uint32_t dist = j < Jr ? cnt_dist[j] : 0;
    long long xf = f, xl = l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long yf = __shfl_up_sync(0xffffffffu, xf, o), yl = __shfl_up_sync(0xffffffffu, xl, o);
      if (lane >= o) { xf += yf; xl += yl; }
    }
    if (lane == 31) { wf[wid] = xf; wl[wid] = xl; }
    __syncthreads();
    long long pf = s_carry_f, pl = s_carry_l;
    for (int w = 0; w < wid; ++w) { pf += wf[w]; pl += wl[w]; }
    const long long F = pf + xf;          // first touches up to and including event j
    const long long Lex = pl + xl - l;    // last touches strictly before event j
    if (j < Jr) {
      atomicMax(&s_lo, dist);
      atomicMax(&s_hi, (uint32_t)(F - Lex));
    }
    __syncthreads();
    if (threadIdx.x == SW_T - 1) { s_carry_f = pf + xf; s_carry_l = pl + xl; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = s_lo; out[1] = s_hi; }
}

// owners come in runs of consecutive local ids: only the first id of a run sets the bit
__global__ void k_present(const uint32_t* lown, uint32_t n_local, uint32_t n_sessions, uint32_t* present) {
  for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n_local; l += gridDim.x * blockDim.x) {
    const uint32_t o = lown[l];
    if (o < n_sessions && (l == 0 || lown[l - 1] != o)) atomicOr(&present[o >> 5], 1u << (o & 31));
  }
}
__global__ void k_flag_present(const uint32_t* call_sess, uint32_t n_calls, const uint32_t* present, uint32_t* flag) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n_calls; c += gridDim.x * blockDim.x) {
    uint32_t s = call_sess[c];
    flag[c] = (present[s >> 5] >> (s & 31)) & 1u;
  }
}
__global__ void k_scatter_flag2(const uint32_t* flag, const uint32_t* pos, uint32_t n, uint32_t* out) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    if (flag[c]) out[pos[c]] = c;
}
__global__ void k_export(const uint32_t* lidf, const uint32_t* nxt, uint64_t n, uint32_t* nu_out, uint32_t* lid_out) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    if (nu_out) nu_out[p] = nxt[p];
    if (lid_out) lid_out[p] = lidf[p] & LID_MASK;
  }
}

unsigned grid_for(uint64_t n, int threads = NTHREADS) {
  uint64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148u * 64u) g = 148u * 64u;
  return (unsigned)g;
}

}  // namespace

saga_status run_next_use(saga_trace* t, uint32_t w, uint32_t* nu_out, uint32_t* lid_out, cudaStream_t s) {
  NodeDev& nd = t->nodes[w];
  const TraceView& v = t->v;
  const uint64_t N = nd.N;
  if (!nd.nu_done) {
    if (!nd.lidf) {
      nd.lidf = dalloc<uint32_t>(t, N);
      nd.nxt = dalloc<uint32_t>(t, N);
      if (!nd.lidf || !nd.nxt) { set_error("out of device memory (next use)"); return SAGA_ERR_OOM; }
    }
    uint32_t key_bits = 32 - __builtin_clz(v.n_blocks > 1 ? v.n_blocks - 1 : 1);
    uint32_t *skey = nullptr, *sval = nullptr, *lown = nullptr, *l2g = nullptr, *tctr = nullptr, *nl = nullptr;
    unsigned long long* status = nullptr;
    const uint64_t tiles = (N + SS_TILE - 1) / SS_TILE;
    SAGA_CK(ws_malloc((void**)&skey, std::max<uint64_t>(N, 1) * 4, s));
    SAGA_CK(ws_malloc((void**)&sval, std::max<uint64_t>(N, 1) * 4, s));
    SAGA_CK(ws_malloc((void**)&lown, std::max<uint64_t>(N, 1) * 4, s));
    SAGA_CK(ws_malloc((void**)&l2g, std::max<uint64_t>(N, 1) * 4, s));
    SAGA_CK(ws_malloc((void**)&status, std::max<uint64_t>(tiles, 1) * 8, s));
    SAGA_CK(ws_malloc((void**)&tctr, 8, s));
    SAGA_CK(ws_malloc((void**)&nl, 4, s));
    SAGA_CK(cudaMemsetAsync(status, 0, std::max<uint64_t>(tiles, 1) * 8, s));
    SAGA_CK(cudaMemsetAsync(tctr, 0, 8, s));
    SAGA_CK(cudaMemsetAsync(nl, 0, 4, s));
    // K4: onesweep sort of (block id, position)
    SAGA_CK(onesweep_sort_pairs(t, nd.block, N, key_bits, skey, sval, s));
    // K5: segmented scans in sorted order
    if (N > 0) {
      prof_begin(SAGA_PROF_SEGSCAN, s);
      k_segscan<<<(unsigned)tiles, SS_T, 0, s>>>(skey, sval, N, v.owner, nd.nxt, nd.lidf, lown, l2g, status, tctr,
                                                        nl);
      prof_end(SAGA_PROF_SEGSCAN, s);
      count_launch();
    }
    // per-event statistics in stream order
    const uint32_t J = nd.J, Jr = nd.J - 1;
    uint64_t* ev_pos = nullptr;
    uint32_t *cd = nullptr, *cf = nullptr, *cl = nullptr, *sw = nullptr;
    SAGA_CK(ws_malloc((void**)&ev_pos, (size_t(J) + 1) * 8, s));
    SAGA_CK(ws_malloc((void**)&cd, size_t(J) * 12 + 16, s));
    cf = cd + J;
    cl = cf + J;
    sw = cl + J;
    SAGA_CK(cudaMemsetAsync(cd, 0, size_t(J) * 12 + 16, s));
    prof_begin(SAGA_PROF_EPOCH, s);
    k_ev_pos<<<grid_for(size_t(J) + 1), NTHREADS, 0, s>>>(nd.g_pos, nd.ev_g, J, ev_pos);
    count_launch();
    if (N > 0) {
      k_epoch_stats<<<(unsigned)((N + SS_TILE - 1) / SS_TILE), SS_T, 0, s>>>(nd.nxt, nd.lidf, nd.ftg, N, ev_pos, J, cd, cf, cl);
      count_launch();
    }
    k_sweep<<<1, SW_T, 0, s>>>(cd, cf, cl, Jr, sw);
    prof_end(SAGA_PROF_EPOCH, s);
    count_launch();
    uint32_t hw[2] = {0, 0}, hn = 0;
    SAGA_CK_LAUNCH();
    SAGA_CK(d2h(hw, sw, 8, s));
    SAGA_CK(d2h(&hn, nl, 4, s));
    SAGA_CK(cudaStreamSynchronize(s));
    nd.w_lo = hw[0];
    nd.w_hi = hw[1];
    nd.n_local = hn;
    nd.lown = dalloc<uint32_t>(t, hn);
    nd.lid2gid = dalloc<uint32_t>(t, hn);
    if (!nd.lown || !nd.lid2gid) { set_error("out of device memory (next use)"); return SAGA_ERR_OOM; }
    SAGA_CK(cudaMemcpyAsync(nd.lown, lown, size_t(hn) * 4, cudaMemcpyDeviceToDevice, s));
    SAGA_CK(cudaMemcpyAsync(nd.lid2gid, l2g, size_t(hn) * 4, cudaMemcpyDeviceToDevice, s));
    // update list: calls of the sessions that own a block at this node (replay session state)
    const uint32_t nc = v.n_calls;
    uint32_t *present = nullptr, *flag = nullptr, *pos = nullptr;
    SAGA_CK(ws_malloc((void**)&present, (size_t(v.n_sessions) / 32 + 1) * 4, s));
    SAGA_CK(ws_malloc((void**)&flag, (size_t(nc) + 1) * 4, s));
    SAGA_CK(ws_malloc((void**)&pos, (size_t(nc) + 1) * 4, s));
    SAGA_CK(cudaMemsetAsync(present, 0, (size_t(v.n_sessions) / 32 + 1) * 4, s));
    k_present<<<grid_for(hn), NTHREADS, 0, s>>>(nd.lown, hn, v.n_sessions, present);
    k_flag_present<<<grid_for(nc), NTHREADS, 0, s>>>(v.call_sess, nc, present, flag);
    count_launch(2);
    SAGA_CK(scan_u32(t, flag, pos, nc));
    uint32_t nu = 0;
    SAGA_CK(d2h(&nu, pos + nc, 4, s));
    SAGA_CK(cudaStreamSynchronize(s));
    nd.n_upd = nu;
    nd.upd_c = dalloc<uint32_t>(t, nu);
    if (!nd.upd_c) { set_error("out of device memory (next use)"); return SAGA_ERR_OOM; }
    k_scatter_flag2<<<grid_for(nc), NTHREADS, 0, s>>>(flag, pos, nc, nd.upd_c);
    count_launch();
    SAGA_CK_LAUNCH();
    ws_free(skey, s);
    ws_free(sval, s);
    ws_free(lown, s);
    ws_free(l2g, s);
    ws_free(status, s);
    ws_free(tctr, s);
    ws_free(nl, s);
    ws_free(ev_pos, s);
    ws_free(cd, s);
    ws_free(present, s);
    ws_free(flag, s);
    ws_free(pos, s);
    nd.nu_done = true;
  }
  if ((nu_out || lid_out) && N > 0) {
    k_export<<<grid_for(N), NTHREADS, 0, s>>>(nd.lidf, nd.nxt, N, nu_out, lid_out);
    count_launch();
    SAGA_CK_LAUNCH();
  }
  return SAGA_OK;
}

}  // namespace saga
