// A4 part 2: Belady next use and derived per-position quantities,
// for all owned nodes of a batch in one launch per kernel (node = segment; a CTA's tile belongs
// to one node, found from the per-node tile offsets passed by value).
//
// k_segscan (sorted order): head flags mark the first occurrence of each block id in the sorted
//   (block, position) sequence; a single-pass decoupled look-back scan of the head count (per
//   node: the look-back stops at the node's first tile) gives the dense local id; the
//   neighbours in sorted order give next_use and the previous occurrence prv; heads are the
//   node's first touches.  Results are scattered to stream order.  128-bit loads.
// k_epoch_stats (stream order, no atomics on the per-position words): a record is the first of
//   its block in its epoch iff its previous occurrence lies before the epoch (-> LID_NFIE
//   otherwise); the last one iff its next use lies after it, so per epoch
//   distinct = #{p : nxt[p] >= end} (-> W_lo); per-epoch counts of first and last touches give
//   the live-block count W_hi by a prefix scan (k_sweep, one CTA per node).
#include <algorithm>
#include <vector>

#include "saga_internal.cuh"

namespace saga {
namespace {

constexpr int SS_T = 256;
constexpr int SS_ITEMS = 16;
constexpr int SS_TILE = SS_T * SS_ITEMS;
constexpr unsigned long long F_AGG = 1ull << 62;
constexpr unsigned long long F_INC = 2ull << 62;
constexpr unsigned long long V_MASK = (1ull << 62) - 1;
constexpr uint32_t MAXN = 32;  // nodes per launch (n_nodes <= 32)

// one node of a batch
struct NuSeg {
  const uint32_t* skey;   // sorted block ids
  const uint32_t* sval;   // positions in sorted order
  uint64_t n;             // accesses
  uint32_t tile0;         // first global tile of the node
  uint32_t J;             // events incl. the sentinel
  uint32_t* nxt;          // [n] next use (stream order)
  uint32_t* prv;          // [n] previous occurrence (stream order), NONE at a first touch
  uint32_t* lidf;         // [n] local id | flags
  const uint32_t* ftg;    // [n/32+1] global-first-touch bits of CALL records
  uint32_t* lown;         // [n] (scratch sized n; first n_local used) owner of local id
  uint32_t* l2g;          // [n] global block id of local id
  uint32_t* nl_out;       // n_local
  const uint64_t* ev_pos; // [J+1] first position of each event
  uint32_t* cd;           // [J] per event: distinct blocks (W_lo)
  uint32_t* cf;           // [J] first touches
  uint32_t* cl;           // [J] last touches
};
struct NuTable { NuSeg s[MAXN]; };  // kernel parameters (by value: no table upload, no sync)

__device__ __forceinline__ uint32_t find_node(const NuSeg (&segs)[MAXN], uint32_t nseg, uint32_t tile) {
  uint32_t lo = 0, hi = nseg;
  while (lo + 1 < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (segs[mid].tile0 <= tile) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(SS_T, 3) k_segscan(const __grid_constant__ NuTable T, uint32_t nseg,
                                                  const uint32_t* __restrict__ owner, unsigned long long* status,
                                                  uint32_t* tile_counter) {
  __shared__ uint32_t s_tile, s_seg;
  __shared__ uint32_t wsum[SS_T / 32];
  __shared__ unsigned long long s_prefix;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    const uint32_t tg = atomicAdd(tile_counter, 1u);
    s_tile = tg;
    s_seg = find_node(T.s, nseg, tg);
  }
  __syncthreads();
  const uint32_t tg = s_tile;
  const NuSeg S = T.s[s_seg];
  const uint32_t tile = tg - S.tile0;
  const uint64_t n = S.n;
  const uint64_t base = (uint64_t)tile * SS_TILE + (uint64_t)threadIdx.x * SS_ITEMS;
  uint32_t k[SS_ITEMS + 1], v[SS_ITEMS];
  if (base + SS_ITEMS <= n) {  // 128-bit loads of keys and of values
    const uint4* k4 = reinterpret_cast<const uint4*>(S.skey + base);
    const uint4* v4 = reinterpret_cast<const uint4*>(S.sval + base);
    uint4 a[SS_ITEMS / 4], c[SS_ITEMS / 4];
#pragma unroll
    for (int q = 0; q < SS_ITEMS / 4; ++q) { a[q] = __ldcs(k4 + q); c[q] = __ldcs(v4 + q); }
#pragma unroll
    for (int q = 0; q < SS_ITEMS / 4; ++q) {
      k[4 * q] = a[q].x; k[4 * q + 1] = a[q].y; k[4 * q + 2] = a[q].z; k[4 * q + 3] = a[q].w;
      v[4 * q] = c[q].x; v[4 * q + 1] = c[q].y; v[4 * q + 2] = c[q].z; v[4 * q + 3] = c[q].w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < SS_ITEMS; ++i) {
      const uint64_t j = base + i;
      k[i] = j < n ? S.skey[j] : 0xFFFFFFFFu;
      v[i] = j < n ? S.sval[j] : 0u;
    }
  }
  k[SS_ITEMS] = (base + SS_ITEMS < n) ? S.skey[base + SS_ITEMS] : 0xFFFFFFFFu;
  const uint32_t prevk = (base > 0 && base - 1 < n) ? S.skey[base - 1] : 0xFFFFFFFFu;
  const uint32_t prevv = (base > 0 && base - 1 < n) ? S.sval[base - 1] : 0u;
  uint32_t heads = 0;
  uint32_t own[SS_ITEMS];  // owners of the head items, loaded before the scan / look-back
#pragma unroll
  for (int i = 0; i < SS_ITEMS; ++i) {
    const uint64_t j = base + i;
    const uint32_t pk = i == 0 ? prevk : k[i - 1];
    const bool head = j < n && (j == 0 || pk != k[i]);
    own[i] = head ? __ldg(&owner[k[i]]) : 0u;
    if (head) ++heads;
  }
  // block exclusive scan of head counts
  uint32_t x = heads;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  for (int w = 0; w < SS_T / 32; ++w) { if (w < wid) wpre += wsum[w]; tot += wsum[w]; }
  const uint32_t texcl = wpre + x - heads;
  // decoupled look-back on the tile total over this node's tiles, 32 predecessors per step
  if (wid == 0) {
    unsigned long long* my = status + tg;
    unsigned long long ex = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed64(my, F_INC | tot);
    } else {
      if (lane == 0) st_relaxed64(my, F_AGG | tot);
      int64_t t2 = (int64_t)tg - 1;
      while (true) {
        const int64_t idx = t2 - lane;
        unsigned long long s = F_INC;  // before the node's first tile: an inclusive zero
        if (idx >= (int64_t)S.tile0) { do { s = ld_relaxed64(status + idx); } while ((s & (F_AGG | F_INC)) == 0); }
        const uint32_t inc = __ballot_sync(0xffffffffu, (s & F_INC) != 0);
        const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest inclusive predecessor, else all 32
        unsigned long long vv = lane <= stop ? (s & V_MASK) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vv += __shfl_xor_sync(0xffffffffu, vv, o);
        ex += vv;
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
    else nv = has_next ? S.sval[j + 1] : 0u;
    S.nxt[pos] = has_next ? nv : INF32;
    S.prv[pos] = head ? NONE : (i == 0 ? prevv : v[i - 1]);
    S.lidf[pos] = l | (head ? LID_FTN : 0u);
    if (head) { S.lown[l] = own[i]; S.l2g[l] = k[i]; }
    if (j == n - 1) *S.nl_out = l + 1;
  }
}

// stream order: NFIE / FTG flags, per-event distinct / first-touch / last-touch counts.  A CTA
// walks ES_TPC consecutive tiles; the event holding a tile's first position is found by a binary
// search for the CTA's first tile of a node and by walking forward from the previous tile after
// that (a tile spans ~1-2 events).
constexpr uint32_t ES_TPC = 4;
__global__ void __launch_bounds__(SS_T) k_epoch_stats(const __grid_constant__ NuTable T, uint32_t nseg, uint32_t tiles) {
  __shared__ uint32_t s_j0, s_seg;
  uint32_t prev_seg = NONE, prev_j0 = 0;
  for (uint32_t tg = blockIdx.x * ES_TPC; tg < min(tiles, (blockIdx.x + 1) * ES_TPC); ++tg) {
    if (threadIdx.x == 0) {
      const uint32_t sg = find_node(T.s, nseg, tg);
      const NuSeg& S = T.s[sg];
      const uint64_t t0 = (uint64_t)(tg - S.tile0) * SS_TILE;
      uint32_t j0;
      if (sg == prev_seg) {  // last j with ev_pos[j] <= t0, forward from the previous tile's
        j0 = prev_j0;
        while (S.ev_pos[j0 + 1] <= t0) ++j0;
      } else {
        uint32_t lo = 0, hi = S.J;
        while (lo + 1 < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (S.ev_pos[mid] <= t0) lo = mid; else hi = mid;
        }
        j0 = lo;
      }
      s_seg = sg;
      s_j0 = j0;
    }
    __syncthreads();
    prev_seg = s_seg;
    prev_j0 = s_j0;
    const NuSeg S = T.s[prev_seg];
    const uint64_t n = S.n;
    const uint64_t p0 = (uint64_t)(tg - S.tile0) * SS_TILE + (uint64_t)threadIdx.x * SS_ITEMS;
    if (p0 < n) {
      uint32_t j = prev_j0;  // walk forward to the event containing p0
      while (S.ev_pos[j + 1] <= p0) ++j;
      uint64_t start = S.ev_pos[j], end = S.ev_pos[j + 1];
      uint32_t q[SS_ITEMS], pv[SS_ITEMS], lf[SS_ITEMS];
      const bool full = p0 + SS_ITEMS <= n;
      if (full) {
        const uint4* n4 = reinterpret_cast<const uint4*>(S.nxt + p0);
        const uint4* r4 = reinterpret_cast<const uint4*>(S.prv + p0);
        const uint4* l4 = reinterpret_cast<const uint4*>(S.lidf + p0);
        uint4 a[SS_ITEMS / 4], c[SS_ITEMS / 4], e[SS_ITEMS / 4];
#pragma unroll
        for (int z = 0; z < SS_ITEMS / 4; ++z) { a[z] = n4[z]; c[z] = r4[z]; e[z] = l4[z]; }
#pragma unroll
        for (int z = 0; z < SS_ITEMS / 4; ++z) {
          q[4 * z] = a[z].x; q[4 * z + 1] = a[z].y; q[4 * z + 2] = a[z].z; q[4 * z + 3] = a[z].w;
          pv[4 * z] = c[z].x; pv[4 * z + 1] = c[z].y; pv[4 * z + 2] = c[z].z; pv[4 * z + 3] = c[z].w;
          lf[4 * z] = e[z].x; lf[4 * z + 1] = e[z].y; lf[4 * z + 2] = e[z].z; lf[4 * z + 3] = e[z].w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < SS_ITEMS; ++i) {
          const bool ok = p0 + i < n;
          q[i] = ok ? S.nxt[p0 + i] : 0u;
          pv[i] = ok ? S.prv[p0 + i] : 0u;
          lf[i] = ok ? S.lidf[p0 + i] : 0u;
        }
      }
      const uint32_t fw = S.ftg[p0 >> 5];  // the SS_ITEMS (16) positions lie in one 32-bit word
      uint32_t cd = 0, cf = 0, cl = 0;
#pragma unroll
      for (int i = 0; i < SS_ITEMS; ++i) {
        const uint64_t p = p0 + i;
        if (p >= n) break;
        while (p >= end) {  // flush and move to the next event
          if (cd) atomicAdd(&S.cd[j], cd);
          if (cf) atomicAdd(&S.cf[j], cf);
          if (cl) atomicAdd(&S.cl[j], cl);
          cd = cf = cl = 0;
          ++j;
          start = end;
          end = S.ev_pos[j + 1];
        }
        if (q[i] == INF32) ++cl;
        if ((uint64_t)q[i] >= end) ++cd;                                   // last record of its block in this epoch
        if (lf[i] & LID_FTN) ++cf;
        if (pv[i] != NONE && (uint64_t)pv[i] >= start) lf[i] |= LID_NFIE;  // the block already came up this epoch
        if ((fw >> ((uint32_t)p & 31u)) & 1u) lf[i] |= LID_FTG;             // global first touch of a CALL record
      }
      if (full) {
        uint4* l4 = reinterpret_cast<uint4*>(S.lidf + p0);
#pragma unroll
        for (int z = 0; z < SS_ITEMS / 4; ++z) l4[z] = make_uint4(lf[4 * z], lf[4 * z + 1], lf[4 * z + 2], lf[4 * z + 3]);
      } else {
        for (int i = 0; i < SS_ITEMS; ++i) if (p0 + i < n) S.lidf[p0 + i] = lf[i];
      }
      if (cd) atomicAdd(&S.cd[j], cd);
      if (cf) atomicAdd(&S.cf[j], cf);
      if (cl) atomicAdd(&S.cl[j], cl);
    }
    __syncthreads();  // s_seg / s_j0 are rewritten for the next tile
  }
}

// W_lo = max distinct; W_hi = max_j (sum_{i<=j} first_i - sum_{i<j} last_i)   (one CTA per node)
constexpr int SW_T = 1024;
__global__ void k_sweep(const __grid_constant__ NuTable T, uint32_t* out /*[nseg][2]*/) {
  __shared__ long long s_carry_f, s_carry_l;
  __shared__ uint32_t s_lo, s_hi;
  __shared__ long long wf[SW_T / 32], wl[SW_T / 32];
  const NuSeg& S = T.s[blockIdx.x];
  const uint32_t Jr = S.J - 1;  // record events (the last one is the sentinel)
  if (threadIdx.x == 0) { s_carry_f = 0; s_carry_l = 0; s_lo = 0; s_hi = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t b = 0; b < Jr; b += SW_T) {
    const uint32_t j = b + threadIdx.x;
    long long f = j < Jr ? S.cf[j] : 0, l = j < Jr ? S.cl[j] : 0;
    uint32_t dist = j < Jr ? S.cd[j] : 0;
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
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = s_lo; out[2 * blockIdx.x + 1] = s_hi; }
}

// per-event record ranges of every node: ev_pos[j] = first position of event j (J+1 entries)
struct EvPosArgs { const uint64_t* g_pos[MAXN]; const uint32_t* ev_g[MAXN]; uint64_t* ev_pos[MAXN]; uint32_t J[MAXN]; };
__global__ void k_ev_pos(const __grid_constant__ EvPosArgs A) {
  const uint32_t w = blockIdx.y;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= A.J[w]; j += gridDim.x * blockDim.x)
    A.ev_pos[w][j] = A.g_pos[w][A.ev_g[w][j]];
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

// A4 of one batch of nodes (all not yet done, all expanded)
saga_status next_use_batch(saga_trace* t, const std::vector<uint32_t>& ws, cudaStream_t s) {
  const TraceView& v = t->v;
  const uint32_t nb = (uint32_t)ws.size();
  const uint32_t key_bits = 32 - __builtin_clz(v.n_blocks > 1 ? v.n_blocks - 1 : 1);
  // scratch layout: every node's slice 16-byte aligned
  std::vector<uint64_t> off(nb);
  uint64_t tot = 0, tiles = 0;
  NuTable T{};
  for (uint32_t i = 0; i < nb; ++i) {
    NodeDev& nd = t->nodes[ws[i]];
    off[i] = tot;
    tot += (nd.N + 3) & ~3ull;
    if (!nd.lidf) {
      nd.lidf = dalloc<uint32_t>(t, nd.N);
      nd.nxt = dalloc<uint32_t>(t, nd.N);
      nd.prv = dalloc<uint32_t>(t, nd.N);
      if (!nd.lidf || !nd.nxt || !nd.prv) { set_error("out of device memory (next use)"); return SAGA_ERR_OOM; }
    }
    T.s[i].n = nd.N;
    T.s[i].tile0 = (uint32_t)tiles;
    T.s[i].J = nd.J;
    tiles += (nd.N + SS_TILE - 1) / SS_TILE;
  }
  uint32_t *skey = nullptr, *sval = nullptr, *lown = nullptr, *l2g = nullptr, *tctr = nullptr, *small = nullptr;
  uint32_t* cnt = nullptr;
  uint64_t* ev_pos = nullptr;
  unsigned long long* status = nullptr;
  uint64_t totJ = 0;
  for (uint32_t i = 0; i < nb; ++i) totJ += t->nodes[ws[i]].J + 1;
  SAGA_CK(ws_malloc((void**)&skey, tot * 4 + 16, s));
  SAGA_CK(ws_malloc((void**)&sval, tot * 4 + 16, s));
  SAGA_CK(ws_malloc((void**)&lown, tot * 4 + 16, s));
  SAGA_CK(ws_malloc((void**)&l2g, tot * 4 + 16, s));
  SAGA_CK(ws_malloc((void**)&status, std::max<uint64_t>(tiles, 1) * 8, s));
  SAGA_CK(ws_malloc((void**)&tctr, 8, s));
  SAGA_CK(ws_malloc((void**)&small, 4 * 3 * MAXN + 16, s));  // [nb][2] sweep, [nb] n_local
  SAGA_CK(ws_malloc((void**)&ev_pos, totJ * 8, s));
  SAGA_CK(ws_malloc((void**)&cnt, totJ * 12 + 16, s));
  SAGA_CK(cudaMemsetAsync(status, 0, std::max<uint64_t>(tiles, 1) * 8, s));
  SAGA_CK(cudaMemsetAsync(tctr, 0, 8, s));
  SAGA_CK(cudaMemsetAsync(small, 0, 4 * 3 * MAXN + 16, s));
  SAGA_CK(cudaMemsetAsync(cnt, 0, totJ * 12 + 16, s));
  // K4: onesweep sort of (block id, position) of every node in one launch per pass
  std::vector<SortJob> jobs(nb);
  for (uint32_t i = 0; i < nb; ++i) {
    const NodeDev& nd = t->nodes[ws[i]];
    jobs[i] = SortJob{nd.block, nd.N, skey + off[i], sval + off[i]};
  }
  SAGA_CK(onesweep_sort_segments(t, jobs.data(), nb, key_bits, s));
  EvPosArgs ep{};
  uint64_t jo = 0;
  uint32_t maxJ = 1;
  for (uint32_t i = 0; i < nb; ++i) {
    NodeDev& nd = t->nodes[ws[i]];
    NuSeg& x = T.s[i];
    x.skey = skey + off[i]; x.sval = sval + off[i];
    x.nxt = nd.nxt; x.prv = nd.prv; x.lidf = nd.lidf; x.ftg = nd.ftg;
    x.lown = lown + off[i]; x.l2g = l2g + off[i]; x.nl_out = small + 2 * MAXN + i;
    x.ev_pos = ev_pos + jo;
    x.cd = cnt + jo; x.cf = cnt + totJ + jo; x.cl = cnt + 2 * totJ + jo;
    ep.g_pos[i] = nd.g_pos; ep.ev_g[i] = nd.ev_g; ep.ev_pos[i] = ev_pos + jo; ep.J[i] = nd.J;
    maxJ = std::max(maxJ, nd.J + 1);
    jo += nd.J + 1;
  }
  if (tiles > 0) {
    // K5: segmented scans in sorted order
    prof_begin(SAGA_PROF_SEGSCAN, s);
    k_segscan<<<(unsigned)tiles, SS_T, 0, s>>>(T, nb, v.owner, status, tctr);
    prof_end(SAGA_PROF_SEGSCAN, s);
    count_launch();
  }
  prof_begin(SAGA_PROF_EPOCH, s);
  k_ev_pos<<<dim3(std::min<unsigned>((maxJ + NTHREADS - 1) / NTHREADS, 1024u), nb), NTHREADS, 0, s>>>(ep);
  count_launch();
  if (tiles > 0) {
    k_epoch_stats<<<(unsigned)((tiles + ES_TPC - 1) / ES_TPC), SS_T, 0, s>>>(T, nb, (uint32_t)tiles);
    count_launch();
  }
  k_sweep<<<nb, SW_T, 0, s>>>(T, small);
  prof_end(SAGA_PROF_EPOCH, s);
  count_launch();
  SAGA_CK_LAUNCH();
  std::vector<uint32_t> hs(3 * MAXN);
  SAGA_CK(d2h(hs.data(), small, 4 * 3 * MAXN, s));
  SAGA_CK(cudaStreamSynchronize(s));
  const uint32_t nc = v.n_calls;
  // update lists of all nodes of the batch: kernels for every node first, then ONE host read of
  // their lengths (each host sync waits for SMs that replays in flight may hold)
  uint32_t* present = nullptr;
  std::vector<uint32_t*> flag(nb, nullptr), pos(nb, nullptr);
  SAGA_CK(ws_malloc((void**)&present, (size_t(v.n_sessions) / 32 + 1) * 4, s));
  for (uint32_t i = 0; i < nb; ++i) {
    SAGA_CK(ws_malloc((void**)&flag[i], (size_t(nc) + 1) * 4, s));
    SAGA_CK(ws_malloc((void**)&pos[i], (size_t(nc) + 1) * 4, s));
  }
  for (uint32_t i = 0; i < nb; ++i) {
    NodeDev& nd = t->nodes[ws[i]];
    nd.w_lo = hs[2 * i];
    nd.w_hi = hs[2 * i + 1];
    const uint32_t hn = nd.N ? hs[2 * MAXN + i] : 0u;
    nd.n_local = hn;
    nd.lown = dalloc<uint32_t>(t, hn);
    nd.lid2gid = dalloc<uint32_t>(t, hn);
    if (!nd.lown || !nd.lid2gid) { set_error("out of device memory (next use)"); return SAGA_ERR_OOM; }
    SAGA_CK(cudaMemcpyAsync(nd.lown, lown + off[i], size_t(hn) * 4, cudaMemcpyDeviceToDevice, s));
    SAGA_CK(cudaMemcpyAsync(nd.lid2gid, l2g + off[i], size_t(hn) * 4, cudaMemcpyDeviceToDevice, s));
    // update list: calls of the sessions that own a block at this node (replay session state)
    SAGA_CK(cudaMemsetAsync(present, 0, (size_t(v.n_sessions) / 32 + 1) * 4, s));
    k_present<<<grid_for(hn), NTHREADS, 0, s>>>(nd.lown, hn, v.n_sessions, present);
    k_flag_present<<<grid_for(nc), NTHREADS, 0, s>>>(v.call_sess, nc, present, flag[i]);
    count_launch(2);
    SAGA_CK(scan_u32(t, flag[i], pos[i], nc));
    SAGA_CK(cudaMemcpyAsync(small + i, pos[i] + nc, 4, cudaMemcpyDeviceToDevice, s));  // (small is free again)
  }
  SAGA_CK(d2h(hs.data(), small, 4 * nb, s));
  for (uint32_t i = 0; i < nb; ++i) {
    NodeDev& nd = t->nodes[ws[i]];
    const uint32_t nu = hs[i];
    nd.n_upd = nu;
    nd.upd_c = dalloc<uint32_t>(t, nu);
    if (!nd.upd_c) { set_error("out of device memory (next use)"); return SAGA_ERR_OOM; }
    k_scatter_flag2<<<grid_for(nc), NTHREADS, 0, s>>>(flag[i], pos[i], nc, nd.upd_c);
    count_launch();
    SAGA_CK_LAUNCH();
    nd.nu_done = true;
  }
  ws_free(skey, s); ws_free(sval, s); ws_free(lown, s); ws_free(l2g, s);
  ws_free(status, s); ws_free(tctr, s); ws_free(small, s); ws_free(ev_pos, s); ws_free(cnt, s);
  ws_free(present, s);
  for (uint32_t i = 0; i < nb; ++i) { ws_free(flag[i], s); ws_free(pos[i], s); }
  return SAGA_OK;
}

}  // namespace

// A4 for several nodes: batches of at most MAXN nodes and ~2^29 accesses (scratch ~24 B/access,
// held by the workspace cache afterwards)
saga_status run_next_use_nodes(saga_trace* t, const uint32_t* nodes, uint32_t n, cudaStream_t s) {
  std::vector<uint32_t> batch;
  uint64_t acc = 0;
  const uint64_t cap = 1ull << 29;
  for (uint32_t i = 0; i <= n; ++i) {
    const bool flush = i == n || batch.size() == MAXN || (!batch.empty() && acc + t->nodes[nodes[i]].N > cap);
    if (flush && !batch.empty()) {
      const saga_status st = next_use_batch(t, batch, s);
      if (st != SAGA_OK) return st;
      batch.clear();
      acc = 0;
    }
    if (i == n) break;
    const NodeDev& nd = t->nodes[nodes[i]];
    if (nd.nu_done || std::find(batch.begin(), batch.end(), nodes[i]) != batch.end()) continue;
    batch.push_back(nodes[i]);
    acc += nd.N;
  }
  return SAGA_OK;
}

saga_status run_next_use(saga_trace* t, uint32_t w, uint32_t* nu_out, uint32_t* lid_out, cudaStream_t s) {
  NodeDev& nd = t->nodes[w];
  if (!nd.nu_done) {
    const saga_status st = run_next_use_nodes(t, &w, 1, s);
    if (st != SAGA_OK) return st;
  }
  const uint64_t N = nd.N;
  if ((nu_out || lid_out) && N > 0) {
    k_export<<<grid_for(N), NTHREADS, 0, s>>>(nd.lidf, nd.nxt, N, nu_out, lid_out);
    count_launch();
    SAGA_CK_LAUNCH();
  }
  return SAGA_OK;
}

}  // namespace saga
