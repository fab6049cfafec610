// A4 part 1: stable LSD "onesweep" radix sort of (block id, position) pairs for sm_100a, over
// several independent segments (one per owned cache node) in ONE launch per digit pass.
//
// One histogram pass reads every key once (128-bit loads) and builds the digit histograms of
// all passes of every segment; then one kernel per 8-bit digit over the tiles of all segments:
// each CTA takes a dynamic tile id (global over the segments, so a segment's tiles start in
// order), loads its keys / values with 128-bit loads and transposes them through shared memory
// into warp-striped order (item i of lane l = element i*32 + l of the warp's sub-tile: ranking in
// memory order keeps the sort stable), ranks them with a ballot multisplit into per-warp
// counters, publishes its per-digit counts, resolves its global offsets by decoupled look-back
// over the predecessor tiles of its own segment (flag | count words, relaxed GPU-scope loads and
// stores), stages the tile in shared memory in digit order and writes it out so that
// consecutive threads write consecutive addresses of a bucket.  Sorting all nodes in one launch
// set replaces n_nodes small launch sets (ramp-up and tail of each) by one grid >> #SMs.
#include <vector>

#include "saga_internal.cuh"

namespace saga {
namespace {

constexpr int RBITS = 8;
constexpr int RADIX = 1 << RBITS;
constexpr int SORT_T = 256;
constexpr int SORT_W = SORT_T / 32;
constexpr int ITEMS = 16;
constexpr int TILE = SORT_T * ITEMS;  // 4096 keys
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1;
constexpr int MAXPASS = 4;
constexpr int HCHUNK = 16384;         // keys per histogram work unit
constexpr uint32_t MAXSEG = 64;       // segments per launch (passed by value as a kernel parameter)

// one segment of one digit pass
struct SortSeg {
  const uint32_t* keys_in;
  const uint32_t* vals_in;   // unused in the first pass (values = positions)
  uint32_t* keys_out;
  uint32_t* vals_out;
  uint64_t n;
  uint32_t tile0;            // first global tile of the segment
  uint32_t chunk0;           // first histogram chunk of the segment
  const uint32_t* bucket_base;  // [RADIX] exclusive scan of this pass's digit histogram
};
struct SegTable { SortSeg s[MAXSEG]; };   // 3.5 KB of kernel parameters (no table upload, no sync)

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// segment of global tile / chunk id x: last entry with start <= x (nseg <= 64, warp-wide search)
template <bool CHUNK>
__device__ __forceinline__ uint32_t find_seg(const SortSeg (&segs)[MAXSEG], uint32_t nseg, uint32_t x) {
  uint32_t lo = 0, hi = nseg;
  while (lo + 1 < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((CHUNK ? segs[mid].chunk0 : segs[mid].tile0) <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// digit histograms of all passes of all segments in one read of the keys
__global__ void __launch_bounds__(SORT_T) k_hist(const __grid_constant__ SegTable T, uint32_t nseg, uint32_t n_chunks,
                                                 int npass, uint32_t* __restrict__ ghist /*[nseg][npass][RADIX]*/) {
  __shared__ uint32_t h[MAXPASS][RADIX];
  const int lane = threadIdx.x & 31;
  for (uint32_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    const uint32_t sg = find_seg<true>(T.s, nseg, ch);
    const SortSeg S = T.s[sg];
    for (int i = threadIdx.x; i < MAXPASS * RADIX; i += SORT_T) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t k0 = (uint64_t)(ch - S.chunk0) * HCHUNK;
    const uint64_t k1 = min(S.n, k0 + HCHUNK);
    const uint4* k4 = reinterpret_cast<const uint4*>(S.keys_in + k0);
    const uint32_t nq = (uint32_t)((k1 - k0) / 4);
    for (uint32_t i = threadIdx.x; i < ((nq + 31) & ~31u); i += SORT_T) {
      const bool ok = i < nq;
      uint4 q = ok ? __ldcs(k4 + i) : make_uint4(0, 0, 0, 0);
      uint32_t kk[4] = {q.x, q.y, q.z, q.w};
      const uint32_t okm = __ballot_sync(0xffffffffu, ok);
#pragma unroll
      for (int p = 0; p < MAXPASS; ++p) {
        if (p >= npass) break;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t d = (kk[j] >> (p * RBITS)) & (RADIX - 1);
          // keys arrive in long ascending runs: high digits are warp-uniform, aggregate them
          const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
          if (__all_sync(0xffffffffu, !ok || d == d0)) {
            if (lane == 0 && okm) atomicAdd(&h[p][d0], (uint32_t)__popc(okm));
          } else if (ok) {
            atomicAdd(&h[p][d], 1u);
          }
        }
      }
    }
    for (uint64_t i = k0 + (uint64_t)nq * 4 + threadIdx.x; i < k1; i += SORT_T)  // tail (< 4 keys)
      for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(S.keys_in[i] >> (p * RBITS)) & (RADIX - 1)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < npass * RADIX; i += SORT_T) {
      const uint32_t c = (&h[0][0])[i];
      if (c) atomicAdd(&ghist[(uint64_t)sg * npass * RADIX + i], c);
    }
    __syncthreads();
  }
}

// exclusive scan of each pass's histogram of each segment -> bucket bases (one CTA per segment)
__global__ void k_hist_scan(uint32_t* ghist, int npass) {
  __shared__ uint32_t s[RADIX];
  uint32_t* g = ghist + (uint64_t)blockIdx.x * npass * RADIX;
  for (int p = 0; p < npass; ++p) {
    const uint32_t v = g[p * RADIX + threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < RADIX; o <<= 1) {
      const uint32_t y = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += y;
      __syncthreads();
    }
    g[p * RADIX + threadIdx.x] = s[threadIdx.x] - v;
    __syncthreads();
  }
}

template <bool FIRST>
__global__ void __launch_bounds__(SORT_T, 4) k_onesweep(const __grid_constant__ SegTable T, uint32_t nseg, int shift,
                                                     uint32_t* status /*[total tiles][RADIX]*/, uint32_t* tile_counter) {
  __shared__ __align__(16) uint32_t s_keys[TILE];
  __shared__ __align__(16) uint32_t s_vals[TILE];
  __shared__ uint32_t s_whist[SORT_W][RADIX];
  __shared__ uint32_t s_excl[RADIX];
  __shared__ uint32_t s_glob[RADIX];
  __shared__ uint32_t s_tile, s_seg;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    const uint32_t tg = atomicAdd(tile_counter, 1u);
    s_tile = tg;
    s_seg = find_seg<false>(T.s, nseg, tg);
  }
  for (int i = threadIdx.x; i < SORT_W * RADIX; i += SORT_T) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tg = s_tile;
  const SortSeg S = T.s[s_seg];
  const uint32_t tile = tg - S.tile0;  // tile index within the segment
  const uint64_t n = S.n;
  const uint64_t base = (uint64_t)tile * TILE;
  const uint64_t wbase = base + (uint64_t)wid * 32 * ITEMS;
  // 128-bit loads of the warp's 32 x ITEMS elements (blocked: lane l holds 4 consecutive
  // elements per load), transposed through the warp's region of s_keys / s_vals to striped order
  uint32_t* wk = s_keys + wid * 32 * ITEMS;
  uint32_t* wv = s_vals + wid * 32 * ITEMS;
  const bool full = wbase + 32 * ITEMS <= n;
#pragma unroll
  for (int q = 0; q < ITEMS / 4; ++q) {
    const uint32_t o = (uint32_t)(q * 128 + lane * 4);  // element offset within the warp's sub-tile
    uint4 kq, vq;
    if (full) {
      kq = __ldcs(reinterpret_cast<const uint4*>(S.keys_in + wbase + o));
      if (!FIRST) vq = __ldcs(reinterpret_cast<const uint4*>(S.vals_in + wbase + o));
    } else {
      uint32_t a[4], b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t idx = wbase + o + j;
        a[j] = idx < n ? S.keys_in[idx] : 0u;
        b[j] = (!FIRST && idx < n) ? S.vals_in[idx] : 0u;
      }
      kq = make_uint4(a[0], a[1], a[2], a[3]);
      vq = make_uint4(b[0], b[1], b[2], b[3]);
    }
    *reinterpret_cast<uint4*>(wk + o) = kq;
    if (!FIRST) *reinterpret_cast<uint4*>(wv + o) = vq;
  }
  __syncwarp();
  uint32_t k[ITEMS], v[ITEMS], r[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    k[i] = wk[i * 32 + lane];
    v[i] = FIRST ? (uint32_t)(wbase + (uint64_t)i * 32 + lane) : wv[i * 32 + lane];
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = wbase + (uint64_t)i * 32 + lane;
    const bool ok = idx < n;
    const uint32_t d = ok ? ((k[i] >> shift) & (RADIX - 1)) : 0x100u;
    // lanes holding the same 9-bit value (0x100 = past the end).  Block ids arrive in ascending
    // runs, so a warp's 32 consecutive keys usually share the digit (high passes) or hold 32
    // consecutive digits (the low pass): two votes settle those; otherwise one match.any
    // (measured 2.50 vs 2.65 ms per C2 sort against 9 ballots, profiles/r02_ab_sort_match_any.log)
    const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
    uint32_t peers;
    if (__all_sync(0xffffffffu, d == d0)) {
      peers = 0xffffffffu;
    } else if (__all_sync(0xffffffffu, d == ((d0 + (uint32_t)lane) & (RADIX - 1)))) {
      peers = 1u << lane;
    } else {
#ifndef SAGA_SORT_BALLOT_RANK
      peers = __match_any_sync(0xffffffffu, d);
#else
      peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < RBITS + 1; ++b) {
        const uint32_t bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
#endif
    }
    const uint32_t leader = 31 - __clz(peers);
    uint32_t c = 0;
    if (ok && lane == leader) {
      c = s_whist[wid][d];
      s_whist[wid][d] = c + __popc(peers);
    }
    c = __shfl_sync(0xffffffffu, c, leader);
    r[i] = c + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: warp exclusive offsets, tile count, look-back
  const int d = threadIdx.x;  // SORT_T == RADIX
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < SORT_W; ++w) {
    const uint32_t x = s_whist[w][d];
    s_whist[w][d] = cnt;
    cnt += x;
  }
  uint32_t* my = status + (uint64_t)tg * RADIX + d;
  if (tile == 0) st_relaxed(my, FLAG_INC | cnt);
  else st_relaxed(my, FLAG_AGG | cnt);
  // tile-local exclusive scan over digits (for staging)
  {
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __shared__ uint32_t wsum[SORT_W];
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < wid; ++w) pre += wsum[w];
    s_excl[d] = pre + x - cnt;
  }
  // decoupled look-back over the predecessor tiles of this segment, for this digit: LB status
  // words per step are loaded together (independent loads), then consumed in order until the
  // first inclusive prefix; an entry not yet published is polled again from there
  constexpr int LB = 8;
  uint32_t excl = 0;
  if (tile > 0) {
    int64_t t2 = (int64_t)tg - 1;
    const int64_t lo = (int64_t)S.tile0;
    while (true) {
      uint32_t st[LB];
#pragma unroll
      for (int k2 = 0; k2 < LB; ++k2)
        st[k2] = (t2 - k2 >= lo) ? ld_relaxed(status + (uint64_t)(t2 - k2) * RADIX + d) : FLAG_INC;
      int used = 0;
      bool done = false;
#pragma unroll
      for (int k2 = 0; k2 < LB; ++k2) {
        if (done || used < k2) continue;               // stopped earlier in this window
        if ((st[k2] & (FLAG_AGG | FLAG_INC)) == 0) continue;  // not ready: poll from here again
        excl += st[k2] & VAL_MASK;
        used = k2 + 1;
        if (st[k2] & FLAG_INC) done = true;
      }
      if (done) break;
      if (used == 0) __nanosleep(64);  // the predecessor has not published yet: back off
      t2 -= used;
    }
    st_relaxed(my, FLAG_INC | (excl + cnt));
  }
  s_glob[d] = S.bucket_base[d] + excl;
  __syncthreads();  // (also: every warp has read its transposed sub-tile before staging overwrites it)
  // stage in digit order
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = wbase + (uint64_t)i * 32 + lane;
    if (idx < n) {
      const uint32_t dd = (k[i] >> shift) & (RADIX - 1);
      const uint32_t p = s_excl[dd] + s_whist[wid][dd] + r[i];
      s_keys[p] = k[i];
      s_vals[p] = v[i];
    }
  }
  __syncthreads();
  const uint32_t valid = (uint32_t)((n - base) < (uint64_t)TILE ? (n - base) : (uint64_t)TILE);
  for (uint32_t j = threadIdx.x; j < valid; j += SORT_T) {
    const uint32_t key = s_keys[j];
    const uint32_t dd = (key >> shift) & (RADIX - 1);
    const uint32_t dst = s_glob[dd] + (j - s_excl[dd]);
    S.keys_out[dst] = key;
    S.vals_out[dst] = s_vals[j];
  }
}

}  // namespace

cudaError_t onesweep_sort_segments(saga_trace* t, const SortJob* jobs, uint32_t nseg, uint32_t key_bits, cudaStream_t s) {
  if (nseg > MAXSEG) {  // more segments than one launch takes: sort them in groups
    for (uint32_t i = 0; i < nseg; i += MAXSEG) {
      const cudaError_t e = onesweep_sort_segments(t, jobs + i, std::min(MAXSEG, nseg - i), key_bits, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  uint64_t total = 0;
  for (uint32_t i = 0; i < nseg; ++i) total += jobs[i].n;
  if (total == 0 || nseg == 0) return cudaSuccess;
  if (key_bits < 1) key_bits = 1;
  ProfScope prof(SAGA_PROF_SORT, s);
  const int npass = (int)((key_bits + RBITS - 1) / RBITS);
  // per-segment tile / chunk layout (segments with n = 0 get no tiles) and ping-pong offsets
  SegTable th{};
  std::vector<SegTable> tp(npass);
  std::vector<uint64_t> off(nseg);
  uint64_t tiles = 0, chunks = 0, tot4 = 0;
  for (uint32_t i = 0; i < nseg; ++i) {
    th.s[i].keys_in = jobs[i].keys_in;
    th.s[i].n = jobs[i].n;
    th.s[i].tile0 = (uint32_t)tiles;
    th.s[i].chunk0 = (uint32_t)chunks;
    tiles += (jobs[i].n + TILE - 1) / TILE;
    chunks += (jobs[i].n + HCHUNK - 1) / HCHUNK;
    off[i] = tot4;
    tot4 += (jobs[i].n + 3) & ~3ull;
  }
  uint32_t *kA = nullptr, *vA = nullptr, *hist = nullptr, *status = nullptr, *tctr = nullptr;
  cudaError_t e;
  if ((e = ws_malloc((void**)&kA, tot4 * 4 + 16, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&vA, tot4 * 4 + 16, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&hist, (size_t)nseg * npass * RADIX * 4, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&status, tiles * RADIX * 4, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&tctr, 4 * MAXPASS, s)) != cudaSuccess) return e;
  cudaMemsetAsync(hist, 0, (size_t)nseg * npass * RADIX * 4, s);
  cudaMemsetAsync(tctr, 0, 4 * MAXPASS, s);
  // pass p writes so that the last pass lands in the caller's outputs and no pass reads and
  // writes the same buffer
  for (uint32_t i = 0; i < nseg; ++i) {
    const uint32_t* ki = jobs[i].keys_in;
    const uint32_t* vi = nullptr;
    for (int p = 0; p < npass; ++p) {
      const bool to_out = (npass - 1 - p) % 2 == 0;
      SortSeg y = th.s[i];
      y.keys_in = ki; y.vals_in = vi;
      y.keys_out = to_out ? jobs[i].keys_out : kA + off[i];
      y.vals_out = to_out ? jobs[i].vals_out : vA + off[i];
      y.bucket_base = hist + ((size_t)i * npass + p) * RADIX;
      tp[p].s[i] = y;
      ki = y.keys_out;
      vi = y.vals_out;
    }
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned hgrid = (unsigned)std::min<uint64_t>(std::max<uint64_t>(chunks, 1), (uint64_t)nsm * 8);
  k_hist<<<hgrid, SORT_T, 0, s>>>(th, nseg, (uint32_t)chunks, npass, hist);
  k_hist_scan<<<nseg, RADIX, 0, s>>>(hist, npass);
  count_launch(2);
  for (int p = 0; p < npass; ++p) {
    cudaMemsetAsync(status, 0, tiles * RADIX * 4, s);  // look-back flags of this pass
    if (p == 0)
      k_onesweep<true><<<(unsigned)tiles, SORT_T, 0, s>>>(tp[p], nseg, p * RBITS, status, tctr + p);
    else
      k_onesweep<false><<<(unsigned)tiles, SORT_T, 0, s>>>(tp[p], nseg, p * RBITS, status, tctr + p);
    count_launch();
  }
  e = cudaGetLastError();
  ws_free(kA, s);
  ws_free(vA, s);
  ws_free(hist, s);
  ws_free(status, s);
  ws_free(tctr, s);
  return e;
}

cudaError_t onesweep_sort_pairs(saga_trace* t, const uint32_t* keys_in, uint64_t n, uint32_t key_bits, uint32_t* keys_out,
                                uint32_t* vals_out, cudaStream_t s) {
  SortJob j{keys_in, n, keys_out, vals_out};
  return onesweep_sort_segments(t, &j, 1, key_bits, s);
}

}  // namespace saga
