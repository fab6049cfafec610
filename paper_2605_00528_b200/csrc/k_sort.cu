// A4 part 1: stable LSD "onesweep" radix sort of (block id, position) pairs for sm_100a.
//
// One histogram pass reads every key once (128-bit loads) and builds the digit histograms of
// all passes; then one kernel per 8-bit digit: each CTA takes a dynamic tile id, ranks its
// keys with warp-level match_any multisplit into per-warp counters, publishes its per-digit
// counts, resolves its global offsets by decoupled look-back over predecessor tiles (flag |
// count words, relaxed GPU-scope loads/stores), stages the tile in shared memory in digit
// order and writes it out so that consecutive threads write consecutive addresses of a bucket.
// Stability follows from ranking in memory order (warp-striped items: item i of lane l is
// element i*32 + l of the warp's sub-tile) and from tile order = look-back order.
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

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// digit histograms of all passes in one read of the keys
__global__ void __launch_bounds__(SORT_T) k_hist(const uint32_t* __restrict__ keys, uint64_t n, int npass,
                                                 uint32_t* __restrict__ ghist /*[npass][RADIX]*/) {
  __shared__ uint32_t h[MAXPASS][RADIX];
  for (int i = threadIdx.x; i < MAXPASS * RADIX; i += SORT_T) (&h[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t n4 = n / 4;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys);
  for (uint64_t i = (uint64_t)blockIdx.x * SORT_T + threadIdx.x; i < ((n4 + 31) & ~31ull); i += (uint64_t)gridDim.x * SORT_T) {
    const bool ok = i < n4;
    uint4 q = ok ? __ldcs(k4 + i) : make_uint4(0, 0, 0, 0);
    uint32_t kk[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int p = 0; p < MAXPASS; ++p) {
      if (p >= npass) break;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t d = (kk[j] >> (p * RBITS)) & (RADIX - 1);
        // keys arrive in long ascending runs: high digits are warp-uniform, aggregate them
        uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
        uint32_t okm = __ballot_sync(0xffffffffu, ok);
        if (__all_sync(0xffffffffu, !ok || d == d0)) {
          if (lane == 0 && okm) atomicAdd(&h[p][d0], (uint32_t)__popc(okm));
        } else if (ok) {
          atomicAdd(&h[p][d], 1u);
        }
      }
    }
  }
  // tail (n % 4 keys)
  if (blockIdx.x == 0) {
    for (uint64_t i = n4 * 4 + threadIdx.x; i < n; i += SORT_T)
      for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(keys[i] >> (p * RBITS)) & (RADIX - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * RADIX; i += SORT_T) {
    uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(&ghist[i], c);
  }
}

// exclusive scan of each pass's histogram -> bucket bases (one CTA of RADIX threads)
__global__ void k_hist_scan(uint32_t* ghist, int npass) {
  __shared__ uint32_t s[RADIX];
  for (int p = 0; p < npass; ++p) {
    uint32_t v = ghist[p * RADIX + threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < RADIX; o <<= 1) {
      uint32_t y = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += y;
      __syncthreads();
    }
    ghist[p * RADIX + threadIdx.x] = s[threadIdx.x] - v;
    __syncthreads();
  }
}

template <bool FIRST>
__global__ void __launch_bounds__(SORT_T) k_onesweep(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                                                     uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                     uint64_t n, int shift, const uint32_t* __restrict__ bucket_base,
                                                     uint32_t* status /*[tiles][RADIX]*/, uint32_t* tile_counter) {
  __shared__ uint32_t s_keys[TILE];
  __shared__ uint32_t s_vals[TILE];
  __shared__ uint32_t s_whist[SORT_W][RADIX];
  __shared__ uint32_t s_excl[RADIX];
  __shared__ uint32_t s_glob[RADIX];
  __shared__ uint32_t s_tile;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = threadIdx.x; i < SORT_W * RADIX; i += SORT_T) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * TILE;
  const uint64_t wbase = base + (uint64_t)wid * 32 * ITEMS;
  uint32_t k[ITEMS], v[ITEMS], r[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = wbase + (uint64_t)i * 32 + lane;
    const bool ok = idx < n;
    k[i] = ok ? __ldcs(keys_in + idx) : 0u;
    if (FIRST) v[i] = (uint32_t)idx;
    else v[i] = ok ? __ldcs(vals_in + idx) : 0u;
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = wbase + (uint64_t)i * 32 + lane;
    const bool ok = idx < n;
    const uint32_t d = ok ? ((k[i] >> shift) & (RADIX - 1)) : 0x100u;
#ifdef SAGA_SORT_MATCH_ANY
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#else
    // lanes holding the same 9-bit value (0x100 = past the end): 9 ballots instead of MATCH
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < RBITS + 1; ++b) {
      const uint32_t bit = (d >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
#endif
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
    uint32_t x = s_whist[w][d];
    s_whist[w][d] = cnt;
    cnt += x;
  }
  uint32_t* my = status + (uint64_t)tile * RADIX + d;
  if (tile == 0) st_relaxed(my, FLAG_INC | cnt);
  else st_relaxed(my, FLAG_AGG | cnt);
  // tile-local exclusive scan over digits (for staging)
  s_excl[d] = cnt;
  __syncthreads();
  {
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __shared__ uint32_t wsum[SORT_W];
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < wid; ++w) pre += wsum[w];
    s_excl[d] = pre + x - cnt;
  }
  // decoupled look-back over predecessor tiles for this digit
  uint32_t excl = 0;
  if (tile > 0) {
    int64_t t2 = (int64_t)tile - 1;
    while (true) {
      uint32_t s;
      do { s = ld_relaxed(status + (uint64_t)t2 * RADIX + d); } while ((s & (FLAG_AGG | FLAG_INC)) == 0);
      excl += s & VAL_MASK;
      if (s & FLAG_INC) break;
      --t2;
    }
    st_relaxed(my, FLAG_INC | (excl + cnt));
  }
  s_glob[d] = bucket_base[d] + excl;
  __syncthreads();
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
    keys_out[dst] = key;
    vals_out[dst] = s_vals[j];
  }
}

}  // namespace

cudaError_t onesweep_sort_pairs(saga_trace* t, const uint32_t* keys_in, uint64_t n, uint32_t key_bits, uint32_t* keys_out,
                                uint32_t* vals_out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (key_bits < 1) key_bits = 1;
  ProfScope prof(SAGA_PROF_SORT, s);
  const int npass = (int)((key_bits + RBITS - 1) / RBITS);
  const uint64_t tiles = (n + TILE - 1) / TILE;
  uint32_t *kA = nullptr, *vA = nullptr, *hist = nullptr, *status = nullptr, *tctr = nullptr;
  cudaError_t e;
  // ping-pong buffers: pass p writes (p odd -> out) so that the last pass lands in *_out
  if ((e = ws_malloc((void**)&kA, n * 4, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&vA, n * 4, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&hist, MAXPASS * RADIX * 4, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&status, tiles * RADIX * 4 * npass, s)) != cudaSuccess) return e;
  if ((e = ws_malloc((void**)&tctr, 4 * MAXPASS, s)) != cudaSuccess) return e;
  cudaMemsetAsync(hist, 0, MAXPASS * RADIX * 4, s);
  cudaMemsetAsync(status, 0, tiles * RADIX * 4 * npass, s);
  cudaMemsetAsync(tctr, 0, 4 * MAXPASS, s);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  uint64_t hb = (n / 4 + SORT_T - 1) / SORT_T;
  unsigned hgrid = (unsigned)std::min<uint64_t>(std::max<uint64_t>(hb, 1), (uint64_t)nsm * 8);
  k_hist<<<hgrid, SORT_T, 0, s>>>(keys_in, n, npass, hist);
  k_hist_scan<<<1, RADIX, 0, s>>>(hist, npass);
  count_launch(2);
  // pass targets: final pass writes keys_out/vals_out
  const uint32_t* ki = keys_in;
  const uint32_t* vi = nullptr;
  for (int p = 0; p < npass; ++p) {
    const bool last = p == npass - 1;
    // choose output so that the last pass ends in *_out and no pass reads and writes the same buffer
    uint32_t* ko = ((npass - 1 - p) % 2 == 0) ? keys_out : kA;
    uint32_t* vo = ((npass - 1 - p) % 2 == 0) ? vals_out : vA;
    (void)last;
    if (p == 0)
      k_onesweep<true><<<(unsigned)tiles, SORT_T, 0, s>>>(ki, nullptr, ko, vo, n, p * RBITS, hist + p * RADIX,
                                                          status + (uint64_t)p * tiles * RADIX, tctr + p);
    else
      k_onesweep<false><<<(unsigned)tiles, SORT_T, 0, s>>>(ki, vi, ko, vo, n, p * RBITS, hist + p * RADIX,
                                                           status + (uint64_t)p * tiles * RADIX, tctr + p);
    count_launch();
    ki = ko;
    vi = vo;
  }
  e = cudaGetLastError();
  ws_free(kA, s);
  ws_free(vA, s);
  ws_free(hist, s);
  ws_free(status, s);
  ws_free(tctr, s);
  return e;
}

}  // namespace saga
