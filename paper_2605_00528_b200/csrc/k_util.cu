// Device-wide exclusive scans (reduce-then-scan, 3 launches) used by the stream-expansion
// bookkeeping of A3 (group sizes, per-node call lists).  Sizes here are O(calls), not O(accesses).
#include "saga_internal.cuh"

namespace saga {

namespace {
constexpr int SCAN_T = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_T * SCAN_ITEMS;

template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_tot[SCAN_T / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T w = lane < SCAN_T / 32 ? warp_tot[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < SCAN_T / 32) warp_tot[lane] = w;
  }
  __syncthreads();
  T base = wid > 0 ? warp_tot[wid - 1] : T(0);
  *total = warp_tot[SCAN_T / 32 - 1];
  __syncthreads();
  return base + x - v;
}

template <class T>
__global__ void __launch_bounds__(SCAN_T) k_tile_reduce(const T* __restrict__ in, uint64_t n, T* __restrict__ sums) {
  uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    uint64_t j = base + (uint64_t)i * SCAN_T + threadIdx.x;
    if (j < n) s += in[j];
  }
  T tot;
  block_excl_scan<T>(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <class T>
__global__ void __launch_bounds__(SCAN_T) k_scan_sums(T* sums, uint64_t nb, T* total_out) {
  // single CTA: exclusive scan of nb tile sums in place
  T carry = 0;
  for (uint64_t b0 = 0; b0 < nb; b0 += SCAN_T) {
    uint64_t j = b0 + threadIdx.x;
    T v = j < nb ? sums[j] : T(0);
    T tot;
    T ex = block_excl_scan<T>(v, &tot);
    if (j < nb) sums[j] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total_out = carry;
}

template <class T>
__global__ void __launch_bounds__(SCAN_T) k_tile_scan(const T* __restrict__ in, uint64_t n, const T* __restrict__ sums,
                                                      T* __restrict__ out) {
  // blocked arrangement: thread owns SCAN_ITEMS consecutive elements
  uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  T v[SCAN_ITEMS];
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = (base + i < n) ? in[base + i] : T(0);
    s += v[i];
  }
  T tot;
  T ex = block_excl_scan<T>(s, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
}

template <class T>
cudaError_t scan_impl(saga_trace* t, const T* in, T* out, uint64_t n) {
  uint64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  T* sums = nullptr;
  cudaError_t e = ws_malloc((void**)&sums, (nb + 1) * sizeof(T), t->stream);
  if (e != cudaSuccess) return e;
  if (nb > 0) {
    k_tile_reduce<T><<<(unsigned)nb, SCAN_T, 0, t->stream>>>(in, n, sums);
    count_launch();
  }
  k_scan_sums<T><<<1, SCAN_T, 0, t->stream>>>(sums, nb, out + n);
  count_launch();
  if (nb > 0) {
    k_tile_scan<T><<<(unsigned)nb, SCAN_T, 0, t->stream>>>(in, n, sums, out);
    count_launch();
  }
  e = cudaGetLastError();
  ws_free(sums, t->stream);
  return e;
}
}  // namespace

cudaError_t scan_u64(saga_trace* t, const uint64_t* in, uint64_t* out, uint64_t n) { return scan_impl<uint64_t>(t, in, out, n); }
cudaError_t scan_u32(saga_trace* t, const uint32_t* in, uint32_t* out, uint64_t n) { return scan_impl<uint32_t>(t, in, out, n); }

}  // namespace saga
