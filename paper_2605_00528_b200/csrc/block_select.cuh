// Block-level building blocks shared by the replay (A7) and the bulk score/select (A5/A6)
// kernels: reductions, an exclusive scan, and radix select of the k largest unique uint64 keys.
//
// Every collective costs ONE __syncthreads: warp partials go to a double-buffered slot in shared
// memory and every warp finishes the combine with shuffles.  A thread can only overwrite a slot
// two collectives later, after the barrier of the collective in between, which every thread
// reaches only once it has read the slot -- so no second barrier is needed.  `Par` carries the
// slot parity; all threads execute the same sequence of collectives, so their parities agree.
#pragma once
#include "saga_internal.cuh"

namespace saga {

struct Add { template <class T> __device__ T operator()(T a, T b) const { return a + b; } };
struct Max { template <class T> __device__ T operator()(T a, T b) const { return a > b ? a : b; } };
struct Or { template <class T> __device__ T operator()(T a, T b) const { return a | b; } };
struct And { template <class T> __device__ T operator()(T a, T b) const { return a & b; } };

struct Par { uint32_t p = 0; };

template <int BT>
struct BlockScratch {
  static constexpr int NW = BT / 32;
  static_assert((NW & (NW - 1)) == 0 && NW <= 32, "block size must be 32 x power of two");
  unsigned long long part[2][NW];
  uint32_t part2[2][NW];  // second value of block_max2
  uint32_t hist[256];
  uint32_t sel_d, sel_above;
};

template <int BT, class T, class Op>
__device__ __forceinline__ T block_reduce(T x, Op op, BlockScratch<BT>& sm, Par& par) {
  constexpr int NW = BT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = op(x, __shfl_xor_sync(0xffffffffu, x, o));
  T* buf = reinterpret_cast<T*>(sm.part[par.p]);
  par.p ^= 1u;
  if (lane == 0) buf[wid] = x;
  __syncthreads();
  T y = buf[lane & (NW - 1)];
#pragma unroll
  for (int o = NW / 2; o > 0; o >>= 1) y = op(y, __shfl_xor_sync(0xffffffffu, y, o));
  return y;
}

// two maxima (int64, uint32) in one collective (one barrier)
template <int BT>
__device__ __forceinline__ void block_max2(long long& x, uint32_t& y, BlockScratch<BT>& sm, Par& par) {
  constexpr int NW = BT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
    y = max(y, __shfl_xor_sync(0xffffffffu, y, o));
  }
  long long* bx = reinterpret_cast<long long*>(sm.part[par.p]);
  uint32_t* by = sm.part2[par.p];
  par.p ^= 1u;
  if (lane == 0) { bx[wid] = x; by[wid] = y; }
  __syncthreads();
  x = bx[lane & (NW - 1)];
  y = by[lane & (NW - 1)];
#pragma unroll
  for (int o = NW / 2; o > 0; o >>= 1) {
    x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
    y = max(y, __shfl_xor_sync(0xffffffffu, y, o));
  }
}

// exclusive scan of one value per thread; *total receives the block sum
template <int BT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total, BlockScratch<BT>& sm, Par& par) {
  constexpr int NW = BT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  uint32_t* buf = reinterpret_cast<uint32_t*>(sm.part[par.p]);
  par.p ^= 1u;
  if (lane == 31) buf[wid] = x;
  __syncthreads();
  const uint32_t y0 = buf[lane & (NW - 1)];
  uint32_t y = y0;
#pragma unroll
  for (int o = 1; o < NW; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, y, o, NW);
    if ((lane & (NW - 1)) >= o) y += t;
  }
  *total = __shfl_sync(0xffffffffu, y, NW - 1);
  return __shfl_sync(0xffffffffu, y - y0, wid) + x - v;
}

// Threshold T with #{i : kb[i] >= T} == k for n keys, 1 <= k <= n, where the keys are unique
// except possibly for copies of the value 0 and T > 0 (the replay pads with zeros).  Radix select
// from the highest bit on which the keys differ, 8-bit digits, early exit when the pivot bucket
// is consumed exactly.  Every pass re-reads kb (L2-resident for replay sizes).
template <int BT>
__device__ uint64_t radix_select(const uint64_t* kb, uint32_t n, uint32_t k, BlockScratch<BT>& sm, Par& par) {
  unsigned long long o = 0, an = ~0ull;
  for (uint32_t i = threadIdx.x; i < n; i += BT) { const uint64_t x = kb[i]; o |= x; an &= x; }
  o = block_reduce<BT, unsigned long long>(o, Or(), sm, par);
  an = block_reduce<BT, unsigned long long>(an, And(), sm, par);
  const unsigned long long diff = o ^ an;
  if (diff == 0) return o;
  const int top = 63 - __clzll(diff);
  const uint64_t above_mask = (top == 63) ? 0ull : ~((2ull << top) - 1ull);
  uint64_t prefix = an & above_mask;   // bits above `top` are common to every key
  uint64_t mask = above_mask;
  int width = min(8, top + 1);
  int shift = top + 1 - width;
  uint32_t rem = k;
  while (true) {
    for (int i = threadIdx.x; i < 256; i += BT) sm.hist[i] = 0;
    __syncthreads();
    const uint32_t dm = (1u << width) - 1u;
    for (uint32_t i = threadIdx.x; i < n; i += BT) {
      const uint64_t x = kb[i];
      if ((x & mask) == prefix) atomicAdd(&sm.hist[(uint32_t)(x >> shift) & dm], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t local[8];
      uint32_t s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { local[j] = sm.hist[255 - (lane * 8 + j)]; s += local[j]; }
      uint32_t x = s;
#pragma unroll
      for (int of = 1; of < 32; of <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, of);
        if (lane >= of) x += y;
      }
      uint32_t above = x - s;  // keys in digits above this lane's first digit
      int found = -1;
      uint32_t above_d = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (found < 0 && above < rem && rem <= above + local[j]) { found = 255 - (lane * 8 + j); above_d = above; }
        above += local[j];
      }
      const uint32_t fm = __ballot_sync(0xffffffffu, found >= 0);
      const int src = __ffs(fm) - 1;
      const int d = __shfl_sync(0xffffffffu, found, src);
      const uint32_t ab = __shfl_sync(0xffffffffu, above_d, src);
      if (lane == 0) { sm.sel_d = (uint32_t)d; sm.sel_above = ab; }
    }
    __syncthreads();
    const uint32_t d = sm.sel_d, ab = sm.sel_above, hd = sm.hist[d];
    __syncthreads();
    rem -= ab;
    prefix |= (uint64_t)d << shift;
    mask |= (uint64_t)dm << shift;
    if (hd == rem || shift == 0) return prefix;
    width = min(8, shift);
    shift -= width;
  }
}

}  // namespace saga
