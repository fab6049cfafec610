// Internal declarations of libsaga (B200 / sm_100a).  Not part of the ABI (see include/saga.h).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "saga.h"

namespace saga {

constexpr uint32_t INF32 = 0xFFFFFFFFu;
constexpr uint32_t NONE = 0xFFFFFFFFu;
// packed per-position word of a node stream after next-use: local id | flags
constexpr uint32_t LID_FTN = 1u << 31;   // first touch of the block at this node
constexpr uint32_t LID_NFIE = 1u << 30;  // NOT the first record of the block in its epoch
constexpr uint32_t LID_FTG = 1u << 29;   // CALL record that is the block's first touch in the whole trace
constexpr uint32_t LID_MASK = (1u << 29) - 1;
constexpr int NTHREADS = 256;

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...);

// Stream-ordered workspace cache (saga_api.cu): blocks are cudaMalloc'ed once and recycled per
// (device, stream), so the hot path never grows a memory pool inside a timed step.
cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t s);
void ws_free(void* p, cudaStream_t s);
void ws_release_stream(cudaStream_t s);  // after a sync of s: its idle blocks serve any stream
size_t ws_idle_bytes();                   // idle cached bytes of the current device

// Small host<->device copies of the host-side control flow (sizes, flags, launch tables).  Both
// wait for the stream first and move the bytes through a pinned bounce buffer, then wait again:
// a copy from or to pageable memory blocks inside the driver's staging path until the stream
// reaches it, which stalls every other host thread's pageable copy behind a long kernel (two
// steps in flight on two streams would serialise).  Synchronous: the bytes are in place on return.
cudaError_t d2h(void* dst, const void* src, size_t n, cudaStream_t s);
cudaError_t h2d(void* dst, const void* src, size_t n, cudaStream_t s);

// device-time profile (saga_profile_enable / saga_profile_read)
void prof_begin(int cat, cudaStream_t s);
void prof_end(int cat, cudaStream_t s);
struct ProfScope {
  int cat;
  cudaStream_t s;
  ProfScope(int c, cudaStream_t st) : cat(c), s(st) { prof_begin(cat, s); }
  ~ProfScope() { prof_end(cat, s); }
};
// NVTX range over a host-side scope (ABI entry points): visible in Nsight timelines (header-only
// NVTX3; no cost without an attached tool)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
#define SAGA_NVTX() saga::NvtxScope _saga_nvtx(__func__)

struct Mig { uint32_t e, s, v, t; };
struct ActRec { uint32_t e, w, mask, pad; };

// ------------------------------------------------------------------------------------------
// device-side view of the trace (all pointers device memory)
// ------------------------------------------------------------------------------------------
struct TraceView {
  uint32_t n_calls, n_sessions, n_types, n_aeg, n_edges, n_ranges, n_blocks, n_nodes, btok;
  int64_t epoch_us;
  uint32_t prefill_tok_s, decode_tok_s;
  const int64_t* call_t;
  const uint32_t* call_sess;
  const uint32_t* call_v;
  const uint32_t* call_prompt;
  const uint32_t* call_out;
  const uint32_t* call_new;
  const uint8_t* call_last;
  const uint32_t* roff;
  const uint32_t* rlo;
  const uint32_t* rlen;
  const uint16_t* styp;
  const uint32_t* slo;
  const uint32_t* slen;
  const uint32_t* eoff;
  const uint32_t* edst;
  const float* ep;
  const uint32_t* eq16;
  const int64_t* ttl;
  const uint32_t* obs;
  const uint8_t* term;
  const uint32_t* tlo;
  const uint32_t* tlen;
  const int64_t* cttl = nullptr;   // optional per-call TTL base (overrides ttl[call_v[c]])
  const uint32_t* cobs = nullptr;  // optional per-call expected observation length
  // derived (A1)
  const uint32_t* ecall;   // admission epoch e(c) = t/E + 1
  const int64_t* tend;     // tool start t_c + prefill(new) + decode(out)
  const uint64_t* rsum;    // blocks accessed by the call
  const uint32_t* owner;   // [n_blocks] session, or n_sessions + type, or NONE
  const uint32_t* fcall;   // [n_blocks] first call (global (t, s) order) touching the block, or NONE
  const uint32_t* sc_off;  // [n_sessions+1] calls of each session (CSR, ascending)
  const uint32_t* sc_call;
  const uint32_t* sc_e;    // [n_calls] admission epoch of sc_call[i] (one load per binary-search step)
  const float* ci_P;       // P_reuse(s) after call c (eq:reuse + eq:overlap), fp32 pinned
  const uint32_t* ci_size; // size(s) after call c in blocks (eq:size numerator)
  const uint8_t* ci_fin;   // is_last or terminal
  const uint32_t* pf_e = nullptr;    // [n_calls] PREFETCH boundary of the call (0 = none; SAGA_LOAD_PREFETCH)
  const uint32_t* pf_len = nullptr;  // [n_calls] blocks of its predicted prefix
};

struct NodeDev {
  bool owned = false;
  bool expanded = false;       // A3 done (deferred with SAGA_LOAD_DEFER_EXPAND)
  uint64_t N = 0;          // accesses
  uint32_t J = 0;          // events incl. the trailing sentinel
  uint32_t G = 0;          // record groups
  uint32_t n_inv = 0;
  uint64_t max_group = 0;      // largest block set one call brings to the node (CALL / MIG / PREFETCH group)
  uint32_t* block = nullptr;
  uint32_t* ftg = nullptr;     // [N/32+1] bit p: CALL record p is its block's global first touch
  uint64_t* g_pos = nullptr;   // [G+1]
  int64_t* g_t = nullptr;      // [G]
  uint32_t* g_call = nullptr;  // [G]
  uint32_t* g_kind = nullptr;  // [G] 0 CALL, 1 MIG
  uint32_t* g_e = nullptr;     // [G]
  uint32_t* ev_e = nullptr;    // [J]
  uint32_t* ev_g = nullptr;    // [J+1]
  uint32_t* ev_inv = nullptr;  // [J+1]
  uint32_t* ev_act = nullptr;  // [J]
  uint32_t* inv_s = nullptr;   // [n_inv]
  uint32_t* inv_e = nullptr;   // [n_inv]
  // A4 products
  bool nu_done = false;
  uint32_t n_local = 0, w_lo = 0, w_hi = 0;
  uint32_t* lidf = nullptr;    // [N] local id | LID_FTN | LID_NFIE
  uint32_t* nxt = nullptr;     // [N] next use
  uint32_t* prv = nullptr;     // [N] previous occurrence of the position's block (NONE at a first touch)
  uint32_t* lown = nullptr;    // [n_local] owner of the local block
  uint32_t* lid2gid = nullptr; // [n_local] global block id of the local block (ascending)
  uint32_t n_upd = 0;
  uint32_t* upd_c = nullptr;   // calls of sessions present at the node (call order)
  // replay index (built once per node by the first saga_replay, DESIGN.md §6 "replay state")
  bool rp_done = false;
  uint32_t n_units = 0;        // maximal runs of positions with the same (record group, owner)
  uint32_t max_ev_units = 0;   // most units in one event
  uint64_t* ev_pos = nullptr;  // [J+1] first position of event j
  uint32_t* ev_unit = nullptr; // [J+1] first unit of event j
  uint32_t* ev_upd = nullptr;  // [J] end of the session-update list for event j
  uint32_t* u_of = nullptr;    // [N] unit of position p | KIND_MIG
  uint32_t* upu = nullptr;     // [N] unit of prv[p]
  void* urec = nullptr;        // [n_units] UnitRec (k_replay.cu): t, position range, local owner
  uint32_t n_lo = 0;           // private owners (sessions) with blocks at this node
  uint32_t* upd_lo = nullptr;  // [n_upd] local owner id of each session-update call
};

}  // namespace saga

struct saga_trace {
  int device = 0;
  cudaStream_t stream = nullptr;
  // the replay kernel's own stream, at the device's lowest priority (joined to and from `stream`
  // by events): a launch set of short kernels from other work (the next step's expansion and
  // sort) takes SMs the replay's CTAs free before its queued replay CTAs do
  cudaStream_t replay_stream = nullptr;
  bool sticky_error = false;
  saga_place_cfg pcfg{};
  uint32_t owned_mask = 0;
  saga::TraceView v{};
  // host metadata
  uint32_t n_calls = 0, n_sessions = 0, n_types = 0, n_nodes = 0;
  // placement outputs
  uint8_t* node_of = nullptr;       // [n_calls]
  saga::Mig* migs = nullptr;        // [n_mig]
  saga::ActRec* act = nullptr;      // [n_act]
  uint32_t n_mig = 0, n_act = 0;
  int64_t n_steals = 0, n_reroutes = 0;
  uint32_t load_flags = 0;          // SAGA_LOAD_* of saga_load_trace_ex
  std::vector<saga::NodeDev> nodes;
  void* callkey = nullptr;          // [n_calls] CallKey (k_replay.cu), built by the first replay
  uint32_t* replay_status = nullptr; // [8] the replay kernels' internal-check words (saga_replay_wait)
  std::vector<void*> allocs;        // every device allocation owned by the handle
};

namespace saga {

template <class T>
T* dalloc(saga_trace* t, size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  // 64 bytes of slack: 16-byte TMA bulk copies may round a range's end up past element n - 1
  if (ws_malloc(&p, n * sizeof(T) + 64, t->stream) != cudaSuccess) return nullptr;
  t->allocs.push_back(p);
  return static_cast<T*>(p);
}

// ------------------------------------------------------------------------------------------
// device helpers shared by the kernels of the CUDA path (not by the oracle)
// ------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }
// TTL base / expected observation length of call c: the per-call override when given, else the
// value of its AEG node
__device__ __forceinline__ int64_t call_ttl_base(const TraceView& v, uint32_t c) {
  return v.cttl ? v.cttl[c] : v.ttl[v.call_v[c]];
}
__device__ __forceinline__ uint32_t call_obs(const TraceView& v, uint32_t c) {
  return v.cobs ? v.cobs[c] : v.obs[v.call_v[c]];
}

// ---- 1-D TMA bulk copies (cp.async.bulk) global -> shared, completed on an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: expect `bytes` on bar, then copy [src, src + bytes) to dst (16-byte aligned, bytes % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}

// Per-owner inputs of the WA-LRU key at boundary T_e (resolved by the caller).
struct OwnerKeyIn {
  uint32_t size;     // blocks (eq:size numerator)
  float P;           // P_reuse (eq:reuse), already 0 for finished sessions, act for shared
  bool prot_shared;  // shared prefix: protected iff act
  bool shared;
  bool fin;
  int64_t t_call;    // tool start of c*
  int64_t ttl_base;
};

struct KeyCtx {
  int64_t Te, tau;
  uint32_t smax;
  int64_t den, num;
  int64_t ttl_max;
  float alpha, beta, gamma;
};

// eq:eviction / eq:recency / eq:size in fp32 with explicit round-to-nearest ops (no contraction);
// fd = (float) (T_e - t_last), rounded to nearest (callers that stage candidates keep fd)
__device__ __forceinline__ float wa_lru_score_fd(const KeyCtx& x, float fd, uint32_t size, float P) {
  float R = x.tau > 0 ? fminf(1.0f, __fdiv_rn(fd, __ll2float_rn(x.tau))) : 0.0f;
  float S = __fdiv_rn(__ll2float_rn((long long)size), __ll2float_rn((long long)x.smax));
  float a = __fmul_rn(x.alpha, R);
  float b = __fmul_rn(x.beta, __fsub_rn(1.0f, P));
  float c = __fmul_rn(x.gamma, S);
  return __fadd_rn(__fadd_rn(a, b), c);
}
__device__ __forceinline__ float wa_lru_score(const KeyCtx& x, int64_t t_last, uint32_t size, float P) {
  return wa_lru_score_fd(x, __ll2float_rn(x.Te - t_last), size, P);
}
__device__ __forceinline__ uint32_t quantize_q20(float s) {
  float f = floorf(__fmul_rn(s, 1048576.0f));
  if (!(f > 0.0f)) return 0u;  // also maps NaN to 0
  if (f > 1048576.0f) return 1048576u;
  return (uint32_t)f;
}

// Alg. alg:ttl + eq:pressure as exact integers: el < min(ttl * (1 - m/2), TTL_max),
// m = clamp((occ/C - low) / (high - low), 0, 1) = num / den.
__device__ __forceinline__ bool ttl_protected(const KeyCtx& x, const OwnerKeyIn& o) {
  if (o.shared) return o.prot_shared;
  if (o.fin) return false;
  int64_t el = x.Te - o.t_call;
  if (!(el < x.ttl_max)) return false;
  // 128-bit products: exact for every capacity / TTL the ABI accepts
  return (__int128)2 * x.den * el < (__int128)o.ttl_base * (2 * x.den - x.num);
}

__device__ __forceinline__ uint64_t aeg_key(bool prot, uint32_t q, uint32_t lid) {
  return ((uint64_t)(!prot) << 63) | ((uint64_t)q << 32) | (uint64_t)lid;
}

// ------------------------------------------------------------------------------------------
// host launch helpers (defined in the .cu files)
// ------------------------------------------------------------------------------------------
// exclusive scan of n values into out[0..n] (out[n] = total); scratch handled internally
cudaError_t scan_u64(saga_trace* t, const uint64_t* in, uint64_t* out, uint64_t n);
cudaError_t scan_u32(saga_trace* t, const uint32_t* in, uint32_t* out, uint64_t n);

saga_status load_validate_and_derive(saga_trace* t, const saga_trace_desc* d);
saga_status run_placement(saga_trace* t);
saga_status run_prefetch_plan(saga_trace* t);
saga_status replay_check(saga_trace* t);
saga_status run_expand(saga_trace* t, uint32_t w);
saga_status run_next_use(saga_trace* t, uint32_t w, uint32_t* next_use_out, uint32_t* lid_out, cudaStream_t s);
saga_status run_next_use_nodes(saga_trace* t, const uint32_t* nodes, uint32_t n, cudaStream_t s);
saga_status run_score(const saga_trace* t, const saga_score_batch* b, const saga_replay_cfg* cfg, float* score,
                      uint64_t* key, cudaStream_t s);
saga_status run_select(const uint64_t* key, const uint64_t* seg_off, const uint32_t* k, uint32_t n_seg,
                       const uint64_t* out_off, uint32_t* victim, cudaStream_t s);
// vlog (optional, device): every victim as (epoch << 32) | local id, *vlog_n (device) entries
saga_status run_replay(saga_trace* t, const saga_replay_cfg* cfg, const uint32_t* caps, uint32_t n_caps,
                       const uint32_t* nodes, uint32_t n_owned, int64_t* counters, cudaStream_t s,
                       uint64_t* vlog = nullptr, uint64_t vlog_cap = 0, uint64_t* vlog_n = nullptr);
saga_status run_tool_stats(const saga_trace* t, const uint32_t* label, uint32_t n_labels, uint32_t p_pm, uint32_t window,
                           uint32_t min_samples, uint32_t terms, int64_t* ttl_out, uint32_t* obs_out, cudaStream_t s);
saga_status run_pattern(const saga_trace* t, const uint32_t* label, uint32_t n_labels, const uint8_t* role,
                        uint32_t theta_pm, uint32_t min_tasks, uint64_t* counts, uint32_t* tasks, uint32_t* pred,
                        float* prob, uint64_t* eval, cudaStream_t s);

// radix sort of (key u32, value = position) pairs: sorted keys and values into *_out
cudaError_t onesweep_sort_pairs(saga_trace* t, const uint32_t* keys_in, uint64_t n, uint32_t key_bits,
                                uint32_t* keys_out, uint32_t* vals_out, cudaStream_t s);
// the same over independent segments (one per cache node) in one launch per pass; keys_in /
// keys_out / vals_out of every job 16-byte aligned
struct SortJob {
  const uint32_t* keys_in;
  uint64_t n;
  uint32_t* keys_out;
  uint32_t* vals_out;
};
cudaError_t onesweep_sort_segments(saga_trace* t, const SortJob* jobs, uint32_t nseg, uint32_t key_bits, cudaStream_t s);

}  // namespace saga

#define SAGA_CK(call)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (call);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      saga::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, __LINE__, \
                      cudaGetErrorString(_e));                                                 \
      return SAGA_ERR_CUDA;                                                                    \
    }                                                                                          \
  } while (0)

#define SAGA_CK_LAUNCH() SAGA_CK(cudaGetLastError())
