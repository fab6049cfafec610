// C ABI of libsaga (include/saga.h): argument checks, handle lifetime, stream ordering.
// Every compute step runs in the kernels of k_*.cu; nothing here touches trace data on the host.
#include <cstring>
#include <chrono>
#include <mutex>

#include "saga_internal.cuh"

namespace saga {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

// ---------------- profile: CUDA event pairs per kernel family ----------------
namespace prof_detail {
struct ProfRec { int cat; cudaEvent_t a, b; };
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_prof_pool;
thread_local std::vector<std::pair<int, cudaEvent_t>> g_prof_open;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) { cudaEvent_t e = g_prof_pool.back(); g_prof_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace prof_detail
using namespace prof_detail;

void prof_begin(int cat, cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  cudaEvent_t e = prof_event();
  cudaEventRecord(e, s);
  g_prof_open.push_back({cat, e});
}

void prof_end(int cat, cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  for (size_t i = g_prof_open.size(); i-- > 0;) {
    if (g_prof_open[i].first != cat) continue;
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, s);
    g_prof.push_back({cat, g_prof_open[i].second, b});
    g_prof_open.erase(g_prof_open.begin() + (long)i);
    return;
  }
}

// ---------------- workspace cache ----------------
namespace ws_detail {
struct Blk { void* p; size_t size; int dev; cudaStream_t s; bool used; bool any; };  // any: stream drained
std::mutex g_ws_mu;
std::vector<Blk> g_ws;
}  // namespace ws_detail

cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t s) {
  using namespace ws_detail;
  if (bytes == 0) bytes = 1;
  const size_t gran = bytes <= (1ull << 20) ? 512 : (1ull << 20);
  const size_t want = (bytes + gran - 1) & ~(gran - 1);
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(g_ws_mu);
    size_t best = SIZE_MAX, bi = 0;
    for (size_t i = 0; i < g_ws.size(); ++i) {
      const Blk& b = g_ws[i];
      if (b.used || b.dev != dev || (b.s != s && !b.any) || b.size < want || b.size > 2 * want + gran) continue;
      if (b.size < best) { best = b.size; bi = i; }
    }
    if (best != SIZE_MAX) { g_ws[bi].used = true; g_ws[bi].s = s; g_ws[bi].any = false; *p = g_ws[bi].p; return cudaSuccess; }
  }
  void* q = nullptr;
  static const bool dbg = getenv("SAGA_WS_DEBUG") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMalloc(&q, want);
  if (dbg)
    fprintf(stderr, "[saga ws] cudaMalloc %zu B on stream %p: %.3f ms\n", want, (void*)s,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  if (e != cudaSuccess) {  // release cached idle blocks of this device and retry once
    cudaGetLastError();
    std::vector<void*> drop;
    {
      std::lock_guard<std::mutex> g(g_ws_mu);
      for (size_t i = 0; i < g_ws.size();) {
        if (!g_ws[i].used && g_ws[i].dev == dev) { drop.push_back(g_ws[i].p); g_ws.erase(g_ws.begin() + (long)i); }
        else ++i;
      }
    }
    cudaDeviceSynchronize();
    for (void* x : drop) cudaFree(x);
    e = cudaMalloc(&q, want);
    if (e != cudaSuccess) return e;
  }
  std::lock_guard<std::mutex> g(g_ws_mu);
  g_ws.push_back({q, want, dev, s, true, false});
  *p = q;
  return cudaSuccess;
}

// stream-ordered release: later work on the same stream may reuse the block
void ws_free(void* p, cudaStream_t s) {
  using namespace ws_detail;
  if (!p) return;
  std::lock_guard<std::mutex> g(g_ws_mu);
  for (Blk& b : g_ws)
    if (b.p == p) { b.used = false; b.s = s; b.any = false; return; }
}

// bytes held by idle cached blocks of the current device (ws_malloc releases them when a fresh
// allocation does not fit): memory a large allocation can count on besides cudaMemGetInfo's free
size_t ws_idle_bytes() {
  using namespace ws_detail;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_ws_mu);
  size_t n = 0;
  for (const Blk& b : g_ws)
    if (!b.used && b.dev == dev) n += b.size;
  return n;
}

// after the caller synchronised stream s: its idle blocks may serve any stream
void ws_release_stream(cudaStream_t s) {
  using namespace ws_detail;
  std::lock_guard<std::mutex> g(g_ws_mu);
  for (Blk& b : g_ws)
    if (!b.used && b.s == s) b.any = true;
}

// pinned bounce buffers for d2h / h2d, one per concurrent caller
namespace bounce_detail {
constexpr size_t kBounce = 64 * 1024;
std::mutex g_mu;
std::vector<void*> g_free;
void* take() {
  {
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_free.empty()) { void* p = g_free.back(); g_free.pop_back(); return p; }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, kBounce, cudaHostAllocPortable) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  return p;
}
void give(void* p) {
  std::lock_guard<std::mutex> g(g_mu);
  g_free.push_back(p);
}
}  // namespace bounce_detail

// (stream-ordered copy + one sync: the copy waits for the work queued before it on s)
cudaError_t d2h(void* dst, const void* src, size_t n, cudaStream_t s) {
  using namespace bounce_detail;
  cudaError_t e = cudaSuccess;
  if (n == 0) return cudaStreamSynchronize(s);
  void* b = n <= kBounce ? take() : nullptr;
  if ((e = cudaMemcpyAsync(b ? b : dst, src, n, cudaMemcpyDeviceToHost, s)) == cudaSuccess) e = cudaStreamSynchronize(s);
  if (b) {
    if (e == cudaSuccess) memcpy(dst, b, n);
    give(b);
  }
  return e;
}

cudaError_t h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
  using namespace bounce_detail;
  cudaError_t e = cudaSuccess;
  if (n == 0) return cudaStreamSynchronize(s);
  void* b = n <= kBounce ? take() : nullptr;
  if (b) memcpy(b, src, n);
  if ((e = cudaMemcpyAsync(dst, b ? b : src, n, cudaMemcpyHostToDevice, s)) == cudaSuccess) e = cudaStreamSynchronize(s);
  if (b) give(b);
  return e;
}

static void mempool_setup(int device) {
  static std::mutex mu;
  static uint64_t done_mask = 0;
  std::lock_guard<std::mutex> g(mu);
  if (device < 64 && (done_mask >> device) & 1ull) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;  // keep freed blocks cached in the pool across steps
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (device < 64) done_mask |= 1ull << device;
}

}  // namespace saga

using namespace saga;

#define CHECK_HANDLE(t)                                                        \
  do {                                                                         \
    if (!(t)) { set_error("%s: NULL handle", __func__); return SAGA_ERR_INVALID_ARG; } \
    if ((t)->sticky_error) { set_error("%s: handle is in a CUDA error state", __func__); return SAGA_ERR_CUDA; } \
  } while (0)

#define GUARD(t, call)                                 \
  do {                                                 \
    saga_status _s = (call);                           \
    if (_s == SAGA_ERR_CUDA && (t)) (t)->sticky_error = true; \
    if (_s != SAGA_OK) return _s;                      \
  } while (0)

extern "C" {

const char* saga_last_error(void) { return g_err.c_str(); }

uint64_t saga_kernel_launches(void) { return g_launches.load(); }

void saga_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
}

void saga_profile_read(double* ms_out, uint64_t* n_out) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  double ms[SAGA_PROF_NCAT] = {0};
  uint64_t n[SAGA_PROF_NCAT] = {0};
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    float x = 0.f;
    if (cudaEventElapsedTime(&x, r.a, r.b) == cudaSuccess && r.cat >= 0 && r.cat < SAGA_PROF_NCAT) {
      ms[r.cat] += x;
      n[r.cat] += 1;
    }
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof.clear();
  for (int i = 0; i < SAGA_PROF_NCAT; ++i) {
    if (ms_out) ms_out[i] = ms[i];
    if (n_out) n_out[i] = n[i];
  }
}

void saga_free_trace(saga_trace* t) {
  if (!t) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(t->device);
  for (void* p : t->allocs) ws_free(p, t->stream);
  if (cudaStreamSynchronize(t->stream) == cudaSuccess) ws_release_stream(t->stream);  // reusable by other streams
  if (t->replay_stream) cudaStreamDestroy(t->replay_stream);  // its work was joined back to t->stream
  cudaSetDevice(prev);
  delete t;
}

// A3 of a node on first use when the load deferred it (SAGA_LOAD_DEFER_EXPAND)
static saga_status ensure_expanded(saga_trace* t, uint32_t w) {
  NodeDev& nd = t->nodes[w];
  if (nd.expanded) return SAGA_OK;
  const saga_status st = run_expand(t, w);
  if (st == SAGA_OK) nd.expanded = true;
  return st;
}

saga_status saga_load_trace(const saga_trace_desc* desc, const saga_place_cfg* cfg, uint32_t owned_node_mask, int device,
                            saga_stream_t stream, saga_trace** out) {
  return saga_load_trace_ex(desc, cfg, owned_node_mask, device, stream, 0u, out);
}

saga_status saga_load_trace_ex(const saga_trace_desc* desc, const saga_place_cfg* cfg, uint32_t owned_node_mask,
                               int device, saga_stream_t stream, uint32_t flags, saga_trace** out) {
  SAGA_NVTX();
  g_err.clear();
  if (!desc || !cfg || !out) { set_error("saga_load_trace: NULL argument"); return SAGA_ERR_INVALID_ARG; }
  *out = nullptr;
  if (cfg->epoch_us <= 0 || cfg->epoch_us > 1000000000ll || cfg->kappa == 0 || cfg->prefill_tok_s == 0 ||
      cfg->decode_tok_s == 0) {
    set_error("saga_load_trace: epoch_us must be in (0, 1e9] and kappa, prefill_tok_s, decode_tok_s positive");
    return SAGA_ERR_INVALID_ARG;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    set_error("saga_load_trace: no CUDA device %d", device);
    return SAGA_ERR_INVALID_ARG;
  }
  SAGA_CK(cudaSetDevice(device));
  mempool_setup(device);
  saga_trace* t = new saga_trace();
  t->device = device;
  t->stream = (cudaStream_t)stream;
  t->pcfg = *cfg;
  t->n_calls = desc->n_calls;
  t->n_sessions = desc->n_sessions;
  t->n_types = desc->n_types;
  t->n_nodes = desc->n_nodes;
  t->load_flags = flags;
  saga_status st = load_validate_and_derive(t, desc);
  if (st != SAGA_OK) { saga_free_trace(t); return st; }
  t->owned_mask = owned_node_mask ? owned_node_mask : (desc->n_nodes >= 32 ? 0xFFFFFFFFu : ((1u << desc->n_nodes) - 1u));
  t->nodes.assign(desc->n_nodes, NodeDev());
  st = run_placement(t);
  if (st != SAGA_OK) { saga_free_trace(t); return st; }
  if (flags & SAGA_LOAD_PREFETCH) {
    st = run_prefetch_plan(t);
    if (st != SAGA_OK) { saga_free_trace(t); return st; }
  }
  for (uint32_t w = 0; w < desc->n_nodes; ++w) {
    if (!((t->owned_mask >> w) & 1u)) continue;
    t->nodes[w].owned = true;
    if (flags & SAGA_LOAD_DEFER_EXPAND) continue;
    st = ensure_expanded(t, w);
    if (st != SAGA_OK) { saga_free_trace(t); return st; }
  }
  cudaError_t e = cudaStreamSynchronize(t->stream);
  if (e != cudaSuccess) {
    set_error("saga_load_trace: %s", cudaGetErrorString(e));
    saga_free_trace(t);
    return SAGA_ERR_CUDA;
  }
  *out = t;
  return SAGA_OK;
}

saga_status saga_trace_info(const saga_trace* t, uint32_t node, uint64_t* n_access, uint32_t* n_local_blocks) {
  CHECK_HANDLE(t);
  if (node >= t->n_nodes || !t->nodes[node].owned) { set_error("saga_trace_info: node %u not owned", node); return SAGA_ERR_STATE; }
  saga_trace* tm = const_cast<saga_trace*>(t);  // lazy A3 only; the trace is not otherwise modified
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(tm, ensure_expanded(tm, node));
  const NodeDev& nd = t->nodes[node];
  if (n_access) *n_access = nd.N;
  if (n_local_blocks) *n_local_blocks = nd.nu_done ? nd.n_local : UINT32_MAX;
  return SAGA_OK;
}

saga_status saga_placement(const saga_trace* t, uint8_t* node_host, uint32_t* mig_host, uint64_t mig_cap, int64_t* stats) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  SAGA_CK(cudaSetDevice(t->device));
  if (node_host) SAGA_CK(d2h(node_host, t->node_of, t->n_calls, t->stream));
  if (mig_host && mig_cap) {
    uint64_t n = std::min<uint64_t>(mig_cap, t->n_mig);
    if (n) SAGA_CK(d2h(mig_host, t->migs, n * sizeof(Mig), t->stream));
  }
  SAGA_CK(cudaStreamSynchronize(t->stream));
  if (stats) { stats[0] = t->n_steals; stats[1] = t->n_reroutes; stats[2] = t->n_mig; }
  return SAGA_OK;
}

saga_status saga_node_stream_sizes(const saga_trace* t, uint32_t node, uint64_t* n_access, uint32_t* n_events,
                                   uint32_t* n_groups, uint32_t* n_inv) {
  CHECK_HANDLE(t);
  if (node >= t->n_nodes || !t->nodes[node].owned) { set_error("node %u not owned", node); return SAGA_ERR_STATE; }
  saga_trace* tm = const_cast<saga_trace*>(t);  // lazy A3 only
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(tm, ensure_expanded(tm, node));
  const NodeDev& nd = t->nodes[node];
  if (n_access) *n_access = nd.N;
  if (n_events) *n_events = nd.J;
  if (n_groups) *n_groups = nd.G;
  if (n_inv) *n_inv = nd.n_inv;
  return SAGA_OK;
}

namespace {
// internal work of a handle is ordered on its own stream; callers' streams are joined with events
saga_status join(cudaStream_t from, cudaStream_t to) {
  if (!from || !to || from == to) return SAGA_OK;
  cudaEvent_t ev;
  SAGA_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  SAGA_CK(cudaEventRecord(ev, from));
  SAGA_CK(cudaStreamWaitEvent(to, ev, 0));
  cudaEventDestroy(ev);
  return SAGA_OK;
}
__global__ void k_pack_ev(const uint32_t* ev_e, const uint32_t* ev_g, uint32_t J, uint32_t* out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < J; j += gridDim.x * blockDim.x) {
    out[3 * j] = ev_e[j];
    out[3 * j + 1] = ev_g[j];
    out[3 * j + 2] = ev_g[j + 1] - ev_g[j];
  }
}
__global__ void k_pack_grp(const uint64_t* g_pos, const uint32_t* g_kind, uint32_t G, uint64_t* out) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    out[2 * g] = g_pos[g];
    out[2 * g + 1] = g_kind[g];
  }
}
}  // namespace

saga_status saga_node_stream(const saga_trace* t, uint32_t node, uint32_t* block_dev, uint32_t* ev_dev, uint64_t* grp_dev,
                             int64_t* grp_t_dev, uint32_t* inv_dev, saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if (node >= t->n_nodes || !t->nodes[node].owned) { set_error("node %u not owned", node); return SAGA_ERR_STATE; }
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(const_cast<saga_trace*>(t), join(t->stream, (cudaStream_t)stream));
  cudaStream_t s = stream ? (cudaStream_t)stream : t->stream;
  const NodeDev& nd = t->nodes[node];
  if (block_dev && nd.N) SAGA_CK(cudaMemcpyAsync(block_dev, nd.block, nd.N * 4, cudaMemcpyDeviceToDevice, s));
  if (ev_dev && nd.J) { k_pack_ev<<<(nd.J + 255) / 256, 256, 0, s>>>(nd.ev_e, nd.ev_g, nd.J, ev_dev); count_launch(); }
  if (grp_dev && nd.G) { k_pack_grp<<<(nd.G + 255) / 256, 256, 0, s>>>(nd.g_pos, nd.g_kind, nd.G, grp_dev); count_launch(); }
  if (grp_t_dev && nd.G) SAGA_CK(cudaMemcpyAsync(grp_t_dev, nd.g_t, size_t(nd.G) * 8, cudaMemcpyDeviceToDevice, s));
  if (inv_dev && nd.n_inv) SAGA_CK(cudaMemcpyAsync(inv_dev, nd.inv_s, size_t(nd.n_inv) * 4, cudaMemcpyDeviceToDevice, s));
  SAGA_CK_LAUNCH();
  // the handle's stream waits for these reads: saga_free_trace (which syncs it) cannot recycle
  // the trace's buffers while the caller's stream still reads them
  GUARD(const_cast<saga_trace*>(t), join(s, t->stream));
  return SAGA_OK;
}

saga_status saga_belady_next_use(saga_trace* t, uint32_t node, uint32_t* next_use_dev, uint32_t* local_id_dev,
                                 saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if (node >= t->n_nodes || !t->nodes[node].owned) { set_error("saga_belady_next_use: node %u not owned", node); return SAGA_ERR_STATE; }
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(t, join((cudaStream_t)stream, t->stream));
  GUARD(t, ensure_expanded(t, node));
  GUARD(t, run_next_use(t, node, next_use_dev, local_id_dev, t->stream));
  GUARD(t, join(t->stream, (cudaStream_t)stream));
  return SAGA_OK;
}

saga_status saga_belady_next_use_nodes(saga_trace* t, const uint32_t* nodes, uint32_t n_nodes, saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if (n_nodes && !nodes) { set_error("saga_belady_next_use_nodes: NULL argument"); return SAGA_ERR_INVALID_ARG; }
  for (uint32_t i = 0; i < n_nodes; ++i)
    if (nodes[i] >= t->n_nodes || !t->nodes[nodes[i]].owned) {
      set_error("saga_belady_next_use_nodes: node %u not owned", nodes[i]);
      return SAGA_ERR_STATE;
    }
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(t, join((cudaStream_t)stream, t->stream));
  for (uint32_t i = 0; i < n_nodes; ++i) GUARD(t, ensure_expanded(t, nodes[i]));
  GUARD(t, run_next_use_nodes(t, nodes, n_nodes, t->stream));
  GUARD(t, join(t->stream, (cudaStream_t)stream));
  return SAGA_OK;
}

saga_status saga_sweep_range(const saga_trace* t, uint32_t node, uint32_t* w_lo, uint32_t* w_hi) {
  CHECK_HANDLE(t);
  if (node >= t->n_nodes || !t->nodes[node].owned) { set_error("saga_sweep_range: node %u not owned", node); return SAGA_ERR_STATE; }
  const NodeDev& nd = t->nodes[node];
  if (!nd.nu_done) { set_error("saga_sweep_range: call saga_belady_next_use(node %u) first", node); return SAGA_ERR_STATE; }
  if (w_lo) *w_lo = nd.w_lo;
  if (w_hi) *w_hi = nd.w_hi;
  return SAGA_OK;
}

saga_status saga_aeg_score(const saga_trace* t, const saga_score_batch* batch, const saga_replay_cfg* cfg, float* score_dev,
                           uint64_t* key_dev, saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if (!batch || !cfg || !key_dev) { set_error("saga_aeg_score: NULL argument"); return SAGA_ERR_INVALID_ARG; }
  if (batch->policy != SAGA_POLICY_AEG && batch->policy != SAGA_POLICY_BELADY) {
    set_error("saga_aeg_score: policy must be AEG or BELADY");
    return SAGA_ERR_INVALID_ARG;
  }
  if (batch->policy == SAGA_POLICY_AEG)
    for (uint32_t w = 0; w < t->n_nodes; ++w)
      if (t->nodes[w].owned && !t->nodes[w].nu_done) {
        set_error("saga_aeg_score: saga_belady_next_use(node %u) must run first", w);
        return SAGA_ERR_STATE;
      }
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(const_cast<saga_trace*>(t), join(t->stream, (cudaStream_t)stream));
  GUARD(const_cast<saga_trace*>(t), run_score(t, batch, cfg, score_dev, key_dev, stream ? (cudaStream_t)stream : t->stream));
  GUARD(const_cast<saga_trace*>(t), join((cudaStream_t)stream, t->stream));  // see saga_node_stream
  return SAGA_OK;
}

saga_status saga_evict_select(const uint64_t* key_dev, const uint64_t* seg_off_dev, const uint32_t* k_dev, uint32_t n_seg,
                              const uint64_t* out_off_dev, uint32_t* victim_idx_dev, saga_stream_t stream) {
  SAGA_NVTX();
  g_err.clear();
  if (n_seg && (!key_dev || !seg_off_dev || !k_dev || !out_off_dev || !victim_idx_dev)) {
    set_error("saga_evict_select: NULL argument");
    return SAGA_ERR_INVALID_ARG;
  }
  return run_select(key_dev, seg_off_dev, k_dev, n_seg, out_off_dev, victim_idx_dev, (cudaStream_t)stream);
}

saga_status saga_pattern_infer(const saga_trace* t, const uint32_t* call_label_dev, uint32_t n_labels,
                               const uint8_t* session_role_dev, uint32_t theta_pm, uint32_t min_tasks,
                               uint64_t* counts_dev, uint32_t* tasks_dev, uint32_t* pred_dev, float* prob_dev,
                               uint64_t* eval_dev, saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if ((t->n_calls && !call_label_dev) || (t->n_sessions && !session_role_dev) || !counts_dev || !tasks_dev || !pred_dev) {
    set_error("saga_pattern_infer: NULL argument");
    return SAGA_ERR_INVALID_ARG;
  }
  if (n_labels == 0 || n_labels > 64 || theta_pm == 0 || theta_pm > 1000) {
    set_error("saga_pattern_infer: need 1 <= n_labels <= 64 and 1 <= theta_pm <= 1000");
    return SAGA_ERR_INVALID_ARG;
  }
  SAGA_CK(cudaSetDevice(t->device));
  const cudaStream_t s = stream ? (cudaStream_t)stream : t->stream;
  GUARD(const_cast<saga_trace*>(t), join(t->stream, s));
  GUARD(const_cast<saga_trace*>(t), run_pattern(t, call_label_dev, n_labels, session_role_dev, theta_pm, min_tasks,
                                                counts_dev, tasks_dev, pred_dev, prob_dev, eval_dev, s));
  GUARD(const_cast<saga_trace*>(t), join(s, t->stream));  // see saga_node_stream
  return SAGA_OK;
}

saga_status saga_tool_stats(const saga_trace* t, const uint32_t* call_label_dev, uint32_t n_labels, uint32_t p_pm,
                            uint32_t window, uint32_t min_samples, uint32_t ema_terms, int64_t* ttl_out_dev,
                            uint32_t* obs_out_dev, saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if ((t->n_calls && (!call_label_dev || !ttl_out_dev || !obs_out_dev))) {
    set_error("saga_tool_stats: NULL argument");
    return SAGA_ERR_INVALID_ARG;
  }
  if (n_labels == 0 || n_labels > 64 || p_pm == 0 || p_pm > 1000 || window == 0 || window > 1024 || ema_terms > 256) {
    set_error("saga_tool_stats: need 1 <= n_labels <= 64, 1 <= p_pm <= 1000, 1 <= window <= 1024, ema_terms <= 256");
    return SAGA_ERR_INVALID_ARG;
  }
  SAGA_CK(cudaSetDevice(t->device));
  const cudaStream_t s = stream ? (cudaStream_t)stream : t->stream;
  GUARD(const_cast<saga_trace*>(t), join(t->stream, s));
  GUARD(const_cast<saga_trace*>(t), run_tool_stats(t, call_label_dev, n_labels, p_pm, window, min_samples, ema_terms,
                                                   ttl_out_dev, obs_out_dev, s));
  GUARD(const_cast<saga_trace*>(t), join(s, t->stream));  // see saga_node_stream
  return SAGA_OK;
}

saga_status saga_replay_victims(saga_trace* t, const saga_replay_cfg* cfg, uint32_t cap, uint32_t node,
                                uint64_t* log_dev, uint64_t log_cap, uint64_t* n_logged, int64_t* counters_dev,
                                saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if (!cfg || !counters_dev || !n_logged || (log_cap && !log_dev)) { set_error("saga_replay_victims: NULL argument"); return SAGA_ERR_INVALID_ARG; }
  const uint32_t pm = cfg->policy_mask & 31u;
  if (cfg->policy_mask != pm || pm == 0 || (pm & (pm - 1))) { set_error("saga_replay_victims: exactly one policy"); return SAGA_ERR_INVALID_ARG; }
  if (cfg->p_high_pm <= cfg->p_low_pm || cfg->p_high_pm > 1000) { set_error("saga_replay_victims: need p_low_pm < p_high_pm <= 1000"); return SAGA_ERR_INVALID_ARG; }
  if (cap == 0 || cap > (1u << 28)) { set_error("saga_replay_victims: capacity %u out of range (1..2^28)", cap); return SAGA_ERR_CAPACITY; }
  if (node >= t->n_nodes || !t->nodes[node].owned) { set_error("saga_replay_victims: node %u not owned", node); return SAGA_ERR_STATE; }
  if (!t->nodes[node].nu_done) { set_error("saga_replay_victims: saga_belady_next_use(node %u) must run first", node); return SAGA_ERR_STATE; }
  if (cap < t->nodes[node].max_group) {
    set_error("saga_replay_victims: capacity %u is below the %llu blocks of a single call", cap,
              (unsigned long long)t->nodes[node].max_group);
    return SAGA_ERR_CAPACITY;
  }
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(t, join((cudaStream_t)stream, t->stream));
  uint64_t* cnt = nullptr;
  SAGA_CK(ws_malloc((void**)&cnt, 8, t->stream));
  SAGA_CK(cudaMemsetAsync(cnt, 0, 8, t->stream));
  const saga_status st = run_replay(t, cfg, &cap, 1, &node, 1, counters_dev, t->stream, log_dev, log_cap, cnt);
  if (st == SAGA_OK) SAGA_CK(d2h(n_logged, cnt, 8, t->stream));
  ws_free(cnt, t->stream);
  GUARD(t, st);
  GUARD(t, replay_check(t));
  GUARD(t, join(t->stream, (cudaStream_t)stream));
  return SAGA_OK;
}

saga_status saga_replay(saga_trace* t, const saga_replay_cfg* cfg, const uint32_t* caps, uint32_t n_caps,
                        const uint32_t* nodes, uint32_t n_owned, int64_t* counters_dev, saga_stream_t stream) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  if (!cfg || (n_caps && !caps) || (n_owned && !nodes) || !counters_dev) { set_error("saga_replay: NULL argument"); return SAGA_ERR_INVALID_ARG; }
  if ((cfg->policy_mask & ~31u) || !(cfg->policy_mask & 31u)) { set_error("saga_replay: bad policy_mask"); return SAGA_ERR_INVALID_ARG; }
  if (cfg->p_high_pm <= cfg->p_low_pm || cfg->p_high_pm > 1000) { set_error("saga_replay: need p_low_pm < p_high_pm <= 1000"); return SAGA_ERR_INVALID_ARG; }
  for (uint32_t i = 0; i < n_caps; ++i)
    if (caps[i] == 0 || caps[i] > (1u << 28)) { set_error("saga_replay: capacity %u out of range (1..2^28)", caps[i]); return SAGA_ERR_CAPACITY; }
  for (uint32_t i = 0; i < n_owned; ++i) {
    if (nodes[i] >= t->n_nodes || !t->nodes[nodes[i]].owned) { set_error("saga_replay: node %u not owned", nodes[i]); return SAGA_ERR_STATE; }
    if (!t->nodes[nodes[i]].nu_done) { set_error("saga_replay: saga_belady_next_use(node %u) must run first", nodes[i]); return SAGA_ERR_STATE; }
    for (uint32_t c = 0; c < n_caps; ++c)
      if (caps[c] < t->nodes[nodes[i]].max_group) {  // SPEC CapacityError: one call does not fit
        set_error("saga_replay: capacity %u is below the %llu blocks of a single call at node %u", caps[c],
                  (unsigned long long)t->nodes[nodes[i]].max_group, nodes[i]);
        return SAGA_ERR_CAPACITY;
      }
  }
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(t, join((cudaStream_t)stream, t->stream));
  GUARD(t, run_replay(t, cfg, caps, n_caps, nodes, n_owned, counters_dev, t->stream));
  GUARD(t, join(t->stream, (cudaStream_t)stream));
  return SAGA_OK;
}

saga_status saga_replay_wait(saga_trace* t) {
  SAGA_NVTX();
  CHECK_HANDLE(t);
  SAGA_CK(cudaSetDevice(t->device));
  GUARD(t, replay_check(t));
  return SAGA_OK;
}

}  // extern "C"
