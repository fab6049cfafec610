/*
 * saga.h -- C ABI of libsaga, the B200 (sm_100a) hot path of SAGA's trace-driven KV-cache
 * policy evaluation (arXiv 2605.00528, "SAGA: Workflow-Atomic Scheduling for AI Agent
 * Inference on GPU Clusters").  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n;
 * "DESIGN.md R-x" names a reading of a passage the paper leaves open.
 *
 * Pipeline:
 *   saga_load_trace      A1 ingest + validate, A2 placement (eq:routing P:735-743, work stealing
 *                        P:748-766), A3 per-node access streams (sigma of P:881-885)
 *   saga_belady_next_use A4 Belady next-use: onesweep radix sort + segmented scans
 *   saga_sweep_range     W_lo / W_hi of a node (feasibility floor / compulsory-only ceiling)
 *   saga_aeg_score       A5 WA-LRU key (eq:eviction P:659-662, eq:recency/eq:size P:665-670,
 *                        eq:reuse P:673-678, eq:overlap P:680-685, Alg. ttl P:696-708,
 *                        eq:pressure P:710-715) over a batch of eviction candidates
 *   saga_evict_select    A6 capacity-bounded top-k (evict the largest keys)
 *   saga_replay          A7 epoch-synchronous replay of hits/misses per (policy, node, capacity)
 *   saga_allreduce_counters  A8 counter reduction over NCCL (NVLink / NVSwitch)
 *   saga_pattern_infer   F3 pattern-based AEG inference from observed label sequences
 *
 * Conventions for every function:
 *   - Return a saga_status; nothing aborts, exits or throws across the ABI.  The message of the
 *     last failure on the calling thread is saga_last_error().
 *   - "_dev" pointers are device pointers on the handle's device, allocated and owned by the
 *     caller (e.g. torch tensors' data_ptr()); "_host" / plain pointers are host memory.  The
 *     library never frees or retains caller memory.
 *   - Calls taking a stream are stream-ordered and asynchronous unless stated ("syncs").
 *   - SAGA_ERR_CUDA is sticky for a handle: free it.
 *   - A handle is bound to one device and must not be used by two threads at once.
 *   - All outputs are bit-identical across runs and across 1/2/4/8 GPUs.
 */
#ifndef SAGA_H_
#define SAGA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* saga_stream_t; /* identical to cudaStream_t */

typedef enum {
  SAGA_OK = 0,
  SAGA_ERR_INVALID_ARG = 1, /* bad pointer / size / option; nothing was modified            */
  SAGA_ERR_TRACE = 2,       /* trace failed validation (message says which rule); outputs untouched */
  SAGA_ERR_CAPACITY = 3,    /* a capacity below a single call's block count (S:209 CapacityError) */
  SAGA_ERR_STATE = 4,       /* call order violated (e.g. replay before next-use) or internal limit */
  SAGA_ERR_OOM = 5,         /* device allocation failed                                        */
  SAGA_ERR_CUDA = 6,        /* CUDA runtime error (sticky)                                     */
  SAGA_ERR_NCCL = 7         /* NCCL error                                                      */
} saga_status;

typedef enum {
  SAGA_POLICY_AEG = 1,      /* WA-LRU with AEG predictions (eq:eviction) + tool-call TTL (Alg. 1) */
  SAGA_POLICY_BELADY = 2,   /* epoch-batched farthest-next-use (Belady)                  */
  SAGA_POLICY_EVICT_ALL = 4, /* test policy: evict every non-requested block each epoch (Obs. 1) */
  SAGA_POLICY_LRU = 8,       /* baseline "Standard LRU" of Table tab:competitive: the
                                block whose latest access is earliest in the node stream goes first */
  SAGA_POLICY_LRU_PREFIX = 16 /* baseline "LRU + Prefix (vLLM v0.5)": LRU over private blocks;
                                shared-prefix blocks only when no private candidate is left */
} saga_policy;

/* Counter slots, int64 each, SAGA_NCOUNT per (policy, capacity, node) replay: SURVEY §8.C.7's
 * list (its reserved slot holding the peak resident count), then the PREFETCH record counts of F4.
 * Identity: ACCESSES = HITS + MISSES + MIG_HITS + MIG_MISSES + PF_HITS + PF_MISSES.  Unavoidable vs regenerated prefill follows P:881 ("tokens prefilled") and
 * Observation 1: a CALL miss is compulsory only at the block's first touch in the
 * whole trace (first call in (t, s) order touching it); every other CALL miss -- including the
 * re-prefill of a rerouted session at its new node -- is regeneration. */
enum {
  SAGA_C_ACCESSES = 0,
  SAGA_C_HITS = 1,              /* CALL records found resident                                  */
  SAGA_C_MISSES = 2,            /* CALL records not resident (tokens prefilled)          */
  SAGA_C_COMPULSORY_GLOBAL = 3, /* CALL misses at the block's first touch in the whole trace    */
  SAGA_C_COMPULSORY_NODE = 4,   /* misses (CALL or MIG) at the node's first touch of the block  */
  SAGA_C_MIG_HITS = 5,          /* MIG (migrated-in) records found resident                     */
  SAGA_C_MIG_MISSES = 6,
  SAGA_C_INVALIDATED = 7,       /* residents dropped because their session migrated away (R1)   */
  SAGA_C_EVICTIONS = 8,
  SAGA_C_EVICT_PROTECTED = 9,   /* AEG victims that were TTL-protected (hard pressure)   */
  SAGA_C_EVICT_EVENTS = 10,
  SAGA_C_REGEN_TOKENS = 11,     /* block_tokens x (MISSES - COMPULSORY_GLOBAL)                  */
  SAGA_C_REGEN_US = 12,         /* their prefill time at prefill_tok_s                          */
  SAGA_C_VICTIM_HASH = 13,      /* sum over victims of splitmix64((epoch << 32) | local id)     */
  SAGA_C_INFEASIBLE_EPOCH = 14, /* first epoch whose requests exceed the capacity, else 0       */
  SAGA_C_PEAK_RESIDENT = 15,    /* max |S| after an epoch (<= capacity)                         */
  SAGA_C_PF_HITS = 16,          /* PREFETCH records found resident (SAGA_LOAD_PREFETCH)          */
  SAGA_C_PF_MISSES = 17,        /* PREFETCH records loaded ahead of the predicted next step     */
  SAGA_C_RESERVED18 = 18,
  SAGA_C_RESERVED19 = 19,
  SAGA_NCOUNT = 20
};

/* Columnar trace (host pointers; deep-copied by saga_load_trace).  Validation rules
 * (SAGA_ERR_TRACE otherwise), DESIGN.md §3 "Trace format":
 *   1 <= n_nodes <= 32, 1 <= n_types <= 32, block_tokens >= 1;
 *   calls strictly increasing in (call_t_us, call_session), 0 <= t < 2^50, session < n_sessions,
 *   aeg node < n_aeg_nodes, prompt >= 1, new <= prompt;
 *   call_range_off is a CSR of n_calls+1 strictly increasing offsets from 0 to n_ranges (>= 1 range per call);
 *   every range has len >= 1 and lies inside its session's private span
 *   [session_block_lo, +session_block_len) or its type's shared span [type_shared_lo, +len);
 *   all spans are inside [0, n_blocks) and pairwise disjoint;
 *   AEG: CSR aeg_edge_off, edge_dst < n_aeg_nodes, edge_p in [0,1], out-mass <= 1 + 1e-6,
 *   edge_shared_q16 <= 65536 (65536 = whole context shared), 0 <= node_ttl_base_us <= 1e9;
 *   each call's work (prefill + decode microseconds) < 2^32. */
typedef struct {
  uint32_t n_calls, n_sessions, n_types, n_aeg_nodes, n_edges, n_ranges, n_blocks, n_nodes, block_tokens;
  const int64_t* call_t_us;           /* [n_calls] arrival time of the LLM call (us)          */
  const uint32_t* call_session;       /* [n_calls] session (agent task) id                     */
  const uint32_t* call_aeg_node;      /* [n_calls] AEG node v_s of the call (explicit hints) */
  const uint32_t* call_prompt_tokens; /* [n_calls] prompt tokens                               */
  const uint32_t* call_output_tokens; /* [n_calls] generated tokens                            */
  const uint32_t* call_new_tokens;    /* [n_calls] tokens to prefill if the context is cached  */
  const uint8_t* call_is_last;        /* [n_calls] 1 on the session's final call               */
  const uint32_t* call_range_off;     /* [n_calls+1] CSR into the ranges                      */
  const uint32_t* range_block_lo;     /* [n_ranges] first global block id                     */
  const uint32_t* range_len;          /* [n_ranges] blocks (accessed in order)                 */
  const uint16_t* session_type;       /* [n_sessions] agent type / tenant                     */
  const uint32_t* session_block_lo;   /* [n_sessions] private block span                      */
  const uint32_t* session_block_len;
  const uint32_t* aeg_edge_off;       /* [n_aeg_nodes+1] CSR of E                              */
  const uint32_t* edge_dst;           /* [n_edges] successor u                                 */
  const float* edge_p;                /* [n_edges] P(v -> u) (Def. AEG)               */
  const uint32_t* edge_shared_q16;    /* [n_edges] shared-prefix fraction x 65536       */
  const int64_t* node_ttl_base_us;    /* [n_aeg_nodes] Percentile_p of the node's tool (Alg.1 l.2) */
  const uint32_t* node_obs_tokens;    /* [n_aeg_nodes] expected observation length n_obs */
  const uint8_t* node_terminal;       /* [n_aeg_nodes] terminal node                          */
  const uint32_t* type_shared_lo;     /* [n_types] shared-prefix span of the agent type        */
  const uint32_t* type_shared_len;
  /* Optional per-call overrides (NULL = the call's AEG node values), e.g. the online statistics
   * of saga_tool_stats (F4): call_ttl_base_us replaces node_ttl_base_us[v_c] wherever call c's
   * TTL base is read (placement's cached(w,s), the Alg. 1 protection of its session's blocks),
   * in [0, 1e9]; call_obs_tokens replaces node_obs_tokens[v_c] in eq:overlap. */
  const int64_t* call_ttl_base_us;    /* [n_calls] or NULL */
  const uint32_t* call_obs_tokens;    /* [n_calls] or NULL */
} saga_trace_desc;

/* Placement configuration (DESIGN.md R-load, R-steal): 100 ms epochs, kappa
 * concurrent requests per node, theta and R_max in per-mille, T_idle. */
typedef struct {
  int64_t epoch_us;        /* 100000; must be in (0, 1e9] (SAGA_ERR_INVALID_ARG otherwise) */
  uint32_t kappa;          /* 32; at most 256 */
  uint32_t prefill_tok_s;  /* 5000 */
  uint32_t decode_tok_s;   /* 30 */
  uint32_t theta_pm;       /* 800  */
  uint32_t rmax_pm;        /* 2000 */
  int64_t t_idle_us;       /* 100000 */
  uint64_t seed;           /* victim choice splitmix64(seed ^ e*phi ^ thief) */
} saga_place_cfg;

/* Replay / score configuration: weights of eq:eviction, pressure thresholds of
 * eq:pressure in per-mille, TTL_max of Alg. 1. */
typedef struct {
  uint32_t policy_mask;    /* OR of saga_policy */
  float alpha, beta, gamma;/* 0.3, 0.5, 0.2 */
  uint32_t p_low_pm;       /* 700 */
  uint32_t p_high_pm;      /* 900 */
  int64_t ttl_max_us;      /* 300000000 */
  uint32_t flags;          /* reserved, 0 */
} saga_replay_cfg;

/* A batch of eviction candidates for saga_aeg_score (all device pointers).  Segment i holds
 * candidates [seg_off[i], seg_off[i+1]) of node seg_node[i] at boundary epoch seg_epoch[i]
 * (T_e = epoch * epoch_us) with |S| = seg_occ[i], capacity seg_cap[i] and shared-prefix
 * activity mask seg_act[i] (bit a = an unfinished session of type a has affinity there).
 * cand_lid are node-local block ids from saga_belady_next_use; cand_t_last the last access
 * time (us) and cand_nu the next use position (BELADY key). */
typedef struct {
  uint32_t n_seg;
  uint32_t policy;                 /* SAGA_POLICY_AEG or SAGA_POLICY_BELADY */
  const uint32_t* seg_node;
  const uint32_t* seg_epoch;
  const uint32_t* seg_occ;
  const uint32_t* seg_cap;
  const uint32_t* seg_act;
  const uint64_t* seg_off;         /* [n_seg+1] */
  const uint32_t* cand_lid;
  const int64_t* cand_t_last;
  const uint32_t* cand_nu;
} saga_score_batch;

typedef struct saga_trace saga_trace;
typedef struct saga_comm saga_comm;

/* Thread-local message of the last failure ("" if none).  Never NULL. */
const char* saga_last_error(void);

/* A1-A3.  Deep-copies *desc to `device`, validates it (one sync to report SAGA_ERR_TRACE),
 * runs placement (replicated on every rank: capacity- and policy-independent) and expands the
 * access streams of the nodes set in owned_node_mask (0 = all nodes).  Syncs. */
saga_status saga_load_trace(const saga_trace_desc* desc, const saga_place_cfg* cfg, uint32_t owned_node_mask,
                            int device, saga_stream_t stream, saga_trace** out);

/* saga_load_trace with flags.  SAGA_LOAD_DEFER_EXPAND: return after validation and placement
 * (still syncs); each owned node's stream (A3) is expanded on the handle's stream by the first
 * call that needs it (saga_trace_info, saga_node_stream*, saga_belady_next_use).  Lets a caller
 * with several traces in flight run one trace's single-SM placement beside another's replay and
 * start the SM-hungry expansion / next-use only when that replay is done (stream-ordered). */
enum { SAGA_LOAD_DEFER_EXPAND = 1, SAGA_LOAD_PREFETCH = 2 };
/* SAGA_LOAD_PREFETCH (F4, speculative prefetching, §4.3; SPEC prefetch_target
 * S:235-243; DESIGN.md R-prefetch): every node stream also carries PREFETCH records.  When call c
 * of session s (AEG node v, not is_last, v not terminal, v with successors) finishes inference,
 * its tool starts at t_end(c); at the boundary e_pf = t_end(c) / epoch_us + 1 the node that
 * served c prefetches the prefix of the predicted successor u = argmax_u' P(v -> u') (ties: the
 * lowest node id): the first floor(n_sh / block_tokens) blocks of c's block list, n_sh =
 * (prompt_c + output_c) * edge_shared_q16(v -> u) >> 16.  Emitted only if e_pf > e(c) and s's
 * next call is admitted after e_pf.  Per epoch a node's records are MIG (ascending session),
 * PREFETCH (call order), CALL (call order); PREFETCH records write t_last = T_e and count as
 * PF_HITS / PF_MISSES (not CALL misses, never compulsory). */
saga_status saga_load_trace_ex(const saga_trace_desc* desc, const saga_place_cfg* cfg, uint32_t owned_node_mask,
                               int device, saga_stream_t stream, uint32_t flags, saga_trace** out);

/* Sizes of node `node`'s stream: accesses and (after saga_belady_next_use) distinct blocks
 * (UINT32_MAX before).  Syncs.  SAGA_ERR_STATE if the node is not owned. */
saga_status saga_trace_info(const saga_trace* t, uint32_t node, uint64_t* n_access, uint32_t* n_local_blocks);

/* Placement outputs (host copies, syncs): node_host[n_calls] (nullable), migrations as
 * (epoch, session, from, to) quadruples into mig_host[4*mig_cap] (nullable), and
 * stats[3] = {steals, reroutes, n_migrations}. */
saga_status saga_placement(const saga_trace* t, uint8_t* node_host, uint32_t* mig_host, uint64_t mig_cap,
                           int64_t* stats);

/* Node stream structure (device outputs, nullable, sized via saga_node_stream_sizes):
 * block_dev[n_access] global block ids; ev_dev[3*n_events] (epoch, first group, n_groups);
 * grp_dev[n_groups*2] (first position, kind 0 CALL / 1 MIG) and grp_t_dev[n_groups] (t_last
 * value written by the group's records).  Invalidations are attached to the first record epoch
 * at or after their own epoch (DESIGN.md R-inv); a final sentinel event (epoch UINT32_MAX, no
 * groups) carries trailing ones. */
saga_status saga_node_stream_sizes(const saga_trace* t, uint32_t node, uint64_t* n_access, uint32_t* n_events,
                                   uint32_t* n_groups, uint32_t* n_inv);
saga_status saga_node_stream(const saga_trace* t, uint32_t node, uint32_t* block_dev, uint32_t* ev_dev,
                             uint64_t* grp_dev, int64_t* grp_t_dev, uint32_t* inv_dev, saga_stream_t stream);

/* A4.  For node `node`: stable LSD onesweep radix sort of the stream by global block id, then
 * segmented scans.  Writes next_use_dev[p] = min{q > p : block(q) = block(p)} (0xFFFFFFFF if
 * none) and local_id_dev[p] = rank of block(p) among the node's distinct ids (both nullable,
 * n_access entries), and keeps them (plus first-touch flags and W_lo/W_hi) for saga_replay. */
saga_status saga_belady_next_use(saga_trace* t, uint32_t node, uint32_t* next_use_dev, uint32_t* local_id_dev,
                                 saga_stream_t stream);

/* A4 for several owned nodes at once (no outputs; results kept as by saga_belady_next_use): the
 * nodes' streams are sorted and scanned as segments of one launch per kernel (K4 onesweep passes,
 * K5 segmented scan, per-epoch statistics), in batches of up to 32 nodes / 2^29 accesses.  A node
 * already done is skipped.  Syncs once per batch (sizes of the derived tables). */
saga_status saga_belady_next_use_nodes(saga_trace* t, const uint32_t* nodes, uint32_t n_nodes, saga_stream_t stream);

/* W_lo = max over record epochs of distinct blocks requested, W_hi = max over record epochs of
 * blocks live across it (first touch <= epoch end and last touch >= epoch start).  Syncs.
 * SAGA_ERR_STATE before saga_belady_next_use(node). */
saga_status saga_sweep_range(const saga_trace* t, uint32_t node, uint32_t* w_lo, uint32_t* w_hi);

/* A5.  Keys of every candidate of every segment: AEG key = (!prot << 63) | (q << 32) | lid with
 * q = floor(score * 2^20) of the fp32 WA-LRU score (pinned op order);
 * BELADY key = (nu << 32) | lid.  score_dev (fp32, nullable) receives the AEG score.
 * Requires saga_belady_next_use for every node referenced. */
saga_status saga_aeg_score(const saga_trace* t, const saga_score_batch* batch, const saga_replay_cfg* cfg,
                           float* score_dev, uint64_t* key_dev, saga_stream_t stream);

/* A6.  For each segment i of keys [seg_off_dev[i], seg_off_dev[i+1]) select the k_dev[i] largest
 * keys (keys must be unique within a segment) and write their indices relative to the segment
 * start, in descending key order, to victim_idx_dev[out_off_dev[i] ...].  k > segment size
 * is clamped (the tail of the output range is left untouched).  Syncs once before the launch
 * (reads seg_off_dev to size the scratch of segments whose winners exceed shared memory). */
saga_status saga_evict_select(const uint64_t* key_dev, const uint64_t* seg_off_dev, const uint32_t* k_dev,
                              uint32_t n_seg, const uint64_t* out_off_dev, uint32_t* victim_idx_dev,
                              saga_stream_t stream);

/* A7.  Replays policies x caps x nodes.  caps (host, n_caps) uniform across nodes; nodes (host,
 * n_owned) must be owned and have had saga_belady_next_use.  counters_dev is
 * int64[n_pol][n_caps][n_nodes][SAGA_NCOUNT] with n_pol = popcount(policy_mask), policies in
 * the order AEG, BELADY, EVICT_ALL, LRU, LRU_PREFIX; cells of nodes not listed are left untouched (zero them
 * first; then an all-reduce sum over ranks is an exact gather).  A capacity below a node's
 * W_lo is data, not an error: INFEASIBLE_EPOCH is set and that replay stops counting.
 * SAGA_ERR_CAPACITY if a capacity is below the block count of a single call (or
 * migration / prefetch group) at a replayed node (S:209 CapacityError).  Stream-ordered and asynchronous once the node's replay
 * index exists (the first call for a node builds it and syncs for its sizes); the kernel's
 * internal invariant checks are reported by saga_replay_wait.  The replay kernel itself runs on a
 * stream the handle owns, at the device's lowest priority, event-joined after the work queued on
 * the handle's stream and before any work queued there later (ordering is unchanged; other
 * streams' short kernels take freed SMs first; SAGA_REPLAY_SAME_STREAM=1 keeps it on the handle's
 * stream).  Set SAGA_REPLAY_TRACE=1 to print per-item / per-phase SM cycles to stderr (syncs). */
saga_status saga_replay(saga_trace* t, const saga_replay_cfg* cfg, const uint32_t* caps, uint32_t n_caps,
                        const uint32_t* nodes, uint32_t n_owned, int64_t* counters_dev, saga_stream_t stream);

/* Waits for the handle's stream and reports the replay kernels' internal checks (SAGA_ERR_STATE
 * with the failing check in saga_last_error()).  Syncs. */
saga_status saga_replay_wait(saga_trace* t);

/* One (policy, capacity, node) replay of A7 that also logs its victims (SURVEY §1.2's victim
 * logs; the sketch's SAGA_LOG_VICTIMS): cfg->policy_mask must name exactly one policy.
 * log_dev (uint64, log_cap entries, nullable when log_cap = 0) receives every victim as
 * (epoch << 32) | local id, epochs ascending; within an epoch the order is unspecified (the set
 * is unique, the order of equal-epoch entries is not: sort to compare); *n_logged (host) is
 * the number of victims, which may exceed log_cap (then only log_cap were written).
 * counters_dev int64[n_nodes][SAGA_NCOUNT]: the node's row as saga_replay writes it.  Syncs. */
saga_status saga_replay_victims(saga_trace* t, const saga_replay_cfg* cfg, uint32_t cap, uint32_t node,
                                uint64_t* log_dev, uint64_t log_cap, uint64_t* n_logged, int64_t* counters_dev,
                                saga_stream_t stream);

/* F3.  Pattern-based AEG inference, observability tier (b) of §3.3 (P:645:
 * "extracting tool-type patterns, computing transition probabilities, and retaining edges
 * exceeding theta_conf = 0.7"; cold start "until 30 tasks complete") and the next-step accuracy
 * of tab:pattern ("fraction of correctly predicted next-step node transitions in
 * held-out traces").  Readings R-pattern in DESIGN.md §3: first-order (bigram) transitions of
 * the observed label sequence of each session, "exceeding" read as >=, the end of a completed
 * task is successor y = n_labels.
 *   call_label_dev  uint32[n_calls] observed label (tool type) of each call, < n_labels <= 64
 *   session_role_dev uint8[n_sessions]: 0 ignored, 1 training, 2 held-out
 *   theta_pm        theta_conf in per-mille (700), 1..1000; min_tasks the cold start (30)
 * Outputs (device, overwritten):
 *   counts_dev uint64[n_types][n_labels][n_labels+1]: over the calls of training sessions of
 *              type a, consecutive calls labelled x then y, and y = n_labels for a session's
 *              final call when it carries call_is_last;
 *   tasks_dev  uint32[n_types]: completed training sessions of each type;
 *   pred_dev   uint32[n_types][n_labels]: when tasks[a] >= min_tasks, the successor y with
 *              1000 * counts[a][x][y] >= theta_pm * sum_y counts[a][x][y] and the largest count
 *              (smallest y on ties); SAGA_PATTERN_NONE otherwise;
 *   prob_dev   float[n_types][n_labels][n_labels+1] (nullable): (float)counts / (float)total of
 *              every retained edge (fp32 round-to-nearest division), 0 elsewhere;
 *   eval_dev   uint64[n_types][4] (nullable): over held-out sessions, {transitions (same
 *              definition as counts), predicted (pred != NONE), correct (pred == y), 0}.
 * Integer outputs are exact.  SAGA_ERR_INVALID_ARG for a label >= n_labels (checked on the
 * device; syncs once at the end) or arguments out of range. */
enum { SAGA_PATTERN_NONE = 0xFFFFFFFFu };

/* F4, online tool statistics: the per-call TTL base of Alg. 1 line 2
 * ("ttl_base <- Percentile(H_t, p)") and the expected observation length of
 * eq:overlap ("tool-type-specific distributions maintained via exponential moving averages",
 * P:685), from the history the trace itself reveals.  Readings R-online in DESIGN.md §3.
 *   A sample of tool x: a call d labelled x with a successor d' in its session; latency
 *   t(d') - t_end(d) clamped to [0, 2^32 - 1] (t_end = tool start, A1), observation
 *   call_new_tokens[d'], completed at t(d').  For call c (tool x = call_label[c]) the history H is
 *   the samples of x completed at or before t_end(c), in completion (trace) order; k = |H|.
 *   ttl_out_dev[c] (int64) = the nearest-rank p_pm/1000 percentile of the latencies of the last
 *     min(k, window) samples (ascending, rank ceil(p_pm n / 1000)), capped at 1e9; the node's
 *     node_ttl_base_us when fewer than min_samples (cold start).
 *   obs_out_dev[c] (uint32) = floor(E + 0.5), E = the alpha = 0.2 EMA started at the node's
 *     node_obs_tokens and truncated to the newest ema_terms samples:
 *     E = [k <= ema_terms] 0.8^k n0 + sum_{i = m-1 .. 0} (0.2 0.8^i) obs_{k-1-i}, m = min(k, ema_terms),
 *     evaluated in fp64 in that order (weights by repeated multiplication, no contraction).
 * Labels as saga_pattern_infer (n_labels <= 64); 1 <= window <= 1024; ema_terms <= 256.  Both
 * outputs are exact (integer results of pinned fp64 arithmetic).  Feed them back through
 * saga_trace_desc.call_ttl_base_us / call_obs_tokens.  Syncs once (label check). */
saga_status saga_tool_stats(const saga_trace* t, const uint32_t* call_label_dev, uint32_t n_labels, uint32_t p_pm,
                            uint32_t window, uint32_t min_samples, uint32_t ema_terms, int64_t* ttl_out_dev,
                            uint32_t* obs_out_dev, saga_stream_t stream);
saga_status saga_pattern_infer(const saga_trace* t, const uint32_t* call_label_dev, uint32_t n_labels,
                               const uint8_t* session_role_dev, uint32_t theta_pm, uint32_t min_tasks,
                               uint64_t* counts_dev, uint32_t* tasks_dev, uint32_t* pred_dev, float* prob_dev,
                               uint64_t* eval_dev, saga_stream_t stream);

/* A8.  NCCL communicator from a 128-byte ncclUniqueId exchanged by the caller (e.g. over
 * torch.distributed).  The library dlopen()s libnccl.so.2 (the process's copy if loaded). */
saga_status saga_comm_unique_id(void* id128);
saga_status saga_comm_init(const void* id128, int rank, int nranks, int device, saga_comm** out);
/* In-place all-reduce of n int64 on the stream; op 0 = sum, 1 = max. */
saga_status saga_allreduce_counters(saga_comm* c, int64_t* buf_dev, size_t n, int op, saga_stream_t stream);
void saga_comm_destroy(saga_comm* c);

/* Number of libsaga kernels launched by this process so far (for bench.py's gpu_launches). */
uint64_t saga_kernel_launches(void);

/* Optional device-time profile (CUDA events recorded on the launching stream around each kernel
 * family).  saga_profile_read syncs, writes the accumulated milliseconds and launch counts of
 * every category into ms_out[SAGA_PROF_NCAT] / n_out[SAGA_PROF_NCAT] (nullable), and resets. */
enum {
  SAGA_PROF_LOAD = 0,      /* A1 validate + derive (includes the H2D copy of the descriptor)   */
  SAGA_PROF_PLACE = 1,     /* A2 placement kernel                                             */
  SAGA_PROF_EXPAND = 2,    /* A3 stream expansion (span of its launches)                      */
  SAGA_PROF_SORT = 3,      /* A4 histogram + onesweep passes                                  */
  SAGA_PROF_SEGSCAN = 4,   /* A4 segmented scans -> next_use / local ids                      */
  SAGA_PROF_EPOCH = 5,     /* A4 per-epoch statistics (first-in-epoch, W_lo / W_hi)          */
  SAGA_PROF_REPLAY = 6,    /* A5-A7 replay kernel                                             */
  SAGA_PROF_SCORE = 7,     /* A5 bulk score                                                   */
  SAGA_PROF_SELECT = 8,    /* A6 bulk select                                                  */
  SAGA_PROF_PATTERN = 9,   /* F3 pattern inference (count + predict + evaluate)               */
  SAGA_PROF_NCAT = 10
};
void saga_profile_enable(int on);
void saga_profile_read(double* ms_out, uint64_t* n_out);

void saga_free_trace(saga_trace* t);

#ifdef __cplusplus
}
#endif
#endif /* SAGA_H_ */
