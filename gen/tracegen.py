"""Seeded synthetic agent-workflow traces for the SAGA hot path (input generator only).

This module builds the *inputs* of the pipeline -- a columnar call table, an
Agent Execution Graph (AEG) in CSR form and per-session / per-type block spans.
It contains none of the method's arithmetic (no placement, no next-use, no
WA-LRU score, no replay): both the CUDA path and the CPU oracle read what it
produces, and nothing here depends on either of them.

Workload recipes follow SURVEY.md §8.D.1 and DESIGN.md "Input recipe":

* AEG (Def. "Agent Execution Graph", §3.2): V = LLM steps,
  E with transition probabilities P, tool type phi(v).  ReAct agents form a
  chain with P(v_i -> v_{i+1}) ~= 1 - p_term; tree-of-thought style
  branching for WebArena.
* Tool gaps: log-normal fits of Table 1, mu = ln P50,
  sigma = ln(P95/P50)/z_0.95.  Per AEG node the generator emits
  ttl_base = Percentile_95 of the node's tool law (Alg. 1 line 2) as
  integer microseconds; the device never evaluates transcendentals.
* Workloads: SWE-bench mean 37 / max 100 steps, 2-4K prompts,
  100-500 output tokens; WebArena mean ~18 steps, 4-8K prompts incl. page,
  50-200 output tokens; BurstGPT-derived multi-tenant 3/4/3 tenants at
  16/8/4 tasks/min with 100/30/10-step agents.
* Open-loop timestamps: t_next = t_c + ceil(new*1e6/5000)
  + ceil(out*1e6/30) + gap.

All block ids are global; a block is 16 tokens (BASELINE.json configs).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np
from scipy.special import ndtri, ndtr

BLOCK_TOKENS = 16
EPOCH_US = 100_000
PREFILL_TOK_S = 5000
DECODE_TOK_S = 30
Z95 = float(ndtri(0.95))  # 1.6448536...

# Table 1: (P50 ms, P95 ms)
TOOLS = {
    "CodeExec": (180.0, 2400.0),
    "FileOps": (45.0, 320.0),
    "WebApi": (850.0, 4500.0),
    "Database": (120.0, 890.0),
}
TOOL_ORDER = ["FileOps", "CodeExec", "WebApi", "Database"]
# observable tool-type labels of calls (F3 pattern inference): Table 1's classes + run_test
TOOL_LABELS = TOOL_ORDER + ["RunTest"]


def tool_params(name: str):
    """(mu, sigma) of the log-normal in ln(ms)."""
    p50, p95 = TOOLS[name]
    return math.log(p50), math.log(p95 / p50) / Z95


@dataclasses.dataclass
class TraceDesc:
    """Columnar trace, mirrors saga_trace_desc of include/saga.h field by field."""
    name: str
    n_nodes: int
    n_blocks: int
    call_t_us: np.ndarray
    call_session: np.ndarray
    call_aeg_node: np.ndarray
    call_prompt_tokens: np.ndarray
    call_output_tokens: np.ndarray
    call_new_tokens: np.ndarray
    call_is_last: np.ndarray
    call_range_off: np.ndarray
    range_block_lo: np.ndarray
    range_len: np.ndarray
    session_type: np.ndarray
    session_block_lo: np.ndarray
    session_block_len: np.ndarray
    aeg_edge_off: np.ndarray
    edge_dst: np.ndarray
    edge_p: np.ndarray
    edge_shared_q16: np.ndarray
    node_ttl_base_us: np.ndarray
    node_obs_tokens: np.ndarray
    node_terminal: np.ndarray
    type_shared_lo: np.ndarray
    type_shared_len: np.ndarray
    block_tokens: int = BLOCK_TOKENS
    seed: int = 0
    # generator metadata, not part of saga_trace_desc: tool type phi(v) of each AEG node, the label
    # a request stream exposes (F3); index into TOOL_LABELS
    node_tool: Optional[np.ndarray] = None
    # optional per-call overrides of the node TTL base / observation length (saga_trace_desc)
    call_ttl_base_us: Optional[np.ndarray] = None
    call_obs_tokens: Optional[np.ndarray] = None

    @property
    def n_calls(self):
        return int(self.call_t_us.shape[0])

    @property
    def n_sessions(self):
        return int(self.session_type.shape[0])

    @property
    def n_types(self):
        return int(self.type_shared_lo.shape[0])

    @property
    def n_aeg_nodes(self):
        return int(self.node_terminal.shape[0])

    @property
    def n_edges(self):
        return int(self.edge_dst.shape[0])

    @property
    def n_ranges(self):
        return int(self.range_len.shape[0])

    @property
    def n_accesses(self):
        return int(self.range_len.astype(np.int64).sum())

    def arrays(self) -> Dict[str, np.ndarray]:
        return {f.name: getattr(self, f.name) for f in dataclasses.fields(self)
                if isinstance(getattr(self, f.name), np.ndarray)}

    def save(self, path):
        meta = np.array([self.n_nodes, self.n_blocks, self.block_tokens, self.seed], dtype=np.int64)
        np.savez(path, __meta=meta, __name=np.array(self.name), **self.arrays())

    @staticmethod
    def load(path) -> "TraceDesc":
        z = np.load(path)
        meta = z["__meta"]
        kw = {k: z[k] for k in z.files if not k.startswith("__")}
        return TraceDesc(name=str(z["__name"]), n_nodes=int(meta[0]), n_blocks=int(meta[1]),
                         block_tokens=int(meta[2]), seed=int(meta[3]), **kw)


def default_place_cfg(seed: int = 0) -> dict:
    """saga_place_cfg defaults."""
    return dict(epoch_us=EPOCH_US, kappa=32, prefill_tok_s=PREFILL_TOK_S, decode_tok_s=DECODE_TOK_S,
                theta_pm=800, rmax_pm=2000, t_idle_us=100_000, seed=seed)


def default_replay_cfg(policy_mask: int = 3) -> dict:
    """saga_replay_cfg defaults: alpha/beta/gamma, thresholds, TTL_max."""
    return dict(policy_mask=policy_mask, alpha=0.3, beta=0.5, gamma=0.2, p_low_pm=700, p_high_pm=900,
                ttl_max_us=300_000_000, flags=0)


# ----------------------------------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------------------------------

def pattern_labels(d: TraceDesc) -> np.ndarray:
    """Observed label of each call (F3): the tool type phi(v) of its AEG node, uint32."""
    if d.node_tool is None:
        return np.zeros(d.n_calls, np.uint32)
    return np.asarray(d.node_tool, np.uint32)[np.asarray(d.call_aeg_node, np.int64)]


def pattern_roles(d: TraceDesc, held_out_frac: float = 0.5, seed: int = 12345) -> np.ndarray:
    """Session roles for F3 (uint8): a seeded random held_out_frac of the sessions is held out (2),
    the others train (1)."""
    rng = np.random.default_rng(seed)
    return np.where(rng.random(d.n_sessions) < held_out_frac, 2, 1).astype(np.uint8)


def make_label_markov(seed: int, n_sessions: int, trans: np.ndarray, start: int = 0, n_types: int = 1,
                      max_len: int = 200) -> TraceDesc:
    """Sessions whose label sequences follow a first-order Markov chain over labels (F3 pins):
    trans[x][y] for y < L is P(x -> y), trans[x][L] the probability that the task ends.  AEG node
    of a call = its label (node_tool = identity); one private block per call, one node; session
    s has type s % n_types; calls spaced so that sessions interleave."""
    rng = np.random.default_rng(seed)
    trans = np.asarray(trans, np.float64)
    L = trans.shape[0]
    b = _AEGBuilder()
    for x in range(L):
        b.add_node(1_000_000, 0, False, tool=x)
    for x in range(L):
        for y in range(L):
            if trans[x, y] > 0:
                b.add_edge(x, y, float(trans[x, y]))
    aeg = b.finish()
    t, s, v, last = [], [], [], []
    for ss in range(n_sessions):
        x = start
        for j in range(max_len):
            t.append(1 + ss * 7_919 + j * 1_000_003); s.append(ss); v.append(x)
            y = int(rng.choice(L + 1, p=trans[x] / trans[x].sum()))
            if y == L or j == max_len - 1:
                last.append(1)
                break
            last.append(0)
            x = y
    order = np.lexsort((np.array(s), np.array(t)))
    n = len(t)
    cnt = np.bincount(np.array(s), minlength=n_sessions)
    slo = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.uint32)
    # call k of session s touches private block slo[s] + (its index within the session)
    s_arr = np.array(s)[order]
    idx = np.zeros(n, np.int64)
    seen = np.zeros(n_sessions, np.int64)
    for i, ss in enumerate(s_arr):
        idx[i] = seen[ss]; seen[ss] += 1
    return TraceDesc(
        name="label_markov", n_nodes=1, n_blocks=int(n) + 1, seed=seed,
        call_t_us=np.array(t, np.int64)[order], call_session=s_arr.astype(np.uint32),
        call_aeg_node=np.array(v, np.uint32)[order], call_prompt_tokens=np.full(n, 16, np.uint32),
        call_output_tokens=np.full(n, 1, np.uint32), call_new_tokens=np.full(n, 16, np.uint32),
        call_is_last=np.array(last, np.uint8)[order], call_range_off=np.arange(n + 1, dtype=np.uint32),
        range_block_lo=(slo[s_arr] + idx).astype(np.uint32), range_len=np.ones(n, np.uint32),
        session_type=(np.arange(n_sessions) % n_types).astype(np.uint16),
        session_block_lo=slo, session_block_len=cnt.astype(np.uint32),
        type_shared_lo=np.zeros(n_types, np.uint32), type_shared_len=np.zeros(n_types, np.uint32), **aeg)


def _seg(n_steps: np.ndarray):
    """flat (session, step) index arrays for sessions with n_steps[s] steps."""
    n_steps = n_steps.astype(np.int64)
    sess = np.repeat(np.arange(n_steps.size, dtype=np.int64), n_steps)
    start = np.concatenate([[0], np.cumsum(n_steps)[:-1]])
    step = np.arange(sess.size, dtype=np.int64) - start[sess]
    return sess, step, start


def _segcumsum(x: np.ndarray, start: np.ndarray, sess: np.ndarray) -> np.ndarray:
    """inclusive cumulative sum restarted at each session."""
    c = np.cumsum(x.astype(np.int64))
    base = np.concatenate([[0], c])[start]  # sum before each segment
    return c - base[sess]


def _lognormal_us(rng, mu, sigma, size, lo_ms=None, hi_ms=None):
    """log-normal tool latency in integer microseconds (optionally truncated by inverse CDF)."""
    if lo_ms is None:
        z = rng.standard_normal(size)
    else:
        a = ndtr((math.log(lo_ms) - mu) / sigma)
        b = ndtr((math.log(hi_ms) - mu) / sigma)
        z = ndtri(a + rng.random(size) * (b - a))
    ms = np.exp(mu + sigma * z)
    return np.maximum(1, np.rint(ms * 1000.0)).astype(np.int64)


def _p95_us(mu, sigma, lo_ms=None, hi_ms=None) -> int:
    if lo_ms is None:
        ms = math.exp(mu + sigma * Z95)
    else:
        a = float(ndtr((math.log(lo_ms) - mu) / sigma))
        b = float(ndtr((math.log(hi_ms) - mu) / sigma))
        ms = math.exp(mu + sigma * float(ndtri(a + 0.95 * (b - a))))
    return int(round(ms * 1000.0))


def _poisson_arrivals_us(rng, n, rate_per_min):
    gaps = rng.exponential(60.0 / rate_per_min, size=n)
    return np.rint(np.cumsum(gaps) * 1e6).astype(np.int64)


def _ceil_div(a, b):
    return -(-a // b)


class _AEGBuilder:
    def __init__(self):
        self.edges: List[List[tuple]] = []
        self.ttl: List[int] = []
        self.obs: List[int] = []
        self.term: List[int] = []
        self.tool: List[int] = []

    def add_node(self, ttl_us, obs, terminal, tool=0):
        self.edges.append([])
        self.ttl.append(int(ttl_us))
        self.obs.append(int(obs))
        self.term.append(int(terminal))
        self.tool.append(int(tool))
        return len(self.edges) - 1

    def add_edge(self, u, v, p, q16=65536):
        self.edges[u].append((v, np.float32(p), int(q16)))

    def finish(self):
        off = [0]
        dst, p, q = [], [], []
        for es in self.edges:
            for (v, pp, qq) in es:
                dst.append(v); p.append(pp); q.append(qq)
            off.append(len(dst))
        return dict(aeg_edge_off=np.array(off, np.uint32), edge_dst=np.array(dst, np.uint32),
                    edge_p=np.array(p, np.float32), edge_shared_q16=np.array(q, np.uint32),
                    node_ttl_base_us=np.array(self.ttl, np.int64), node_obs_tokens=np.array(self.obs, np.uint32),
                    node_terminal=np.array(self.term, np.uint8), node_tool=np.array(self.tool, np.uint32))


# ----------------------------------------------------------------------------------------------
# session-type generators: return per-call dict (flat, session-local indices) + per-session span
# ----------------------------------------------------------------------------------------------

def _swe_aeg(b: _AEGBuilder, max_steps=100, p_geo=1 / 29.24):
    """ReAct chain v0..v99 (Fig. 2): read_file -> edit_code -> run_test."""
    cyc = ["read_file", "edit_code", "run_test"]
    ttl = {"read_file": _p95_us(*tool_params("FileOps")),
           "edit_code": _p95_us(*tool_params("CodeExec")),
           "run_test": _p95_us(math.log(2400.0), 1.0)}
    obs = {"read_file": 1250, "edit_code": 175, "run_test": 850}
    label = {"read_file": TOOL_LABELS.index("FileOps"), "edit_code": TOOL_LABELS.index("CodeExec"),
             "run_test": TOOL_LABELS.index("RunTest")}
    base = len(b.edges)
    for i in range(max_steps):
        k = cyc[i % 3]
        b.add_node(ttl[k], obs[k], i == max_steps - 1, tool=label[k])
    for i in range(max_steps - 1):
        b.add_edge(base + i, base + i + 1, 1.0 if i < 9 else 1.0 - p_geo)
    return base


def _gen_swe(rng, n, aeg_base, shared_tokens=1024, cap_tokens=32768, p_geo=1 / 29.24, max_steps=100):
    n_steps = np.minimum(10 + (rng.geometric(p_geo, size=n) - 1), max_steps)
    p0 = rng.integers(2000, 4001, size=n)
    h0 = p0 - shared_tokens
    sess, step, start = _seg(n_steps)
    F = sess.size
    out = rng.integers(100, 501, size=F)
    kind = step % 3
    obs = np.where(kind == 0, rng.integers(500, 2001, size=F),
                   np.where(kind == 1, rng.integers(50, 301, size=F), rng.integers(200, 1501, size=F)))
    cs_out = _segcumsum(out, start, sess)
    cs_obs_ex = _segcumsum(obs, start, sess) - obs
    X = h0[sess] + cs_out + cs_obs_ex                      # private tokens after call j (incl. output)
    W = cap_tokens - shared_tokens
    lo = np.maximum(0, X - W)
    prompt = shared_tokens + (X - lo) - out
    prev_obs = np.concatenate([[0], obs[:-1]])
    new = np.where(step == 0, prompt, np.minimum(prompt, prev_obs))
    mu_f, s_f = tool_params("FileOps")
    mu_c, s_c = tool_params("CodeExec")
    gap = np.where(kind == 0, _lognormal_us(rng, mu_f, s_f, F),
                   np.where(kind == 1, _lognormal_us(rng, mu_c, s_c, F),
                            _lognormal_us(rng, math.log(2400.0), 1.0, F)))
    span = _ceil_div(np.maximum.reduceat(X, start), BLOCK_TOKENS)
    ranges = [("shared", None, None), ("priv", lo // BLOCK_TOKENS, _ceil_div(X, BLOCK_TOKENS) - lo // BLOCK_TOKENS)]
    return dict(n_steps=n_steps, sess=sess, step=step, start=start, node=aeg_base + step, prompt=prompt,
                out=out, new=new, gap=gap, span=span, ranges=ranges)


def _webarena_aeg(b: _AEGBuilder, max_steps=60, p_geo=1 / 18, shares=(0.45, 0.55, 0.65)):
    """Branching AEG: per step 3 actions {navigate, click, type}; edges to step i+1 with
    p = (1 - 1/18) * (0.5, 0.3, 0.2); per-branch shared-prefix fraction."""
    tools = [("WebApi", 0), ("Database", 1), ("FileOps", 2)]
    ttl = [_p95_us(*tool_params(t), lo_ms=50.0, hi_ms=30000.0) for t, _ in tools]
    base = len(b.edges)
    for i in range(max_steps):
        for a in range(3):
            b.add_node(ttl[a], 6000, i == max_steps - 1, tool=TOOL_LABELS.index(tools[a][0]))
    probs = (0.5, 0.3, 0.2)
    for i in range(max_steps - 1):
        for a in range(3):
            for a2 in range(3):
                b.add_edge(base + 3 * i + a, base + 3 * (i + 1) + a2, (1.0 - p_geo) * probs[a2],
                           int(round(shares[a2] * 65536)))
    return base


def _gen_webarena(rng, n, aeg_base, shared_tokens=1536, p_geo=1 / 18, max_steps=60):
    n_steps = np.clip(rng.geometric(p_geo, size=n), 1, max_steps)
    sess, step, start = _seg(n_steps)
    F = sess.size
    act = rng.choice(3, size=F, p=[0.5, 0.3, 0.2])
    h0 = rng.integers(200, 601, size=n)
    g = rng.integers(150, 351, size=F)
    out = rng.integers(50, 201, size=F)
    page = rng.integers(4000, 8001, size=F)
    X = h0[sess] + _segcumsum(g, start, sess)             # history tokens after call j
    Xprev = X - g
    prompt = shared_tokens + Xprev + page
    prev_g = np.concatenate([[0], g[:-1]])
    prev_out = np.concatenate([[0], out[:-1]])
    new = np.where(step == 0, prompt, np.minimum(prompt, page + prev_g - prev_out))
    gap = np.empty(F, np.int64)
    for a, t in enumerate(["WebApi", "Database", "FileOps"]):
        m = act == a
        gap[m] = _lognormal_us(rng, *tool_params(t), int(m.sum()), lo_ms=50.0, hi_ms=30000.0)
    hist_blocks = _ceil_div(np.maximum.reduceat(X, start), BLOCK_TOKENS)
    pblk = _ceil_div(page, BLOCK_TOKENS)
    poff = hist_blocks[sess] + _segcumsum(pblk, start, sess) - pblk
    span = hist_blocks + np.add.reduceat(pblk, start)
    ranges = [("shared", None, None), ("priv", np.zeros(F, np.int64), _ceil_div(X, BLOCK_TOKENS)),
              ("priv", poff, pblk)]
    return dict(n_steps=n_steps, sess=sess, step=step, start=start, node=aeg_base + 3 * step + act, prompt=prompt,
                out=out, new=new, gap=gap, span=span, ranges=ranges)


def _chain_aeg(b: _AEGBuilder, n_steps, rng, obs_tokens):
    """Single chain with P = 1 (ReAct); tool of each node uniform over Table 1 classes."""
    base = len(b.edges)
    tools = rng.integers(0, 4, size=n_steps)
    for i in range(n_steps):
        b.add_node(_p95_us(*tool_params(TOOL_ORDER[tools[i]])), obs_tokens, i == n_steps - 1, tool=int(tools[i]))
    for i in range(n_steps - 1):
        b.add_edge(base + i, base + i + 1, 1.0)
    return base, tools


def _gen_tenant(rng, n, aeg_base, node_tools, n_steps_fixed, shared_tokens=256, cap_tokens=8192):
    n_steps = np.full(n, n_steps_fixed, np.int64)
    sess, step, start = _seg(n_steps)
    F = sess.size
    h0 = rng.integers(512, 2049, size=n)
    out = rng.integers(64, 257, size=F)
    obs = rng.integers(64, 257, size=F)
    g = out + obs                                          # context growth per step in [128, 512]
    X = h0[sess] + _segcumsum(g, start, sess) - obs        # private tokens after call j incl. output
    W = cap_tokens - shared_tokens
    lo = np.maximum(0, X - W)
    prompt = shared_tokens + (X - lo) - out
    prev_obs = np.concatenate([[0], obs[:-1]])
    new = np.where(step == 0, prompt, np.minimum(prompt, prev_obs))
    tl = node_tools[step]
    gap = np.empty(F, np.int64)
    for k in range(4):
        m = tl == k
        gap[m] = _lognormal_us(rng, *tool_params(TOOL_ORDER[k]), int(m.sum()))
    span = _ceil_div(np.maximum.reduceat(X, start), BLOCK_TOKENS)
    ranges = [("shared", None, None), ("priv", lo // BLOCK_TOKENS, _ceil_div(X, BLOCK_TOKENS) - lo // BLOCK_TOKENS)]
    return dict(n_steps=n_steps, sess=sess, step=step, start=start, node=aeg_base + step, prompt=prompt,
                out=out, new=new, gap=gap, span=span, ranges=ranges)


# ----------------------------------------------------------------------------------------------
# assembly
# ----------------------------------------------------------------------------------------------

def _assemble(name, n_nodes, seed, parts, arrivals, types, shared_tokens, aeg, shared_blocks_override=None):
    """parts: list (per type) of per-call dicts for the sessions of that type; arrivals[type] per session."""
    n_types = len(shared_tokens)
    shared_len = [(_ceil_div(t, BLOCK_TOKENS) if shared_blocks_override is None else shared_blocks_override[i])
                  for i, t in enumerate(shared_tokens)]
    type_lo = np.concatenate([[0], np.cumsum(shared_len)[:-1]]).astype(np.int64)
    next_block = int(np.sum(shared_len))
    # global session order = arrival order (stable over type, local index)
    all_arr = np.concatenate(arrivals)
    all_typ = np.concatenate([np.full(len(a), t) for t, a in enumerate(arrivals)])
    all_loc = np.concatenate([np.arange(len(a)) for a in arrivals])
    order = np.lexsort((all_loc, all_typ, all_arr))
    n_sess = order.size
    gsid = np.empty(n_sess, np.int64)
    gsid[order] = np.arange(n_sess)
    sess_type = all_typ[order].astype(np.uint16)
    # spans in global session order
    spans = np.concatenate([p["span"] for p in parts])
    span_g = np.empty(n_sess, np.int64)
    span_g[gsid] = spans
    sess_lo = next_block + np.concatenate([[0], np.cumsum(span_g)[:-1]])
    n_blocks = next_block + int(span_g.sum())
    assert n_blocks < 2 ** 32
    # flat calls
    cols = {k: [] for k in ("t", "s", "v", "prompt", "out", "new", "last", "nr")}
    rng_lists = []
    off = 0
    for t, p in enumerate(parts):
        g_of_local = gsid[off:off + len(arrivals[t])]
        off += len(arrivals[t])
        s = g_of_local[p["sess"]]
        inc = (p["new"] * (10 ** 6 // PREFILL_TOK_S) + _ceil_div(p["out"] * 10 ** 6, DECODE_TOK_S) + p["gap"])
        tt = arrivals[t][p["sess"]] + _segcumsum(inc, p["start"], p["sess"]) - inc
        last = (p["step"] == p["n_steps"][p["sess"]] - 1)
        cols["t"].append(tt); cols["s"].append(s); cols["v"].append(p["node"]); cols["prompt"].append(p["prompt"])
        cols["out"].append(p["out"]); cols["new"].append(p["new"]); cols["last"].append(last)
        rl = []
        for (kind, lo, ln) in p["ranges"]:
            if kind == "shared":
                if shared_len[t] == 0:
                    continue
                rl.append((np.full(s.size, type_lo[t]), np.full(s.size, shared_len[t])))
            else:
                rl.append((sess_lo[s] + lo, ln))
        rng_lists.append(rl)
        cols["nr"].append(np.full(s.size, len(rl)))
    cat = {k: np.concatenate(v) for k, v in cols.items()}
    order_c = np.lexsort((cat["s"], cat["t"]))
    # ranges: per-type lists have equal count per call; build flat (call, k) arrays
    lo_all, ln_all = [], []
    for rl in rng_lists:
        lo_all.append(np.stack([r[0] for r in rl], axis=1) if rl else np.zeros((0, 0)))
        ln_all.append(np.stack([r[1] for r in rl], axis=1) if rl else np.zeros((0, 0)))
    nr_max = max(a.shape[1] for a in lo_all)
    LO = np.zeros((cat["t"].size, nr_max), np.int64)
    LN = np.zeros((cat["t"].size, nr_max), np.int64)
    r0 = 0
    for a, b_ in zip(lo_all, ln_all):
        LO[r0:r0 + a.shape[0], :a.shape[1]] = a
        LN[r0:r0 + b_.shape[0], :b_.shape[1]] = b_
        r0 += a.shape[0]
    LO = LO[order_c]
    LN = LN[order_c]
    valid = LN > 0
    nr = valid.sum(axis=1)
    range_off = np.concatenate([[0], np.cumsum(nr)]).astype(np.uint32)
    desc = TraceDesc(
        name=name, n_nodes=n_nodes, n_blocks=n_blocks, seed=seed,
        call_t_us=cat["t"][order_c].astype(np.int64),
        call_session=cat["s"][order_c].astype(np.uint32),
        call_aeg_node=cat["v"][order_c].astype(np.uint32),
        call_prompt_tokens=cat["prompt"][order_c].astype(np.uint32),
        call_output_tokens=cat["out"][order_c].astype(np.uint32),
        call_new_tokens=cat["new"][order_c].astype(np.uint32),
        call_is_last=cat["last"][order_c].astype(np.uint8),
        call_range_off=range_off,
        range_block_lo=LO[valid].astype(np.uint32),
        range_len=LN[valid].astype(np.uint32),
        session_type=sess_type,
        session_block_lo=sess_lo.astype(np.uint32),
        session_block_len=span_g.astype(np.uint32),
        type_shared_lo=type_lo.astype(np.uint32),
        type_shared_len=np.array(shared_len, np.uint32),
        **aeg)
    return desc


# ----------------------------------------------------------------------------------------------
# the five configs (BASELINE.json "configs")
# ----------------------------------------------------------------------------------------------

def make_c1(limit_case: bool = False) -> TraceDesc:
    """C1 tiny: 8 sessions x 10 calls, 1 node, deterministic (no RNG).

    Call j of session s at t = s*250 ms + j*1.5 s; AEG = 10-node chain with P = 1,
    v9 terminal; block 0 is the shared prefix; session s owns ids 1+11s .. 11+11s;
    call j touches [0] + [1+11s, 3+11s+j).  Tools alternate FileOps (even j) /
    CodeExec (odd j): ttl_base 320 ms / 2.4 s (Table 1 P95).  limit_case: all
    ttl_base = 10 s (SURVEY §8.C.10 Theorem 2 limit case)."""
    b = _AEGBuilder()
    for j in range(10):
        ttl = 10_000_000 if limit_case else (320_000 if j % 2 == 0 else 2_400_000)
        b.add_node(ttl, 160 if j % 2 == 0 else 64, j == 9, tool=j % 2)
    for j in range(9):
        b.add_edge(j, j + 1, 1.0)
    aeg = b.finish()
    t, s, v, pr, out, new, last, lo, ln = [], [], [], [], [], [], [], [], []
    for ss in range(8):
        for j in range(10):
            t.append(ss * 250_000 + j * 1_500_000); s.append(ss); v.append(j)
            pr.append(16 * (2 + j)); out.append(16); new.append(32 if j == 0 else 16); last.append(j == 9)
    order = np.lexsort((np.array(s), np.array(t)))
    ranges = []
    for i in order:
        ss, j = s[i], v[i]
        ranges.append([(0, 1), (1 + 11 * ss, 2 + j)])
    off = np.concatenate([[0], np.cumsum([len(r) for r in ranges])]).astype(np.uint32)
    return TraceDesc(
        name="C1" + ("_limit" if limit_case else ""), n_nodes=1, n_blocks=1 + 11 * 8, seed=0,
        call_t_us=np.array(t, np.int64)[order], call_session=np.array(s, np.uint32)[order],
        call_aeg_node=np.array(v, np.uint32)[order], call_prompt_tokens=np.array(pr, np.uint32)[order],
        call_output_tokens=np.array(out, np.uint32)[order], call_new_tokens=np.array(new, np.uint32)[order],
        call_is_last=np.array(last, np.uint8)[order], call_range_off=off,
        range_block_lo=np.array([a for r in ranges for a, _ in r], np.uint32),
        range_len=np.array([b_ for r in ranges for _, b_ in r], np.uint32),
        session_type=np.zeros(8, np.uint16),
        session_block_lo=np.array([1 + 11 * k for k in range(8)], np.uint32),
        session_block_len=np.full(8, 11, np.uint32),
        type_shared_lo=np.array([0], np.uint32), type_shared_len=np.array([1], np.uint32), **aeg)


def make_c2(n_sessions: int = 2000, n_nodes: int = 8, seed: int = 2) -> TraceDesc:
    """C2 SWE-bench-shaped: Poisson 8 tasks/min, steps 10+Geom(1/29.24) <= 100 (mean 37)."""
    rng = np.random.default_rng(seed)
    b = _AEGBuilder()
    base = _swe_aeg(b)
    arr = _poisson_arrivals_us(rng, n_sessions, 8.0)
    part = _gen_swe(rng, n_sessions, base)
    return _assemble("C2", n_nodes, seed, [part], [arr], [0], [1024], b.finish())


def make_c3(n_sessions: int = 5000, n_nodes: int = 16, seed: int = 3) -> TraceDesc:
    """C3 WebArena-shaped: 8 tasks/min, Geom(1/18) in [1,60] steps, branching AEG, 50 ms-30 s gaps."""
    rng = np.random.default_rng(seed)
    b = _AEGBuilder()
    base = _webarena_aeg(b)
    arr = _poisson_arrivals_us(rng, n_sessions, 8.0)
    part = _gen_webarena(rng, n_sessions, base)
    return _assemble("C3", n_nodes, seed, [part], [arr], [0], [1536], b.finish())


def make_c4(n_sessions: int = 20000, n_nodes: int = 16, seed: int = 4) -> TraceDesc:
    """C4 64-GPU cluster (16 TP-4 instances): 50% SWE + 50% WebArena types, 16 tasks/min."""
    rng = np.random.default_rng(seed)
    b = _AEGBuilder()
    base0 = _swe_aeg(b)
    base1 = _webarena_aeg(b)
    arr = _poisson_arrivals_us(rng, n_sessions, 16.0)
    typ = rng.integers(0, 2, size=n_sessions)
    a0, a1 = arr[typ == 0], arr[typ == 1]
    p0 = _gen_swe(rng, a0.size, base0)
    p1 = _gen_webarena(rng, a1.size, base1)
    return _assemble("C4", n_nodes, seed, [p0, p1], [a0, a1], [0, 1], [1024, 1536], b.finish())


def make_c5(n_sessions: int = 100_000, n_nodes: int = 32, seed: int = 5) -> TraceDesc:
    """C5 multi-tenant: 10 tenants 3 heavy/4 medium/3 light, 16/8/4 tasks/min, 100/30/10-step chains."""
    rng = np.random.default_rng(seed)
    classes = [100] * 3 + [30] * 4 + [10] * 3
    rates = np.array([16.0] * 3 + [8.0] * 4 + [4.0] * 3)
    b = _AEGBuilder()
    bases, tools = [], []
    for k in classes:
        base, tl = _chain_aeg(b, k, rng, obs_tokens=160)
        bases.append(base); tools.append(tl)
    tot = rates.sum()
    gaps = rng.exponential(60.0 / tot, size=n_sessions)
    arr_all = np.rint(np.cumsum(gaps) * 1e6).astype(np.int64)
    ten = rng.choice(10, size=n_sessions, p=rates / tot)
    parts, arrs = [], []
    for t in range(10):
        a = arr_all[ten == t]
        arrs.append(a)
        parts.append(_gen_tenant(rng, a.size, bases[t], tools[t], classes[t]))
    return _assemble("C5", n_nodes, seed, parts, arrs, list(range(10)), [256] * 10, b.finish())


# kappa (concurrent requests per node) per config: light load for C1-C3; C4/C5 contended
# ("roughly 80% of peak") so that rerouting and work stealing are exercised.
PLACE_KAPPA = {"C1": 32, "C2": 32, "C3": 32, "C4": 8, "C5": 24}


def place_cfg_for(desc_or_name) -> dict:
    name = desc_or_name if isinstance(desc_or_name, str) else desc_or_name.name
    base = name.split("_")[0]
    seed = 0 if isinstance(desc_or_name, str) else desc_or_name.seed
    cfg = default_place_cfg(seed)
    cfg["kappa"] = PLACE_KAPPA.get(base, 32)
    return cfg


CONFIGS = {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}
PHYSICAL_CAP = {"C1": 64, "C2": 32768, "C3": 32768, "C4": None, "C5": None}
N_SWEEP = {"C1": 8, "C2": 8, "C3": 8, "C4": 32, "C5": 32}


def make(name: str, n_sessions: Optional[int] = None, n_nodes: Optional[int] = None, seed: Optional[int] = None,
         **kw) -> TraceDesc:
    f = CONFIGS[name]
    if name == "C1":
        return f(**kw)
    args = {}
    if n_sessions is not None:
        args["n_sessions"] = n_sessions
    if n_nodes is not None:
        args["n_nodes"] = n_nodes
    if seed is not None:
        args["seed"] = seed
    d = f(**args)
    if n_sessions is not None:
        d.name = f"{name}_s{n_sessions}"
    return d


# ----------------------------------------------------------------------------------------------
# fixtures for pins
# ----------------------------------------------------------------------------------------------

def make_obs1(k: int, c: int, n_sessions: int = 2) -> TraceDesc:
    """Observation 1 fixture: k-step chains, each step adds c blocks (call j touches c*(j+1)
    private blocks), sessions interleaved so every call sits in its own epoch, one node, no shared prefix."""
    b = _AEGBuilder()
    for j in range(k):
        b.add_node(1_000_000_000, 0, j == k - 1)
    for j in range(k - 1):
        b.add_edge(j, j + 1, 1.0)
    aeg = b.finish()
    t, s, v, lo, ln = [], [], [], [], []
    for j in range(k):
        for ss in range(n_sessions):
            t.append((j * n_sessions + ss) * EPOCH_US + 1); s.append(ss); v.append(j)
            lo.append(ss * c * k); ln.append(c * (j + 1))
    n = len(t)
    return TraceDesc(
        name=f"obs1_k{k}_c{c}", n_nodes=1, n_blocks=n_sessions * c * k, seed=0,
        call_t_us=np.array(t, np.int64), call_session=np.array(s, np.uint32), call_aeg_node=np.array(v, np.uint32),
        call_prompt_tokens=np.array([16 * x for x in ln], np.uint32), call_output_tokens=np.full(n, 1, np.uint32),
        call_new_tokens=np.full(n, 16, np.uint32),
        call_is_last=np.array([vv == k - 1 for vv in v], np.uint8),
        call_range_off=np.arange(n + 1, dtype=np.uint32), range_block_lo=np.array(lo, np.uint32),
        range_len=np.array(ln, np.uint32), session_type=np.zeros(n_sessions, np.uint16),
        session_block_lo=np.array([ss * c * k for ss in range(n_sessions)], np.uint32),
        session_block_len=np.full(n_sessions, c * k, np.uint32),
        type_shared_lo=np.array([0], np.uint32), type_shared_len=np.array([0], np.uint32), **aeg)


def make_chain_limit(seed: int, n_sessions: int = 6, max_steps: int = 8) -> TraceDesc:
    """Theorem 2 limit-case fixture: one node, single-chain AEGs with P = 1 and the
    terminal node at the end of every session's chain, TTL >> every gap, no context cap, no shared prefix.
    Each call j of a session touches all of its blocks [0, n_j) with n_j strictly growing."""
    rng = np.random.default_rng(seed)
    b = _AEGBuilder()
    steps = rng.integers(1, max_steps + 1, size=n_sessions)
    bases = []
    for ss in range(n_sessions):
        base = len(b.edges)
        for j in range(steps[ss]):
            b.add_node(1_000_000_000, int(rng.integers(0, 64)), j == steps[ss] - 1)
        for j in range(steps[ss] - 1):
            b.add_edge(base + j, base + j + 1, 1.0)
        bases.append(base)
    aeg = b.finish()
    t, s, v, ln = [], [], [], []
    spans = []
    for ss in range(n_sessions):
        tt = int(rng.integers(0, 10)) * EPOCH_US + int(rng.integers(0, EPOCH_US))
        nb = 0
        for j in range(steps[ss]):
            nb += int(rng.integers(1, 4))
            t.append(tt); s.append(ss); v.append(bases[ss] + j); ln.append(nb)
            tt += int(rng.integers(1, 5)) * EPOCH_US + int(rng.integers(0, EPOCH_US))
        spans.append(nb)
    lo_s = np.concatenate([[0], np.cumsum(spans)[:-1]])
    order = np.lexsort((np.array(s), np.array(t)))
    t = np.array(t, np.int64)[order]; s = np.array(s)[order]; v = np.array(v)[order]; ln = np.array(ln)[order]
    last = np.array([v[i] == bases[s[i]] + steps[s[i]] - 1 for i in range(len(t))], np.uint8)
    n = len(t)
    return TraceDesc(
        name=f"limit_{seed}", n_nodes=1, n_blocks=int(sum(spans)), seed=seed,
        call_t_us=t, call_session=s.astype(np.uint32), call_aeg_node=v.astype(np.uint32),
        call_prompt_tokens=(16 * ln).astype(np.uint32), call_output_tokens=np.full(n, 1, np.uint32),
        call_new_tokens=np.full(n, 16, np.uint32), call_is_last=last,
        call_range_off=np.arange(n + 1, dtype=np.uint32), range_block_lo=lo_s[s].astype(np.uint32),
        range_len=ln.astype(np.uint32), session_type=np.zeros(n_sessions, np.uint16),
        session_block_lo=lo_s.astype(np.uint32), session_block_len=np.array(spans, np.uint32),
        type_shared_lo=np.array([0], np.uint32), type_shared_len=np.array([0], np.uint32), **aeg)


def make_random_small(seed: int, n_sessions: int = 5, n_nodes: int = 2, max_calls: int = 4,
                      max_blocks: int = 6, n_types: int = 2, epochs: int = 12) -> TraceDesc:
    """Tiny random traces with every feature (shared prefixes, branching AEG, several nodes) for
    brute-force and GPU==oracle cases.  Times are drawn so that several calls share epochs."""
    rng = np.random.default_rng(seed)
    b = _AEGBuilder()
    n_aeg = 6
    for i in range(n_aeg):
        b.add_node(int(rng.choice([50_000, 150_000, 400_000, 2_000_000])), int(rng.integers(0, 400)), i == n_aeg - 1,
                   tool=i % len(TOOL_LABELS))
    for i in range(n_aeg - 1):
        ds = sorted(set(int(x) for x in rng.integers(i + 1, n_aeg, size=int(rng.integers(1, 3)))))
        ps = rng.dirichlet(np.ones(len(ds) + 1))[:len(ds)]
        for d, p in zip(ds, ps):
            b.add_edge(i, d, float(p), int(rng.integers(0, 65537)))
    aeg = b.finish()
    shared = [int(rng.integers(0, 3)) for _ in range(n_types)]
    type_lo = np.concatenate([[0], np.cumsum(shared)[:-1]])
    nb = int(sum(shared))
    styp = rng.integers(0, n_types, size=n_sessions)
    spans = rng.integers(1, max_blocks + 1, size=n_sessions)
    slo = nb + np.concatenate([[0], np.cumsum(spans)[:-1]])
    nblocks = int(nb + spans.sum())
    calls = []
    for ss in range(n_sessions):
        nc = int(rng.integers(1, max_calls + 1))
        tt = int(rng.integers(0, 3 * EPOCH_US))
        v = 0
        for j in range(nc):
            a = int(rng.integers(0, spans[ss])); z = int(rng.integers(a + 1, spans[ss] + 1))
            rr = []
            if shared[styp[ss]] > 0 and rng.random() < 0.8:
                rr.append((int(type_lo[styp[ss]]), shared[styp[ss]]))
            rr.append((int(slo[ss] + a), z - a))
            calls.append((tt, ss, v, rr, j == nc - 1))
            tt += int(rng.integers(1, 4 * EPOCH_US))
            v = min(n_aeg - 1, v + 1)
    calls.sort(key=lambda x: (x[0], x[1]))
    n = len(calls)
    rr = [r for c in calls for r in c[3]]
    return TraceDesc(
        name=f"rand_{seed}", n_nodes=n_nodes, n_blocks=nblocks, seed=seed,
        call_t_us=np.array([c[0] for c in calls], np.int64), call_session=np.array([c[1] for c in calls], np.uint32),
        call_aeg_node=np.array([c[2] for c in calls], np.uint32),
        call_prompt_tokens=np.array([16 * sum(x[1] for x in c[3]) for c in calls], np.uint32),
        call_output_tokens=np.array([int(rng.integers(1, 40)) for _ in calls], np.uint32),
        call_new_tokens=np.full(n, 16, np.uint32), call_is_last=np.array([c[4] for c in calls], np.uint8),
        call_range_off=np.concatenate([[0], np.cumsum([len(c[3]) for c in calls])]).astype(np.uint32),
        range_block_lo=np.array([x[0] for x in rr], np.uint32), range_len=np.array([x[1] for x in rr], np.uint32),
        session_type=styp.astype(np.uint16), session_block_lo=slo.astype(np.uint32),
        session_block_len=spans.astype(np.uint32), type_shared_lo=type_lo.astype(np.uint32),
        type_shared_len=np.array(shared, np.uint32), **aeg)


def make_stream_trace(seq, epochs=None, n_nodes: int = 1, n_shared: int = 0) -> TraceDesc:
    """A one-node trace whose node-0 stream is exactly `seq` (block ids): access i is a one-block
    call of a single session at boundary epochs[i] (default: every access in its own epoch).
    Blocks 0 .. n_shared-1 are the shared prefix of the session's agent type, the rest its own.
    Used to feed hand-written access sequences (e.g. SPEC S:252 "A B C A B") to next-use / MIN."""
    seq = [int(x) for x in seq]
    n = len(seq)
    if epochs is None:
        epochs = list(range(1, n + 1))
    nb = max(max(seq) + 1 if seq else 1, n_shared)
    b = _AEGBuilder()
    b.add_node(1_000_000, 0, False)
    aeg = b.finish()
    t = [(int(e) - 1) * EPOCH_US + 1 + i for i, e in enumerate(epochs)]  # admitted at boundary e
    return TraceDesc(
        name="stream", n_nodes=n_nodes, n_blocks=nb, seed=0,
        call_t_us=np.array(t, np.int64), call_session=np.zeros(n, np.uint32), call_aeg_node=np.zeros(n, np.uint32),
        call_prompt_tokens=np.full(n, 16, np.uint32), call_output_tokens=np.full(n, 1, np.uint32),
        call_new_tokens=np.full(n, 16, np.uint32), call_is_last=np.zeros(n, np.uint8),
        call_range_off=np.arange(n + 1, dtype=np.uint32), range_block_lo=np.array(seq, np.uint32),
        range_len=np.ones(n, np.uint32), session_type=np.zeros(1, np.uint16),
        session_block_lo=np.array([n_shared], np.uint32),
        session_block_len=np.array([max(nb - n_shared, 0)], np.uint32),
        type_shared_lo=np.array([0], np.uint32), type_shared_len=np.array([n_shared], np.uint32), **aeg)


def make_hand_trace(calls, nodes, n_nodes: int = 1, shared=None, session_types=None) -> TraceDesc:
    """A hand-written trace for pins whose expected result is derived by hand.

    calls: list of dicts (t, s, v, prompt, out, new=prompt, last=0, blocks=[(lo, len), ...]), any
           order (sorted here by (t, s)); block ids are global.
    nodes: AEG nodes, list of dicts (ttl, obs, term=0, edges=[(dst, p, q16=65536), ...]).
    shared: per agent type (lo, len) shared-prefix span (default: one type without a prefix).
    Each session's private span is the hull of its blocks outside the shared spans."""
    calls = sorted(calls, key=lambda c: (c["t"], c["s"]))
    shared = shared or [(0, 0)]
    ns = max(c["s"] for c in calls) + 1
    styp = np.array(session_types if session_types is not None else [0] * ns, np.uint16)
    b = _AEGBuilder()
    for nd in nodes:
        b.add_node(nd["ttl"], nd.get("obs", 0), bool(nd.get("term", 0)))
    for u, nd in enumerate(nodes):
        for e in nd.get("edges", []):
            b.add_edge(u, e[0], e[1], e[2] if len(e) > 2 else 65536)
    aeg = b.finish()
    in_shared = lambda x: any(lo <= x < lo + ln for lo, ln in shared)
    lo_s = [None] * ns
    hi_s = [None] * ns
    off, rlo, rln = [0], [], []
    for c in calls:
        for lo, ln in c["blocks"]:
            rlo.append(lo); rln.append(ln)
            for x in (lo, lo + ln - 1):
                if not in_shared(x):
                    s = c["s"]
                    lo_s[s] = x if lo_s[s] is None else min(lo_s[s], x)
                    hi_s[s] = x if hi_s[s] is None else max(hi_s[s], x)
        off.append(len(rlo))
    nb = max([lo + ln for lo, ln in zip(rlo, rln)] + [lo + ln for lo, ln in shared] + [1])
    slo = np.array([0 if lo_s[s] is None else lo_s[s] for s in range(ns)], np.uint32)
    sln = np.array([0 if lo_s[s] is None else hi_s[s] - lo_s[s] + 1 for s in range(ns)], np.uint32)
    n = len(calls)
    return TraceDesc(
        name="hand", n_nodes=n_nodes, n_blocks=int(nb), seed=0,
        call_t_us=np.array([c["t"] for c in calls], np.int64),
        call_session=np.array([c["s"] for c in calls], np.uint32),
        call_aeg_node=np.array([c["v"] for c in calls], np.uint32),
        call_prompt_tokens=np.array([c["prompt"] for c in calls], np.uint32),
        call_output_tokens=np.array([c["out"] for c in calls], np.uint32),
        call_new_tokens=np.array([c.get("new", c["prompt"]) for c in calls], np.uint32),
        call_is_last=np.array([c.get("last", 0) for c in calls], np.uint8),
        call_range_off=np.array(off, np.uint32), range_block_lo=np.array(rlo, np.uint32),
        range_len=np.array(rln, np.uint32), session_type=styp, session_block_lo=slo, session_block_len=sln,
        type_shared_lo=np.array([lo for lo, _ in shared], np.uint32),
        type_shared_len=np.array([ln for _, ln in shared], np.uint32), **aeg)
