"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  It loads oracle/libsaga_oracle.so (plain C++17 written from PAPER.md; see
saga_oracle.cpp header) and never touches paper_2605_00528_b200/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "saga_oracle.cpp")
LIB = os.path.join(HERE, "libsaga_oracle.so")

POL_AEG, POL_BELADY, POL_EVICT_ALL, POL_LRU, POL_LRU_PREFIX = 1, 2, 4, 8, 16
INF = 0xFFFFFFFF
COUNTERS = ["ACCESSES", "HITS", "MISSES", "COMPULSORY_GLOBAL", "COMPULSORY_NODE", "MIG_HITS", "MIG_MISSES",
            "INVALIDATED", "EVICTIONS", "EVICT_PROTECTED", "EVICT_EVENTS", "REGEN_TOKENS", "REGEN_US", "VICTIM_HASH",
            "INFEASIBLE_EPOCH", "PEAK_RESIDENT", "PF_HITS", "PF_MISSES", "RESERVED18", "RESERVED19"]
NCOUNT = len(COUNTERS)
CI = {n: i for i, n in enumerate(COUNTERS)}

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -ffp-contract=off, no -ffast-math, no SIMD intrinsics).

    SAGA_ORACLE_LIB names a prebuilt library instead (scripts/mutate_oracle.py loads mutants)."""
    if os.environ.get("SAGA_ORACLE_LIB"):
        return os.environ["SAGA_ORACLE_LIB"]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", LIB, SRC, "-lpthread"])
    return LIB


class ODesc(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("n_calls", "n_sessions", "n_types", "n_aeg_nodes", "n_edges",
                                          "n_ranges", "n_blocks", "n_nodes", "block_tokens")] + [
        ("call_t_us", C.c_void_p), ("call_session", C.c_void_p), ("call_aeg_node", C.c_void_p),
        ("call_prompt_tokens", C.c_void_p), ("call_output_tokens", C.c_void_p), ("call_new_tokens", C.c_void_p),
        ("call_is_last", C.c_void_p), ("call_range_off", C.c_void_p), ("range_block_lo", C.c_void_p),
        ("range_len", C.c_void_p), ("session_type", C.c_void_p), ("session_block_lo", C.c_void_p),
        ("session_block_len", C.c_void_p), ("aeg_edge_off", C.c_void_p), ("edge_dst", C.c_void_p),
        ("edge_p", C.c_void_p), ("edge_shared_q16", C.c_void_p), ("node_ttl_base_us", C.c_void_p),
        ("node_obs_tokens", C.c_void_p), ("node_terminal", C.c_void_p), ("type_shared_lo", C.c_void_p),
        ("type_shared_len", C.c_void_p), ("call_ttl_base_us", C.c_void_p), ("call_obs_tokens", C.c_void_p)]


class OPlace(C.Structure):
    _fields_ = [("epoch_us", C.c_int64), ("kappa", C.c_uint32), ("prefill_tok_s", C.c_uint32),
                ("decode_tok_s", C.c_uint32), ("theta_pm", C.c_uint32), ("rmax_pm", C.c_uint32),
                ("t_idle_us", C.c_int64), ("seed", C.c_uint64)]


class OReplay(C.Structure):
    _fields_ = [("policy", C.c_uint32), ("alpha", C.c_float), ("beta", C.c_float), ("gamma", C.c_float),
                ("p_low_pm", C.c_uint32), ("p_high_pm", C.c_uint32), ("ttl_max_us", C.c_int64)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            vp = C.c_void_p
            L.oracle_new.restype = vp
            L.oracle_new.argtypes = [C.POINTER(ODesc), C.POINTER(OPlace), C.POINTER(C.c_int)]
            L.oracle_new_nodes.restype = vp
            L.oracle_new_nodes.argtypes = [C.POINTER(ODesc), C.POINTER(OPlace), C.c_uint32, C.c_uint32,
                                           C.POINTER(C.c_int)]
            L.oracle_prefetch.argtypes = [vp, vp, vp]
            L.oracle_free.argtypes = [vp]
            L.oracle_placement.argtypes = [vp, vp, vp]
            L.oracle_migrations.argtypes = [vp, vp]
            L.oracle_n_act.restype = C.c_uint64
            L.oracle_n_act.argtypes = [vp]
            L.oracle_act.argtypes = [vp, vp]
            for f in ("oracle_stream_len", "oracle_n_events", "oracle_n_groups", "oracle_n_inv"):
                getattr(L, f).restype = C.c_uint64
                getattr(L, f).argtypes = [vp, C.c_uint32]
            L.oracle_stream.argtypes = [vp, C.c_uint32, vp, vp, vp, vp]
            L.oracle_n_local.restype = C.c_uint32
            L.oracle_n_local.argtypes = [vp, C.c_uint32]
            L.oracle_next_use.argtypes = [vp, C.c_uint32, vp, vp, vp, vp]
            L.oracle_lid_owner.argtypes = [vp, C.c_uint32, vp]
            L.oracle_sweep_range.argtypes = [vp, C.c_uint32, vp, vp]
            L.oracle_replay.restype = C.c_uint64
            L.oracle_replay.argtypes = [vp, C.POINTER(OReplay), C.c_uint32, C.c_uint32, vp, vp, C.c_uint64]
            L.oracle_replay_log.restype = C.c_uint64
            L.oracle_replay_log.argtypes = [vp, C.POINTER(OReplay), C.c_uint32, C.c_uint32, vp, vp, C.c_uint64]
            L.oracle_replay_many.argtypes = [vp, C.POINTER(OReplay), C.c_uint32, vp, C.c_uint32, vp, C.c_uint32,
                                             vp, C.c_int]
            L.oracle_min_misses.restype = C.c_int64
            L.oracle_min_misses.argtypes = [vp, C.c_uint32, C.c_uint32]
            L.oracle_keys.argtypes = [vp, C.POINTER(OReplay), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_uint32, vp, vp, vp, C.c_uint64, vp, vp, vp]
            L.oracle_score32.restype = C.c_float
            L.oracle_score32.argtypes = [C.c_float] * 3 + [C.c_int64, C.c_int64, C.c_uint32, C.c_uint32, C.c_float,
                                                            C.POINTER(C.c_uint32)]
            L.oracle_reuse32.restype = C.c_float
            L.oracle_reuse32.argtypes = [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32]
            L.oracle_ttl_protect.restype = C.c_int
            L.oracle_ttl_protect.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_uint32]
            L.oracle_splitmix64.restype = C.c_uint64
            L.oracle_splitmix64.argtypes = [C.c_uint64]
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def replay_cfg(policy=POL_AEG, alpha=0.3, beta=0.5, gamma=0.2, p_low_pm=700, p_high_pm=900,
               ttl_max_us=300_000_000, **_):
    return OReplay(policy, alpha, beta, gamma, p_low_pm, p_high_pm, ttl_max_us)


class Oracle:
    """Owns one oracle instance over a TraceDesc (validation, placement and expansion run at build)."""

    def __init__(self, desc, place_cfg: dict, node_mask: int = 0, prefetch: bool = False):
        self.desc = desc
        self._keep = {}
        arrs = {}
        for f, _ in ODesc._fields_[9:]:
            a = getattr(desc, f, None)  # the per-call overrides are optional
            arrs[f] = None if a is None else np.ascontiguousarray(a)
        self._keep = arrs
        d = ODesc(desc.n_calls, desc.n_sessions, desc.n_types, desc.n_aeg_nodes, desc.n_edges, desc.n_ranges,
                  desc.n_blocks, desc.n_nodes, desc.block_tokens, *[_p(arrs[f]) for f, _ in ODesc._fields_[9:]])
        p = OPlace(place_cfg["epoch_us"], place_cfg["kappa"], place_cfg["prefill_tok_s"], place_cfg["decode_tok_s"],
                   place_cfg["theta_pm"], place_cfg["rmax_pm"], place_cfg["t_idle_us"], place_cfg["seed"])
        self.place_cfg = dict(place_cfg)
        err = C.c_int(0)
        self.h = lib().oracle_new_nodes(C.byref(d), C.byref(p), node_mask, 2 if prefetch else 0, C.byref(err))
        self.err = err.value
        if not self.h:
            raise ValueError(f"oracle: invalid trace (code {self.err})")

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_free(self.h)
            self.h = None

    # ---- placement ----
    def placement(self):
        node = np.zeros(self.desc.n_calls, np.uint8)
        st = np.zeros(3, np.int64)
        lib().oracle_placement(self.h, _p(node), st.ctypes.data)
        mig = np.zeros((int(st[2]), 4), np.uint32)
        if st[2]:
            lib().oracle_migrations(self.h, mig.ctypes.data)
        return node, mig, int(st[0]), int(st[1])

    def act_log(self):
        n = lib().oracle_n_act(self.h)
        out = np.zeros((n, 3), np.uint32)
        if n:
            lib().oracle_act(self.h, out.ctypes.data)
        return out

    # ---- streams ----
    def stream(self, w):
        L = lib()
        n = L.oracle_stream_len(self.h, w)
        ne = L.oracle_n_events(self.h, w)
        ng = L.oracle_n_groups(self.h, w)
        ni = L.oracle_n_inv(self.h, w)
        block = np.zeros(n, np.uint32)
        ev = np.zeros((ne, 4), np.uint32)
        grp = np.zeros((ng, 4), np.int64)
        inv = np.zeros(ni, np.uint32)
        L.oracle_stream(self.h, w, _p(block), _p(ev), _p(grp), _p(inv))
        return dict(block=block, events=ev, groups=grp, inv=inv)

    def next_use(self, w):
        L = lib()
        n = L.oracle_stream_len(self.h, w)
        nu = np.zeros(n, np.uint32)
        lid = np.zeros(n, np.uint32)
        ftn = np.zeros(n, np.uint8)
        fie = np.zeros(n, np.uint8)
        L.oracle_next_use(self.h, w, _p(nu), _p(lid), _p(ftn), _p(fie))
        return dict(next_use=nu, local_id=lid, ftn=ftn, fie=fie)

    def n_local(self, w):
        return lib().oracle_n_local(self.h, w)

    def lid_owner(self, w):
        n = self.n_local(w)
        out = np.zeros(n, np.uint32)
        lib().oracle_lid_owner(self.h, w, _p(out))
        return out

    def sweep_range(self, w):
        a, b = C.c_uint32(0), C.c_uint32(0)
        lib().oracle_sweep_range(self.h, w, C.byref(a), C.byref(b))
        return a.value, b.value

    # ---- replay ----
    def replay(self, policy, w, cap, rcfg: dict | None = None, log=False):
        cfg = replay_cfg(**(rcfg or {}))
        cfg.policy = policy
        ctr = np.zeros(NCOUNT, np.int64)
        if log:
            cap_log = 1 << 22
            buf = np.zeros(cap_log, np.uint32)
            n = lib().oracle_replay(self.h, C.byref(cfg), w, cap, ctr.ctypes.data, buf.ctypes.data, cap_log)
            return ctr, buf[:n].copy()
        lib().oracle_replay(self.h, C.byref(cfg), w, cap, ctr.ctypes.data, None, 0)
        return ctr

    def replay_log(self, policy, w, cap, rcfg: dict | None = None):
        """(counters, victims as uint64 (epoch << 32) | local id in eviction order)."""
        cfg = replay_cfg(**(rcfg or {}))
        cfg.policy = policy
        ctr = np.zeros(NCOUNT, np.int64)
        cap_log = 1 << 22
        buf = np.zeros(cap_log, np.uint64)
        n = lib().oracle_replay_log(self.h, C.byref(cfg), w, cap, ctr.ctypes.data, buf.ctypes.data, cap_log)
        assert n <= cap_log
        return ctr, buf[:n].copy()

    def replay_many(self, policy_mask, caps, nodes=None, rcfg: dict | None = None, nthreads=None):
        cfg = replay_cfg(**(rcfg or {}))
        caps = np.ascontiguousarray(caps, np.uint32)
        nodes = np.arange(self.desc.n_nodes, dtype=np.uint32) if nodes is None else np.ascontiguousarray(nodes, np.uint32)
        npol = bin(policy_mask & 31).count("1")
        out = np.zeros((npol, caps.size, self.desc.n_nodes, NCOUNT), np.int64)
        lib().oracle_replay_many(self.h, C.byref(cfg), policy_mask, caps.ctypes.data, caps.size, nodes.ctypes.data,
                                 nodes.size, out.ctypes.data, int(nthreads or os.cpu_count() or 1))
        return out

    def prefetch_plan(self):
        """Per call (PREFETCH epoch or 0, prefix blocks) -- with prefetch=True."""
        e = np.zeros(self.desc.n_calls, np.uint32)
        n = np.zeros(self.desc.n_calls, np.uint32)
        lib().oracle_prefetch(self.h, _p(e), _p(n))
        return e, n

    def min_misses(self, w, cap):
        return lib().oracle_min_misses(self.h, w, cap)

    def keys(self, policy, w, e, occ, cap, act, lid, t_last, nu, rcfg: dict | None = None):
        cfg = replay_cfg(**(rcfg or {}))
        cfg.policy = policy
        lid = np.ascontiguousarray(lid, np.uint32)
        t_last = np.ascontiguousarray(t_last, np.int64)
        nu = np.ascontiguousarray(nu, np.uint32)
        n = lid.size
        key = np.zeros(n, np.uint64)
        s32 = np.zeros(n, np.float32)
        s64 = np.zeros(n, np.float64)
        lib().oracle_keys(self.h, C.byref(cfg), w, e, occ, cap, act, _p(lid), _p(t_last), _p(nu), n,
                          _p(key), _p(s32), _p(s64))
        return key, s32, s64


def select_topk(keys: np.ndarray, k: int) -> np.ndarray:
    """A6 plain definition: indices of the k largest keys, in descending key order (full sort)."""
    idx = np.argsort(np.asarray(keys, np.uint64), kind="stable")[::-1]
    return idx[:k]


# scalar entry points (SPEC worked examples): thin callers of the oracle's score() / reuse() / prot()
def score32(alpha, beta, gamma, d, tau, size, smax, P):
    """eq:eviction of a private unfinished candidate idle d of tau_max, size of size_max: (fp32, q)."""
    q = C.c_uint32(0)
    s = lib().oracle_score32(alpha, beta, gamma, d, tau, size, smax, P, C.byref(q))
    return s, q.value


def reuse32(p, q16, ncur, nobs):
    p = np.ascontiguousarray(p, np.float32)
    q16 = np.ascontiguousarray(q16, np.uint32)
    return lib().oracle_reuse32(_p(p), _p(q16), p.size, ncur, nobs)


def ttl_protect(el, ttl_base, ttl_max, occ, cap, low_pm=700, high_pm=900):
    return bool(lib().oracle_ttl_protect(el, ttl_base, ttl_max, occ, cap, low_pm, high_pm))


def splitmix64(x):
    return lib().oracle_splitmix64(x)
