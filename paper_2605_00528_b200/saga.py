"""Thin ctypes binding of libsaga (include/saga.h): argument marshalling only.

Every step of the hot path runs in libsaga's sm_100a kernels.  PyTorch is used for device
memory, streams and process groups.  There is no CPU fallback: importing this module on a box
without the built extension raises immediately, and calling it without a CUDA device fails.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsaga.so")

POLICY_AEG, POLICY_BELADY, POLICY_EVICT_ALL, POLICY_LRU, POLICY_LRU_PREFIX = 1, 2, 4, 8, 16
NCOUNT = 20
COUNTERS = ["ACCESSES", "HITS", "MISSES", "COMPULSORY_GLOBAL", "COMPULSORY_NODE", "MIG_HITS", "MIG_MISSES",
            "INVALIDATED", "EVICTIONS", "EVICT_PROTECTED", "EVICT_EVENTS", "REGEN_TOKENS", "REGEN_US", "VICTIM_HASH",
            "INFEASIBLE_EPOCH", "PEAK_RESIDENT", "PF_HITS", "PF_MISSES", "RESERVED18", "RESERVED19"]
CI = {n: i for i, n in enumerate(COUNTERS)}
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "TRACE", 3: "CAPACITY", 4: "STATE", 5: "OOM", 6: "CUDA", 7: "NCCL"}

DESC_ARRAYS = [("call_t_us", np.int64), ("call_session", np.uint32), ("call_aeg_node", np.uint32),
               ("call_prompt_tokens", np.uint32), ("call_output_tokens", np.uint32), ("call_new_tokens", np.uint32),
               ("call_is_last", np.uint8), ("call_range_off", np.uint32), ("range_block_lo", np.uint32),
               ("range_len", np.uint32), ("session_type", np.uint16), ("session_block_lo", np.uint32),
               ("session_block_len", np.uint32), ("aeg_edge_off", np.uint32), ("edge_dst", np.uint32),
               ("edge_p", np.float32), ("edge_shared_q16", np.uint32), ("node_ttl_base_us", np.int64),
               ("node_obs_tokens", np.uint32), ("node_terminal", np.uint8), ("type_shared_lo", np.uint32),
               ("type_shared_len", np.uint32),
               # optional per-call overrides (None = the AEG node values)
               ("call_ttl_base_us", np.int64), ("call_obs_tokens", np.uint32)]
OPTIONAL_ARRAYS = {"call_ttl_base_us", "call_obs_tokens"}


class SagaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"saga status {STATUS.get(status, status)}: {msg}")
        self.status = status


class TraceDescC(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("n_calls", "n_sessions", "n_types", "n_aeg_nodes", "n_edges", "n_ranges",
                                          "n_blocks", "n_nodes", "block_tokens")] + [(n, C.c_void_p) for n, _ in DESC_ARRAYS]


class PlaceCfgC(C.Structure):
    _fields_ = [("epoch_us", C.c_int64), ("kappa", C.c_uint32), ("prefill_tok_s", C.c_uint32),
                ("decode_tok_s", C.c_uint32), ("theta_pm", C.c_uint32), ("rmax_pm", C.c_uint32),
                ("t_idle_us", C.c_int64), ("seed", C.c_uint64)]


class ReplayCfgC(C.Structure):
    _fields_ = [("policy_mask", C.c_uint32), ("alpha", C.c_float), ("beta", C.c_float), ("gamma", C.c_float),
                ("p_low_pm", C.c_uint32), ("p_high_pm", C.c_uint32), ("ttl_max_us", C.c_int64), ("flags", C.c_uint32)]


class ScoreBatchC(C.Structure):
    _fields_ = [("n_seg", C.c_uint32), ("policy", C.c_uint32), ("seg_node", C.c_void_p), ("seg_epoch", C.c_void_p),
                ("seg_occ", C.c_void_p), ("seg_cap", C.c_void_p), ("seg_act", C.c_void_p), ("seg_off", C.c_void_p),
                ("cand_lid", C.c_void_p), ("cand_t_last", C.c_void_p), ("cand_nu", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsaga.so not built ({LIB_PATH}); run __graft_entry__.build() or "
                          f"python paper_2605_00528_b200/build.py")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    sigs = {
        "saga_last_error": (C.c_char_p, []),
        "saga_kernel_launches": (u64, []),
        "saga_load_trace": (i32, [C.POINTER(TraceDescC), C.POINTER(PlaceCfgC), u32, i32, vp, C.POINTER(vp)]),
        "saga_load_trace_ex": (i32, [C.POINTER(TraceDescC), C.POINTER(PlaceCfgC), u32, i32, vp, u32, C.POINTER(vp)]),
        "saga_trace_info": (i32, [vp, u32, C.POINTER(u64), C.POINTER(u32)]),
        "saga_placement": (i32, [vp, vp, vp, u64, vp]),
        "saga_node_stream_sizes": (i32, [vp, u32, C.POINTER(u64), C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
        "saga_node_stream": (i32, [vp, u32, vp, vp, vp, vp, vp, vp]),
        "saga_belady_next_use": (i32, [vp, u32, vp, vp, vp]),
        "saga_belady_next_use_nodes": (i32, [vp, vp, u32, vp]),
        "saga_replay_wait": (i32, [vp]),
        "saga_sweep_range": (i32, [vp, u32, C.POINTER(u32), C.POINTER(u32)]),
        "saga_aeg_score": (i32, [vp, C.POINTER(ScoreBatchC), C.POINTER(ReplayCfgC), vp, vp, vp]),
        "saga_evict_select": (i32, [vp, vp, vp, u32, vp, vp, vp]),
        "saga_replay": (i32, [vp, C.POINTER(ReplayCfgC), vp, u32, vp, u32, vp, vp]),
        "saga_replay_victims": (i32, [vp, C.POINTER(ReplayCfgC), u32, u32, vp, u64, C.POINTER(u64), vp, vp]),
        "saga_pattern_infer": (i32, [vp, vp, u32, vp, u32, u32, vp, vp, vp, vp, vp, vp]),
        "saga_tool_stats": (i32, [vp, vp, u32, u32, u32, u32, u32, vp, vp, vp]),
        "saga_comm_unique_id": (i32, [vp]),
        "saga_comm_init": (i32, [vp, i32, i32, i32, C.POINTER(vp)]),
        "saga_allreduce_counters": (i32, [vp, vp, C.c_size_t, i32, vp]),
        "saga_comm_destroy": (None, [vp]),
        "saga_free_trace": (None, [vp]),
        "saga_profile_enable": (None, [i32]),
        "saga_profile_read": (None, [vp, vp]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def _check(st):
    if st != 0:
        raise SagaError(st, lib.saga_last_error().decode(errors="replace"))


def kernel_launches() -> int:
    return int(lib.saga_kernel_launches())


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def place_cfg_c(cfg: dict) -> PlaceCfgC:
    return PlaceCfgC(cfg["epoch_us"], cfg["kappa"], cfg["prefill_tok_s"], cfg["decode_tok_s"], cfg["theta_pm"],
                     cfg["rmax_pm"], cfg["t_idle_us"], cfg["seed"])


def replay_cfg_c(cfg: dict) -> ReplayCfgC:
    return ReplayCfgC(cfg.get("policy_mask", 3), cfg.get("alpha", 0.3), cfg.get("beta", 0.5), cfg.get("gamma", 0.2),
                      cfg.get("p_low_pm", 700), cfg.get("p_high_pm", 900), cfg.get("ttl_max_us", 300_000_000),
                      cfg.get("flags", 0))


class HostDesc:
    """Keeps the host arrays (numpy or pinned torch tensors) alive while the C struct points at them."""

    def __init__(self, desc, pinned: bool = False):
        import torch
        self.keep = []
        ptrs = []
        for name, dt in DESC_ARRAYS:
            if name in OPTIONAL_ARRAYS and getattr(desc, name, None) is None:
                ptrs.append(None)
                continue
            a = np.ascontiguousarray(getattr(desc, name), dtype=dt)
            if pinned:
                t = torch.from_numpy(a.view(np.uint8) if a.size else np.zeros(1, np.uint8)).pin_memory()
                self.keep.append(t)
                ptrs.append(t.data_ptr())
            else:
                self.keep.append(a)
                ptrs.append(a.ctypes.data if a.size else None)
        self.c = TraceDescC(desc.n_calls, desc.n_sessions, desc.n_types, desc.n_aeg_nodes, desc.n_edges, desc.n_ranges,
                            desc.n_blocks, desc.n_nodes, desc.block_tokens, *ptrs)
        self.nbytes = sum(int(k.numel() if hasattr(k, "numel") else k.nbytes) for k in self.keep)


class Trace:
    """A loaded trace handle (saga_load_trace).  All methods are stream-ordered on `stream`."""

    def __init__(self, desc, place_cfg: dict, owned_mask: int = 0, device: int = 0, stream=None, host=None,
                 defer_expand: bool = False, prefetch: bool = False):
        import torch
        self.desc = desc
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self._host = host if host is not None else HostDesc(desc)
        self._pc = place_cfg_c(place_cfg)
        h = C.c_void_p()
        _check(lib.saga_load_trace_ex(C.byref(self._host.c), C.byref(self._pc), owned_mask, device,
                                      _stream_ptr(self.stream), (1 if defer_expand else 0) | (2 if prefetch else 0),
                                      C.byref(h)))
        self.h = h

    def free(self):
        if getattr(self, "h", None):
            lib.saga_free_trace(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def info(self, node):
        n = C.c_uint64()
        nl = C.c_uint32()
        _check(lib.saga_trace_info(self.h, node, C.byref(n), C.byref(nl)))
        return n.value, (None if nl.value == 0xFFFFFFFF else nl.value)

    def placement(self):
        node = np.zeros(self.desc.n_calls, np.uint8)
        st = np.zeros(3, np.int64)
        _check(lib.saga_placement(self.h, node.ctypes.data if node.size else None, None, 0, st.ctypes.data))
        mig = np.zeros((int(st[2]), 4), np.uint32)
        if st[2]:
            _check(lib.saga_placement(self.h, None, mig.ctypes.data, int(st[2]), st.ctypes.data))
        return node, mig, int(st[0]), int(st[1])

    def node_stream(self, node):
        import torch
        n, J, G, I = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib.saga_node_stream_sizes(self.h, node, C.byref(n), C.byref(J), C.byref(G), C.byref(I)))
        dev = torch.device("cuda", self.device)
        block = torch.empty(max(n.value, 1), dtype=torch.int32, device=dev)
        ev = torch.empty(max(J.value, 1) * 3, dtype=torch.int32, device=dev)
        grp = torch.empty(max(G.value, 1) * 2, dtype=torch.int64, device=dev)
        grp_t = torch.empty(max(G.value, 1), dtype=torch.int64, device=dev)
        inv = torch.empty(max(I.value, 1), dtype=torch.int32, device=dev)
        _check(lib.saga_node_stream(self.h, node, block.data_ptr(), ev.data_ptr(), grp.data_ptr(), grp_t.data_ptr(),
                                    inv.data_ptr(), _stream_ptr(self.stream)))
        self.stream.synchronize()
        u32 = lambda t: t.cpu().numpy().view(np.uint32)
        return dict(block=u32(block)[:n.value], events=u32(ev)[:3 * J.value].reshape(-1, 3),
                    groups=grp.cpu().numpy()[:2 * G.value].reshape(-1, 2), group_t=grp_t.cpu().numpy()[:G.value],
                    inv=u32(inv)[:I.value])

    def next_use(self, node, next_use_out=None, local_id_out=None):
        """A4 for one node; optional int32 torch outputs receive next_use / local_id (uint32 bits)."""
        _check(lib.saga_belady_next_use(self.h, node, next_use_out.data_ptr() if next_use_out is not None else None,
                                        local_id_out.data_ptr() if local_id_out is not None else None,
                                        _stream_ptr(self.stream)))

    def next_use_nodes(self, nodes):
        """A4 for several nodes in one launch set per kernel (saga_belady_next_use_nodes)."""
        nodes = np.ascontiguousarray(nodes, np.uint32)
        _check(lib.saga_belady_next_use_nodes(self.h, nodes.ctypes.data if nodes.size else None, nodes.size,
                                              _stream_ptr(self.stream)))

    def sweep_range(self, node):
        a, b = C.c_uint32(), C.c_uint32()
        _check(lib.saga_sweep_range(self.h, node, C.byref(a), C.byref(b)))
        return a.value, b.value

    def replay(self, rcfg: dict, caps, nodes, counters, wait: bool = True):
        """A7 (saga_replay, asynchronous); wait=True also runs saga_replay_wait (sync + checks)."""
        caps = np.ascontiguousarray(caps, np.uint32)
        nodes = np.ascontiguousarray(nodes, np.uint32)
        cfg = replay_cfg_c(rcfg)
        _check(lib.saga_replay(self.h, C.byref(cfg), caps.ctypes.data, caps.size, nodes.ctypes.data, nodes.size,
                               counters.data_ptr(), _stream_ptr(self.stream)))
        if wait:
            self.replay_wait()

    def replay_wait(self):
        _check(lib.saga_replay_wait(self.h))

    def pattern_infer(self, label, n_labels: int, role, theta_pm: int = 700, min_tasks: int = 30,
                      want_prob: bool = True, want_eval: bool = True):
        """F3 (saga_pattern_infer): label uint32/int32 cuda tensor [n_calls], role uint8 cuda tensor
        [n_sessions] (0 ignored, 1 training, 2 held-out).  Returns a dict of cuda tensors: counts
        int64 [T, L, L+1], tasks int32 [T], pred int32 [T, L] (-1 = none), prob float32
        [T, L, L+1], eval int64 [T, 4] (transitions, predicted, correct, 0)."""
        import torch
        dev = label.device
        T, L = self.desc.n_types, int(n_labels)
        out = dict(counts=torch.empty((T, L, L + 1), dtype=torch.int64, device=dev),
                   tasks=torch.empty(T, dtype=torch.int32, device=dev),
                   pred=torch.empty((T, L), dtype=torch.int32, device=dev))
        if want_prob:
            out["prob"] = torch.empty((T, L, L + 1), dtype=torch.float32, device=dev)
        if want_eval:
            out["eval"] = torch.empty((T, 4), dtype=torch.int64, device=dev)
        ptr = lambda k: out[k].data_ptr() if k in out else None
        _check(lib.saga_pattern_infer(self.h, label.data_ptr(), L, role.data_ptr(), int(theta_pm), int(min_tasks),
                                      ptr("counts"), ptr("tasks"), ptr("pred"), ptr("prob"), ptr("eval"),
                                      _stream_ptr(self.stream)))
        return out

    def replay_victims(self, rcfg: dict, cap: int, node: int, log_cap: int = 1 << 22):
        """One (policy, cap, node) replay with its victim log.  Returns (counters int64[NCOUNT] numpy,
        victims uint64 numpy of (epoch << 32) | local id, epochs ascending)."""
        import torch
        cfg = replay_cfg_c(rcfg)
        ctr = torch.zeros((self.desc.n_nodes, NCOUNT), dtype=torch.int64, device=f"cuda:{self.device}")
        log = torch.empty(max(1, log_cap), dtype=torch.int64, device=f"cuda:{self.device}")
        n = C.c_uint64(0)
        _check(lib.saga_replay_victims(self.h, C.byref(cfg), int(cap), int(node), log.data_ptr(), int(log_cap),
                                       C.byref(n), ctr.data_ptr(), _stream_ptr(self.stream)))
        if n.value > log_cap:
            raise SagaError(4, f"victim log needs {n.value} entries (log_cap {log_cap})")
        return ctr[node].cpu().numpy(), log[:n.value].cpu().numpy().view(np.uint64)

    def tool_stats(self, label, n_labels: int, p_pm: int = 950, window: int = 256, min_samples: int = 20,
                   ema_terms: int = 64):
        """F4 (saga_tool_stats): label int32 cuda tensor [n_calls].  Returns (ttl int64 [n_calls],
        obs int32 [n_calls] (uint32 bits)) cuda tensors."""
        import torch
        n = self.desc.n_calls
        ttl = torch.empty(max(n, 1), dtype=torch.int64, device=label.device)
        obs = torch.empty(max(n, 1), dtype=torch.int32, device=label.device)
        _check(lib.saga_tool_stats(self.h, label.data_ptr(), int(n_labels), int(p_pm), int(window), int(min_samples),
                                   int(ema_terms), ttl.data_ptr(), obs.data_ptr(), _stream_ptr(self.stream)))
        return ttl[:n], obs[:n]

    def aeg_score(self, batch: dict, rcfg: dict, key_out, score_out=None, policy=POLICY_AEG):
        """batch: dict of int/uint torch tensors seg_node, seg_epoch, seg_occ, seg_cap, seg_act (int32),
        seg_off (int64, n_seg+1), cand_lid (int32), cand_t_last (int64), cand_nu (int32)."""
        b = ScoreBatchC(int(batch["seg_off"].numel() - 1), policy, *[batch[k].data_ptr() for k in
                        ("seg_node", "seg_epoch", "seg_occ", "seg_cap", "seg_act", "seg_off", "cand_lid",
                         "cand_t_last", "cand_nu")])
        cfg = replay_cfg_c(rcfg)
        _check(lib.saga_aeg_score(self.h, C.byref(b), C.byref(cfg),
                                  score_out.data_ptr() if score_out is not None else None, key_out.data_ptr(),
                                  _stream_ptr(self.stream)))


def evict_select(keys, seg_off, k, out_off, victims, stream=None):
    _check(lib.saga_evict_select(keys.data_ptr(), seg_off.data_ptr(), k.data_ptr(), int(seg_off.numel() - 1),
                                 out_off.data_ptr(), victims.data_ptr(), _stream_ptr(stream)))


class Comm:
    """In-library NCCL communicator; the unique id is broadcast over torch.distributed."""

    def __init__(self, rank: int, world: int, device: int):
        import torch
        import torch.distributed as dist
        buf = (C.c_char * 128)()
        if rank == 0:
            _check(lib.saga_comm_unique_id(buf))
        t = torch.frombuffer(bytearray(bytes(buf)), dtype=torch.uint8).clone()
        if dist.is_available() and dist.is_initialized() and world > 1:
            obj = [bytes(t.numpy())]
            dist.broadcast_object_list(obj, src=0)
            raw = obj[0]
        else:
            raw = bytes(t.numpy())
        idb = (C.c_char * 128).from_buffer_copy(raw)
        h = C.c_void_p()
        _check(lib.saga_comm_init(idb, rank, world, device, C.byref(h)))
        self.h = h

    def allreduce(self, buf, op: int = 0, stream=None):
        _check(lib.saga_allreduce_counters(self.h, buf.data_ptr(), buf.numel(), op, _stream_ptr(stream)))

    def destroy(self):
        if getattr(self, "h", None):
            lib.saga_comm_destroy(self.h)
            self.h = None
