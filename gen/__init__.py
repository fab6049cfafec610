"""Seeded synthetic input generators shared by the CUDA path, the oracle and the tests.

Holds no arithmetic of the method itself (see tracegen.py docstring)."""
from .tracegen import (TraceDesc, make, make_c1, make_c2, make_c3, make_c4, make_c5, make_obs1,
                       make_chain_limit, make_random_small, make_stream_trace, default_place_cfg, default_replay_cfg,
                       PHYSICAL_CAP, N_SWEEP, CONFIGS, PLACE_KAPPA, place_cfg_for,
                       TOOL_LABELS, pattern_labels, pattern_roles, make_label_markov, make_hand_trace)
import math


def sweep_caps(w_lo: int, w_hi: int, k: int, physical=None):
    """Capacity sweep C_k = round_half_up(W_lo * (W_hi/W_lo)^(k/(K-1))), k = 0..K-1 (fp64, host),
    plus the physical point when given.  An input list to both arms."""
    if w_lo <= 0:
        w_lo = 1
    if w_hi < w_lo:
        w_hi = w_lo
    if k == 1:
        caps = [int(w_lo)]
    else:
        caps = [int(math.floor(w_lo * (w_hi / w_lo) ** (i / (k - 1)) + 0.5)) for i in range(k)]
    if physical is not None:
        caps.append(int(physical))
    return caps
