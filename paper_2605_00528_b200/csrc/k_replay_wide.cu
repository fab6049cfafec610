// The replay kernel (k_replay.cu) compiled a second time for launches with more items than SMs:
// 256 threads and two CTAs per SM (128 registers, 40 KB of TMA staging + 48 KB of dynamic shared
// memory each), so two items' barrier- and latency-bound epoch chains share an SM.  Same source,
// same results; run_replay dispatches here (DESIGN.md §6 "Replay occupancy").
#define SAGA_REPLAY_RT 256
#define SAGA_REPLAY_MINB 2
#define SAGA_REPLAY_PF 1024
#define SAGA_REPLAY_DYN_KB 48
#define SAGA_REPLAY_ENTRY run_replay_wide
#define SAGA_REPLAY_IS_WIDE 1
#include "k_replay.cu"
