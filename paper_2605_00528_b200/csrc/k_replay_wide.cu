// The replay kernel (k_replay.cu) compiled a second time for launches with more items than SMs:
// 256 threads and two CTAs per SM (128 registers, 40 KB of TMA staging + 16 KB of dynamic shared
// memory each), so two items' barrier- and latency-bound epoch chains share an SM.  Same source,
// same results; run_replay dispatches here (DESIGN.md §6 "Replay occupancy").
#ifndef SAGA_WIDE_RT  // overridable for occupancy experiments (SAGA_NVCC_EXTRA="-DSAGA_WIDE_RT=128 ...")
#define SAGA_WIDE_RT 256
#define SAGA_WIDE_MINB 2
#define SAGA_WIDE_PF 1024
#define SAGA_WIDE_DYN_KB 16
#endif
#define SAGA_REPLAY_RT SAGA_WIDE_RT
#define SAGA_REPLAY_MINB SAGA_WIDE_MINB
#define SAGA_REPLAY_PF SAGA_WIDE_PF
#define SAGA_REPLAY_DYN_KB SAGA_WIDE_DYN_KB
#define SAGA_REPLAY_ENTRY run_replay_wide
#define SAGA_REPLAY_IS_WIDE 1
#include "k_replay.cu"
