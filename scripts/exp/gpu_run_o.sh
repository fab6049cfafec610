#!/bin/bash
# replay A/B: TMA staging depth (C2 has many 2,049-record epochs: a 32K-token window + 1) and UNR
cd ${GRAFT_REPO_ROOT:-.}
VARIANTS="-DSAGA_REPLAY_PF=2304;-DSAGA_REPLAY_PF=2304 -DSAGA_REPLAY_UNR=3;-DSAGA_REPLAY_PF=3072 -DSAGA_REPLAY_UNR=3" bash scripts/gpu_ab2.sh
