#!/bin/bash
# replay A/B: speculative L2 prefetch of the list-head units' alive words and lidf / nxt
cd ${GRAFT_REPO_ROOT:-.}
VARIANTS="-DSAGA_REPLAY_PF_VICTIM" bash scripts/gpu_ab2.sh
