#!/bin/bash
# replay A/B: hierarchical-bitmap take batch (c1 blocks whose word loads are issued together)
cd ${GRAFT_REPO_ROOT:-.}
VARIANTS="-DSAGA_HB_BATCH=8;-DSAGA_HB_BATCH=16" bash scripts/gpu_ab2.sh
